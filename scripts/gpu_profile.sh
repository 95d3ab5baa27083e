# ncu captures behind profiles/r02 (one gpurun call; summaries are copied to profiles/ by scripts/ncu_summary.py):
#   launch list (time + DRAM bytes per launch) of 2 smoothing steps + 1 V-cycle of config1,
#   full sections of one fused Cartesian sweep, one 2D cut colour step, one 3D cut colour step (config2).
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --profile-from-start off --csv --log-file gpurun_out/launches.csv python scripts/profile_step.py --steps 2 --vcycle > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_cart_fused_tma -c 1 \
    -o gpurun_out/cart -f python scripts/profile_step.py --steps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_cut_step7 -s 3 -c 1 \
    -o gpurun_out/cut7 -f python scripts/profile_step.py --steps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_cut_colour3 -s 1 -c 1 \
    -o gpurun_out/cut3d -f python scripts/profile_step.py --steps 1 --workload CONFIG2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --profile-from-start off --csv --log-file gpurun_out/launches3d.csv python scripts/profile_step.py --steps 1 --workload CONFIG2 > /dev/null 2>&1
for r in cart cut7 cut3d; do
  ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
done
python scripts/launch_summary.py gpurun_out/launches.csv
python scripts/launch_summary.py gpurun_out/launches3d.csv
