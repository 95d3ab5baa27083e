# ncu captures behind profiles/r01 (one gpurun call; summaries are copied to profiles/ by hand):
#   launch list (time + DRAM bytes per launch) of 2 smoothing steps + 1 V-cycle of config1,
#   full sections of one fused Cartesian sweep and one cut colour step.
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --profile-from-start off --csv --log-file gpurun_out/launches.csv python scripts/profile_step.py --steps 2 --vcycle > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_cart_fused_tma -c 1 \
    -o gpurun_out/cart -f python scripts/profile_step.py --steps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_cut_step7 -s 3 -c 1 \
    -o gpurun_out/cut7 -f python scripts/profile_step.py --steps 1 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches.csv
