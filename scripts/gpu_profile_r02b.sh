# round-2 (second session) evidence: bench line, ncu launch list of 2 smoothing steps + 1 V-cycle,
# full ncu sections of one k_cut_sweep and one k_cart_fused_tma launch (config1)
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_r02d.json 2> gpurun_out/bench_r02d.err; tail -2 gpurun_out/bench_r02d.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --profile-from-start off --csv --log-file gpurun_out/launches_r02d.csv python scripts/profile_step.py --steps 2 --vcycle > /dev/null 2>&1
for k in k_cut_sweep k_cart_fused_tma; do
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:$k -c 1 \
      -o gpurun_out/$k -f python scripts/profile_step.py --steps 1 > /dev/null 2>&1
  ncu -i gpurun_out/$k.ncu-rep --page details --csv > gpurun_out/${k}_details.csv 2>/dev/null
  ncu -i gpurun_out/$k.ncu-rep --page raw --csv > gpurun_out/${k}_raw.csv 2>/dev/null
done
python scripts/launch_summary.py gpurun_out/launches_r02d.csv > gpurun_out/launches_r02d.md
python scripts/ncu_summary.py --traffic gpurun_out/traffic_r02d.json gpurun_out/k_cart_fused_tma_raw.csv gpurun_out/k_cut_sweep_raw.csv > gpurun_out/ncu_r02d.md
cat gpurun_out/launches_r02d.md gpurun_out/ncu_r02d.md
