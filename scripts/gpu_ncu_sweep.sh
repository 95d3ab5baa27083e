# ncu of the one-launch cut sweep (full sections, one launch of config1's finest level) + launch list
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_cut_sweep -s 0 -c 1 \
    -o gpurun_out/sweep -f python scripts/profile_step.py --steps 1 > gpurun_out/ncu_sweep.log 2>&1
ncu -i gpurun_out/sweep.ncu-rep --page details --csv > gpurun_out/sweep_details.csv 2>/dev/null
ncu -i gpurun_out/sweep.ncu-rep --page raw --csv > gpurun_out/sweep_raw.csv 2>/dev/null
ncu -i gpurun_out/sweep.ncu-rep --page source --csv > gpurun_out/sweep_source.csv 2>/dev/null
