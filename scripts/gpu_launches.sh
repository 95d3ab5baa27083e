# launch list (ncu gpu__time_duration + dram bytes per launch) of 2 smoothing steps + 1 V-cycle of config1
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --profile-from-start off --csv --log-file gpurun_out/launches.csv python scripts/profile_step.py --steps 2 --vcycle > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches.csv
