python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_v12.csv python scripts/profile_step.py --steps 2 --vcycle > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_cut_step7 -s 3 -c 1 -o gpurun_out/cut7_v12 -f python scripts/profile_step.py --steps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_cart_fused_tma -c 1 -o gpurun_out/cart_v12 -f python scripts/profile_step.py --steps 1 > /dev/null 2>&1
ls gpurun_out
