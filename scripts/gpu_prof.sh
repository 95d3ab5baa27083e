python -m pytest tests/test_gpu_slab.py -x -q -k "world1 or layout" > gpurun_out/slab1.log 2>&1; tail -3 gpurun_out/slab1.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 scripts/nccl_selftest.py > gpurun_out/nccl2.log 2>&1; grep -i "rank\|error" gpurun_out/nccl2.log | tail -8
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_v9.csv python scripts/profile_step.py --steps 2 --vcycle > /dev/null 2>&1; wc -l gpurun_out/launches_v9.csv
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_cut_step6 -s 3 -c 1 -o gpurun_out/cut6_v9 -f python scripts/profile_step.py --steps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_cart_fused_tma -c 1 -o gpurun_out/cart_v9 -f python scripts/profile_step.py --steps 1 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
