mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; tail -3 gpurun_out/gputests.log
grep -E "passed|failed|PASS|FAIL" gpurun_out/gputests.log | tail -3
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
timeout 1200 bash scripts/gpu_profile.sh > gpurun_out/profile_summary.txt 2>&1; tail -30 gpurun_out/profile_summary.txt
