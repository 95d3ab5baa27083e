# One gpurun call: GPU tests, bench line, smoke (outputs under gpurun_out/).
#   /usr/local/graft/bin/gpurun --timeout 1500 -- 'bash scripts/gpu_check.sh'
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; tail -1 gpurun_out/gputests.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
