python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; tail -1 gpurun_out/gputests.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
