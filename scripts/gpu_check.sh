python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; tail -2 gpurun_out/gputests.log
