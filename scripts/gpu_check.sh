python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; tail -3 gpurun_out/gputests.log
timeout 900 python scripts/ab.py variants/v16.so variants/v17.so
