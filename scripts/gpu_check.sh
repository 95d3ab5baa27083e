python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; tail -3 gpurun_out/gputests.log
timeout 900 python scripts/ab.py variants/v11.so variants/v12.so
