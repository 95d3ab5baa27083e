python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; tail -15 gpurun_out/gputests.log
timeout 900 python scripts/ab.py variants/base.so variants/base.so:CUTFEM_CUTMAP=0
