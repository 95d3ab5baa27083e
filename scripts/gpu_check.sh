python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; tail -3 gpurun_out/gputests.log
timeout 900 python scripts/ab.py variants/v18.so variants/v20.so variants/v20.so:CUTFEM_TILEAPPLY_MIN=1 variants/v20.so:CUTFEM_TILEAPPLY_MIN=100000
