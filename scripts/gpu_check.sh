python -m pytest tests/test_gpu_modes.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/t1.log 2>&1; tail -5 gpurun_out/t1.log
timeout 900 python scripts/ab.py variants/base.so variants/base.so:CUTFEM_CUT_GRID=0 variants/base.so:CUTFEM_CUT_GRID_MIN_N=256
