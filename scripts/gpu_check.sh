python -m pytest tests/test_gpu_modes.py tests/test_gpu_fullsize.py -x -q > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
timeout 900 python scripts/ab.py variants/v27_g1.so variants/v27.so
