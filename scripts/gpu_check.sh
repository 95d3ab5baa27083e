python -m pytest tests/test_gpu_3d.py tests/test_gpu_slab.py -x -q -k "3d" > gpurun_out/t3.log 2>&1; tail -3 gpurun_out/t3.log
timeout 900 python scripts/ab.py --w CONFIG2 variants/v18.so variants/v19.so
