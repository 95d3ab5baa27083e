python -m pytest tests/test_gpu_slab.py -x -q > gpurun_out/slab.log 2>&1; tail -25 gpurun_out/slab.log
