python -m pytest tests/test_gpu_slab.py -x -q -k "3d" > gpurun_out/s3.log 2>&1; tail -30 gpurun_out/s3.log
