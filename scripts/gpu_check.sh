python -m pytest tests/test_gpu_slab.py -x -q -k "fullsize" > gpurun_out/fs.log 2>&1; tail -15 gpurun_out/fs.log
