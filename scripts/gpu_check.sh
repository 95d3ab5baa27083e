python -m pytest tests/test_gpu_slab.py -x -q -k "errors or layout or world1" > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
