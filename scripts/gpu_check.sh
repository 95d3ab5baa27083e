timeout 900 python scripts/large_size.py 2>&1 | tail -3
python -m pytest tests/test_gpu_modes.py tests/test_gpu_fullsize.py -x -q > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
