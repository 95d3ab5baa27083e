python -m pytest tests/test_gpu_parity.py -x -q -k "non_dof" > gpurun_out/t.log 2>&1; tail -25 gpurun_out/t.log
