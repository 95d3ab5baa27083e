python -m pytest tests/test_gpu_modes.py -x -q -k "vcycle_cluster" > gpurun_out/vc.log 2>&1; tail -15 gpurun_out/vc.log
python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; tail -15 gpurun_out/gputests.log
timeout 900 python scripts/ab.py variants/v12.so variants/v13.so variants/v13.so:CUTFEM_VC_MAX_N=128 variants/v13.so:CUTFEM_VC_MAX_N=32
