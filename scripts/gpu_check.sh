python -m pytest tests/test_gpu_slab.py tests/test_gpu_modes.py -x -q > gpurun_out/slab.log 2>&1; tail -15 gpurun_out/slab.log
python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; tail -3 gpurun_out/gputests.log
python bench.py --steps 200 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 600 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 900 python scripts/ab.py variants/base.so variants/base.so:CUTFEM_TC32_MIN_N=100000 variants/base.so:CUTFEM_TC32_MIN_N=256
