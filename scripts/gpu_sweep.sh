# sweep iteration: the one-launch cut sweep tests, CTA-count scan, phase timeline
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_sweep.py -x -q --timeout 120 > gpurun_out/sweep_tests.log 2>&1; tail -2 gpurun_out/sweep_tests.log
timeout 300 python scripts/sweep_ng.py ${NGS:-0} 2>&1 | tail -8
NOFLUSH=1 CUTFEM_LIB_OVERRIDE=$PWD/paper_2508_11608_b200/libcutfem_timing.so timeout 200 python scripts/sweep_timeline.py 2>&1 | tail -16
