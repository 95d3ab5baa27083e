python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; tail -15 gpurun_out/gputests.log
timeout 900 python scripts/ab.py variants/base.so variants/base.so:CUTFEM_CUTMAP=0
python bench.py --steps 200 --no-3d > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_cut_step7 -s 3 -c 1 -o gpurun_out/cut7_v11 -f python scripts/profile_step.py --steps 1 > /dev/null 2>&1
