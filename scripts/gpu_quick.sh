# quick GPU iteration: the tests named by $1 (pytest -k), the full GPU suite, bench
mkdir -p gpurun_out
export CUTFEM_VERBOSE=${CUTFEM_VERBOSE:-0}
timeout 900 python -m pytest tests -m gpu -x -q -k "${1:-dataflow}" > gpurun_out/quick_tests.log 2>&1; tail -3 gpurun_out/quick_tests.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; tail -3 gpurun_out/gputests.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
python -c "
import json;d=json.load(open('gpurun_out/bench.json'))
print('value',d['value'],'ms',d['ms_per_step'],'vcycle',d.get('vcycle'),'cg',d.get('cg_mg',{}).get('time_to_solution_ms'))
print(json.dumps(d.get('kernels'))[:600])"
