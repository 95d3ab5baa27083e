"""A/B timing of library variants (CUTFEM_LIB_OVERRIDE) on one workload:
alternates the variants for several rounds in fresh processes and prints
smoothing step, fused Cartesian sweep, cut sweeps and V-cycle (us).
usage: python scripts/ab.py [--w CONFIG1|CONFIG2] lib1.so[:ENV=V,ENV2=V] ..."""
import json
import os
import subprocess
import sys

CHILD = r'''
import os, sys, json
sys.path.insert(0, os.getcwd())
import torch, workloads
from paper_2508_11608_b200 import cutfem
w = getattr(workloads, sys.argv[1])
g = cutfem.Problem.from_workload(w)
L = w.n_levels - 1
x = g.to_device(workloads.lattice_vector(w, 1)); b = g.to_device(workloads.lattice_vector(w, 2))
def t(fn, n):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n * 1e3
n = 100 if w.dim == 2 else 10
r = dict(smooth=t(lambda: g.smooth(L, x, b), n), cart=t(lambda: g.colour_step(L, 2 if w.dim == 2 else 0, 0, x, b), n),
         cut=t(lambda: g.colour_step(L, 3 if w.dim == 2 else 1, 0, x, b), n))
z = g.zeros()
r["vcycle"] = t(lambda: g.vcycle(z, b), 10 if w.dim == 2 else 3)
print(json.dumps(r))
'''

args = sys.argv[1:]
wname = "CONFIG1"
if args and args[0] == "--w":
    wname, args = args[1], args[2:]
libs = args
res = {l: [] for l in libs}
for rnd in range(3):
    for lib in libs:
        path, _, envs = lib.partition(":")
        env = dict(os.environ, CUTFEM_LIB_OVERRIDE=os.path.abspath(path))
        env.update(dict(kv.split("=") for kv in envs.split(",") if kv))
        out = subprocess.run([sys.executable, "-c", CHILD, wname], env=env, capture_output=True, text=True, timeout=600)
        line = [s for s in out.stdout.splitlines() if s.startswith("{")]
        if not line:
            print(lib, "FAILED", out.stderr[-2000:])
            continue
        res[lib].append(json.loads(line[-1]))
for lib, rs in res.items():
    if not rs:
        continue
    keys = rs[0].keys()
    print(lib, " ".join(f"{k}={min(r[k] for r in rs):.1f}/{sorted(r[k] for r in rs)[len(rs)//2]:.1f}" for k in keys))
