"""Run the bench workload's smoothing step under the CUDA profiler range
(for `ncu --profile-from-start off`): setup and warm-up are outside the
range, `--steps` smoothing steps (and optionally one V-cycle) inside."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2508_11608_b200 import cutfem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--vcycle", action="store_true")
ap.add_argument("--workload", default="CONFIG1")
args = ap.parse_args()
w = getattr(workloads, args.workload)
g = cutfem.Problem.from_workload(w)
L = w.n_levels - 1
x = g.to_device(workloads.lattice_vector(w, 1))
b = g.to_device(workloads.lattice_vector(w, 2))
for _ in range(3):
    g.smooth(L, x, b)
    if args.vcycle:
        g.vcycle(x, b)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(args.steps):
    g.smooth(L, x, b)
if args.vcycle:
    g.vcycle(x, b)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done", cutfem.launch_count())
