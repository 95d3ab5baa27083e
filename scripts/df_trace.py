"""CUTFEM_DF_TRACE=1: per-phase globaltimer stamps of the dataflow cut sweep
(max over segments, us from the first CTA start) on every level of a workload."""
import os
import sys

os.environ["CUTFEM_DF_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2508_11608_b200 import cutfem  # noqa: E402

w = getattr(workloads, sys.argv[1]) if len(sys.argv) > 1 else workloads.CONFIG1
g = cutfem.Problem.from_workload(w)
sys.stderr.write("columns: start blob-loaded pdl-done b-gathered | per step: waited gathered written released\n")
for l in range(1, w.n_levels):
    x = g.to_device(workloads.lattice_vector(w, 1, l), l)
    b = g.to_device(workloads.lattice_vector(w, 2, l), l)
    for _ in range(3):
        g.colour_step(l, 3, 0, x, b)
        torch.cuda.synchronize()
