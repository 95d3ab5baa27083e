import sys; sys.path.insert(0,'/root/repo')
import workloads, torch, numpy as np
from paper_2508_11608_b200 import cutfem
w = workloads.paper_level(1, 7)
g = cutfem.Problem.from_workload(w)
print("built", flush=True)
for l in range(w.n_levels):
    x = g.to_device(workloads.lattice_vector(w, 1, l), l)
    y = g.zeros(l)
    g.apply_operator(l, x, y)
    torch.cuda.synchronize()
    print("level", l, "ok", flush=True)
