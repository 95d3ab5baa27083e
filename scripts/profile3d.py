import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
from paper_2508_11608_b200 import cutfem
w = workloads.CONFIG2
nlev = int(sys.argv[1]) if len(sys.argv) > 1 else 6
w = workloads.Workload(w.name, w.x0, w.y0, w.length, w.n_coarse, nlev, w.cx, w.cy, w.r, w.p, w.n_c, w.tol, 3, w.z0, w.cz)
g = cutfem.Problem.from_workload(w)
L = nlev - 1
x = g.to_device(workloads.lattice_vector(w, 1)); b = g.to_device(workloads.lattice_vector(w, 2))
g.smooth(L, x, b); torch.cuda.synchronize()
torch.cuda.profiler.start()
g.smooth(L, x, b)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
