import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
from paper_2508_11608_b200 import cutfem
w = workloads.CONFIG1
g = cutfem.Problem.from_workload(w)
b = g.to_device(workloads.lattice_vector(w, 2))
z = g.zeros()
for _ in range(3):
    g.vcycle(z, b)
torch.cuda.synchronize()
torch.cuda.profiler.start()
g.vcycle(z, b)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
