"""Two NCCL ranks on ONE GPU (torchrun --nproc-per-node 2, both on cuda:0):
checks whether this NCCL accepts it (it normally refuses duplicate GPUs) and,
if it does, that the slab-partitioned smoothing step / V-cycle / CG over the
NCCL endpoint match the single-rank path bit-exactly."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import workloads  # noqa: E402
from paper_2508_11608_b200 import cutfem  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("gloo")
w = workloads.paper_level(2, 9)
L = w.n_levels - 1
g = cutfem.Problem.from_workload(w)
try:
    comm = cutfem.Comm.nccl_from_torch(dist)
except Exception as e:  # noqa: BLE001
    print(f"rank {rank}: NCCL endpoint refused: {e}", flush=True)
    sys.exit(0)
g.partition(comm)
g1 = cutfem.Problem.from_workload(w)
x0, b0 = workloads.lattice_vector(w, 1), workloads.lattice_vector(w, 2)
res = []
for h in (g1, g):
    x = h.to_device(x0)
    b = h.to_device(b0)
    h.smooth(L, x, b)
    h.vcycle(x, b)
    xs = h.zeros()
    it, rel = h.solve_cg_mg(xs, b, tol=1e-9)
    torch.cuda.synchronize()
    res.append((h.to_host(x), it, h.to_host(xs)))
info = g.partition_info(L)
nl = g.lattice_shape(L)[0]
o = slice(info["r0"] * nl, info["r1"] * nl)
ok = np.array_equal(res[0][0][o], res[1][0][o]) and res[0][1] == res[1][1]
err = np.abs(res[0][2][o] - res[1][2][o]).max() / np.abs(res[0][2]).max()
print(f"rank {rank}/{world}: rows [{info['r0']},{info['r1']}) smooth+vcycle bit-exact={ok} cg its {res[1][1]} "
      f"(single {res[0][1]}) sol err {err:.1e}", flush=True)
dist.destroy_process_group()
