"""Step timeline of the cluster-resident cut sweeps (variant build with
-DCF_TIMING): globaltimer stamps of CTA 0..15 at entry, after pdl_wait, after
the first five step barriers, at exit (ns).
usage: CUTFEM_LIB_OVERRIDE=variants/timing.so python scripts/cluster_timeline.py [level]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2508_11608_b200 import cutfem  # noqa: E402

w = workloads.CONFIG1
g = cutfem.Problem.from_workload(w)
lib = ctypes.CDLL(os.environ["CUTFEM_LIB_OVERRIDE"])
lib.cutfem_debug_timers.argtypes = [ctypes.c_void_p, ctypes.c_int]
L = int(sys.argv[1]) if len(sys.argv) > 1 else 5
x = g.to_device(workloads.lattice_vector(w, 1, L), L)
b = g.to_device(workloads.lattice_vector(w, 2, L), L)
for rep in range(3):
    g.colour_step(L, 3, 0, x, b)
    torch.cuda.synchronize()
buf = np.zeros((8192, 8), dtype=np.uint64)
lib.cutfem_debug_timers(buf.ctypes.data, 16)
t = buf[:16].astype(np.int64)
t0 = t[:, 0].min()
print(f"level {L}, cut patches per colour {list(g.level_info(L).n_cutp)[:4]}")
print("CTA stamps relative to first entry (ns): entry, waited, step1..5, exit")
for r in range(16):
    print(r, (t[r] - t0).tolist())
