"""Phase timeline of one k_cart_fused_tma launch (debug build -DCF_TIMING via
CUTFEM_LIB_OVERRIDE): per CTA globaltimer stamps 0 start, 1 vertex kinds
staged, 2 patch lists compacted (+ dependency wait), 3 x/b regions landed,
4 two passes done, 5 four passes done, 6 neighbour flags seen, 7 stored."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2508_11608_b200 import cutfem  # noqa: E402

w = getattr(workloads, os.environ.get("WL", "CONFIG1"))
lvl = int(os.environ.get("LEVEL", w.n_levels - 1))
g = cutfem.Problem.from_workload(w)
x = g.to_device(workloads.lattice_vector(w, 1, lvl), lvl)
b = g.to_device(workloads.lattice_vector(w, 2, lvl), lvl)
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
lib = cutfem._lib
lib.cutfem_debug_timers.argtypes = [ctypes.c_void_p, ctypes.c_int]
n = int(os.environ.get("NCTA", "252"))
for it in range(4):
    if not os.environ.get("NOFLUSH"):
        flush.fill_(1.0)
    torch.cuda.synchronize()
    g.colour_step(lvl, 2, 0, x, b)
    torch.cuda.synchronize()
buf = np.zeros((n, 8), dtype=np.uint64)
assert lib.cutfem_debug_timers(buf.ctypes.data, n) == 0
t = (buf.astype(np.int64) - int(buf[:, 0].min())) / 1e3
names = ["start", "vk", "lists", "loaded", "2pass", "4pass", "flags", "stored"]
for k in range(8):
    c = t[:, k]
    print(f"{names[k]:7s} min {c.min():7.2f}  med {np.median(c):7.2f}  max {c.max():7.2f}")
d = np.diff(t, axis=1)
for k in range(7):
    print(f"{names[k]}->{names[k + 1]:7s} med {np.median(d[:, k]):7.2f} max {d[:, k].max():7.2f}")
