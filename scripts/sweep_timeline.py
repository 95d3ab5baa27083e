"""Phase timeline of one k_cut_sweep launch (debug build with -DCF_TIMING,
loaded through CUTFEM_LIB_OVERRIDE): per CTA globaltimer stamps
0 start (before the dependency wait), 1 slots loaded, 2 step 0 done,
3 step 1 done, 4 half the steps done, 5 all steps done, 6 grid counter
passed, 7 stores done.  Prints the distribution over CTAs (us from the
earliest start)."""
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
info = g.level_info(lvl)
n = info.sweep_ctas[0]
x = g.to_device(workloads.lattice_vector(w, 1, lvl), lvl)
b = g.to_device(workloads.lattice_vector(w, 2, lvl), lvl)
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
lib = cutfem._lib
lib.cutfem_debug_timers.argtypes = [ctypes.c_void_p, ctypes.c_int]
for it in range(4):
    if not os.environ.get("NOFLUSH"):
        flush.fill_(1.0)
    torch.cuda.synchronize()
    if os.environ.get("STEP"):
        g.smooth(lvl, x, b)
    else:
        g.colour_step(lvl, 3, 0, x, b)
    torch.cuda.synchronize()
buf = np.zeros((n, 8), dtype=np.uint64)
assert lib.cutfem_debug_timers(buf.ctypes.data, n) == 0
t = (buf.astype(np.int64) - int(buf[:, 0].min())) / 1e3
print(f"level {lvl}: {n} CTAs, redundancy {info.sweep_redundancy[0]:.2f}")
names = ["start", "slots", "step1", "half", "steps", "gridwait", "stored", "-"]
for k in range(7):
    c = t[:, k]
    print(f"{names[k]:9s} min {c.min():7.2f}  med {np.median(c):7.2f}  max {c.max():7.2f}")
b2 = np.zeros((4096 + n, 8), dtype=np.uint64)
assert lib.cutfem_debug_timers(b2.ctypes.data, 4096 + n) == 0
acc = b2[4096:, :7].astype(np.float64)
for i, nm in enumerate(["data wait", "gather", "rows", "arrive"]):
    print(f"consumer 0 cycles in {nm:10s}: med {np.median(acc[:, i]):8.0f} max {acc[:, i].max():8.0f}")
print(f"chunks per CTA: med {np.median(acc[:, 4]):.0f} max {acc[:, 4].max():.0f}; runs med {np.median(acc[:, 5]):.0f} "
      f"max {acc[:, 5].max():.0f}; bytes med {np.median(acc[:, 6]) / 1e3:.0f} KB max {acc[:, 6].max() / 1e3:.0f} KB")
b3 = np.zeros((5012, 8), dtype=np.uint64)
assert lib.cutfem_debug_timers(b3.ctypes.data, 5012) == 0
iss, ful, don = (b3[5000:5004].ravel().astype(np.int64), b3[5004:5008].ravel().astype(np.int64),
                 b3[5008:5012].ravel().astype(np.int64))
base = iss[0]
for k in range(min(32, int(acc[0, 4]))):
    print(f"chunk {k:2d}: issued {iss[k] - base:7d}  landed+seen {ful[k] - base:7d}  done {don[k] - base:7d}  "
          f"lat {ful[k] - iss[k]:6d}")
d = np.diff(t, axis=1)
for k in range(6):
    print(f"{names[k]}->{names[k + 1]:9s} med {np.median(d[:, k]):7.2f} max {d[:, k].max():7.2f}")
