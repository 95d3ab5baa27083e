"""Phase timeline of one 2D cut colour step (variant build with -DCF_TIMING):
per-block globaltimer stamps -> distribution of phase durations (ns).
usage: CUTFEM_LIB_OVERRIDE=variants/timing.so python scripts/cut_timeline.py [level]"""
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
L = int(sys.argv[1]) if len(sys.argv) > 1 else w.n_levels - 1
info = g.level_info(L)
x = g.to_device(workloads.lattice_vector(w, 1, L), L)
b = g.to_device(workloads.lattice_vector(w, 2, L), L)
V5 = os.environ.get("CUTFEM_CUT2", "5") != "4"
names = (["entry->desc", "desc->pdlwait", "pdlwait->loaded", "faces+cells", "gather", "inverse->end"] if V5 else
         ["entry->desc", "desc->pdlwait", "pdlwait->loaded", "loaded->inverse", "inverse->end"])
for rep in range(3):
    g.colour_step(L, 1, 0, x, b)   # one cut colour (colour 0), non-ping-pong path? uses kind 1
    torch.cuda.synchronize()
np_ = info.n_cutp[0]
buf = np.zeros((8192, 8), dtype=np.uint64)
lib.cutfem_debug_timers(buf.ctypes.data, 8192)
t = buf[:np_, :len(names) + 1].astype(np.int64)
t0 = t[:, 0].min()
print(f"level {L}: {np_} patches; span entry-first -> end-last {(t[:, len(names)].max() - t0)} ns")
for k, nm in enumerate(names):
    d = t[:, k + 1] - t[:, k]
    print(f"  {nm:16s} median {np.median(d):7.0f}  p90 {np.percentile(d, 90):7.0f}  max {d.max():7.0f}")
print("  block start spread (ns): median", np.median(t[:, 0] - t0), "max", (t[:, 0] - t0).max())
