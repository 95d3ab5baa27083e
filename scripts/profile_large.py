"""One fused Cartesian sweep + one cut step at n = 4096 (Q2) inside the profiler range."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2508_11608_b200 import cutfem  # noqa: E402

nlev = int(sys.argv[1]) if len(sys.argv) > 1 else 12
w = workloads.Workload("large", -1.105, -1.105, 2.21, 2, nlev, 0.0, 0.0, 1.0, 2)
g = cutfem.Problem.from_workload(w)
L = nlev - 1
info = g.level_info(L)
x = g.to_device(np.random.default_rng(1).standard_normal(info.nl * info.nl))
b = g.to_device(np.random.default_rng(2).standard_normal(info.nl * info.nl))
g.smooth(L, x, b)
torch.cuda.synchronize()
torch.cuda.profiler.start()
g.smooth(L, x, b)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
