"""Per coarse level of config1: the one-launch cut sweep's device time for
forced CTA counts (CUTFEM_SWEEP_NG), measured as a CUDA graph of 20 sweeps
(launch overhead amortised, PDL between them), warm."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2508_11608_b200 import cutfem  # noqa: E402

w = workloads.CONFIG1
res = {}
for ng in sys.argv[1:] or ["0", "1", "2", "4", "8", "16", "32"]:
    if ng == "0":
        os.environ.pop("CUTFEM_SWEEP_NG", None)
    else:
        os.environ["CUTFEM_SWEEP_NG"] = ng
    g = cutfem.Problem.from_workload(w)
    row = []
    for l in range(1, w.n_levels):
        x = g.to_device(workloads.lattice_vector(w, 1, l), l)
        b = g.to_device(workloads.lattice_vector(w, 2, l), l)
        for _ in range(3):
            g.colour_step(l, 3, 0, x, b)
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=s):
                for _ in range(20):
                    g.colour_step(l, 3, 0, x, b, stream=s.cuda_stream)
        torch.cuda.synchronize()
        gr.replay()
        torch.cuda.synchronize()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            gr.replay()
        e.record()
        torch.cuda.synchronize()
        row.append((g.level_info(l).sweep_ctas[0], a.elapsed_time(e) * 1e3 / 100))
    print(f"ng={ng:>3s}: " + "  ".join(f"L{l + 1}:{c:3d}/{t:5.1f}us" for l, (c, t) in enumerate(row)), flush=True)
    g.close()
