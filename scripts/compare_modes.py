"""Time one smoothing step / V-cycle of config1 for the launch modes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2508_11608_b200 import cutfem  # noqa: E402

w = getattr(workloads, sys.argv[1] if len(sys.argv) > 1 else "CONFIG1")
MODES = {"default": dict(CUTFEM_FUSED="1", CUTFEM_PDL="1", CUTFEM_MMA="1", CUTFEM_PINGPONG="1", CUTFEM_TMA="1", CUTFEM_CTACUT="1"),
         "node apply": dict(CUTFEM_TILEAPPLY="0"),
         "warp per cut patch": dict(CUTFEM_TILEAPPLY="1", CUTFEM_CTACUT="0"),
         "no tma": dict(CUTFEM_CTACUT="1", CUTFEM_TMA="0"),
         "no mma (FD)": dict(CUTFEM_TMA="1", CUTFEM_MMA="0"),
         "no pdl": dict(CUTFEM_MMA="1", CUTFEM_PDL="0")}
for mode, env in MODES.items():
    for cut_mode in (0,):
        os.environ.update(env)
        g = cutfem.Problem.from_workload(w, cut_mode=cut_mode)
        L = w.n_levels - 1
        x = g.to_device(workloads.lattice_vector(w, 1))
        b = g.to_device(workloads.lattice_vector(w, 2))
        for _ in range(5):
            g.smooth(L, x, b)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(200):
            g.smooth(L, x, b)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 200
        z = g.zeros()
        for _ in range(3):
            g.vcycle(z, b)
        torch.cuda.synchronize()
        s.record()
        for _ in range(20):
            g.vcycle(z, b)
        e.record()
        torch.cuda.synchronize()
        vms = s.elapsed_time(e) / 20
        xs = g.zeros()
        it, rel = g.solve_cg_mg(xs, b, tol=w.tol)
        torch.cuda.synchronize()
        s.record()
        it, rel = g.solve_cg_mg(xs, b, tol=w.tol)
        e.record()
        torch.cuda.synchronize()
        print(f"mode={mode} cut_mode={cut_mode}: smooth {ms*1e3:.1f} us, vcycle {vms*1e3:.1f} us, "
              f"cg {s.elapsed_time(e):.2f} ms ({it} it)", flush=True)
        g.close()
