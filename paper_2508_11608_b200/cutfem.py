"""Thin ctypes binding of libcutfem_mg.so (include/cutfem_mg.h).

Argument marshalling only: every step of the path runs in the CUDA kernels
of the library.  Device vectors are torch CUDA float64 tensors holding a
level's lattice vector (NL x LD, see `lattice_shape`); PyTorch provides the
device memory and the current stream.  There is no CPU fallback: importing
this module fails loudly when the shared library is missing.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("CUTFEM_LIB_OVERRIDE") or os.path.join(_HERE, "libcutfem_mg.so")


class CutfemError(RuntimeError):
    pass


def _load():
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} is missing: run `python paper_2508_11608_b200/build.py` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    return ctypes.CDLL(_LIB_PATH)


_lib = _load()


class Params(ctypes.Structure):
    _fields_ = [("x0", ctypes.c_double), ("y0", ctypes.c_double), ("length", ctypes.c_double),
                ("n_coarse", ctypes.c_int), ("n_levels", ctypes.c_int), ("degree", ctypes.c_int),
                ("cx", ctypes.c_double), ("cy", ctypes.c_double), ("r", ctypes.c_double),
                ("gamma_D", ctypes.c_double), ("gamma_k", ctypes.c_double * 4), ("sigma", ctypes.c_int),
                ("n_q", ctypes.c_int), ("n_c", ctypes.c_int), ("symmetric", ctypes.c_int),
                ("cut_mode", ctypes.c_int), ("dim", ctypes.c_int), ("z0", ctypes.c_double),
                ("cz", ctypes.c_double), ("domain", ctypes.c_int)]


class LevelInfo(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int), ("n", ctypes.c_int), ("nl", ctypes.c_int), ("ld", ctypes.c_int), ("n_dofs", ctypes.c_int64),
                ("n_inside", ctypes.c_int), ("n_cut", ctypes.c_int), ("n_ghost_faces", ctypes.c_int),
                ("n_cart", ctypes.c_int * 8), ("n_cutp", ctypes.c_int * 8), ("n_vol_qp", ctypes.c_int64),
                ("n_surf_qp", ctypes.c_int64), ("h", ctypes.c_double), ("cut_step_bytes", ctypes.c_int64 * 8),
                ("cut_method_bytes", ctypes.c_int64 * 8), ("sweep_ctas", ctypes.c_int * 2),
                ("sweep_redundancy", ctypes.c_double * 2), ("sweep_map_bytes", ctypes.c_int64 * 2),
                ("host_span_doubles", ctypes.c_int64)]


_P = ctypes.c_void_p
_D = ctypes.c_void_p
_sig = {
    "cutfem_setup_mesh": [ctypes.POINTER(Params), _P, ctypes.POINTER(_P)],
    "cutfem_build_patches": [_P, _P],
    "cutfem_destroy": [_P],
    "cutfem_level_info_get": [_P, ctypes.c_int, ctypes.POINTER(LevelInfo)],
    "cutfem_apply_operator": [_P, ctypes.c_int, _D, _D, _P],
    "cutfem_smooth": [_P, ctypes.c_int, _D, _D, ctypes.c_int, _P],
    "cutfem_vcycle": [_P, _D, _D, _P],
    "cutfem_colour_step": [_P, ctypes.c_int, ctypes.c_int, ctypes.c_int, _D, _D, _P],
    "cutfem_solve_cg_mg": [_P, _D, _D, ctypes.c_double, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                           ctypes.POINTER(ctypes.c_double), _P],
    "cutfem_smooth_host": [_P, ctypes.c_int, _D, _D, ctypes.c_int, _P],
    "cutfem_solve_cg_mg_host": [_P, _D, _D, ctypes.c_double, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                ctypes.POINTER(ctypes.c_double), _P],
    "cutfem_prolongate_add": [_P, ctypes.c_int, _D, _D, _P],
    "cutfem_restrict": [_P, ctypes.c_int, _D, _D, _P],
    "cutfem_export_cell_types": [_P, ctypes.c_int, _D],
    "cutfem_export_dof_mask": [_P, ctypes.c_int, _D],
    "cutfem_export_patches": [_P, ctypes.c_int, ctypes.c_int, ctypes.c_int, _D, ctypes.POINTER(ctypes.c_int)],
    "cutfem_export_cut_interior": [_P, ctypes.c_int, _D, _D, ctypes.POINTER(ctypes.c_int),
                                   ctypes.POINTER(ctypes.c_int64)],
    "cutfem_comm_local_create": [ctypes.c_int, ctypes.POINTER(_P)],
    "cutfem_comm_nccl_unique_id": [ctypes.c_char_p],
    "cutfem_comm_nccl_create": [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_P)],
    "cutfem_comm_destroy": [_P],
    "cutfem_partition": [_P, _P],
    "cutfem_partition_info": [_P, ctypes.c_int, ctypes.POINTER(ctypes.c_int)],
    "cutfem_halo_exchange": [_P, ctypes.c_int, _D, _P],
    "cutfem_sweep_plan": [ctypes.c_int] * 8 + [_D] * 5 + [ctypes.c_double, ctypes.c_double, _D, _D, _D, ctypes.c_int,
                                               _D, _D, ctypes.c_int],
    "cutfem_slab_plan": [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                         ctypes.POINTER(ctypes.c_int64)],
}
for _name, _args in _sig.items():
    getattr(_lib, _name).argtypes = _args
    getattr(_lib, _name).restype = ctypes.c_int
_lib.cutfem_last_error.restype = ctypes.c_char_p
_lib.cutfem_last_error.argtypes = []
_lib.cutfem_launch_count.restype = ctypes.c_int64
_lib.cutfem_launch_count.argtypes = []

EXPORTED = list(_sig) + ["cutfem_last_error", "cutfem_launch_count"]


def _check(rc):
    if rc != 0:
        raise CutfemError(f"cutfem status {rc}: {_lib.cutfem_last_error().decode()}")


def _stream(stream):
    if stream is not None:
        return ctypes.c_void_p(int(stream))
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dptr(t):
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise CutfemError("vectors must be contiguous CUDA float64 torch tensors")
    return ctypes.c_void_p(t.data_ptr())


def launch_count():
    return int(_lib.cutfem_launch_count())


def make_params(x0, y0, length, n_coarse, n_levels, degree, cx, cy, r, gamma_D=0.0, gamma_k=(-1, -1, -1, -1),
                sigma=-1, n_q=0, n_c=2, symmetric=1, cut_mode=0, dim=2, z0=0.0, cz=0.0, domain=0):
    g = (ctypes.c_double * 4)(*[float(v) for v in (list(gamma_k) + [-1] * 4)[:4]])
    return Params(x0, y0, length, n_coarse, n_levels, degree, cx, cy, r, gamma_D, g, sigma, n_q, n_c, symmetric,
                  cut_mode, dim, z0, cz, domain)


NCCL_ID_BYTES = 128


def sweep_plan(n, p, ld, S, reverse, nsm, force_ng, ijc, in_lists, ex_lists, ca, cb):
    """Host-only planner of the one-launch cut sweep (cutfem_sweep_plan):
    patches given as ijc (k, 3) = (I, J, colour) and per-patch lists of
    interior / coupled exterior lattice nodes (b * ld + a).  Returns (owned,
    cones): owned[g] = nodes of CTA g, cones[g][s] = patch indices of its
    step-s cone."""
    npatch = len(in_lists)
    ijc = np.ascontiguousarray(np.asarray(ijc, dtype=np.int32).reshape(npatch, 3))
    in_off = np.zeros(npatch + 1, np.int32)
    ex_off = np.zeros(npatch + 1, np.int32)
    in_off[1:] = np.cumsum([len(v) for v in in_lists])
    ex_off[1:] = np.cumsum([len(v) for v in ex_lists])
    in_nodes = np.ascontiguousarray(np.concatenate([np.asarray(v, np.int32) for v in in_lists] or [np.zeros(0, np.int32)]))
    ex_nodes = np.ascontiguousarray(np.concatenate([np.asarray(v, np.int32) for v in ex_lists] or [np.zeros(0, np.int32)]))
    own_cap = int(in_off[-1]) + 1
    task_cap = max(1, npatch * S * nsm)
    ncta = ctypes.c_int(0)
    own_off = np.zeros(nsm + 1, np.int32)
    own_nodes = np.zeros(own_cap, np.int32)
    task_off = np.zeros(nsm * S + 1, np.int32)
    task_patch = np.zeros(task_cap, np.int32)
    d = lambda a: a.ctypes.data_as(_D)
    _check(_lib.cutfem_sweep_plan(n, p, ld, S, int(reverse), nsm, force_ng, npatch, d(ijc), d(in_off), d(in_nodes),
                                  d(ex_off), d(ex_nodes), float(ca), float(cb), ctypes.byref(ncta), d(own_off),
                                  d(own_nodes), own_cap, d(task_off), d(task_patch), task_cap))
    g = ncta.value
    owned = [own_nodes[own_off[i]:own_off[i + 1]].tolist() for i in range(g)]
    cones = [[task_patch[task_off[i * S + s]:task_off[i * S + s + 1]].tolist() for s in range(S)] for i in range(g)]
    return owned, cones


def slab_plan(n_cells, degree, world, rank, halo_cells):
    """The partition's slab plan of one level (host only): owned / valid
    lattice rows and the row bands exchanged with the neighbours."""
    out = (ctypes.c_int64 * 17)()
    _check(_lib.cutfem_slab_plan(n_cells, degree, world, rank, halo_cells, out))
    v = list(out)
    xf = [dict(zip(("peer", "send_off", "send_n", "recv_off", "recv_n"), v[7 + 5 * i:12 + 5 * i]))
          for i in range(v[6])]
    return dict(c0=v[0], c1=v[1], r0=v[2], r1=v[3], v0=v[4], v1=v[5], xfers=xf)


class Comm:
    """One rank's communicator endpoint (cutfem_comm), handed to
    Problem.partition, which takes ownership."""

    def __init__(self, handle):
        self._h = handle

    @staticmethod
    def local(world):
        """`world` endpoints of an in-process group (ranks = threads sharing one device)."""
        arr = (_P * world)()
        _check(_lib.cutfem_comm_local_create(world, arr))
        return [Comm(_P(arr[r])) for r in range(world)]

    @staticmethod
    def nccl_unique_id():
        buf = ctypes.create_string_buffer(NCCL_ID_BYTES)
        _check(_lib.cutfem_comm_nccl_unique_id(buf))
        return buf.raw

    @staticmethod
    def nccl(uid, rank, world):
        """NCCL endpoint; uid = the bytes of rank 0's nccl_unique_id() (collective)."""
        h = _P()
        _check(_lib.cutfem_comm_nccl_create(ctypes.c_char_p(bytes(uid)), rank, world, ctypes.byref(h)))
        return Comm(h)

    @staticmethod
    def nccl_from_torch(dist):
        """NCCL endpoint of the current torch.distributed group (id broadcast over it)."""
        from .dist import broadcast_nccl_id
        uid = broadcast_nccl_id(dist, Comm.nccl_unique_id)
        return Comm.nccl(uid, dist.get_rank(), dist.get_world_size())

    def close(self):
        if self._h:
            _check(_lib.cutfem_comm_destroy(self._h))
            self._h = _P()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Problem:
    """Handle on a set-up problem (setup_mesh + build_patches)."""

    def __init__(self, params, stream=None, build=True):
        self._h = _P()
        _check(_lib.cutfem_setup_mesh(ctypes.byref(params), _stream(stream), ctypes.byref(self._h)))
        self.params = params
        self.n_levels = params.n_levels
        if build:
            self.build_patches(stream)

    @classmethod
    def from_workload(cls, w, stream=None, **kw):
        prm = make_params(w.x0, w.y0, w.length, w.n_coarse, w.n_levels, w.p, w.cx, w.cy, w.r, n_c=w.n_c,
                          dim=getattr(w, "dim", 2), z0=getattr(w, "z0", 0.0), cz=getattr(w, "cz", 0.0),
                          domain=1 if getattr(w, "domain", "cut") == "fitted" else 0, **kw)
        return cls(prm, stream)

    def build_patches(self, stream=None):
        _check(_lib.cutfem_build_patches(self._h, _stream(stream)))

    def close(self):
        if self._h:
            _check(_lib.cutfem_destroy(self._h))
            self._h = _P()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --- queries
    def level_info(self, level=-1):
        level = level % self.n_levels
        info = LevelInfo()
        _check(_lib.cutfem_level_info_get(self._h, level, ctypes.byref(info)))
        return info

    def lattice_shape(self, level=-1):
        i = self.level_info(level)
        return i.nl, i.ld

    def _rows(self, level):
        i = self.level_info(level)
        return i.nl ** (i.dim - 1), i.nl, i.ld

    def zeros(self, level=-1):
        import torch
        rows, nl, ld = self._rows(level)
        return torch.zeros(rows * ld, dtype=torch.float64, device="cuda")

    def to_device(self, lattice_np, level=-1):
        """(NL^dim,) numpy lattice vector (x fastest) -> padded device vector."""
        import torch
        rows, nl, ld = self._rows(level)
        a = np.zeros((rows, ld))
        a[:, :nl] = np.asarray(lattice_np, dtype=np.float64).reshape(rows, nl)
        return torch.from_numpy(a.ravel()).cuda()

    def to_host(self, t, level=-1):
        """padded device vector -> (NL^dim,) numpy lattice vector."""
        rows, nl, ld = self._rows(level)
        return t.detach().cpu().numpy().reshape(rows, ld)[:, :nl].ravel().copy()

    # --- slab partition
    def partition(self, comm):
        _check(_lib.cutfem_partition(self._h, comm._h))
        comm._h = _P()   # owned by the problem

    def partition_info(self, level=-1):
        """dict(part, r0, r1, v0, v1, rank, world, halo): owned / valid lattice rows of `level`."""
        out = (ctypes.c_int * 8)()
        _check(_lib.cutfem_partition_info(self._h, level % self.n_levels, out))
        return dict(zip(("part", "r0", "r1", "v0", "v1", "rank", "world", "halo"), list(out)))

    def halo_exchange(self, level, v, stream=None):
        _check(_lib.cutfem_halo_exchange(self._h, level % self.n_levels, _dptr(v), _stream(stream)))

    # --- hot path (names of the C ABI)
    def apply_operator(self, level, x, y, stream=None):
        _check(_lib.cutfem_apply_operator(self._h, level % self.n_levels, _dptr(x), _dptr(y), _stream(stream)))

    def smooth(self, level, x, b, reverse=False, stream=None):
        _check(_lib.cutfem_smooth(self._h, level % self.n_levels, _dptr(x), _dptr(b), int(reverse), _stream(stream)))

    def colour_step(self, level, kind, colour, x, b, stream=None):
        _check(_lib.cutfem_colour_step(self._h, level % self.n_levels, kind, colour, _dptr(x), _dptr(b),
                                       _stream(stream)))

    def vcycle(self, x, b, stream=None):
        _check(_lib.cutfem_vcycle(self._h, _dptr(x), _dptr(b), _stream(stream)))

    def solve_cg_mg(self, x, b, tol=1e-8, max_it=500, stream=None):
        it = ctypes.c_int(0)
        rel = ctypes.c_double(0.0)
        _check(_lib.cutfem_solve_cg_mg(self._h, _dptr(x), _dptr(b), tol, max_it, ctypes.byref(it),
                                       ctypes.byref(rel), _stream(stream)))
        return it.value, rel.value

    def smooth_host(self, level, x_np, b_np, reverse=False, stream=None):
        """x_np, b_np: C-contiguous float64 numpy arrays of NL*LD entries."""
        _check(_lib.cutfem_smooth_host(self._h, level % self.n_levels, x_np.ctypes.data_as(_D),
                                       b_np.ctypes.data_as(_D), int(reverse), _stream(stream)))

    def solve_cg_mg_host(self, x_np, b_np, tol=1e-8, max_it=500, stream=None):
        it = ctypes.c_int(0)
        rel = ctypes.c_double(0.0)
        _check(_lib.cutfem_solve_cg_mg_host(self._h, x_np.ctypes.data_as(_D), b_np.ctypes.data_as(_D), tol,
                                            max_it, ctypes.byref(it), ctypes.byref(rel), _stream(stream)))
        return it.value, rel.value

    def prolongate_add(self, level, x_coarse, x_fine, stream=None):
        _check(_lib.cutfem_prolongate_add(self._h, level, _dptr(x_coarse), _dptr(x_fine), _stream(stream)))

    def restrict(self, level, r_fine, b_coarse, stream=None):
        _check(_lib.cutfem_restrict(self._h, level, _dptr(r_fine), _dptr(b_coarse), _stream(stream)))

    # --- exports (host)
    def cell_types(self, level=-1):
        i = self.level_info(level)
        out = np.zeros(i.n ** i.dim, dtype=np.int8)
        _check(_lib.cutfem_export_cell_types(self._h, level % self.n_levels, out.ctypes.data_as(_D)))
        return out.reshape((i.n,) * i.dim)

    def dof_mask(self, level=-1):
        i = self.level_info(level)
        out = np.zeros(i.nl ** i.dim, dtype=np.uint8)
        _check(_lib.cutfem_export_dof_mask(self._h, level % self.n_levels, out.ctypes.data_as(_D)))
        return out.reshape((i.nl,) * i.dim).astype(bool)

    def patches(self, level, kind, colour):
        level = level % self.n_levels
        cnt = ctypes.c_int(0)
        _check(_lib.cutfem_export_patches(self._h, level, kind, colour, None, ctypes.byref(cnt)))
        out = np.zeros(max(cnt.value, 1), dtype=np.int32)
        _check(_lib.cutfem_export_patches(self._h, level, kind, colour, out.ctypes.data_as(_D), ctypes.byref(cnt)))
        return out[:cnt.value]

    def cut_interior(self, level=-1):
        level = level % self.n_levels
        npat = ctypes.c_int(0)
        nent = ctypes.c_int64(0)
        _check(_lib.cutfem_export_cut_interior(self._h, level, None, None, ctypes.byref(npat), ctypes.byref(nent)))
        off = np.zeros(npat.value + 1, dtype=np.int64)
        nodes = np.zeros(max(nent.value, 1), dtype=np.int32)
        _check(_lib.cutfem_export_cut_interior(self._h, level, off.ctypes.data_as(_D), nodes.ctypes.data_as(_D),
                                               ctypes.byref(npat), ctypes.byref(nent)))
        return off, nodes[:nent.value]
