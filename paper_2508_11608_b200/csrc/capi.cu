// capi.cu — extern "C" boundary of libcutfem_mg.so (include/cutfem_mg.h).
// Argument validation, exception -> status-code translation, host-pointer
// variants.  Single translation unit: includes the kernels and the host
// orchestration.
#include "../../include/cutfem_mg.h"
#include "problem.cuh"

struct cutfem_problem_s {
  cf::Problem p;
};

struct cutfem_comm_s {
  cf::Comm* c;
};

static thread_local std::string g_err;

template <class F>
static int guarded(F&& f) {
  try {
    f();
    return CUTFEM_OK;
  } catch (const cf::Error& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return CUTFEM_ERR_STATE;
  }
}

static void check_level(cutfem_problem pb, int level) {
  cf::require(pb != nullptr, cf::ERR_ARG, "null problem handle");
  cf::require(!pb->p.broken, cf::ERR_STATE, "a failed cutfem_partition left this problem unusable; destroy it");
  cf::require(level >= 0 && level < (int)pb->p.lv.size(), cf::ERR_ARG, "level out of range");
}
static void check_built(cutfem_problem pb) {
  cf::require(pb != nullptr, cf::ERR_ARG, "null problem handle");
  cf::require(pb->p.built, cf::ERR_STATE, "cutfem_build_patches has not been called");
  cf::require(!pb->p.broken, cf::ERR_STATE, "a failed cutfem_partition left this problem unusable; destroy it");
}
static void use_stream(cutfem_problem pb, void* stream) { pb->p.st = (cudaStream_t)stream; }

extern "C" {

const char* cutfem_last_error(void) { return g_err.c_str(); }
int64_t cutfem_launch_count(void) { return cf::g_launches; }

#ifdef CF_TIMING
// debug builds only: copy the per-block phase timestamps of the last instrumented launch
int cutfem_debug_timers(unsigned long long* host, int nblocks) {
  return cudaMemcpyFromSymbol(host, g_dbg, sizeof(unsigned long long) * 8 * nblocks) == cudaSuccess ? 0 : -1;
}
#endif

int cutfem_setup_mesh(const cutfem_params* prm, void* stream, cutfem_problem* out) {
  return guarded([&]() {
    cf::require(prm != nullptr && out != nullptr, cf::ERR_ARG, "null argument");
    cf::require(prm->degree >= 1 && prm->degree <= CF_MAXP, cf::ERR_ARG, "degree must be 1..4");
    cf::require(prm->dim == 0 || prm->dim == 2 || prm->dim == 3, cf::ERR_ARG, "dim must be 2 or 3");
    cf::require(prm->dim != 3 || prm->degree <= 3, cf::ERR_ARG, "3D supports degree 1..3");
    cf::require(prm->n_coarse >= 1 && prm->n_levels >= 1 && prm->n_levels <= 16, cf::ERR_ARG, "bad level counts");
    cf::require(((int64_t)prm->n_coarse << (prm->n_levels - 1)) * prm->degree < 60000, cf::ERR_SIZE,
                "finest lattice too large");
    cf::require(prm->domain == 0 || prm->domain == 1, cf::ERR_ARG, "domain must be 0 (level set) or 1 (fitted box)");
    cf::require(prm->length > 0 && (prm->domain == 1 || prm->r > 0), cf::ERR_ARG,
                "box length and radius must be positive");
    cf::require(prm->n_q >= 0 && prm->n_q <= CF_MAXNQ, cf::ERR_ARG, "n_q must be 0..12");
    cf::require(prm->n_c >= 1, cf::ERR_ARG, "n_c must be >= 1");
    *out = nullptr;
    auto* pb = new cutfem_problem_s();
    cf::Params& P = pb->p.prm;
    P.dim = prm->dim == 3 ? 3 : 2;
    P.x0 = prm->x0;
    P.y0 = prm->y0;
    P.z0 = prm->z0;
    P.cz = prm->cz;
    P.length = prm->length;
    P.cx = prm->cx;
    P.cy = prm->cy;
    P.r = prm->r;
    P.n_coarse = prm->n_coarse;
    P.n_levels = prm->n_levels;
    P.p = prm->degree;
    P.gamma_D = prm->gamma_D > 0 ? prm->gamma_D : 5.0 * P.p * (P.p + 1);
    for (int k = 0; k < CF_MAXP; ++k) P.gamma_k[k] = prm->gamma_k[k] >= 0 ? prm->gamma_k[k] : 0.1;
    P.sigma = prm->sigma;
    P.n_q = prm->n_q > 0 ? prm->n_q : P.p + 1;
    P.n_c = prm->n_c;
    P.symmetric = prm->symmetric;
    cf::require(prm->cut_mode == 0 || prm->cut_mode == 1, cf::ERR_ARG, "cut_mode must be 0 or 1");
    P.cut_mode = prm->cut_mode;
    P.domain = prm->domain;
    use_stream(pb, stream);
    try {
      pb->p.setup_mesh();
    } catch (...) {
      delete pb;
      throw;
    }
    *out = pb;
  });
}

int cutfem_build_patches(cutfem_problem pb, void* stream) {
  return guarded([&]() {
    cf::require(pb != nullptr, cf::ERR_ARG, "null problem handle");
    cf::require(!pb->p.built, cf::ERR_STATE, "patches already built");
    use_stream(pb, stream);
    pb->p.build_patches();
  });
}

int cutfem_destroy(cutfem_problem pb) {
  return guarded([&]() { delete pb; });
}

int cutfem_level_info_get(cutfem_problem pb, int level, cutfem_level_info* out) {
  return guarded([&]() {
    check_level(pb, level);
    cf::require(out != nullptr, cf::ERR_ARG, "null output");
    const cf::LevelData& D = pb->p.lv[level];
    out->n = D.a.n;
    out->nl = D.a.nl;
    out->ld = D.a.ld;
    out->n_dofs = D.n_dofs;
    out->n_inside = D.n_inside;
    out->n_cut = D.a.n_cut;
    out->n_ghost_faces = D.a.n_ghost;
    out->dim = pb->p.prm.dim;
    for (int c = 0; c < 8; ++c) {
      out->n_cart[c] = D.n_cart[c];
      out->n_cutp[c] = D.n_cutp[c];
    }
    for (int c = 0; c < 8; ++c) out->cut_step_bytes[c] = D.gmap ? D.cut_bytes[c] : 0;
    for (int c = 0; c < 8; ++c) out->cut_method_bytes[c] = D.cut_method_bytes[c];
    if (pb->p.prm.dim == 2) pb->p.build_spans(const_cast<cf::LevelData&>(D));
    out->host_span_doubles = D.span_doubles;
    for (int d = 0; d < 2; ++d) {
      out->sweep_ctas[d] = D.sw[d].ok ? D.sw[d].ncta : 0;
      out->sweep_redundancy[d] = D.sw[d].ok ? D.sw[d].redundancy : 0.0;
      out->sweep_map_bytes[d] = D.sw[d].ok ? D.sw[d].map_bytes_total : 0;
    }
    out->n_vol_qp = D.n_vq;
    out->n_surf_qp = D.n_sq;
    out->h = D.a.h;
  });
}

int cutfem_apply_operator(cutfem_problem pb, int level, const double* x, double* y, void* stream) {
  return guarded([&]() {
    check_level(pb, level);
    cf::require(x && y && x != y, cf::ERR_ARG, "x, y must be distinct non-null device pointers");
    use_stream(pb, stream);
    pb->p.apply_entry(level, x, y);
  });
}

int cutfem_smooth(cutfem_problem pb, int level, double* x, const double* b, int reverse, void* stream) {
  return guarded([&]() {
    check_built(pb);
    check_level(pb, level);
    cf::require(x && b && (const double*)x != b, cf::ERR_ARG, "x, b must be distinct non-null device pointers");
    use_stream(pb, stream);
    pb->p.graphed(1, x, b, level * 2 + (reverse ? 1 : 0), [&]() {
      pb->p.zero_boundary(level, x);
      pb->p.smooth(level, x, b, reverse);
    });
  });
}

int cutfem_colour_step(cutfem_problem pb, int level, int kind, int colour, double* x, const double* b, void* stream) {
  return guarded([&]() {
    check_built(pb);
    check_level(pb, level);
    cf::require(kind >= 0 && kind <= 3 && colour >= 0 && colour < 8, cf::ERR_ARG, "bad kind/colour");
    cf::require(!pb->p.lv[level].part || (pb->p.prm.dim == 2 && kind >= 2), cf::ERR_STATE,
                "a partitioned level only exposes the whole sweeps (kind 2, 3)");
    cf::require(x && b && (const double*)x != b, cf::ERR_ARG, "x, b must be distinct non-null device pointers");
    use_stream(pb, stream);
    pb->p.zero_boundary(level, x);
    if (pb->p.prm.dim == 3) {
      cf::require(kind <= 1 && colour < 8, cf::ERR_ARG, "3D colour step: kind 0/1, colour 0..7");
      if (kind == 0) pb->p.cart_step3(level, colour, x, b);
      else pb->p.cut_step3(level, colour, x, b);
    } else if (kind == 3) {
      cf::require(pb->p.pingpong, cf::ERR_STATE, "kind 3 needs the ping-pong cut sweeps");
      pb->p.cut_sweeps(level, x, b, colour & 1);
    } else if (kind == 0) pb->p.cart_step(level, colour, x, b);
    else if (kind == 1 && pb->p.pingpong) {
      cf::require(colour < 4, cf::ERR_ARG, "2D colours are 0..3");
      cf::LevelData& D = pb->p.lv[level];
      CF_CUDA(cudaMemcpyAsync(D.xs, x, (size_t)pb->p.vsize(level) * sizeof(double), cudaMemcpyDeviceToDevice, pb->p.st));
      pb->p.cut_pp_step(level, colour, -1, D.xs, x, b);
    } else if (kind == 1) pb->p.cut_step(level, colour, x, b);
    else pb->p.cart_fused(level, x, b, colour & 1);
  });
}

int cutfem_comm_local_create(int world, cutfem_comm* out) {
  return guarded([&]() {
    cf::require(world >= 1 && out != nullptr, cf::ERR_ARG, "world must be >= 1, out non-null");
    auto* hub = new cf::LocalHub(world);
    for (int r = 0; r < world; ++r) out[r] = new cutfem_comm_s{new cf::LocalComm(hub, r)};
  });
}

int cutfem_comm_nccl_unique_id(unsigned char* id_out) {
  return guarded([&]() {
    cf::require(id_out != nullptr, cf::ERR_ARG, "null output");
    static_assert(sizeof(ncclUniqueId) == CUTFEM_NCCL_ID_BYTES, "ncclUniqueId size");
    ncclUniqueId id;
    CF_NCCL(cf::nccl_api().GetUniqueId(&id));
    std::memcpy(id_out, &id, sizeof(id));
  });
}

int cutfem_comm_nccl_create(const unsigned char* id, int rank, int world, cutfem_comm* out) {
  return guarded([&]() {
    cf::require(id != nullptr && out != nullptr, cf::ERR_ARG, "null argument");
    cf::require(world >= 1 && rank >= 0 && rank < world, cf::ERR_ARG, "bad rank / world");
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    *out = new cutfem_comm_s{new cf::NcclComm(uid, rank, world)};
  });
}

int cutfem_comm_destroy(cutfem_comm comm) {
  return guarded([&]() {
    if (!comm) return;
    delete comm->c;
    delete comm;
  });
}

int cutfem_partition(cutfem_problem pb, cutfem_comm comm) {
  return guarded([&]() {
    check_built(pb);
    cf::require(comm != nullptr && comm->c != nullptr, cf::ERR_ARG, "null or already attached comm");
    try {
      pb->p.partition(comm->c);
    } catch (...) {
      // some levels may already hold rank-restricted work lists: refuse further use
      if (pb->p.comm == nullptr) pb->p.broken = true;
      throw;
    }
    comm->c = nullptr;   // owned by the problem now
    delete comm;
  });
}

int cutfem_partition_info(cutfem_problem pb, int level, int* out) {
  return guarded([&]() {
    check_level(pb, level);
    cf::require(out != nullptr, cf::ERR_ARG, "null output");
    const cf::LevelData& D = pb->p.lv[level];
    const int nl = D.a.nl;
    out[0] = D.part;
    out[1] = D.part ? D.r0 : 0;
    out[2] = D.part ? D.r1 : nl;
    out[3] = D.part ? D.v0 : 0;
    out[4] = D.part ? D.v1 : nl;
    out[5] = pb->p.comm ? pb->p.comm->rank : 0;
    out[6] = pb->p.comm ? pb->p.comm->world : 1;
    out[7] = D.part ? D.hw : 0;
  });
}

int cutfem_slab_plan(int n_cells, int degree, int world, int rank, int halo_cells, int64_t* out) {
  return guarded([&]() {
    cf::require(out != nullptr, cf::ERR_ARG, "null output");
    cf::require(n_cells >= 1 && degree >= 1 && world >= 1 && rank >= 0 && rank < world && halo_cells >= 0, cf::ERR_ARG,
                "bad slab plan arguments");
    cf::require(n_cells % world == 0 && n_cells / world >= halo_cells + 1, cf::ERR_ARG,
                "slabs must be whole and thicker than the halo");
    const cf::SlabPlan s = cf::slab_plan(n_cells, degree, world, rank, halo_cells, 1);
    const int64_t head[7] = {s.c0, s.c1, s.r0, s.r1, s.v0, s.v1, (int64_t)s.xf.size()};
    for (int i = 0; i < 7; ++i) out[i] = head[i];
    for (int i = 0; i < 2; ++i) {
      const bool has = i < (int)s.xf.size();
      out[7 + 5 * i + 0] = has ? s.xf[i].peer : -1;
      out[7 + 5 * i + 1] = has ? s.xf[i].send_off : 0;
      out[7 + 5 * i + 2] = has ? s.xf[i].send_n : 0;
      out[7 + 5 * i + 3] = has ? s.xf[i].recv_off : 0;
      out[7 + 5 * i + 4] = has ? s.xf[i].recv_n : 0;
    }
  });
}

int cutfem_sweep_plan(int n, int p, int ld, int S, int reverse, int nsm, int force_ng, int npatch, const int* ijc,
                      const int* in_off, const int* in_nodes, const int* ex_off, const int* ex_nodes, double ca,
                      double cb, int* ncta, int* own_off, int* own_nodes, int own_cap, int* task_off, int* task_patch,
                      int task_cap) {
  return guarded([&]() {
    cf::require(n >= 1 && p >= 1 && p <= 3 && ld >= n * p + 1 && S >= 4 && S % 4 == 0 && nsm >= 1 && npatch >= 0,
                cf::ERR_ARG, "bad sweep plan arguments");
    cf::require(ijc && in_off && ex_off && ncta && own_off && own_nodes && task_off && task_patch, cf::ERR_ARG,
                "null argument");
    std::vector<cf::host::SweepPatch> P(npatch);
    long long blk = 0;
    for (int k = 0; k < npatch; ++k) {
      cf::host::SweepPatch& q = P[k];
      q.I = ijc[3 * k];
      q.J = ijc[3 * k + 1];
      q.colour = ijc[3 * k + 2];
      q.in.assign(in_nodes + in_off[k], in_nodes + in_off[k + 1]);
      q.ex.assign(ex_nodes + ex_off[k], ex_nodes + ex_off[k + 1]);
      cf::require(!q.in.empty(), cf::ERR_ARG, "a patch without interior nodes");
      // map blocks laid out consecutively (the planner only needs their sizes)
      q.blk0 = blk;
      q.rows = blk + cf::map_hdr_d((int)q.ex.size());
      q.blk1 = q.rows + cf::map_rows_d((int)q.in.size(), (int)(q.in.size() + q.ex.size()), 0);
      blk = q.blk1;
    }
    cf::host::SweepPlan plan;
    const cf::host::SweepProgram R = cf::host::build_sweep(P, n, p, ld, S, reverse, nsm, 232448, force_ng, false, ca, cb,
                                                          -1, -1, 0, &plan);
    cf::require(plan.ng > 0, cf::ERR_ARG, "no plan: " + R.why);
    *ncta = plan.ng;
    int no = 0, nt = 0;
    own_off[0] = 0;
    task_off[0] = 0;
    for (int g = 0; g < plan.ng; ++g) {
      for (int nd : plan.owned[g]) {
        cf::require(no < own_cap, cf::ERR_SIZE, "own_cap too small");
        own_nodes[no++] = nd;
      }
      own_off[g + 1] = no;
      for (int s2 = 0; s2 < S; ++s2) {
        for (int k : plan.cones[g][s2]) {
          cf::require(nt < task_cap, cf::ERR_SIZE, "task_cap too small");
          task_patch[nt++] = k;
        }
        task_off[g * S + s2 + 1] = nt;
      }
    }
  });
}

int cutfem_halo_exchange(cutfem_problem pb, int level, double* v, void* stream) {
  return guarded([&]() {
    check_level(pb, level);
    cf::require(v != nullptr, cf::ERR_ARG, "null vector");
    use_stream(pb, stream);
    pb->p.halo(level, v);
  });
}

int cutfem_vcycle(cutfem_problem pb, double* x, const double* b, void* stream) {
  return guarded([&]() {
    check_built(pb);
    cf::require(x && b && (const double*)x != b, cf::ERR_ARG, "x, b must be distinct non-null device pointers");
    use_stream(pb, stream);
    const int L = pb->p.prm.n_levels - 1;
    pb->p.graphed(2, x, b, 0, [&]() {
      pb->p.zero_boundary(L, x);
      pb->p.vcycle(L, x, b);
    });
  });
}

int cutfem_solve_cg_mg(cutfem_problem pb, double* x, const double* b, double tol, int max_it, int* iters,
                       double* rel_res, void* stream) {
  return guarded([&]() {
    check_built(pb);
    cf::require(x && b, cf::ERR_ARG, "null vector");
    cf::require(tol >= 0 && max_it >= 0, cf::ERR_ARG, "tol and max_it must be non-negative");
    use_stream(pb, stream);
    pb->p.solve_cg(x, b, tol, max_it, iters, rel_res);
  });
}

static void host_buffers(cutfem_problem pb) {
  if (!pb->p.hx) {
    const int64_t nv = pb->p.vsize(pb->p.prm.n_levels - 1);
    pb->p.hx = pb->p.alloc<double>(nv);
    pb->p.hb = pb->p.alloc<double>(nv);
  }
}

// host memory the device can address directly (pinned, mapped: cudaHostAlloc /
// cudaHostRegister under unified addressing): its device pointer, else null
static const double* mapped(const void* h) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, h) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return a.type == cudaMemoryTypeHost && a.devicePointer ? (const double*)a.devicePointer : nullptr;
}

int cutfem_smooth_host(cutfem_problem pb, int level, double* x_host, const double* b_host, int reverse,
                       void* stream) {
  return guarded([&]() {
    check_built(pb);
    check_level(pb, level);
    cf::require(x_host && b_host, cf::ERR_ARG, "null vector");
    use_stream(pb, stream);
    host_buffers(pb);
    const size_t bytes = (size_t)pb->p.vsize(level) * sizeof(double);
    const double *mx = mapped(x_host), *mb = mapped(b_host);
    if (mx && mb && pb->p.prm.dim == 2 && pb->p.prm.domain == 0) {
      // pinned host vectors: only the DoF span of every row crosses PCIe (the
      // library ignores non-DoF entries on input and leaves them unchanged)
      pb->p.copy_spans(level, mx, pb->p.hx, mb, pb->p.hb);
      double* dx = pb->p.hx;
      const double* db = pb->p.hb;
      pb->p.graphed(1, dx, db, level * 2 + (reverse ? 1 : 0), [&]() { pb->p.smooth(level, dx, db, reverse); });
      pb->p.copy_spans(level, pb->p.hx, (double*)mx);
      pb->p.sync();
      return;
    }
    CF_CUDA(cudaMemcpyAsync(pb->p.hx, x_host, bytes, cudaMemcpyHostToDevice, pb->p.st));
    CF_CUDA(cudaMemcpyAsync(pb->p.hb, b_host, bytes, cudaMemcpyHostToDevice, pb->p.st));
    double* dx = pb->p.hx;
    const double* db = pb->p.hb;
    pb->p.graphed(1, dx, db, level * 2 + (reverse ? 1 : 0), [&]() {
      pb->p.zero_boundary(level, dx);
      pb->p.smooth(level, dx, db, reverse);
    });
    CF_CUDA(cudaMemcpyAsync(x_host, pb->p.hx, bytes, cudaMemcpyDeviceToHost, pb->p.st));
    pb->p.sync();
  });
}

int cutfem_solve_cg_mg_host(cutfem_problem pb, double* x_host, const double* b_host, double tol, int max_it,
                            int* iters, double* rel_res, void* stream) {
  return guarded([&]() {
    check_built(pb);
    cf::require(x_host && b_host, cf::ERR_ARG, "null vector");
    use_stream(pb, stream);
    host_buffers(pb);
    const size_t bytes = (size_t)pb->p.vsize(pb->p.prm.n_levels - 1) * sizeof(double);
    CF_CUDA(cudaMemcpyAsync(pb->p.hb, b_host, bytes, cudaMemcpyHostToDevice, pb->p.st));
    pb->p.solve_cg(pb->p.hx, pb->p.hb, tol, max_it, iters, rel_res);
    CF_CUDA(cudaMemcpyAsync(x_host, pb->p.hx, bytes, cudaMemcpyDeviceToHost, pb->p.st));
    pb->p.sync();
  });
}

int cutfem_prolongate_add(cutfem_problem pb, int level, const double* x_coarse, double* x_fine, void* stream) {
  return guarded([&]() {
    check_level(pb, level);
    cf::require(level >= 1, cf::ERR_ARG, "level must be >= 1");
    cf::require(x_coarse && x_fine, cf::ERR_ARG, "null vector");
    use_stream(pb, stream);
    pb->p.prolongate_add(level, x_coarse, x_fine);
  });
}

int cutfem_restrict(cutfem_problem pb, int level, const double* r_fine, double* b_coarse, void* stream) {
  return guarded([&]() {
    check_level(pb, level);
    cf::require(level >= 1, cf::ERR_ARG, "level must be >= 1");
    cf::require(r_fine && b_coarse, cf::ERR_ARG, "null vector");
    use_stream(pb, stream);
    pb->p.restrict_(level, r_fine, b_coarse);
  });
}

int cutfem_export_cell_types(cutfem_problem pb, int level, int8_t* host_out) {
  return guarded([&]() {
    check_level(pb, level);
    cf::require(host_out != nullptr, cf::ERR_ARG, "null output");
    const cf::LevelData& D = pb->p.lv[level];
    const size_t nc = (size_t)D.a.n * D.a.n * (pb->p.prm.dim == 3 ? D.a.n : 1);
    CF_CUDA(cudaMemcpy(host_out, D.ctype, nc, cudaMemcpyDeviceToHost));
  });
}

int cutfem_export_dof_mask(cutfem_problem pb, int level, uint8_t* host_out) {
  return guarded([&]() {
    check_level(pb, level);
    cf::require(host_out != nullptr, cf::ERR_ARG, "null output");
    const cf::LevelArgs& L = pb->p.lv[level].a;
    const int rows = L.nl * (pb->p.prm.dim == 3 ? L.nl : 1);
    CF_CUDA(cudaMemcpy2D(host_out, L.nl, pb->p.lv[level].mask, L.ld, L.nl, rows, cudaMemcpyDeviceToHost));
  });
}

int cutfem_export_patches(cutfem_problem pb, int level, int kind, int colour, int32_t* host_out, int* count) {
  return guarded([&]() {
    check_built(pb);
    check_level(pb, level);
    cf::require((kind == 0 || kind == 1) && colour >= 0 && colour < (pb->p.prm.dim == 3 ? 8 : 4) && count, cf::ERR_ARG,
                "bad kind/colour");
    const cf::LevelData& D = pb->p.lv[level];
    const int* off = kind == 0 ? D.cart_off : D.cutp_off;
    const int* list = kind == 0 ? D.cart_list : D.cutp_list;
    *count = off[colour + 1] - off[colour];
    if (host_out && *count)
      CF_CUDA(cudaMemcpy(host_out, list + off[colour], sizeof(int) * (*count), cudaMemcpyDeviceToHost));
  });
}

int cutfem_export_cut_interior(cutfem_problem pb, int level, int64_t* host_offsets, int32_t* host_nodes,
                               int* n_patches, int64_t* n_entries) {
  return guarded([&]() {
    check_built(pb);
    check_level(pb, level);
    const cf::LevelData& D = pb->p.lv[level];
    const int ncp = D.cutp_off[pb->p.prm.dim == 3 ? 8 : 4];
    if (n_patches) *n_patches = ncp;
    if (n_entries) *n_entries = D.n_ent;
    if (host_offsets) CF_CUDA(cudaMemcpy(host_offsets, D.cutp_ent, sizeof(int64_t) * (ncp + 1), cudaMemcpyDeviceToHost));
    if (host_nodes && D.n_ent) {
      std::vector<int32_t> tmp(D.n_ent);
      CF_CUDA(cudaMemcpy(tmp.data(), D.ent_node, sizeof(int32_t) * D.n_ent, cudaMemcpyDeviceToHost));
      for (int64_t e = 0; e < D.n_ent; ++e) {
        int b = tmp[e] / D.a.ld, a = tmp[e] % D.a.ld;   // b = row (c nl + b in 3D)
        host_nodes[e] = b * D.a.nl + a;
      }
    }
  });
}

}  // extern "C"
