// problem.cuh — host orchestration: setup of the hierarchy (P l.65-69),
// patches (P l.141-179), V-cycle (P l.124), CG; CUDA-graph caching of the
// launch sequences.  Every arithmetic step runs in the kernels of
// kernels.cuh / setup.cuh; the host only sequences launches.
#pragma once
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>
#include <vector>

#include "internal.cuh"
#include "kernels.cuh"
#include "smoother2.cuh"
#include "dim3.cuh"
#include "tables.cuh"
#include "comm.cuh"
#include "sweep.cuh"

namespace cf {

int64_t g_launches = 0;

#define CF_DISPATCH(p, ...)                               \
  switch (p) {                                            \
    case 1: { constexpr int P = 1; __VA_ARGS__; } break;  \
    case 2: { constexpr int P = 2; __VA_ARGS__; } break;  \
    case 3: { constexpr int P = 3; __VA_ARGS__; } break;  \
    case 4: { constexpr int P = 4; __VA_ARGS__; } break;  \
    default: throw Error(ERR_ARG, "degree must be 1..4"); \
  }

#define CF_DISPATCH3(p, ...)                              \
  switch (p) {                                            \
    case 1: { constexpr int P = 1; __VA_ARGS__; } break;  \
    case 2: { constexpr int P = 2; __VA_ARGS__; } break;  \
    case 3: { constexpr int P = 3; __VA_ARGS__; } break;  \
    default: throw Error(ERR_ARG, "3D supports degree 1..3"); \
  }

template <int P> constexpr int cart_tp() { return P == 1 ? 16 : (P == 2 ? 8 : (P == 3 ? 7 : 6)); }
constexpr int CUT_WPB = 4;
#ifndef CF_CART_NT32
#define CF_CART_NT32 256   // threads of the fused Cartesian CTA with 32-cell tiles (512 measured slower)
#endif
// fused Cartesian tile (cells per side); p = 2 uses 32-cell tiles on large
// levels of the TMA/tensor-core sweep (Problem::tc_big_n) and 16 otherwise
template <int P> constexpr int fused_tc() { return P == 1 ? 32 : (P <= 3 ? 16 : 8); }

struct GraphRec {
  cudaGraphExec_t exec = nullptr;
  int64_t launches = 0;
};

struct Problem {
  Params prm;
  std::vector<LevelData> lv;
  cudaStream_t st = nullptr;
  cudaStream_t cap_st = nullptr;
  bool built = false;
  bool broken = false;      // a partition failed half-way (capi refuses further hot-path calls)
  bool fused = true;        // fused Cartesian colours (env CUTFEM_FUSED=0 disables)
  bool use_mma = true;      // Cartesian patch map on fp64 tensor cores (env CUTFEM_MMA=0 disables)
  bool pingpong = true;     // cut steps without a scatter kernel (env CUTFEM_PINGPONG=0 disables)
  bool use_tma = true;      // TMA tile loads in the fused Cartesian sweep (env CUTFEM_TMA=0 disables)
  bool cta_cut = true;      // CTA of 64 threads per cut patch (env CUTFEM_CTACUT=0: one warp per patch)
  int cut3_v = 3;           // 3D cut-patch kernel version (env CUTFEM_CUT3=2: lane-parallel jump array)
  bool tile_apply = true;   // TMA-tiled operator (env CUTFEM_TILEAPPLY=0: node-centric global gather)
  bool cart_split = false;  // force the two-launch Cartesian sweep through xs (env CUTFEM_CART_SPLIT=1)
  bool wide_halo = true;    // partition: wide-halo cut sweeps where the slabs are thick enough (env CUTFEM_WIDE_HALO=0)
  bool cut_map = true;      // cut steps through the precomputed dense patch maps, p <= 3 (env CUTFEM_CUTMAP=0)
  int tc_big_n = 512;       // levels with n >= this use 32-cell fused tiles for p = 2 (env CUTFEM_TC32_MIN_N)
  int tc_small_n = 128;     // Q2 levels with 16 <= n <= this use 8 x 8-cell fused tiles (env CUTFEM_TC8_MAX_N; V-cycle 658 -> 640 us)
  int tile_apply_min_tiles = 148;   // TMA-tiled operator on levels with >= this many 16x16 tiles (env CUTFEM_TILEAPPLY_MIN)
  int tcx_big = 24;         // ... TCX x 32 cells, TCX in {16, 24, 32} (env CUTFEM_TCX; 24: 18.5 us vs 21.5 us for 32 x 32 at config1)
  bool verbose = false;     // launch decisions on stderr (env CUTFEM_VERBOSE=1)
  bool sym_packed = false;  // 3D: always pack the local inverses symmetric (env CUTFEM_SYM_PACKED=1)
  bool one_sweep = true;    // 2D cut sweeps in one launch (k_cut_sweep; env CUTFEM_SWEEP=0: one launch per step)
  int sweep_ng = 0;         // force the CTA count of k_cut_sweep (env CUTFEM_SWEEP_NG)
  // slab partition: comm != nullptr after partition()
  Comm* comm = nullptr;
  static constexpr int HALO = 4;   // halo width in cells (the fused Cartesian apron)
  // coarse
  int n0 = 0;
  int* c_nodes = nullptr;
  double* c_inv = nullptr;
  // CG
  double *cg_x = nullptr, *cg_r = nullptr, *cg_z = nullptr, *cg_p = nullptr, *cg_q = nullptr;
  double *part = nullptr, *sc = nullptr, *sc_host = nullptr;
  // host-pointer entry points
  double *hx = nullptr, *hb = nullptr;
  // scratch
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  int* d_count = nullptr;
  std::vector<void*> allocs;
  std::map<std::tuple<int, const void*, const void*, int>, GraphRec> graphs;

  ~Problem() {
    delete comm;
    for (auto& g : graphs)
      if (g.second.exec) cudaGraphExecDestroy(g.second.exec);
    for (void* p : allocs) cudaFree(p);
    if (sc_host) cudaFreeHost(sc_host);
    if (cap_st) cudaStreamDestroy(cap_st);
  }

  template <class T>
  T* alloc(int64_t n) {
    void* p = nullptr;
    if (n <= 0) n = 1;
    CF_CUDA(cudaMalloc(&p, (size_t)n * sizeof(T)));
    allocs.push_back(p);
    return (T*)p;
  }
  void* scratch(size_t bytes) {
    if (bytes > tmp_bytes) {
      if (tmp) cudaFree(tmp);
      tmp = nullptr;
      CF_CUDA(cudaMalloc(&tmp, bytes));
      tmp_bytes = bytes;
    }
    return tmp;
  }
  void sync() { CF_CUDA(cudaStreamSynchronize(st)); }

  int read_count() {
    int h = 0;
    CF_CUDA(cudaMemcpyAsync(&h, d_count, sizeof(int), cudaMemcpyDeviceToHost, st));
    sync();
    return h;
  }

  // indices i in [0, n) with flag[i] != 0, in increasing order
  int select(const uint8_t* flags, int n, int* out) {
    size_t bytes = 0;
    thrust::counting_iterator<int> it(0);
    CF_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, it, flags, out, d_count, n, st));
    CF_CUDA(cub::DeviceSelect::Flagged(scratch(bytes), bytes, it, flags, out, d_count, n, st));
    return read_count();
  }
  // exclusive scan of n ints into n+1 int64 offsets; returns the total.  The
  // ints are widened first: CUB accumulates in the input type, and sums such
  // as the local-inverse sizes (3D Q3: sum m_j^2 ~ 5e9) overflow 32 bits
  int64_t scan64(const int* in, int n, int64_t* out) {
    size_t bytes = 0;
    CF_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), st));
    if (n == 0) return 0;
    k_widen<<<ceil_div(n, 256), 256, 0, st>>>(in, n, out + 1);
    CF_LAUNCHED();
    CF_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, out + 1, out + 1, n, st));
    CF_CUDA(cub::DeviceScan::InclusiveSum(scratch(bytes), bytes, out + 1, out + 1, n, st));
    int64_t tot = 0;
    CF_CUDA(cudaMemcpyAsync(&tot, out + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    sync();
    return tot;
  }
  int64_t scan32(const int* in, int n, int* out) {
    size_t bytes = 0;
    CF_CUDA(cudaMemsetAsync(out, 0, sizeof(int), st));
    if (n == 0) return 0;
    CF_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, in, out + 1, n, st));
    CF_CUDA(cub::DeviceScan::InclusiveSum(scratch(bytes), bytes, in, out + 1, n, st));
    int tot = 0;
    CF_CUDA(cudaMemcpyAsync(&tot, out + n, sizeof(int), cudaMemcpyDeviceToHost, st));
    sync();
    return tot;
  }

  // launch with programmatic dependent launch (PDL) when enabled: the kernel
  // may start while its predecessor drains; it calls griddepcontrol.wait
  // before touching data the predecessor writes
  bool pdl = true;
  template <typename... KArgs, typename... Args>
  void launch(void (*kern)(KArgs...), dim3 g, dim3 b, size_t smem, Args... args) {
    launch_ex(false, kern, g, b, smem, args...);
  }
  // coop = cooperative launch (all CTAs co-resident; the kernel may grid-sync)
  template <typename... KArgs, typename... Args>
  void launch_ex(bool coop, void (*kern)(KArgs...), dim3 g, dim3 b, size_t smem, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = g;
    cfg.blockDim = b;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (pdl) {
      attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[na].val.programmaticStreamSerializationAllowed = 1;
      ++na;
    }
    if (coop) {
      attr[na].id = cudaLaunchAttributeCooperative;
      attr[na].val.cooperative = 1;
      ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    CF_CUDA(cudaLaunchKernelEx(&cfg, kern, ((KArgs)args)...));
  }
  int num_sms() {
    int dev = 0, nsm = 0;
    CF_CUDA(cudaGetDevice(&dev));
    CF_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    return nsm;
  }
  // CTAs of `kern` (256 threads, smem bytes) that fit on the device at once
  template <typename K>
  int coresident(K kern, size_t smem, int threads = 256) {
    int nsm = 0, dev = 0, per = 0;
    CF_CUDA(cudaGetDevice(&dev));
    CF_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    CF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, threads, smem));
    return per * nsm;
  }


  // ---------------------------------------------------------------- setup
  void setup_mesh() {
    if (const char* e = std::getenv("CUTFEM_FUSED")) fused = std::atoi(e) != 0;
    if (const char* e = std::getenv("CUTFEM_PDL")) pdl = std::atoi(e) != 0;
    if (const char* e = std::getenv("CUTFEM_MMA")) use_mma = std::atoi(e) != 0;
    if (const char* e = std::getenv("CUTFEM_PINGPONG")) pingpong = std::atoi(e) != 0;
    if (const char* e = std::getenv("CUTFEM_TMA")) use_tma = std::atoi(e) != 0;
    if (const char* e = std::getenv("CUTFEM_CTACUT")) cta_cut = std::atoi(e) != 0;
    if (const char* e = std::getenv("CUTFEM_CUT3")) cut3_v = std::atoi(e);
    if (const char* e = std::getenv("CUTFEM_TILEAPPLY")) tile_apply = std::atoi(e) != 0;
    if (const char* e = std::getenv("CUTFEM_CART_SPLIT")) cart_split = std::atoi(e) != 0;
    if (const char* e = std::getenv("CUTFEM_WIDE_HALO")) wide_halo = std::atoi(e) != 0;
    if (const char* e = std::getenv("CUTFEM_CUTMAP")) cut_map = std::atoi(e) != 0;
    if (const char* e = std::getenv("CUTFEM_VERBOSE")) verbose = std::atoi(e) != 0;
    if (const char* e = std::getenv("CUTFEM_SYM_PACKED")) sym_packed = std::atoi(e) != 0;
    if (const char* e = std::getenv("CUTFEM_SWEEP")) one_sweep = std::atoi(e) != 0;
    if (const char* e = std::getenv("CUTFEM_SWEEP_NG")) sweep_ng = std::atoi(e);
    if (const char* e = std::getenv("CUTFEM_TC32_MIN_N")) tc_big_n = std::atoi(e);
    if (const char* e = std::getenv("CUTFEM_TCX")) tcx_big = std::atoi(e);
    if (const char* e = std::getenv("CUTFEM_TILEAPPLY_MIN")) tile_apply_min_tiles = std::atoi(e);
    if (const char* e = std::getenv("CUTFEM_TC8_MAX_N")) tc_small_n = std::atoi(e);
    require(tcx_big == 16 || tcx_big == 24 || tcx_big == 32, ERR_ARG, "CUTFEM_TCX must be 16, 24 or 32");
    if (prm.dim == 3) {
      setup_mesh3();
      return;
    }
    host::upload_tables();
    host::cart_map(prm.p);  // dense Cartesian patch map (p <= 3), built outside any graph capture
    d_count = alloc<int>(1);
    const int p = prm.p;
    lv.resize(prm.n_levels);
    for (int l = 0; l < prm.n_levels; ++l) {
      LevelData& D = lv[l];
      LevelArgs& L = D.a;
      std::memset(&L, 0, sizeof(L));
      L.n = prm.n_coarse << l;
      L.p = p;
      L.fitted = prm.domain == 1;
      L.nl = L.n * p + 1;
      L.ld = (L.nl + 1) & ~1;
      L.h = prm.length / L.n;
      L.x0 = prm.x0;
      L.y0 = prm.y0;
      L.cx = prm.cx;
      L.cy = prm.cy;
      L.r = prm.r;
      L.map_one_lane = L.n >= MAP_ONE_LANE_MIN_N ? 1 : 0;
      L.gDh = prm.gamma_D / L.h;
      for (int k = 1; k <= p; ++k) {
        double f = 1.0;
        for (int q = 2; q <= k; ++q) f *= q;
        L.gs[k] = prm.gamma_k[k - 1] * std::pow(L.h, prm.sigma + 1) / (f * f);
      }
      const int n = L.n;
      dim3 b2(16, 16), gcell(ceil_div(n, 16), ceil_div(n, 16));
      D.ctype = alloc<int8_t>((int64_t)n * n);
      k_classify<<<gcell, b2, 0, st>>>(L, D.ctype);
      CF_LAUNCHED();
      L.ctype = D.ctype;
      D.mask = alloc<uint8_t>((int64_t)L.nl * L.ld);
      CF_CUDA(cudaMemsetAsync(d_count, 0, sizeof(int), st));
      k_mask<<<dim3(ceil_div(L.ld, 16), ceil_div(L.nl, 16)), b2, 0, st>>>(L, D.ctype, D.mask, d_count);
      CF_LAUNCHED();
      L.mask = D.mask;
      D.n_dofs = read_count();
      require(D.n_dofs > 0, ERR_GEOMETRY, "a level has no DoF: the domain does not meet the background box");
      if (l > 0) {
        CF_CUDA(cudaMemsetAsync(d_count, 0, sizeof(int), st));
        k_parent_check<<<gcell, b2, 0, st>>>(L, D.ctype, lv[l - 1].a.n, lv[l - 1].ctype, d_count);
        CF_LAUNCHED();
        require(read_count() == 0, ERR_GEOMETRY, "a fine active cell has an inactive parent (Omega_l not in Omega_{l-1})");
      }
      // cut cells and inside count
      uint8_t* flags = alloc<uint8_t>(2 * (int64_t)n * n);
      int* tmpi = alloc<int>(2 * (int64_t)n * n);
      k_iota_flags_cells<<<ceil_div((int64_t)n * n, 256), 256, 0, st>>>(n, D.ctype, INSIDE, flags);
      CF_LAUNCHED();
      D.n_inside = select(flags, n * n, tmpi);
      k_iota_flags_cells<<<ceil_div((int64_t)n * n, 256), 256, 0, st>>>(n, D.ctype, CUT, flags);
      CF_LAUNCHED();
      L.n_cut = select(flags, n * n, tmpi);
      D.cut_list = alloc<int>(L.n_cut);
      CF_CUDA(cudaMemcpyAsync(D.cut_list, tmpi, sizeof(int) * L.n_cut, cudaMemcpyDeviceToDevice, st));
      L.cut_list = D.cut_list;
      D.cut_id = alloc<int>((int64_t)n * n);
      k_fill<<<ceil_div((int64_t)n * n, 256), 256, 0, st>>>(D.cut_id, (int64_t)n * n, -1);
      CF_LAUNCHED();
      if (L.n_cut) {
        k_scatter_id<<<ceil_div(L.n_cut, 256), 256, 0, st>>>(D.cut_list, L.n_cut, D.cut_id);
        CF_LAUNCHED();
      }
      L.cut_id = D.cut_id;
      // ghost faces
      k_ghost_flags<<<ceil_div(2 * (int64_t)n * n, 256), 256, 0, st>>>(L, D.ctype, flags);
      CF_LAUNCHED();
      L.n_ghost = select(flags, 2 * n * n, tmpi);
      D.ghost_list = alloc<int>(L.n_ghost);
      CF_CUDA(cudaMemcpyAsync(D.ghost_list, tmpi, sizeof(int) * L.n_ghost, cudaMemcpyDeviceToDevice, st));
      L.ghost_list = D.ghost_list;
      D.gx_id = alloc<int>((int64_t)n * n);
      D.gy_id = alloc<int>((int64_t)n * n);
      k_fill<<<ceil_div((int64_t)n * n, 256), 256, 0, st>>>(D.gx_id, (int64_t)n * n, -1);
      CF_LAUNCHED();
      k_fill<<<ceil_div((int64_t)n * n, 256), 256, 0, st>>>(D.gy_id, (int64_t)n * n, -1);
      CF_LAUNCHED();
      if (L.n_ghost) {
        k_ghost_maps<<<ceil_div(L.n_ghost, 256), 256, 0, st>>>(D.ghost_list, L.n_ghost, n, D.gx_id, D.gy_id);
        CF_LAUNCHED();
      }
      L.gx_id = D.gx_id;
      L.gy_id = D.gy_id;
      D.ccode = alloc<uint8_t>((int64_t)n * n);
      k_cell_codes<<<ceil_div((int64_t)n * n, 256), 256, 0, st>>>(L, D.ccode);
      CF_LAUNCHED();
      L.ccode = D.ccode;
      // cut-cell quadrature (R6)
      D.q_off = alloc<int>(L.n_cut + 1);
      D.s_off = alloc<int>(L.n_cut + 1);
      int* vc = tmpi;
      int* scn = tmpi + n * n;
      if (L.n_cut) {
        k_cut_count<<<ceil_div(L.n_cut, 128), 128, 0, st>>>(L, prm.n_q, vc, scn);
        CF_LAUNCHED();
      }
      D.n_vq = scan32(vc, L.n_cut, D.q_off);
      D.n_sq = scan32(scn, L.n_cut, D.s_off);
      L.q_off = D.q_off;
      L.s_off = D.s_off;
      D.qbuf = alloc<double>(3 * D.n_vq);
      D.sbuf = alloc<double>(5 * D.n_sq);
      L.qx = D.qbuf;
      L.qy = D.qbuf + D.n_vq;
      L.qw = D.qbuf + 2 * D.n_vq;
      L.sx = D.sbuf;
      L.sy = D.sbuf + D.n_sq;
      L.sw = D.sbuf + 2 * D.n_sq;
      L.snx = D.sbuf + 3 * D.n_sq;
      L.sny = D.sbuf + 4 * D.n_sq;
      if (L.n_cut) {
        k_cut_fill<<<ceil_div(L.n_cut, 128), 128, 0, st>>>(L, prm.n_q, D.qbuf, D.qbuf + D.n_vq, D.qbuf + 2 * D.n_vq,
                                                           D.sbuf, D.sbuf + D.n_sq, D.sbuf + 2 * D.n_sq,
                                                           D.sbuf + 3 * D.n_sq, D.sbuf + 4 * D.n_sq);
        CF_LAUNCHED();
      }
      {
        const int NB = (p + 1) * (p + 1);
        D.ecut = alloc<double>((int64_t)L.n_cut * NB * NB);
        L.ecut = D.ecut;
        if (L.n_cut) {
          CF_DISPATCH(p, (k_cut_elem<P><<<ceil_div((int64_t)L.n_cut * NB, 4), 128, 0, st>>>(L, D.ecut)));
          CF_LAUNCHED();
        }
      }
      D.ycut = alloc<double>((int64_t)L.n_cut * (p + 1) * (p + 1));
      D.jm = alloc<double>((int64_t)L.n_ghost * p * (p + 1));
      L.ycut = D.ycut;
      L.jm = D.jm;
      const int64_t nv = (int64_t)L.nl * L.ld;
      D.x = alloc<double>(nv);
      D.b = alloc<double>(nv);
      D.r = alloc<double>(nv);
      CF_CUDA(cudaMemsetAsync(D.x, 0, nv * 8, st));
      CF_CUDA(cudaMemsetAsync(D.b, 0, nv * 8, st));
      CF_CUDA(cudaMemsetAsync(D.r, 0, nv * 8, st));
      sync();
      cudaFree(flags);
      cudaFree(tmpi);
      allocs.erase(std::remove(allocs.begin(), allocs.end(), (void*)flags), allocs.end());
      allocs.erase(std::remove(allocs.begin(), allocs.end(), (void*)tmpi), allocs.end());
    }
  }

  void build_patches() {
    if (prm.dim == 3) {
      build_patches3();
      return;
    }
    const int p = prm.p;
    for (int l = 0; l < prm.n_levels; ++l) {
      LevelData& D = lv[l];
      LevelArgs& L = D.a;
      const int n = L.n, nv = (n + 1) * (n + 1);
      D.vkind = alloc<uint8_t>(nv);
      k_vertex_kind<<<dim3(ceil_div(n + 1, 16), ceil_div(n + 1, 16)), dim3(16, 16), 0, st>>>(L, D.ctype, D.vkind);
      CF_LAUNCHED();
      uint8_t* fl = alloc<uint8_t>(nv);
      int* tmpi = alloc<int>(nv);
      for (int kind = V_CART; kind <= V_CUT; ++kind) {
        std::vector<int> all;
        int* off = kind == V_CART ? D.cart_off : D.cutp_off;
        int* cnt = kind == V_CART ? D.n_cart : D.n_cutp;
        off[0] = 0;
        std::vector<int> hostlists;
        for (int c = 0; c < 4; ++c) {
          k_vertex_flags<<<ceil_div(nv, 256), 256, 0, st>>>(n, D.vkind, (uint8_t)kind, c, fl);
          CF_LAUNCHED();
          cnt[c] = select(fl, nv, tmpi);
          std::vector<int> h(cnt[c]);
          if (cnt[c]) CF_CUDA(cudaMemcpyAsync(h.data(), tmpi, sizeof(int) * cnt[c], cudaMemcpyDeviceToHost, st));
          sync();
          hostlists.insert(hostlists.end(), h.begin(), h.end());
          off[c + 1] = off[c] + cnt[c];
        }
        int* dl = alloc<int>(hostlists.size());
        if (!hostlists.empty())
          CF_CUDA(cudaMemcpyAsync(dl, hostlists.data(), sizeof(int) * hostlists.size(), cudaMemcpyHostToDevice, st));
        (kind == V_CART ? D.cart_list : D.cutp_list) = dl;
      }
      // Cartesian tiles
      int TP = 0;
      CF_DISPATCH(p, TP = cart_tp<P>());
      std::vector<int> tiles;
      D.cart_tile_off[0] = 0;
      for (int c = 0; c < 4; ++c) {
        int cxo = c & 1, cyo = c >> 1;
        int npx = (n - cxo) / 2 + 1, npy = (n - cyo) / 2 + 1;
        int tx = ceil_div(npx, TP), ty = ceil_div(npy, TP);
        uint8_t* tf = alloc<uint8_t>((int64_t)tx * ty);
        int* ts = alloc<int>((int64_t)tx * ty);
        k_tile_flags<<<ceil_div((int64_t)tx * ty, 128), 128, 0, st>>>(n, D.vkind, c, TP, tx, ty, tf);
        CF_LAUNCHED();
        int ns = select(tf, tx * ty, ts);
        if (ns) {
          k_pack_tiles<<<ceil_div(ns, 128), 128, 0, st>>>(ts, ns, tx, ts);
          CF_LAUNCHED();
        }
        std::vector<int> h(ns);
        if (ns) CF_CUDA(cudaMemcpyAsync(h.data(), ts, sizeof(int) * ns, cudaMemcpyDeviceToHost, st));
        sync();
        tiles.insert(tiles.end(), h.begin(), h.end());
        D.n_cart_tiles[c] = ns;
        D.cart_tile_off[c + 1] = D.cart_tile_off[c] + ns;
      }
      {
        int TC = 0;
        CF_DISPATCH(p, TC = fused_tc<P>());
        int TCX = TC;
        if (p == 2 && use_mma && use_tma && n >= tc_big_n) {   // (p = 3: 32-cell tiles exceed shared memory)
          TC = 32;
          // 24 x 32 balances the single co-resident wave at 512^2; on larger
          // levels (several waves through the split sweep) 32 x 32 has less
          // apron overhead: 4096^2 sweep 662 vs 746 us
          TCX = n >= 1024 ? 32 : tcx_big;
        } else if (p == 2 && use_mma && use_tma && n <= tc_small_n && n >= 16) {
          TC = TCX = 8;   // small levels: more, smaller tiles (more CTAs in flight)
        }
        D.tc = TC;
        D.tcx = TCX;
        const int tx = ceil_div(n, TCX), ty = ceil_div(n, TC), nt = tx * ty;
        uint8_t* tf = alloc<uint8_t>(nt);
        int* ts = alloc<int>(nt);
        k_fused_tile_flags<<<ceil_div(nt, 128), 128, 0, st>>>(n, D.vkind, TCX, TC, tx, tf, nt);
        CF_LAUNCHED();
        uint8_t* tfe = alloc<uint8_t>(nt);
        k_dilate_tile_flags<<<ceil_div(nt, 128), 128, 0, st>>>(tx, ty, tf, tfe);
        CF_LAUNCHED();
        D.n_fused_tiles = select(tf, nt, ts);
        if (D.n_fused_tiles) {
          k_pack_tiles<<<ceil_div(D.n_fused_tiles, 128), 128, 0, st>>>(ts, D.n_fused_tiles, tx, ts);
          CF_LAUNCHED();
        }
        D.fused_tiles = ts;
        int* te = alloc<int>(nt);
        D.n_fused_ext = select(tfe, nt, te);
        if (D.n_fused_ext) {
          k_pack_tiles<<<ceil_div(D.n_fused_ext, 128), 128, 0, st>>>(te, D.n_fused_ext, tx, te);
          CF_LAUNCHED();
        }
        D.fused_ext = te;
        D.tflag_stride = tx + 2;
        D.tflag = alloc<unsigned>((int64_t)(tx + 2) * (ty + 2));
        if (p <= 3) {   // patch lists of every (direction, tile, pass) of the in-place TMA sweep
          const int H = 4, RWX = (TCX + 2 * H) * p + 1, RWP = (RWX + 1) & ~1;
          const int maxp = ((TCX + 7) / 2 + 1) * ((TC + 7) / 2 + 1);
          D.fpl_tx = tx;
          D.fpl_nt = nt;
          D.fpl_maxp = maxp;
          D.fpl = alloc<int>((int64_t)2 * nt * 4 * maxp);
          D.fpc = alloc<int>((int64_t)2 * nt * 4);
          k_fused_plists<<<ceil_div(2 * nt * 4, 128), 128, 0, st>>>(n, p, TC, TCX, H, RWP, maxp, D.vkind, tx, ty, D.fpl,
                                                                     D.fpc);
          CF_LAUNCHED();
        }
        reset_tile_flags(D, ty);
      }
      D.cart_tiles = alloc<int>(tiles.size());
      if (!tiles.empty())
        CF_CUDA(cudaMemcpyAsync(D.cart_tiles, tiles.data(), sizeof(int) * tiles.size(), cudaMemcpyHostToDevice, st));
      // cut patch interior sets (R3)
      const int ncp = D.cutp_off[4];
      int* mcount = alloc<int>(ncp);
      D.cutp_ent = alloc<int64_t>(ncp + 1);
      if (ncp) {
        k_cut_interior<false><<<ceil_div(ncp, 128), 128, 0, st>>>(L, D.ctype, D.cutp_list, ncp, mcount, nullptr,
                                                                   nullptr, nullptr, nullptr);
        CF_LAUNCHED();
      }
      D.n_ent = scan64(mcount, ncp, D.cutp_ent);
      for (int c = 0; c <= 4; ++c) {
        D.ent_col_off[c] = 0;
        if (ncp) CF_CUDA(cudaMemcpyAsync(&D.ent_col_off[c], D.cutp_ent + D.cutp_off[c], sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      }
      sync();
      D.ent_node = alloc<int32_t>(D.n_ent);
      D.ent_loc = alloc<uint16_t>(D.n_ent);
      D.ent_patch = alloc<int32_t>(D.n_ent);
      D.zbuf = alloc<double>(D.n_ent);
      if (ncp) {
        k_cut_interior<true><<<ceil_div(ncp, 128), 128, 0, st>>>(L, D.ctype, D.cutp_list, ncp, nullptr, D.cutp_ent,
                                                                  D.ent_node, D.ent_loc, D.ent_patch);
        CF_LAUNCHED();
      }
      // local matrices and their inverses (P l.193, R10)
      int* msq = alloc<int>(ncp);
      D.cutp_inv = alloc<int64_t>(ncp + 1);
      int mmax = 0;
      if (ncp) {
        k_square<<<ceil_div(ncp, 128), 128, 0, st>>>(mcount, ncp, msq);
        CF_LAUNCHED();
        std::vector<int> hm(ncp);
        CF_CUDA(cudaMemcpyAsync(hm.data(), mcount, sizeof(int) * ncp, cudaMemcpyDeviceToHost, st));
        sync();
        for (int v : hm) mmax = std::max(mmax, v);
      }
      D.n_inv = scan64(msq, ncp, D.cutp_inv);
      D.inv = alloc<double>(D.n_inv);
      if (D.n_ent) {
        CF_DISPATCH(p, (k_local_matrix<P, CUT_WPB><<<ceil_div(D.n_ent, CUT_WPB), 32 * CUT_WPB, 0, st>>>(
                           L, D.cutp_list, D.cutp_ent, D.ent_loc, D.ent_patch, D.n_ent, D.cutp_inv, D.inv)));
        CF_LAUNCHED();
        size_t smb = (size_t)(mmax * mmax + 2 * mmax) * sizeof(double);
        CF_CUDA(cudaFuncSetAttribute(k_batched_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(smb, 48 * 1024)));
        k_batched_inverse<<<ncp, 128, smb, st>>>(D.cutp_ent, D.cutp_inv, D.inv, ncp);
        CF_LAUNCHED();
      }
      D.desc = alloc<CutDesc>(ncp);
      if (ncp) {
        CF_DISPATCH(p, (k_cut_desc<P><<<ceil_div(ncp, 128), 128, 0, st>>>(L, D.cutp_list, ncp, D.cutp_ent, D.ent_loc,
                                                                          D.cutp_inv, (CutDesc*)D.desc)));
        CF_LAUNCHED();
      }
      if (ncp && cut_map && prm.cut_mode == 0 && p <= 3) build_cut_maps(D, ncp);
      D.act_desc = D.desc;
      for (int c = 0; c < 5; ++c) D.act_off[c] = D.cutp_off[c];
      build_copy_lists(D, D.ent_node, D.ent_col_off, (const CutDesc*)D.desc, ncp);
      if (ncp) method_bytes(D, ncp);
      if (ncp && D.gmap && one_sweep) build_sweeps(D, ncp);
      sync();
    }
    build_coarse();
    // CG workspace on the finest level
    const int64_t nvf = vsize(prm.n_levels - 1);
    cg_x = alloc<double>(nvf);
    cg_r = alloc<double>(nvf);
    cg_z = alloc<double>(nvf);
    cg_p = alloc<double>(nvf);
    cg_q = alloc<double>(nvf);
    part = alloc<double>(DOT_BLOCKS);
    sc = alloc<double>(8);
    if (!sc_host) CF_CUDA(cudaMallocHost(&sc_host, 8 * sizeof(double)));
    for (double* v : {cg_x, cg_r, cg_z, cg_p, cg_q}) CF_CUDA(cudaMemsetAsync(v, 0, nvf * 8, st));
    sync();
    built = true;
  }

  // tile counters of the in-place fused sweep (k_cart_fused_tma): 0 on the
  // tiles of D.fused_tiles, 0x7fffffff elsewhere (border and absent tiles
  // never hold a launch back); stream-ordered after every launch so far
  void reset_tile_flags(LevelData& D, int ty) {
    const int stride = D.tflag_stride;
    std::vector<unsigned> h((size_t)stride * (ty + 2), 0x7fffffffu);
    std::vector<int> t(D.n_fused_tiles);
    if (D.n_fused_tiles) CF_CUDA(cudaMemcpyAsync(t.data(), D.fused_tiles, sizeof(int) * D.n_fused_tiles,
                                                 cudaMemcpyDeviceToHost, st));
    sync();
    for (int v : t) h[(size_t)((v >> 16) + 1) * stride + (v & 0xffff) + 1] = 0u;
    CF_CUDA(cudaMemcpyAsync(D.tflag, h.data(), sizeof(unsigned) * h.size(), cudaMemcpyHostToDevice, st));
    sync();
  }

  // ping-pong copy lists (see k_cut_step): [prev][cur] = N_prev \ N_cur for
  // prev, cur colours, and [4][cur] = band \ N_cur for the first step
  // dense affine maps G_j = [A_j^{-1} | -A_j^{-1} A_{I,W}] of the cut patches
  // (k_cut_map; offsets stored in the descriptors)
  void build_cut_maps(LevelData& D, int ncp) {
    const int p = prm.p, WS = 4 * p + 1, WW = WS * WS;
    std::vector<CutDesc> hd(ncp);
    CF_CUDA(cudaMemcpy(hd.data(), D.desc, sizeof(CutDesc) * ncp, cudaMemcpyDeviceToHost));
    // dense maps first (k_cut_map), then the compressed blocks
    std::vector<int64_t> dense(ncp + 1, 0);
    std::vector<int> hm(ncp);
    for (int k = 0; k < ncp; ++k) {
      hm[k] = __builtin_popcountll(hd[k].mask[0]) + __builtin_popcountll(hd[k].mask[1]);
      hd[k].map_off = dense[k];
      dense[k + 1] = dense[k] + (int64_t)hm[k] * (hm[k] + WW);
    }
    CF_CUDA(cudaMemcpy(D.desc, hd.data(), sizeof(CutDesc) * ncp, cudaMemcpyHostToDevice));
    double* Gd = alloc<double>(dense[ncp]);
    int64_t* doff = alloc<int64_t>(ncp + 1);
    int* nnz = alloc<int>(ncp);
    CF_CUDA(cudaMemcpy(doff, dense.data(), sizeof(int64_t) * (ncp + 1), cudaMemcpyHostToDevice));
    std::vector<int> hn(ncp);
    CF_DISPATCH(p, {
      if constexpr (P <= 3) {
        const size_t smb = CutGroup6<P>::bytes;
        CF_CUDA(cudaFuncSetAttribute(k_cut_map<P, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb));
        k_cut_map<P, 64><<<dim3(ncp, WW + 1), 64, smb, st>>>(D.a, (const CutDesc*)D.desc, (const double*)D.ecut,
                                                              (const double*)D.inv, Gd);
        CF_LAUNCHED();
        k_map_nnz<P><<<ncp, 128, 0, st>>>((const CutDesc*)D.desc, doff, Gd, nnz);
        CF_LAUNCHED();
        CF_CUDA(cudaMemcpyAsync(hn.data(), nnz, sizeof(int) * ncp, cudaMemcpyDeviceToHost, st));
        sync();
        int64_t off = 0;
        for (int c = 0; c < 8; ++c) D.cut_bytes[c] = 0;
        // map blocks of each colour stored in the order of the vertex angle about the
        // level-set centre: the cut patches along a stretch of the boundary have
        // adjacent maps (k_cut_sweep moves a CTA's maps with a few large bulk copies)
        std::vector<int> ord(ncp);
        for (int k = 0; k < ncp; ++k) ord[k] = k;
        auto angle = [&](int k) {
          return std::atan2(D.a.y0 + hd[k].J * D.a.h - D.a.cy, D.a.x0 + hd[k].I * D.a.h - D.a.cx);
        };
        for (int c = 0; c < 4; ++c)
          std::stable_sort(ord.begin() + D.cutp_off[c], ord.begin() + D.cutp_off[c + 1],
                           [&](int a, int b2) { return angle(a) < angle(b2); });
        for (int q = 0; q < ncp; ++q) {
          const int k = ord[q];
          hd[k].map_off = off | ((int64_t)hn[k] << 48);
          const int64_t blk = map_hdr_d(hn[k]) + map_rows_d(hm[k], hm[k] + hn[k], D.a.map_one_lane);
          off += blk;
          // algorithmic bytes of the patch in its colour step: descriptor, map block,
          // gathered window and b values, written interior values
          int c = 0;
          while (c < 3 && k >= D.cutp_off[c + 1]) ++c;
          D.cut_bytes[c] += 64 + 8 * blk + 8 * (int64_t)hn[k] + 16 * (int64_t)hm[k];
        }
        CF_CUDA(cudaMemcpy(D.desc, hd.data(), sizeof(CutDesc) * ncp, cudaMemcpyHostToDevice));
        require(off < (1ll << 48), ERR_SIZE, "cut-patch maps exceed 2^48 doubles");
        D.gmap = alloc<double>(off);
        D.n_gmap = off;
        k_map_compact<P><<<ncp, 128, 0, st>>>((const CutDesc*)D.desc, doff, Gd, D.gmap, D.a.map_one_lane);
        CF_LAUNCHED();
      }
    });
    sync();
    for (void* q : {(void*)Gd, (void*)doff, (void*)nnz}) {
      cudaFree(q);
      allocs.erase(std::remove(allocs.begin(), allocs.end(), q), allocs.end());
    }
  }

  // DoF spans of the lattice rows of a 2D level (from the DoF mask; rows
  // without DoF: empty), for the host-vector paths
  void build_spans(LevelData& D) {
    if (D.span) return;
    const LevelArgs& L = D.a;
    const int64_t rows = prm.dim == 3 ? (int64_t)L.nl * L.nl : L.nl;
    std::vector<uint8_t> m((size_t)rows * L.ld);
    CF_CUDA(cudaMemcpy(m.data(), D.mask, m.size(), cudaMemcpyDeviceToHost));
    std::vector<int> sp(2 * rows, 0);
    int64_t tot = 0;
    for (int64_t b = 0; b < rows; ++b) {
      int a0 = -1, a1 = -1;
      for (int a = 0; a < L.nl; ++a)
        if (m[(size_t)b * L.ld + a]) {
          if (a0 < 0) a0 = a;
          a1 = a + 1;
        }
      if (a0 < 0) a0 = a1 = 0;
      sp[2 * b] = a0;
      sp[2 * b + 1] = a1;
      tot += a1 - a0;
    }
    D.span = alloc<int>(2 * rows);
    CF_CUDA(cudaMemcpy(D.span, sp.data(), sizeof(int) * sp.size(), cudaMemcpyHostToDevice));
    D.span_doubles = tot;
  }
  // copy the DoF spans of a lattice vector of level l (src / dst: device or
  // mapped pinned host memory); src2 / dst2: a second vector in the same launch
  void copy_spans(int l, const double* src, double* dst, const double* src2 = nullptr, double* dst2 = nullptr) {
    LevelData& D = lv[l];
    build_spans(D);
    const int64_t rows = prm.dim == 3 ? (int64_t)D.a.nl * D.a.nl : D.a.nl;
    for (int64_t r0 = 0; r0 < rows; r0 += 65535) {
      const int nb = (int)std::min<int64_t>(65535, rows - r0);
      k_copy_spans<<<dim3(nb, src2 ? 2 : 1), 256, 0, st>>>(src, dst, D.span, D.a.ld, (int)r0, src2, dst2);
      CF_LAUNCHED();
    }
  }

  // programs of the one-launch cut sweeps (sweep.cuh) of a 2D level, both
  // directions: the patches (interior nodes in map row order, the coupled
  // exterior nodes in map column order, map rows) go to the host builder,
  // the program arrays come back to the device
  void build_sweeps(LevelData& D, int ncp, int own_b0 = -1, int own_b1 = -1, int max_ctas = 0) {
    const auto t_start = std::chrono::steady_clock::now();
    const LevelArgs& L = D.a;
    const int p = prm.p, BS = 2 * p + 1, WS = 4 * p + 1, WW = WS * WS;
    std::vector<CutDesc> hd(ncp);
    CF_CUDA(cudaMemcpy(hd.data(), D.desc, sizeof(CutDesc) * ncp, cudaMemcpyDeviceToHost));
    uint8_t* dix = alloc<uint8_t>((int64_t)ncp * WW);
    k_map_idx<<<ceil_div(ncp, 128), 128, 0, st>>>((const CutDesc*)D.desc, ncp, (const double*)D.gmap, WW, dix);
    CF_LAUNCHED();
    std::vector<uint8_t> hix((size_t)ncp * WW);
    CF_CUDA(cudaMemcpyAsync(hix.data(), dix, hix.size(), cudaMemcpyDeviceToHost, st));
    sync();
    cudaFree(dix);
    allocs.erase(std::remove(allocs.begin(), allocs.end(), (void*)dix), allocs.end());
    std::vector<host::SweepPatch> P;
    for (int k = 0; k < ncp; ++k) {
      const CutDesc& d = hd[k];
      const int nnz = (int)(d.map_off >> 48);
      host::SweepPatch q;
      q.I = d.I;
      q.J = d.J;
      q.colour = (d.I & 1) + 2 * (d.J & 1);
      for (int loc = 0; loc < BS * BS; ++loc)
        if ((d.mask[loc >> 6] >> (loc & 63)) & 1ull)
          q.in.push_back((p * (d.J - 1) + loc / BS) * L.ld + p * (d.I - 1) + loc % BS);
      if (q.in.empty()) continue;
      for (int j = 0; j < nnz; ++j) {
        const int w = hix[(size_t)k * WW + j];
        q.ex.push_back((p * (d.J - 2) + w / WS) * L.ld + p * (d.I - 2) + w % WS);
      }
      q.blk0 = d.map_off & ((1ll << 48) - 1);
      q.rows = q.blk0 + map_hdr_d(nnz);
      q.blk1 = q.rows + map_rows_d((int)q.in.size(), (int)(q.in.size() + q.ex.size()), L.map_one_lane);
      P.push_back(std::move(q));
    }
    int dev = 0, nsm = 0, smax = 0;
    CF_CUDA(cudaGetDevice(&dev));
    CF_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    CF_CUDA(cudaDeviceGetAttribute(&smax, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    if (max_ctas > 0) nsm = std::min(nsm, max_ctas);
    static const char attr_key = 0;   // per-device attribute (dev_once)
    dev_once(&attr_key, [&] {
      CF_CUDA(cudaFuncSetAttribute(k_cut_sweep, cudaFuncAttributeMaxDynamicSharedMemorySize, smax - 1024));
    });
    for (int dir = 0; dir < 2; ++dir) {
      host::SweepProgram R = host::build_sweep(P, L.n, p, L.ld, 4 * prm.n_c, dir, nsm, (size_t)smax, sweep_ng, verbose,
                                               (L.cx - L.x0) / L.h * p, (L.cy - L.y0) / L.h * p, own_b0, own_b1,
                                               L.map_one_lane);
      LevelData::Sweep& W = D.sw[dir];
      W.ok = R.ok;
      if (!R.ok) {
        if (verbose) std::fprintf(stderr, "[cutfem] sweep n=%d dir=%d not built: %s\n", L.n, dir, R.why.c_str());
        continue;
      }
      SweepArgs A = {};
      auto up = [&](const auto& v) {
        using T = typename std::decay_t<decltype(v)>::value_type;
        T* d = alloc<T>((int64_t)v.size());
        if (!v.empty()) CF_CUDA(cudaMemcpyAsync(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, st));
        return d;
      };
      A.cta = up(R.cta);
      A.chunk = up(R.chunk);
      A.run = up(R.run);
      A.aux = (const unsigned char*)up(R.aux);
      A.slot_node = up(R.slot_node);
      A.own = up(R.own);
      A.gmap = D.gmap;
      A.gbar = alloc<unsigned long long>(1);
      CF_CUDA(cudaMemsetAsync(A.gbar, 0, sizeof(unsigned long long), st));
      A.S = R.S;
      A.one_lane = L.map_one_lane;
      A.nch = R.nch;
      A.cb = R.cb;
      A.off_chunk = R.off_chunk;
      A.off_run = R.off_run;
      A.off_xs = R.off_xs;
      A.off_bs = R.off_bs;
      A.off_v = R.off_v;
      A.off_ring = R.off_ring;
      static_assert(sizeof(SweepArgs) <= sizeof(W.args), "SweepArgs fits LevelData::Sweep::args");
      std::memcpy(W.args, &A, sizeof(A));
      W.ncta = R.ncta;
      W.smem = R.smem;
      W.est_us = R.est_us;
      W.redundancy = R.redundancy;
      W.map_bytes_total = R.map_bytes_total;
      sync();
    }
    if (verbose)
      std::fprintf(stderr, "[cutfem] sweep programs n=%d built in %.1f ms\n", L.n,
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count());
  }

  // method bytes of one cut colour step: per
  // patch the paper's local solver streams A_j^{-1} (m^2), the element
  // matrices of its cut cells ((p+1)^4 each), reads b_I and the coupled window
  // values x_I, x_E (m + nnz) and writes x_I (m): 8 (m^2 + n_cut (p+1)^4 +
  // 3 m + nnz) bytes, whatever the implementation (the patch maps of R13 are
  // an implementation choice and are not counted)
  void method_bytes(LevelData& D, int ncp) {
    const int p = prm.p, e4 = (p + 1) * (p + 1) * (p + 1) * (p + 1);
    std::vector<CutDesc> hd(ncp);
    CF_CUDA(cudaMemcpy(hd.data(), D.desc, sizeof(CutDesc) * ncp, cudaMemcpyDeviceToHost));
    for (int c = 0; c < 8; ++c) D.cut_method_bytes[c] = 0;
    for (int c = 0; c < 4; ++c)
      for (int k = D.cutp_off[c]; k < D.cutp_off[c + 1]; ++k) {
        const CutDesc& d = hd[k];
        const long long m = __builtin_popcountll(d.mask[0]) + __builtin_popcountll(d.mask[1]);
        const long long nnz = d.map_off >= 0 ? (long long)(d.map_off >> 48) : 0;
        int ncut = 0;
        for (int q = 0; q < 4; ++q) ncut += d.cid[q] >= 0;
        D.cut_method_bytes[c] += 8 * (m * (m + 1) / 2 + (long long)ncut * e4 + 3 * m + nnz);
      }
  }



  // 3D: per patch 8 (m^2 + n_cut (p+1)^6 + (2p+1)^3 + 2 m): inverse, cut-cell
  // matrices, the patch block of x (the residual's reach through the patch
  // cells), b_I, written correction
  void method_bytes3(LevelData& D, int ncp) {
    const int p = prm.p, e6 = (int)std::pow(p + 1, 6), bs3 = (2 * p + 1) * (2 * p + 1) * (2 * p + 1);
    std::vector<CutDesc3> hd(ncp);
    CF_CUDA(cudaMemcpy(hd.data(), D.desc, sizeof(CutDesc3) * ncp, cudaMemcpyDeviceToHost));
    for (int c = 0; c < 8; ++c) {
      D.cut_method_bytes[c] = 0;
      for (int k = D.cutp_off[c]; k < D.cutp_off[c + 1]; ++k) {
        const CutDesc3& d = hd[k];
        long long m = 0;
        for (int w = 0; w < 6; ++w) m += __builtin_popcountll(d.mask[w]);
        int ncut = 0;
        for (int q = 0; q < 8; ++q) ncut += d.cid[q] >= 0;
        D.cut_method_bytes[c] += 8 * (m * (m + 1) / 2 + (long long)ncut * e6 + bs3 + 2 * m);   // (symmetric A_j^{-1}: m (m+1) / 2)
      }
    }
  }

  // (ent_node, col_off[0..4]: the interior nodes of the swept patches per
  // colour; desc/ncp: their descriptors)
  void build_copy_lists(LevelData& D, const int32_t* ent_node, const int64_t* col_off, const CutDesc* desc, int ncp) {
    const LevelArgs& L = D.a;
    const int64_t nv = (int64_t)L.nl * L.ld;
    if (!D.xs) {
      D.xs = alloc<double>(nv);
      CF_CUDA(cudaMemsetAsync(D.xs, 0, nv * 8, st));
    }
    uint8_t* marks = alloc<uint8_t>(5 * nv);
    CF_CUDA(cudaMemsetAsync(marks, 0, 5 * nv, st));
    for (int c = 0; c < 4; ++c)
      if (col_off[c + 1] > col_off[c]) {
        k_mark_entries<<<ceil_div(col_off[c + 1] - col_off[c], 256), 256, 0, st>>>(ent_node, col_off[c], col_off[c + 1],
                                                                                 marks + c * nv);
        CF_LAUNCHED();
      }
    if (ncp) {
      k_mark_band<<<ncp, 128, 0, st>>>(desc, ncp, L, marks + 4 * nv);
      CF_LAUNCHED();
    }
    uint8_t* fl = alloc<uint8_t>(nv);
    int* tmp = alloc<int>(nv);
    std::vector<int> all;
    for (int pv = 0; pv < 5; ++pv)
      for (int c = 0; c < 4; ++c) {
        D.copy_off[pv][c] = (int)all.size();
        D.copy_n[pv][c] = 0;
        if (pv == c) continue;
        k_andnot_flags<<<ceil_div(nv, 256), 256, 0, st>>>(marks + pv * nv, marks + c * nv, nv, fl);
        CF_LAUNCHED();
        const int cnt = select(fl, (int)nv, tmp);
        std::vector<int> h(cnt);
        if (cnt) CF_CUDA(cudaMemcpyAsync(h.data(), tmp, sizeof(int) * cnt, cudaMemcpyDeviceToHost, st));
        sync();
        all.insert(all.end(), h.begin(), h.end());
        D.copy_n[pv][c] = cnt;
      }
    D.copy_lists = alloc<int32_t>(all.size());
    if (!all.empty())
      CF_CUDA(cudaMemcpyAsync(D.copy_lists, all.data(), sizeof(int) * all.size(), cudaMemcpyHostToDevice, st));
    sync();
    for (void* q : {(void*)marks, (void*)fl, (void*)tmp}) {
      cudaFree(q);
      allocs.erase(std::remove(allocs.begin(), allocs.end(), q), allocs.end());
    }
  }

  // Wide-halo cut sweeps of a partitioned level: step s (of S = 4 n_c, per
  // direction) runs the patches of its colour with vertex rows
  // [c0 - e_s, c1 + e_s], e_s = 1 + 3 (S-1-s).  A patch reads the cell rows
  // [J-2, J+2) and a node is final after step s if every step-s patch whose
  // interior holds it ran, i.e. on the cell rows [c0 - e_s + 1, c1 + e_s - 1):
  // exactly the rows step s+1 reads.  So one exchange of HW = e_0 + 2 = 3 S
  // cells before the sweeps replaces the 4 n_c per-step exchanges, and the
  // last step (e = 1) leaves the owned rows final.  Copy lists per step:
  // N_{s-1} \ N_s, each N restricted to its step (for s = 0: the band of the
  // windows of every patch of the sweep \ N_0).
  void build_wide(LevelData& D, const std::vector<CutDesc>& hd, const std::vector<int64_t>& he,
                  const std::vector<int32_t>& hn) {
    const LevelArgs& L = D.a;
    const int S = 4 * prm.n_c;
    const int64_t nv = (int64_t)L.nl * L.ld;
    std::vector<CutDesc> kd;
    std::vector<std::vector<int32_t>> nodes;   // per (d, s)
    for (int d = 0; d < 2; ++d) {
      D.wd_off[d].assign(S + 1, 0);
      for (int s = 0; s < S; ++s) {
        const int c = d ? 3 - (s & 3) : (s & 3), e = 1 + 3 * (S - 1 - s);
        D.wd_off[d][s] = (int)kd.size();
        std::vector<int32_t> nn;
        for (int k = D.cutp_off[c]; k < D.cutp_off[c + 1]; ++k)
          if (hd[k].J >= D.c0 - e && hd[k].J <= D.c1 + e) {
            kd.push_back(hd[k]);
            nn.insert(nn.end(), hn.begin() + he[k], hn.begin() + he[k + 1]);
          }
        nodes.push_back(nn);
      }
      D.wd_off[d][S] = (int)kd.size();
    }
    CutDesc* dd = alloc<CutDesc>(kd.size());
    if (!kd.empty()) CF_CUDA(cudaMemcpy(dd, kd.data(), sizeof(CutDesc) * kd.size(), cudaMemcpyHostToDevice));
    D.wdesc = dd;
    // marks of N_(d,s) and of the band of step 0, then the set differences
    uint8_t* mk = alloc<uint8_t>(3 * nv);
    uint8_t* fl = alloc<uint8_t>(nv);
    int* tmp = alloc<int>(nv);
    int32_t* dn = alloc<int32_t>(1);
    std::vector<int32_t> all;
    for (int d = 0; d < 2; ++d) {
      D.wc_off[d].assign(S, 0);
      D.wc_n[d].assign(S, 0);
      for (int s = 0; s < S; ++s) {
        CF_CUDA(cudaMemsetAsync(mk, 0, 2 * nv, st));
        // mk[0] = previous set (band of step 0 for s = 0), mk[nv] = N_s
        auto mark = [&](const std::vector<int32_t>& v, uint8_t* m) {
          if (v.empty()) return;
          int32_t* buf = alloc<int32_t>(v.size());
          CF_CUDA(cudaMemcpy(buf, v.data(), sizeof(int32_t) * v.size(), cudaMemcpyHostToDevice));
          k_mark_entries<<<ceil_div((int64_t)v.size(), 256), 256, 0, st>>>(buf, 0, (int64_t)v.size(), m);
          CF_LAUNCHED();
          sync();
          cudaFree(buf);
          allocs.erase(std::remove(allocs.begin(), allocs.end(), (void*)buf), allocs.end());
        };
        if (s == 0) {   // the read band: windows of every patch the sweep runs
          const int n0 = D.wd_off[d][S] - D.wd_off[d][0];
          if (n0) {
            k_mark_band<<<n0, 128, 0, st>>>(dd + D.wd_off[d][0], n0, L, mk);
            CF_LAUNCHED();
          }
        } else {
          mark(nodes[d * S + s - 1], mk);
        }
        mark(nodes[d * S + s], mk + nv);
        k_andnot_flags<<<ceil_div(nv, 256), 256, 0, st>>>(mk, mk + nv, nv, fl);
        CF_LAUNCHED();
        const int cnt = select(fl, (int)nv, tmp);
        std::vector<int32_t> h(cnt);
        if (cnt) CF_CUDA(cudaMemcpy(h.data(), tmp, sizeof(int) * cnt, cudaMemcpyDeviceToHost));
        D.wc_off[d][s] = (int)all.size();
        D.wc_n[d][s] = cnt;
        all.insert(all.end(), h.begin(), h.end());
      }
    }
    D.wcopy = alloc<int32_t>(all.size());
    if (!all.empty()) CF_CUDA(cudaMemcpy(D.wcopy, all.data(), sizeof(int32_t) * all.size(), cudaMemcpyHostToDevice));
    for (void* q : {(void*)mk, (void*)fl, (void*)tmp, (void*)dn}) {
      cudaFree(q);
      allocs.erase(std::remove(allocs.begin(), allocs.end(), q), allocs.end());
    }
  }

  // ------------------------------------------------------- slab partition
  // Rank c->rank of c->world owns the cell rows [c0, c1) = [rank s, (rank+1) s),
  // s = n / world, of every level whose slabs are whole fused Cartesian tiles
  // (s % TC == 0) at least HALO + 1 cells thick, from the finest level down;
  // the coarser levels (and level 0, the exact coarse solve) are replicated on
  // every rank.  Each rank keeps the whole hierarchy (setup is replicated) and
  // restricts its work lists to its rows: fused tiles of its rows, cut patches
  // whose interiors meet its rows (vertex rows [c0 - 1, c1]: the patches on
  // the slab boundary are computed by both neighbours, identically), cut cells
  // and ghost faces within HALO cells.  Lattice vectors are full-size; the
  // rows [v0, v1) = owned rows + HALO cells are valid after a halo exchange.
  // doubles per lattice row of the partitioned direction (a row in 2D, a plane in 3D)
  int64_t rowsz(int l) const {
    const LevelArgs& L = lv[l].a;
    return (int64_t)L.ld * (prm.dim == 3 ? L.nl : 1);
  }

  // 3D: slabs of z-planes; narrow halo, one exchange per colour step; the
  // rank runs the Cartesian and cut patches with vertex planes [c0 - 1, c1]
  // (compact descriptor / scatter lists with renumbered zbuf offsets)
  void partition3(Comm* c) {
    const int W = c->world, R = c->rank, p = prm.p;
    bool finer = true;
    for (int l = prm.n_levels - 1; l >= 1; --l) {
      LevelData& D = lv[l];
      const int n = D.a.n, nl = D.a.nl, s = n / W, nv = n + 1;
      const int64_t ps = rowsz(l);
      const bool ok = finer && n % W == 0 && s >= HALO + 1;
      finer = ok;
      if (!ok) continue;
      D.part = 1;
      const SlabPlan sp = slab_plan(n, p, W, R, HALO, ps);
      D.c0 = sp.c0;
      D.c1 = sp.c1;
      D.r0 = sp.r0;
      D.r1 = sp.r1;
      D.wide = 0;
      D.hw = HALO;
      D.v0 = D.v0n = sp.v0;
      D.v1 = D.v1n = sp.v1;
      D.rc0 = p * (D.c0 / 2);
      D.rc1 = R == W - 1 ? lv[l - 1].a.nl : p * (D.c1 / 2);
      D.halo = sp.xf;
      D.halo_n = sp.xf;
      auto keepK = [&](int K) { return K >= D.c0 - 1 && K <= D.c1; };
      // Cartesian patches
      {
        const int nc = D.cart_off[8];
        std::vector<int> h(nc), k;
        if (nc) CF_CUDA(cudaMemcpy(h.data(), D.cart_list, sizeof(int) * nc, cudaMemcpyDeviceToHost));
        D.act_cart_off[0] = 0;
        for (int cc = 0; cc < 8; ++cc) {
          for (int q = D.cart_off[cc]; q < D.cart_off[cc + 1]; ++q)
            if (keepK(h[q] / (nv * nv))) k.push_back(h[q]);
          D.act_cart_off[cc + 1] = (int)k.size();
        }
        int* dl = alloc<int>(k.size());
        if (!k.empty()) CF_CUDA(cudaMemcpy(dl, k.data(), sizeof(int) * k.size(), cudaMemcpyHostToDevice));
        D.act_cart = dl;
      }
      // cut patches: compact descriptors (zbuf offsets renumbered) and scatter list
      {
        const int ncp = D.cutp_off[8];
        std::vector<CutDesc3> hd(ncp), kd;
        std::vector<int64_t> he(ncp + 1);
        std::vector<int32_t> hn(D.n_ent), kn;
        if (ncp) {
          CF_CUDA(cudaMemcpy(hd.data(), D.desc, sizeof(CutDesc3) * ncp, cudaMemcpyDeviceToHost));
          CF_CUDA(cudaMemcpy(he.data(), D.cutp_ent, sizeof(int64_t) * (ncp + 1), cudaMemcpyDeviceToHost));
        }
        if (D.n_ent) CF_CUDA(cudaMemcpy(hn.data(), D.ent_node, sizeof(int32_t) * D.n_ent, cudaMemcpyDeviceToHost));
        D.act_off[0] = 0;
        D.act_ent_off[0] = 0;
        for (int cc = 0; cc < 8; ++cc) {
          for (int k = D.cutp_off[cc]; k < D.cutp_off[cc + 1]; ++k)
            if (keepK(hd[k].K)) {
              CutDesc3 d = hd[k];
              d.e0 = (int)kn.size();
              kd.push_back(d);
              kn.insert(kn.end(), hn.begin() + he[k], hn.begin() + he[k + 1]);
            }
          D.act_off[cc + 1] = (int)kd.size();
          D.act_ent_off[cc + 1] = (int64_t)kn.size();
        }
        CutDesc3* dd = alloc<CutDesc3>(kd.size());
        int32_t* dn = alloc<int32_t>(kn.size());
        if (!kd.empty()) CF_CUDA(cudaMemcpy(dd, kd.data(), sizeof(CutDesc3) * kd.size(), cudaMemcpyHostToDevice));
        if (!kn.empty()) CF_CUDA(cudaMemcpy(dn, kn.data(), sizeof(int32_t) * kn.size(), cudaMemcpyHostToDevice));
        D.act_desc = dd;
        D.act_ent = dn;
      }
      // k_band3 ranges: cut cells and x/y-faces of the planes [c0 - HALO, c1 + HALO),
      // z-faces (k | k+1) with k in [c0 - HALO, c1 + HALO - 1); lists sorted by (k n + j) n + i
      {
        const int lo = std::max(0, D.c0 - HALO), hi = std::min(n, D.c1 + HALO);
        const int zhi = std::max(lo, std::min(n - 1, D.c1 + HALO - 1));
        const int64_t n2 = (int64_t)n * n, n3 = n2 * n;
        std::vector<int64_t> hc(D.a.n_cut), hg(D.a.n_ghost);
        {
          std::vector<int> t(D.a.n_cut), u(D.a.n_ghost);
          if (D.a.n_cut) CF_CUDA(cudaMemcpy(t.data(), D.cut_list, sizeof(int) * D.a.n_cut, cudaMemcpyDeviceToHost));
          if (D.a.n_ghost) CF_CUDA(cudaMemcpy(u.data(), D.ghost_list, sizeof(int) * D.a.n_ghost, cudaMemcpyDeviceToHost));
          for (size_t q = 0; q < t.size(); ++q) hc[q] = (uint32_t)t[q];
          for (size_t q = 0; q < u.size(); ++q) hg[q] = (uint32_t)u[q];
        }
        auto range = [](const std::vector<int64_t>& v, int64_t a, int64_t b, int& first, int& cnt) {
          first = (int)(std::lower_bound(v.begin(), v.end(), a) - v.begin());
          cnt = (int)(std::lower_bound(v.begin(), v.end(), b) - v.begin()) - first;
        };
        range(hc, lo * n2, hi * n2, D.band3[0], D.band3[1]);
        range(hg, 0 * n3 + lo * n2, 0 * n3 + hi * n2, D.band3[2], D.band3[5]);
        range(hg, 1 * n3 + lo * n2, 1 * n3 + hi * n2, D.band3[3], D.band3[6]);
        range(hg, 2 * n3 + lo * n2, 2 * n3 + zhi * n2, D.band3[4], D.band3[7]);
      }
    }
    comm = c;
  }

  void partition(Comm* c) {
    require(prm.dim == 2 || prm.dim == 3, ERR_ARG, "the slab partition needs a 2D or 3D problem");
    require(built, ERR_STATE, "cutfem_build_patches has not been called");
    if (prm.dim == 3) {
      require(comm == nullptr, ERR_STATE, "the problem is already partitioned");
      require(c->world >= 1 && c->rank >= 0 && c->rank < c->world, ERR_ARG, "bad rank / world");
      partition3(c);
      return;
    }
    require(comm == nullptr, ERR_STATE, "the problem is already partitioned");
    require(c->world >= 1 && c->rank >= 0 && c->rank < c->world, ERR_ARG, "bad rank / world");
    const int W = c->world, R = c->rank, p = prm.p;
    fused = true;
    pingpong = true;
    bool finer = true;
    for (int l = prm.n_levels - 1; l >= 1; --l) {
      LevelData& D = lv[l];
      const int n = D.a.n, nl = D.a.nl, ld = D.a.ld, s = n / W, TC = D.tc;
      // With the wide halo (default) only slabs thick enough for it are
      // partitioned: a thinner level would need an exchange per cut step
      // (4 n_c + 1 per smoothing step), which costs more than computing the
      // whole (small) level on every rank; CUTFEM_WIDE_HALO=0 partitions every
      // level of >= HALO + 1 rows with the narrow halo instead.
      const int S = 4 * prm.n_c, HW = 3 * S;   // wide halo: 3 cells per cut step (see build_wide)
      const bool ok = finer && n % W == 0 && s % TC == 0 && s >= (wide_halo ? HW : HALO) + 1;
      finer = ok;
      if (!ok) continue;
      D.part = 1;
      D.wide = wide_halo;
      D.hw = D.wide ? HW : HALO;
      const SlabPlan sw = slab_plan(n, p, W, R, D.hw, ld), sn = slab_plan(n, p, W, R, HALO, ld);
      D.c0 = sw.c0;
      D.c1 = sw.c1;
      D.r0 = sw.r0;
      D.r1 = sw.r1;
      D.v0n = sn.v0;
      D.v1n = sn.v1;
      D.v0 = sw.v0;
      D.v1 = sw.v1;
      D.rc0 = p * (D.c0 / 2);
      D.rc1 = R == W - 1 ? lv[l - 1].a.nl : p * (D.c1 / 2);
      D.halo = sw.xf;
      D.halo_n = sn.xf;
      // fused tiles (packed ti | tj << 16) of the owned rows
      auto own_tiles = [&](int*& list, int& cnt) {
        std::vector<int> h(cnt), keep;
        if (cnt) CF_CUDA(cudaMemcpy(h.data(), list, sizeof(int) * cnt, cudaMemcpyDeviceToHost));
        for (int t : h)
          if ((t >> 16) * TC >= D.c0 && (t >> 16) * TC < D.c1) keep.push_back(t);
        cnt = (int)keep.size();
        list = alloc<int>(cnt);
        if (cnt) CF_CUDA(cudaMemcpy(list, keep.data(), sizeof(int) * cnt, cudaMemcpyHostToDevice));
      };
      own_tiles(D.fused_tiles, D.n_fused_tiles);
      own_tiles(D.fused_ext, D.n_fused_ext);
      // the in-place sweep's tile counters: only the rank's tiles take part now
      if (D.tflag) reset_tile_flags(D, ceil_div(D.a.n, D.tc));
      // cut patches with vertex rows [c0 - 1, c1]
      const int ncp = D.cutp_off[4];
      std::vector<CutDesc> hd(ncp), kd;
      std::vector<int64_t> he(ncp + 1);
      std::vector<int32_t> hn(D.n_ent), kn;
      if (ncp) {
        CF_CUDA(cudaMemcpy(hd.data(), D.desc, sizeof(CutDesc) * ncp, cudaMemcpyDeviceToHost));
        CF_CUDA(cudaMemcpy(he.data(), D.cutp_ent, sizeof(int64_t) * (ncp + 1), cudaMemcpyDeviceToHost));
      }
      if (D.n_ent) CF_CUDA(cudaMemcpy(hn.data(), D.ent_node, sizeof(int32_t) * D.n_ent, cudaMemcpyDeviceToHost));
      int64_t col_off[5] = {0, 0, 0, 0, 0};
      D.act_off[0] = 0;
      for (int cc = 0; cc < 4; ++cc) {
        for (int k = D.cutp_off[cc]; k < D.cutp_off[cc + 1]; ++k)
          if (hd[k].J >= D.c0 - 1 && hd[k].J <= D.c1) {
            kd.push_back(hd[k]);
            kn.insert(kn.end(), hn.begin() + he[k], hn.begin() + he[k + 1]);
          }
        D.act_off[cc + 1] = (int)kd.size();
        col_off[cc + 1] = (int64_t)kn.size();
      }
      CutDesc* dd = alloc<CutDesc>(kd.size());
      int32_t* dn = alloc<int32_t>(kn.size());
      if (!kd.empty()) CF_CUDA(cudaMemcpy(dd, kd.data(), sizeof(CutDesc) * kd.size(), cudaMemcpyHostToDevice));
      if (!kn.empty()) CF_CUDA(cudaMemcpy(dn, kn.data(), sizeof(int32_t) * kn.size(), cudaMemcpyHostToDevice));
      D.act_desc = dd;
      build_copy_lists(D, dn, col_off, dd, (int)kd.size());
      if (D.wide) build_wide(D, hd, he, hn);
      // the one-launch cut sweep over the rank's owned rows (wide halo: every
      // cone input is valid after the one exchange before the sweep); ranks that
      // share a GPU (LocalComm) split its SMs, so every cooperative grid fits
      for (int d2 = 0; d2 < 2; ++d2) D.sw[d2].ok = false;
      if (D.wide && one_sweep && D.gmap && ncp)
        build_sweeps(D, ncp, D.r0, D.r1, dynamic_cast<LocalComm*>(c) ? std::max(1, num_sms() / W) : 0);
      // k_band ranges: cut cells and x-faces in cell rows [c0 - HALO, c1 + HALO),
      // y-faces (j | j+1) with j in [c0 - HALO, c1 + HALO - 1); the lists are sorted by j n + i
      const int lo = std::max(0, D.c0 - HALO), hi = std::min(n, D.c1 + HALO);
      std::vector<int> hc(D.a.n_cut), hg(D.a.n_ghost);
      if (D.a.n_cut) CF_CUDA(cudaMemcpy(hc.data(), D.cut_list, sizeof(int) * D.a.n_cut, cudaMemcpyDeviceToHost));
      if (D.a.n_ghost) CF_CUDA(cudaMemcpy(hg.data(), D.ghost_list, sizeof(int) * D.a.n_ghost, cudaMemcpyDeviceToHost));
      auto range = [](const std::vector<int>& v, int a, int b, int& first, int& cnt) {
        first = (int)(std::lower_bound(v.begin(), v.end(), a) - v.begin());
        cnt = (int)(std::lower_bound(v.begin(), v.end(), b) - v.begin()) - first;
      };
      const int nn = n * n;
      range(hc, lo * n, hi * n, D.band[0], D.band[1]);
      range(hg, lo * n, hi * n, D.band[2], D.band[3]);
      const int yhi = std::max(lo, std::min(n - 1, D.c1 + HALO - 1));
      range(hg, nn + lo * n, nn + yhi * n, D.band[4], D.band[5]);
      // TMA operator tiles (16 cells) covering the cell rows [c0 - 2, c1 + 2)
      const int nt = ceil_div(n, 16);
      D.at0 = std::max(0, (D.c0 - 2) / 16);
      D.at1 = std::min(nt, ceil_div(D.c1 + 2, 16));
    }
    // replicated (coarser) levels keep their whole-level one-launch sweeps; ranks
    // sharing a GPU rebuild them on their share of the SMs
    if (dynamic_cast<LocalComm*>(c) && W > 1)
      for (int l = 1; l < prm.n_levels; ++l) {
        LevelData& D = lv[l];
        if (!D.part && D.sw[0].ok && D.gmap) build_sweeps(D, D.cutp_off[4], -1, -1, std::max(1, num_sms() / W));
      }
    comm = c;
  }

  void build_coarse() {
    LevelData& D = lv[0];
    const int64_t nv = vsize(0);
    int* nodes = alloc<int>(nv);
    n0 = select(D.mask, (int)nv, nodes);
    require(n0 <= 4096, ERR_SIZE, "coarse level has more than 4096 DoFs; use a coarser level 0");
    c_nodes = nodes;
    c_inv = alloc<double>((int64_t)n0 * n0);
    double* e = alloc<double>(nv);
    double* y = alloc<double>(nv);
    std::vector<int> hn(n0);
    CF_CUDA(cudaMemcpyAsync(hn.data(), nodes, sizeof(int) * n0, cudaMemcpyDeviceToHost, st));
    sync();
    for (int i = 0; i < n0; ++i) {
      CF_CUDA(cudaMemsetAsync(e, 0, nv * 8, st));
      k_set_entry<<<1, 1, 0, st>>>(e, hn[i], 1.0);
      CF_LAUNCHED();
      apply(0, e, y, nullptr);
      k_gather_column<<<ceil_div(n0, 128), 128, 0, st>>>(y, nodes, n0, c_inv + (int64_t)i * n0);
      CF_LAUNCHED();
    }
    int64_t* offs = alloc<int64_t>(2);
    int64_t ho[2] = {0, n0}, hz[2] = {0, 0};
    CF_CUDA(cudaMemcpyAsync(offs, ho, sizeof(ho), cudaMemcpyHostToDevice, st));
    int64_t* ioff = alloc<int64_t>(2);
    CF_CUDA(cudaMemcpyAsync(ioff, hz, sizeof(hz), cudaMemcpyHostToDevice, st));
    size_t smb = (size_t)(n0 * n0 + 2 * n0) * sizeof(double);
    if (smb <= 200 * 1024) {
      CF_CUDA(cudaFuncSetAttribute(k_batched_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(smb, 48 * 1024)));
      k_batched_inverse<<<1, 256, smb, st>>>(offs, ioff, c_inv, 1);
    } else {   // (3D Q3: 343 coarse DoFs) in place in global memory
      k_batched_inverse_gmem<<<1, 1024, 2 * n0 * sizeof(double), st>>>(offs, ioff, c_inv, 1, 0);
    }
    CF_LAUNCHED();
    sync();
  }

  // ------------------------------------------------------------- hot path
  // fitted box: the cell kernels read the boundary nodes of their cells, so x
  // must be 0 there (the API ignores non-DoF entries on input): zeroed in place
  // at the public entry points (smooth, vcycle, colour_step); a no-op for the
  // level-set domain, whose kernels never read a non-DoF node
  void zero_boundary(int l, double* x) {
    if (prm.domain != 1) return;
    const LevelArgs& L = lv[l].a;
    const int64_t n = prm.dim == 3 ? 6 * (int64_t)L.nl * L.nl : 4 * (int64_t)L.nl;
    launch(k_zero_boundary, dim3(ceil_div(n, 256)), dim3(256), 0, L, x);
    CF_LAUNCHED();
  }
  // public operator: x is const, so in fitted mode it is copied with the DoF
  // mask into the level's residual workspace first
  void apply_entry(int l, const double* x, double* y) {
    if (prm.domain == 1) {
      LevelData& D = lv[l];
      const int64_t nv = vsize(l);
      k_masked_copy<<<4 * 148, 256, 0, st>>>(D.r, x, D.mask, nv);
      CF_LAUNCHED();
      apply(l, D.r, y, nullptr);
      return;
    }
    apply(l, x, y, nullptr);
  }

  void apply(int l, const double* x, double* y, const double* b) {
    if (prm.dim == 3) {
      apply3(l, x, y, b);
      return;
    }
    const LevelData& D = lv[l];
    const LevelArgs& L = D.a;
    const int p = prm.p;
    // under the slab partition: cut cells / ghost faces and tile rows around
    // the owned rows (the residual is needed 2 cells beyond them by the restriction)
    const BandRange R = D.part ? BandRange{D.band[0], D.band[1], D.band[2], D.band[3], D.band[4], D.band[5]}
                               : BandRange{0, L.n_cut, 0, L.n_ghost, 0, 0};
    const int warps = R.cut_n + ceil_div(R.g_n0 + R.g_n1, 32);
    if (warps) {
      if (prm.cut_mode == 0) {
        CF_DISPATCH(p, launch(k_band<P, false>, dim3(ceil_div(warps, 4)), dim3(128), 0, L, x, R));
      } else {
        CF_DISPATCH(p, launch(k_band<P, true>, dim3(ceil_div(warps, 4)), dim3(128), 0, L, x, R));
      }
      CF_LAUNCHED();
    }
    // TMA tiles of 16 x 16 cells where the level has enough of them to fill the
    // GPU; small levels use one thread per node (shorter per-thread chains)
    bool tile_ok = false;
    CF_DISPATCH(p, tile_ok = L.nl >= ApplySmem<P, 16>::RW && L.ld >= ApplySmem<P, 16>::RWP &&
                             (int64_t)ceil_div(L.n, 16) * ceil_div(L.n, 16) >= tile_apply_min_tiles);
    if (tile_apply && tile_ok) {   // the TMA box must fit inside the lattice
      CF_DISPATCH(p, {
        constexpr int TX = 16;
        using S = ApplySmem<P, TX>;
        const CUtensorMap tm = host::lattice_tmap(x, L.nl, L.ld, S::RWP, S::RW);
        static const char attr_key = 0;   // per-device attribute (dev_once)
        dev_once(&attr_key, [&] {
          CF_CUDA(cudaFuncSetAttribute(k_apply_tile<P, TX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::bytes));
        });
        const int nt = ceil_div(L.n, TX);
        const int ty0 = D.part ? D.at0 : 0, ty1 = D.part ? D.at1 : nt;
        if (ty1 > ty0) launch(k_apply_tile<P, TX>, dim3(nt, ty1 - ty0), dim3(256), S::bytes, tm, L, b, y, ty0);
      });
      CF_LAUNCHED();
      return;
    }
    const int row0 = D.part ? std::max(0, (D.c0 - 2) * p) : 0, row1 = D.part ? std::min(L.nl, (D.c1 + 2) * p + 1) : L.nl;
    CF_DISPATCH(p, launch(k_node_apply<P>, dim3(ceil_div(L.ld, 32), ceil_div(row1 - row0, 8)), dim3(32, 8), 0, L, x, b,
                          y, row0, row1));
    CF_LAUNCHED();
  }

  void cart_step(int l, int c, double* x, const double* b) {
    LevelData& D = lv[l];
    if (!D.n_cart_tiles[c]) return;
    CF_DISPATCH(prm.p, {
      constexpr int TP = cart_tp<P>();
      const size_t smb = CartSmem<P, TP>::doubles * sizeof(double);
      static const char attr_key = 0;   // per-device attribute (dev_once)
      dev_once(&attr_key, [&] {
        CF_CUDA(cudaFuncSetAttribute(k_cart_colour_v2<P, TP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb));
      });
      k_cart_colour_v2<P, TP><<<D.n_cart_tiles[c], TP * TP * (2 * P - 1), smb, st>>>(
          D.a, D.cart_tiles + D.cart_tile_off[c], c, D.vkind, x, b);
    });
    CF_LAUNCHED();
  }

  void cut_step(int l, int c, double* x, const double* b) {
    LevelData& D = lv[l];
    const int np = D.n_cutp[c];
    if (!np) return;
    const int base = D.cutp_off[c];
    const CutDesc* desc = (const CutDesc*)D.desc + base;
    CF_DISPATCH(prm.p, {
      const size_t pw = CutSmem3<P>::per_warp * sizeof(double);
      const int wpb = (int)std::max<size_t>(1, std::min<size_t>(4, (96 * 1024) / pw));
      const size_t smb = wpb * pw;
      static const char attr_key = 0;   // per-device attribute (dev_once)
      dev_once(&attr_key, [&] {
        CF_CUDA(cudaFuncSetAttribute(k_cut_colour_v3<P, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CF_CUDA(cudaFuncSetAttribute(k_cut_colour_v3<P, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      });
      if (prm.cut_mode == 0)
        launch(k_cut_colour_v3<P, false>, dim3(ceil_div(np, wpb)), dim3(128), smb, D.a, desc, np, (const double*)D.ecut,
               (const double*)D.inv, (const double*)x, b, D.zbuf, wpb);
      else
        launch(k_cut_colour_v3<P, true>, dim3(ceil_div(np, wpb)), dim3(128), smb, D.a, desc, np, (const double*)D.ecut,
               (const double*)D.inv, (const double*)x, b, D.zbuf, wpb);
    });
    CF_LAUNCHED();
    const int64_t e0 = D.ent_col_off[c], e1 = D.ent_col_off[c + 1];
    if (e1 <= e0) return;
    launch(k_cut_apply, dim3(ceil_div(e1 - e0, 256)), dim3(256), 0, (const int32_t*)D.ent_node, (const double*)D.zbuf,
           e0, e1, x);
    CF_LAUNCHED();
  }


  // exchange after the Cartesian sweep: none when the wide-halo cut sweeps
  // follow (they start with their own wide exchange), else the narrow halo
  void cart_done(int l, double* x, int reverse) {
    if (!(lv[l].wide && !reverse)) halo_n(l, x);
  }

  // the TMA / tensor-core fused sweep with TC x TC cell tiles (see cart_fused)
  template <int P, int TC, int TCX = TC>
  void cart_fused_tma(int l, double* x, const double* b, int reverse) {
    LevelData& D = lv[l];
    constexpr int NT = P >= 3 ? 128 : (TC >= 32 ? CF_CART_NT32 : 256);   // (Q3: 152 registers of G fragments per thread)
    const double* G = host::cart_map(P);
    using S = CartTmaSmem<P, TC, TCX>;
    const CUtensorMap tmx = host::lattice_tmap(x, D.a.nl, D.a.ld, S::RWP, S::RW);
    const CUtensorMap tmb = host::lattice_tmap(b, D.a.nl, D.a.ld, S::RWP, S::RW);
    static const char cap_key = 0;   // per-device attribute + occupancy (dev_cached)
    const int cap = (int)dev_cached(&cap_key, [&] {
      CF_CUDA(cudaFuncSetAttribute(k_cart_fused_tma<P, TC, NT, TCX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::bytes));
      CF_CUDA(cudaFuncSetAttribute(k_cart_fused_tma<P, TC, NT, TCX>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
      return coresident(k_cart_fused_tma<P, TC, NT, TCX>, S::bytes, NT);
    });
    if (verbose) {
      std::fprintf(stderr, "[cutfem] level %d: %d fused tiles (%d ext), %d co-resident -> %s\n", l,
                   D.n_fused_tiles, D.n_fused_ext, cap, (!cart_split && D.n_fused_tiles <= cap) ? "in place" : "split");
    }
    // forward step followed by the one-launch cut sweep: its patch maps go towards
    // L2 while the Cartesian sweep runs (the sweep streams them right after)
    const bool pf = !reverse && one_sweep && D.sw[0].ok && D.gmap && (!D.part || D.wide);
    const unsigned char* pfp = pf ? (const unsigned char*)D.gmap : nullptr;
    const unsigned long long pfb = pf ? (unsigned long long)D.n_gmap * 8ull : 0ull;
    if (!cart_split && D.n_fused_tiles <= cap) {
      launch_ex(true, k_cart_fused_tma<P, TC, NT, TCX>, dim3(D.n_fused_tiles), dim3(NT), S::bytes, tmx, tmb, D.a,
                (const int*)D.fused_tiles, (const uint8_t*)D.vkind, G, x, reverse, 0, 4, D.tflag, D.tflag_stride, pfp,
                pfb, D.fpl && D.fpl_maxp == S::maxp ? (const int*)D.fpl + (size_t)(reverse ? 1 : 0) * D.fpl_nt * 4 * D.fpl_maxp
                                                    : (const int*)nullptr,
                (const int*)D.fpc + (size_t)(reverse ? 1 : 0) * D.fpl_nt * 4, D.fpl_tx);
      CF_LAUNCHED();
      cart_done(l, x, reverse);
      return;
    }
    const CUtensorMap tms = host::lattice_tmap(D.xs, D.a.nl, D.a.ld, S::RWP, S::RW);
    if (D.n_fused_ext)
      launch(k_cart_fused_tma<P, TC, NT, TCX>, dim3(D.n_fused_ext), dim3(NT), S::bytes, tmx, tmb, D.a,
             (const int*)D.fused_ext, (const uint8_t*)D.vkind, G, D.xs, reverse, 0, 2, (unsigned*)nullptr, 0, pfp, pfb,
             (const int*)nullptr, (const int*)nullptr, 0);
    CF_LAUNCHED();
    halo_n(l, D.xs);
    launch(k_cart_fused_tma<P, TC, NT, TCX>, dim3(D.n_fused_tiles), dim3(NT), S::bytes, tms, tmb, D.a,
           (const int*)D.fused_tiles, (const uint8_t*)D.vkind, G, x, reverse, 2, 4, (unsigned*)nullptr, 0,
           (const unsigned char*)nullptr, 0ull, (const int*)nullptr, (const int*)nullptr, 0);
    CF_LAUNCHED();
    cart_done(l, x, reverse);
    return;
  }

  // all four Cartesian colours in one launch (temporal blocking); p <= 3 on
  // the fp64 tensor cores (dense patch map), p = 4 by fast diagonalisation.
  // The sweep is in place: a cooperative launch whose grid barrier orders
  // every CTA's region load before any write.  When the tiles do not fit on
  // the device at once (or CUTFEM_CART_SPLIT=1) the TMA sweep runs as two
  // launches through the shadow buffer xs (passes 0-1: x -> xs over the tiles
  // dilated by one tile, passes 2-3: xs -> x); the other variants fall back to
  // one launch per colour.
  void cart_fused(int l, double* x, const double* b, int reverse) {
    LevelData& D = lv[l];
    if (!D.n_fused_tiles) return;
    CF_DISPATCH(prm.p, {
      if constexpr (P == 2) {
        if (D.tc == 8) {
          cart_fused_tma<P, 8>(l, x, b, reverse);
          return;
        }
        if (D.tc == 32) {
          if (D.tcx == 16) cart_fused_tma<P, 32, 16>(l, x, b, reverse);
          else if (D.tcx == 24) cart_fused_tma<P, 32, 24>(l, x, b, reverse);
          else cart_fused_tma<P, 32, 32>(l, x, b, reverse);
          return;
        }
      }
      constexpr int TC = fused_tc<P>();
      if constexpr (P <= 3) {
        if (use_mma && use_tma && D.a.nl >= CartTmaSmem<P, TC>::RW && D.a.ld >= CartTmaSmem<P, TC>::RWP) {
          cart_fused_tma<P, TC>(l, x, b, reverse);
          return;
        }
        if (use_mma) {
          const double* G = host::cart_map(P);
          const size_t smb = CartMMASmem<P, TC>::doubles * sizeof(double) + CartMMASmem<P, TC>::ints * sizeof(int);
          static const char cap_key = 0;   // per-device attribute + occupancy (dev_cached)
          const int cap = (int)dev_cached(&cap_key, [&] {
            CF_CUDA(cudaFuncSetAttribute(k_cart_fused_mma<P, TC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb));
            return coresident(k_cart_fused_mma<P, TC>, smb);
          });
          if (!cart_split && D.n_fused_tiles <= cap) {
            launch_ex(true, k_cart_fused_mma<P, TC>, dim3(D.n_fused_tiles), dim3(256), smb, D.a,
                      (const int*)D.fused_tiles, (const uint8_t*)D.vkind, G, x, b, reverse, 1);
            CF_LAUNCHED();
            cart_done(l, x, reverse);
            return;
          }
          for (int s = 0; s < 4; ++s) {
            cart_step(l, reverse ? 3 - s : s, x, b);
            if (s < 3) halo_n(l, x);
          }
          cart_done(l, x, reverse);
          return;
        }
      }
      const size_t smb = CartFusedSmem<P, TC>::doubles * sizeof(double);
      static const char cap2_key = 0;   // per-device attribute + occupancy (dev_cached)
      const int cap2 = (int)dev_cached(&cap2_key, [&] {
        CF_CUDA(cudaFuncSetAttribute(k_cart_fused<P, TC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb));
        return coresident(k_cart_fused<P, TC>, smb);
      });
      if (!cart_split && D.n_fused_tiles <= cap2) {
        launch_ex(true, k_cart_fused<P, TC>, dim3(D.n_fused_tiles), dim3(256), smb, D.a, (const int*)D.fused_tiles,
                  (const uint8_t*)D.vkind, x, b, reverse, 1);
        CF_LAUNCHED();
        cart_done(l, x, reverse);
        return;
      }
      for (int s = 0; s < 4; ++s) {
        cart_step(l, reverse ? 3 - s : s, x, b);
        if (s < 3) halo_n(l, x);
      }
      cart_done(l, x, reverse);
    });
  }

  // one ping-pong cut step: read R, write W (k_cut_step); prev = colour of the
  // previous step (4 = first step of the sweep: copy the read band)
  void cut_pp_step(int l, int c, int prev, const double* R, double* W, const double* b) {
    LevelData& D = lv[l];
    const int np = D.act_off[c + 1] - D.act_off[c];
    const int ncopy = prev < 0 ? 0 : D.copy_n[prev][c];
    const int32_t* cl = D.copy_lists + (prev < 0 ? 0 : D.copy_off[prev][c]);
    cut_pp_launch(l, (const CutDesc*)D.act_desc + D.act_off[c], np, cl, ncopy, R, W, b);
  }
  // one ping-pong cut step over the patches desc[0..np) with the copy list cl[0..ncopy)
  void cut_pp_launch(int l, const CutDesc* desc, int np, const int32_t* cl, int ncopy, const double* R, double* W,
                     const double* b) {
    LevelData& D = lv[l];
    if (!np && !ncopy) return;
    if (D.gmap && cut_map && prm.cut_mode == 0 && cta_cut) {
      CF_DISPATCH(prm.p, {
        if constexpr (P <= 3) {
#ifndef CF_CUT7_NT
#define CF_CUT7_NT 128   // threads per cut patch (p <= 2); 64: V-cycle 671 vs 660 us
#endif
          constexpr int NT = P <= 2 ? CF_CUT7_NT : 128;
          const size_t smb = CutMapSmem<P>::bytes;
          static const char attr7_key = 0;   // per-device attribute (dev_once)
          dev_once(&attr7_key, [&] {
            CF_CUDA(cudaFuncSetAttribute(k_cut_step7<P, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb));
          });
          launch(k_cut_step7<P, NT>, dim3(np + ceil_div(ncopy, NT)), dim3(NT), smb, D.a, desc, np,
                 (const double*)D.gmap, R, W, b, cl, ncopy);
          CF_LAUNCHED();
          return;
        }
      });
    }
    CF_DISPATCH(prm.p, {
      if (prm.cut_mode == 0 && cta_cut) {
        constexpr int NT = 64;
        const int cb = ceil_div(ncopy, NT);
        static const char attr6_key = 0;   // per-device attribute (dev_once)
        dev_once(&attr6_key, [&] {
          CF_CUDA(cudaFuncSetAttribute(k_cut_step6<P, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        });
        launch(k_cut_step6<P, NT>, dim3(np + cb), dim3(NT), (size_t)CutGroup6<P>::bytes, D.a, desc, np,
               (const double*)D.ecut, (const double*)D.inv, R, W, b, cl, ncopy);
      } else {
        const size_t pw = CutSmem3<P>::per_warp * sizeof(double);
        const int wpb = (int)std::max<size_t>(1, std::min<size_t>(4, (96 * 1024) / pw));
        const size_t smb = wpb * pw;
        static const char attr_key = 0;   // per-device attribute (dev_once)
        dev_once(&attr_key, [&] {
          CF_CUDA(cudaFuncSetAttribute(k_cut_step<P, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
          CF_CUDA(cudaFuncSetAttribute(k_cut_step<P, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        });
        const int pb = ceil_div(np, wpb), cb = ceil_div(ncopy, 128);
        if (prm.cut_mode == 0)
          launch(k_cut_step<P, false>, dim3(pb + cb), dim3(128), smb, D.a, desc, np, wpb, pb, (const double*)D.ecut,
                 (const double*)D.inv, R, W, b, cl, ncopy);
        else
          launch(k_cut_step<P, true>, dim3(pb + cb), dim3(128), smb, D.a, desc, np, wpb, pb, (const double*)D.ecut,
                 (const double*)D.inv, R, W, b, cl, ncopy);
      }
    });
    CF_LAUNCHED();
  }





  void cut_sweeps(int l, double* x, const double* b, int reverse) {
    double* bufs[2] = {x, lv[l].xs};
    LevelData& D = lv[l];
    if (comm && D.wide && one_sweep && D.sw[reverse ? 1 : 0].ok) {
      // wide halo: one exchange, the one-launch sweep over the rank's owned
      // nodes and their cones, then the narrow halo
      halo(l, x);
      const LevelData::Sweep& W = D.sw[reverse ? 1 : 0];
      SweepArgs A;
      std::memcpy(&A, W.args, sizeof(A));
      launch_ex(true, k_cut_sweep, dim3(W.ncta), dim3(32 * (SW_NW + 1)), W.smem, A, x, b);
      CF_LAUNCHED();
      halo_n(l, x);
      return;
    }
    if (comm && D.wide) {
      // wide halo: one exchange, then every step on the rank's shrinking
      // redundant patch sets (partition()), then the narrow halo
      halo(l, x);
      const int d = reverse ? 1 : 0, S = 4 * prm.n_c;
      for (int s = 0; s < S; ++s)
        cut_pp_launch(l, (const CutDesc*)D.wdesc + D.wd_off[d][s], D.wd_off[d][s + 1] - D.wd_off[d][s],
                      D.wcopy + D.wc_off[d][s], D.wc_n[d][s], bufs[s & 1], bufs[(s + 1) & 1], b);
      halo_n(l, x);
      return;
    }
    if ((!comm || !D.part) && one_sweep && D.sw[reverse ? 1 : 0].ok) {   // the whole cut sweep in one launch (sweep.cuh)
      const LevelData::Sweep& W = D.sw[reverse ? 1 : 0];
      SweepArgs A;
      std::memcpy(&A, W.args, sizeof(A));
      launch_ex(true, k_cut_sweep, dim3(W.ncta), dim3(32 * (SW_NW + 1)), W.smem, A, x, b);   // co-resident (ticket wait)
      CF_LAUNCHED();
      return;
    }
    int prev = 4, s = 0;
    for (int rep = 0; rep < prm.n_c; ++rep)
      for (int cc = 0; cc < 4; ++cc, ++s) {
        const int c = reverse ? 3 - cc : cc;
        cut_pp_step(l, c, prev, bufs[s & 1], bufs[(s + 1) & 1], b);
        halo_n(l, bufs[(s + 1) & 1]);
        prev = c;
      }
  }

  // halo exchange of a lattice vector of a partitioned level (no-op
  // otherwise): the level's halo (wide on wide levels) / the narrow one
  void halo(int l, double* v) {
    if (comm && lv[l].part) comm->exchange(v, lv[l].halo, st);
  }
  void halo_n(int l, double* v) {
    if (comm && lv[l].part) comm->exchange(v, lv[l].halo_n, st);
  }

  // x <- S(x, b) (P eq. smoother-split, l.196-210; reverse = adjoint order, R9)
  void smooth(int l, double* x, const double* b, int reverse) {
    if (prm.dim == 3) {
      smooth3(l, x, b, reverse);
      return;
    }
    if (lv[l].part) {   // slab partition: fused Cartesian sweep + ping-pong cut steps, halo after each write
      if (!reverse) cart_fused(l, x, b, 0);
      cut_sweeps(l, x, b, reverse);
      if (reverse) cart_fused(l, x, b, 1);
      return;
    }
    if (pingpong && fused) {
      if (!reverse) cart_fused(l, x, b, 0);
      cut_sweeps(l, x, b, reverse);
      if (reverse) cart_fused(l, x, b, 1);
      return;
    }
    if (fused) {
      if (!reverse) cart_fused(l, x, b, 0);
      for (int rep = 0; rep < prm.n_c; ++rep)
        for (int c = 0; c < 4; ++c) cut_step(l, reverse ? 3 - c : c, x, b);
      if (reverse) cart_fused(l, x, b, 1);
      return;
    }
    std::vector<std::pair<int, int>> seq;
    for (int c = 0; c < 4; ++c) seq.push_back({0, c});
    for (int rep = 0; rep < prm.n_c; ++rep)
      for (int c = 0; c < 4; ++c) seq.push_back({1, c});
    if (reverse) std::reverse(seq.begin(), seq.end());
    for (auto& s : seq) {
      if (s.first == 0) cart_step(l, s.second, x, b);
      else cut_step(l, s.second, x, b);
    }
  }

  void restrict_(int l, const double* rf, double* bc, double* xz = nullptr) {
    const LevelArgs &Lf = lv[l].a, &Lc = lv[l - 1].a;
    if (prm.dim == 3) {
      const int64_t nv = (int64_t)Lc.nl * Lc.nl * Lc.ld;
      const LevelData& F = lv[l];
      const int64_t ps = (int64_t)Lc.nl * Lc.ld;
      const int64_t o0 = F.part ? F.rc0 * ps : 0, o1 = F.part ? F.rc1 * ps : nv;
      CF_DISPATCH3(prm.p, (k_restrict3<P><<<ceil_div(o1 - o0, 128), 128, 0, st>>>(Lf, Lc, rf, bc, o0, o1)));
      CF_LAUNCHED();
      return;
    }
    const LevelData& F = lv[l];
    const int row0 = F.part ? F.rc0 : 0, row1 = F.part ? F.rc1 : Lc.nl;
    CF_DISPATCH(prm.p, launch(k_restrict<P>, dim3(ceil_div(Lc.ld, 32), ceil_div(row1 - row0, 8)), dim3(32, 8), 0, Lf,
                              Lc, rf, bc, row0, row1, xz));
    CF_LAUNCHED();
  }
  void prolongate_add(int l, const double* xc, double* xf) {
    const LevelArgs &Lf = lv[l].a, &Lc = lv[l - 1].a;
    if (prm.dim == 3) {
      const int64_t nv = (int64_t)Lf.nl * Lf.nl * Lf.ld;
      const LevelData& F = lv[l];
      const int64_t ps = (int64_t)Lf.nl * Lf.ld;
      const int64_t o0 = F.part ? F.v0n * ps : 0, o1 = F.part ? F.v1n * ps : nv;
      CF_DISPATCH3(prm.p, (k_prolongate_add3<P><<<ceil_div(o1 - o0, 128), 128, 0, st>>>(Lf, Lc, xc, xf, o0, o1)));
      CF_LAUNCHED();
      return;
    }
    const LevelData& F = lv[l];
    const int row0 = F.part ? F.v0n : 0, row1 = F.part ? F.v1n : Lf.nl;
    CF_DISPATCH(prm.p, launch(k_prolongate_add<P>, dim3(ceil_div(Lf.nl, 32), ceil_div(row1 - row0, 8)), dim3(32, 8), 0,
                              Lf, Lc, xc, xf, row0, row1));
    CF_LAUNCHED();
  }
  void coarse_solve(const double* b, double* x) {
    k_coarse_solve<<<1, 256, n0 * sizeof(double), st>>>(c_inv, c_nodes, n0, b, x);
    CF_LAUNCHED();
  }


  // V-cycle on level l with initial guess x (P l.124, l.217)
  void vcycle(int l, double* x, const double* b) {
    if (l == 0) {
      coarse_solve(b, x);
      return;
    }
    LevelData& D = lv[l];
    LevelData& C = lv[l - 1];
    smooth(l, x, b, 0);
    apply(l, x, D.r, b);
    // the restriction also zeroes the coarse initial guess (no memset node
    // between the kernels, which would break the programmatic launch chain)
    const bool zero_in_restrict = !D.part && prm.dim == 2;
    restrict_(l, D.r, C.b, zero_in_restrict ? C.x : nullptr);
    if (D.part) {
      if (C.part) halo(l - 1, C.b);
      else replicate(l - 1, C.b, D.rc0, D.rc1);   // the coarse levels run on every rank
    }
    if (!zero_in_restrict) CF_CUDA(cudaMemsetAsync(C.x, 0, vsize(l - 1) * 8, st));
    vcycle(l - 1, C.x, C.b);
    prolongate_add(l, C.x, x);
    smooth(l, x, b, prm.symmetric ? 1 : 0);
  }

  // run `body` through a cached CUDA graph keyed by (tag, ptrs)
  template <class F>
  void graphed(int tag, const void* p1, const void* p2, int extra, F&& body) {
    if (comm) {   // the halo exchanges synchronise ranks on the host (LocalComm): no capture
      body();
      return;
    }
    auto key = std::make_tuple(tag, p1, p2, extra);
    auto it = graphs.find(key);
    if (it == graphs.end()) {
      // capture on a private stream (the legacy default stream cannot be
      // captured); the instantiated graph is launched on the caller's stream
      if (!cap_st) CF_CUDA(cudaStreamCreateWithFlags(&cap_st, cudaStreamNonBlocking));
      cudaStream_t user = st;
      st = cap_st;
      int64_t before = g_launches;
      cudaGraph_t g;
      CF_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      try {
        body();
      } catch (...) {
        cudaStreamEndCapture(st, &g);
        st = user;
        throw;
      }
      st = user;
      CF_CUDA(cudaStreamEndCapture(cap_st, &g));
      GraphRec rec;
      CF_CUDA(cudaGraphInstantiate(&rec.exec, g, 0));
      cudaGraphDestroy(g);
      rec.launches = g_launches - before;
      g_launches = before;
      it = graphs.emplace(key, rec).first;
    }
    CF_CUDA(cudaGraphLaunch(it->second.exec, st));
    g_launches += it->second.launches;
  }

  // doubles in a lattice vector of level l
  int64_t vsize(int l) const {
    const LevelArgs& L = lv[l].a;
    return (int64_t)L.nl * L.ld * (prm.dim == 3 ? L.nl : 1);
  }

  void dot(const double* a, const double* b, int mode, int slot) {
    const LevelData& F = lv[prm.n_levels - 1];
    if (comm && F.part) {   // owned rows, then the sum over ranks
      const int64_t rs = rowsz(prm.n_levels - 1), o = F.r0 * rs, n = (F.r1 - F.r0) * rs;
      k_dot_partial<<<DOT_BLOCKS, DOT_THREADS, 0, st>>>(a + o, b + o, n, part);
      CF_LAUNCHED();
      k_dot_final<<<1, DOT_THREADS, 0, st>>>(part, sc, 0, 7);
      CF_LAUNCHED();
      comm->allreduce_sum(sc + 7, 1, st);
      k_dot_mode<<<1, 1, 0, st>>>(sc, mode, slot);
      CF_LAUNCHED();
      return;
    }
    k_dot_partial<<<DOT_BLOCKS, DOT_THREADS, 0, st>>>(a, b, vsize(prm.n_levels - 1), part);
    CF_LAUNCHED();
    k_dot_final<<<1, DOT_THREADS, 0, st>>>(part, sc, mode, slot);
    CF_LAUNCHED();
  }

  // v (a replicated level) <- sum over ranks of the rows [r0, r1) each rank computed
  void replicate(int l, double* v, int r0, int r1) {
    const LevelArgs& L = lv[l].a;
    const int64_t rs = rowsz(l);
    if (r0 > 0) CF_CUDA(cudaMemsetAsync(v, 0, (size_t)(r0 * rs) * 8, st));
    if (r1 < L.nl) CF_CUDA(cudaMemsetAsync(v + r1 * rs, 0, (size_t)((L.nl - r1) * rs) * 8, st));
    comm->allreduce_sum(v, vsize(l), st);
  }

  // ================================================================ 3D
  void setup_mesh3() {
    host::upload_tables();
    host::cart_map3(prm.p);
    d_count = alloc<int>(1);
    const int p = prm.p;
    lv.resize(prm.n_levels);
    for (int l = 0; l < prm.n_levels; ++l) {
      LevelData& D = lv[l];
      LevelArgs& L = D.a;
      std::memset(&L, 0, sizeof(L));
      L.dim = 3;
      L.n = prm.n_coarse << l;
      L.p = p;
      L.fitted = prm.domain == 1;
      L.nl = L.n * p + 1;
      L.ld = (L.nl + 1) & ~1;
      L.h = prm.length / L.n;
      L.x0 = prm.x0;
      L.y0 = prm.y0;
      L.z0 = prm.z0;
      L.cx = prm.cx;
      L.cy = prm.cy;
      L.cz = prm.cz;
      L.r = prm.r;
      L.gDh = prm.gamma_D / L.h;
      for (int k = 1; k <= p; ++k) {
        double f = 1.0;
        for (int q = 2; q <= k; ++q) f *= q;
        L.gs[k] = prm.gamma_k[k - 1] * std::pow(L.h, prm.sigma + 2) / (f * f);
      }
      const int n = L.n;
      const int64_t n3 = (int64_t)n * n * n, nv = vsize(l);
      D.ctype = alloc<int8_t>(n3);
      k_classify3<<<ceil_div(n3, 256), 256, 0, st>>>(L, D.ctype);
      CF_LAUNCHED();
      L.ctype = D.ctype;
      D.mask = alloc<uint8_t>(nv);
      CF_CUDA(cudaMemsetAsync(d_count, 0, sizeof(int), st));
      k_mask3<<<ceil_div(nv, 256), 256, 0, st>>>(L, D.ctype, D.mask, d_count);
      CF_LAUNCHED();
      L.mask = D.mask;
      D.n_dofs = read_count();
      require(D.n_dofs > 0, ERR_GEOMETRY, "a level has no DoF: the domain does not meet the background box");
      if (l > 0) {
        CF_CUDA(cudaMemsetAsync(d_count, 0, sizeof(int), st));
        k_parent_check3<<<ceil_div(n3, 256), 256, 0, st>>>(L, lv[l - 1].a, d_count);
        CF_LAUNCHED();
        require(read_count() == 0, ERR_GEOMETRY, "a fine active cell has an inactive parent");
      }
      uint8_t* flags = alloc<uint8_t>(3 * n3);
      int* tmpi = alloc<int>(3 * n3);
      k_cell_flags<<<ceil_div(n3, 256), 256, 0, st>>>(n3, D.ctype, INSIDE, flags);
      CF_LAUNCHED();
      D.n_inside = select(flags, (int)n3, tmpi);
      k_cell_flags<<<ceil_div(n3, 256), 256, 0, st>>>(n3, D.ctype, CUT, flags);
      CF_LAUNCHED();
      L.n_cut = select(flags, (int)n3, tmpi);
      D.cut_list = alloc<int>(L.n_cut);
      CF_CUDA(cudaMemcpyAsync(D.cut_list, tmpi, sizeof(int) * L.n_cut, cudaMemcpyDeviceToDevice, st));
      L.cut_list = D.cut_list;
      D.cut_id = alloc<int>(n3);
      k_fill<<<ceil_div(n3, 256), 256, 0, st>>>(D.cut_id, n3, -1);
      CF_LAUNCHED();
      if (L.n_cut) {
        k_scatter_id<<<ceil_div(L.n_cut, 256), 256, 0, st>>>(D.cut_list, L.n_cut, D.cut_id);
        CF_LAUNCHED();
      }
      L.cut_id = D.cut_id;
      k_ghost_flags3<<<ceil_div(3 * n3, 256), 256, 0, st>>>(L, flags);
      CF_LAUNCHED();
      L.n_ghost = select(flags, (int)(3 * n3), tmpi);
      D.ghost_list = alloc<int>(L.n_ghost);
      CF_CUDA(cudaMemcpyAsync(D.ghost_list, tmpi, sizeof(int) * L.n_ghost, cudaMemcpyDeviceToDevice, st));
      L.ghost_list = D.ghost_list;
      D.gx_id = alloc<int>(n3);
      D.gy_id = alloc<int>(n3);
      D.gz_id = alloc<int>(n3);
      for (int* m : {D.gx_id, D.gy_id, D.gz_id}) {
        k_fill<<<ceil_div(n3, 256), 256, 0, st>>>(m, n3, -1);
        CF_LAUNCHED();
      }
      if (L.n_ghost) {
        k_ghost_maps3<<<ceil_div(L.n_ghost, 256), 256, 0, st>>>(D.ghost_list, L.n_ghost, n, D.gx_id, D.gy_id, D.gz_id);
        CF_LAUNCHED();
      }
      L.gx_id = D.gx_id;
      L.gy_id = D.gy_id;
      L.gz_id = D.gz_id;
      D.q_off = alloc<int>(L.n_cut + 1);
      D.s_off = alloc<int>(L.n_cut + 1);
      int* vc = tmpi;
      int* scn = tmpi + n3;
      if (L.n_cut) {
        k_cut_count3<<<ceil_div(L.n_cut, 64), 64, 0, st>>>(L, prm.n_q, vc, scn);
        CF_LAUNCHED();
      }
      D.n_vq = scan32(vc, L.n_cut, D.q_off);
      D.n_sq = scan32(scn, L.n_cut, D.s_off);
      L.q_off = D.q_off;
      L.s_off = D.s_off;
      D.qbuf = alloc<double>(4 * D.n_vq);
      D.sbuf = alloc<double>(7 * D.n_sq);
      QPtrs3 QP;
      for (int d = 0; d < 4; ++d) QP.q[d] = D.qbuf + d * D.n_vq;
      for (int d = 0; d < 7; ++d) QP.s[d] = D.sbuf + d * D.n_sq;
      L.qx = QP.q[0]; L.qy = QP.q[1]; L.qz = QP.q[2]; L.qw = QP.q[3];
      L.sx = QP.s[0]; L.sy = QP.s[1]; L.sz = QP.s[2]; L.sw = QP.s[3];
      L.snx = QP.s[4]; L.sny = QP.s[5]; L.snz = QP.s[6];
      if (L.n_cut) {
        k_cut_fill3<<<ceil_div(L.n_cut, 64), 64, 0, st>>>(L, prm.n_q, QP);
        CF_LAUNCHED();
      }
      const int NB = (p + 1) * (p + 1) * (p + 1);
      D.ecut = alloc<double>((int64_t)L.n_cut * NB * NB);
      L.ecut = D.ecut;
      if (L.n_cut) {
        CF_DISPATCH3(p, (k_cut_elem3<P><<<ceil_div((int64_t)L.n_cut * NB, 4), 128, 0, st>>>(L, D.ecut)));
        CF_LAUNCHED();
      }
      D.ycut = alloc<double>((int64_t)L.n_cut * NB);
      D.jm = alloc<double>((int64_t)L.n_ghost * p * (p + 1) * (p + 1));
      L.ycut = D.ycut;
      L.jm = D.jm;
      D.x = alloc<double>(nv);
      D.b = alloc<double>(nv);
      D.r = alloc<double>(nv);
      for (double* v : {D.x, D.b, D.r}) CF_CUDA(cudaMemsetAsync(v, 0, nv * 8, st));
      sync();
      cudaFree(flags);
      cudaFree(tmpi);
      allocs.erase(std::remove(allocs.begin(), allocs.end(), (void*)flags), allocs.end());
      allocs.erase(std::remove(allocs.begin(), allocs.end(), (void*)tmpi), allocs.end());
    }
  }

  void build_patches3() {
    const int p = prm.p;
    for (int l = 0; l < prm.n_levels; ++l) {
      LevelData& D = lv[l];
      LevelArgs& L = D.a;
      const int n = L.n;
      const int64_t nvt = (int64_t)(n + 1) * (n + 1) * (n + 1);
      D.vkind = alloc<uint8_t>(nvt);
      k_vertex_kind3<<<ceil_div(nvt, 256), 256, 0, st>>>(L, D.vkind);
      CF_LAUNCHED();
      uint8_t* fl = alloc<uint8_t>(nvt);
      int* tmpi = alloc<int>(nvt);
      for (int kind = V_CART; kind <= V_CUT; ++kind) {
        int* off = kind == V_CART ? D.cart_off : D.cutp_off;
        int* cnt = kind == V_CART ? D.n_cart : D.n_cutp;
        off[0] = 0;
        std::vector<int> hostlists;
        for (int c = 0; c < 8; ++c) {
          k_vertex_flags3<<<ceil_div(nvt, 256), 256, 0, st>>>(n, D.vkind, (uint8_t)kind, c, fl);
          CF_LAUNCHED();
          cnt[c] = select(fl, (int)nvt, tmpi);
          std::vector<int> h(cnt[c]);
          if (cnt[c]) CF_CUDA(cudaMemcpyAsync(h.data(), tmpi, sizeof(int) * cnt[c], cudaMemcpyDeviceToHost, st));
          sync();
          hostlists.insert(hostlists.end(), h.begin(), h.end());
          off[c + 1] = off[c] + cnt[c];
        }
        int* dl = alloc<int>(hostlists.size());
        if (!hostlists.empty())
          CF_CUDA(cudaMemcpyAsync(dl, hostlists.data(), sizeof(int) * hostlists.size(), cudaMemcpyHostToDevice, st));
        (kind == V_CART ? D.cart_list : D.cutp_list) = dl;
      }
      const int ncp = D.cutp_off[8];
      int* mcount = alloc<int>(ncp);
      D.cutp_ent = alloc<int64_t>(ncp + 1);
      if (ncp) {
        k_cut_interior3<false><<<ceil_div(ncp, 64), 64, 0, st>>>(L, D.cutp_list, ncp, mcount, nullptr, nullptr,
                                                                  nullptr, nullptr);
        CF_LAUNCHED();
      }
      D.n_ent = scan64(mcount, ncp, D.cutp_ent);
      for (int c = 0; c <= 8; ++c) {
        D.ent_col_off[c] = 0;
        if (ncp) CF_CUDA(cudaMemcpyAsync(&D.ent_col_off[c], D.cutp_ent + D.cutp_off[c], sizeof(int64_t),
                                         cudaMemcpyDeviceToHost, st));
      }
      sync();
      D.ent_node = alloc<int32_t>(D.n_ent);
      D.ent_loc = alloc<uint16_t>(D.n_ent);
      D.ent_patch = alloc<int32_t>(D.n_ent);
      D.zbuf = alloc<double>(D.n_ent);
      if (ncp) {
        k_cut_interior3<true><<<ceil_div(ncp, 64), 64, 0, st>>>(L, D.cutp_list, ncp, nullptr, D.cutp_ent, D.ent_node,
                                                                 D.ent_loc, D.ent_patch);
        CF_LAUNCHED();
      }
      // local matrices and their inverses (P l.193, R10).  Dense m x m
      // (default, coalesced apply) unless they would take more than 35 % of the
      // free device memory (3D Q3 at 256^3): then they are built in chunks of
      // <= 2 GB of dense matrices and packed symmetric (k_pack_sym, m (m+1) / 2
      // doubles per patch; env CUTFEM_SYM_PACKED=1 forces it)
      D.cutp_inv = alloc<int64_t>(ncp + 1);
      std::vector<int> hm(ncp);
      if (ncp) CF_CUDA(cudaMemcpyAsync(hm.data(), mcount, sizeof(int) * ncp, cudaMemcpyDeviceToHost, st));
      sync();
      std::vector<int64_t> hpk(ncp + 1, 0), hfull(ncp + 1, 0), hent(ncp + 1, 0);
      int mmax = 0;
      for (int k = 0; k < ncp; ++k) {
        hpk[k + 1] = hpk[k] + (int64_t)hm[k] * (hm[k] + 1) / 2;
        hfull[k + 1] = hfull[k] + (int64_t)hm[k] * hm[k];
        hent[k + 1] = hent[k] + hm[k];
        mmax = std::max(mmax, hm[k]);
      }
      size_t mfree = 0, mtot = 0;
      CF_CUDA(cudaMemGetInfo(&mfree, &mtot));
      const bool packed = sym_packed || (double)hfull[ncp] * 8.0 > 0.35 * (double)mfree;
      L.sym_packed = packed;
      const std::vector<int64_t>& hoff = packed ? hpk : hfull;
      if (ncp) CF_CUDA(cudaMemcpy(D.cutp_inv, hoff.data(), sizeof(int64_t) * (ncp + 1), cudaMemcpyHostToDevice));
      D.n_inv = hoff[ncp];
      D.inv = alloc<double>(D.n_inv);
      if (D.n_ent) {
        int mfit = 1;   // local inverses in shared memory up to m = 160 (200 KB), larger ones in global memory
        while ((size_t)((mfit + 1) * (mfit + 1) + 2 * (mfit + 1)) * sizeof(double) <= 200 * 1024) ++mfit;
        const int msm = std::min(mmax, mfit);
        const size_t smb = (size_t)(msm * msm + 2 * msm) * sizeof(double);
        CF_CUDA(cudaFuncSetAttribute(k_batched_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)std::max<size_t>(smb, 48 * 1024)));
        // dense: one chunk built in place in D.inv; packed: chunks through a scratch buffer
        const int64_t CHUNK = packed ? (256ll << 20) : hfull[ncp] + 1;   // doubles of dense matrices per chunk
        int64_t maxfull = 0;
        for (int k0 = 0, k1; k0 < ncp; k0 = k1) {
          for (k1 = k0 + 1; k1 < ncp && hfull[k1 + 1] - hfull[k0] <= CHUNK; ++k1) {
          }
          maxfull = std::max(maxfull, hfull[k1] - hfull[k0]);
        }
        double* full = packed ? alloc<double>(maxfull) : D.inv;
        int64_t* foff = alloc<int64_t>(ncp + 1);
        std::vector<int64_t> hf(ncp + 1);
        for (int k0 = 0, k1; k0 < ncp; k0 = k1) {
          for (k1 = k0 + 1; k1 < ncp && hfull[k1 + 1] - hfull[k0] <= CHUNK; ++k1) {
          }
          const int nk = k1 - k0;
          for (int k = k0; k <= k1; ++k) hf[k - k0] = hfull[k] - hfull[k0];
          CF_CUDA(cudaMemcpyAsync(foff, hf.data(), sizeof(int64_t) * (nk + 1), cudaMemcpyHostToDevice, st));
          const int64_t e_lo = hent[k0], ne = hent[k1] - hent[k0];
          if (ne) {
            CF_DISPATCH3(p, (k_local_matrix3<P><<<ceil_div(ne, 2), 64, 0, st>>>(
                                L, D.cutp_list, D.cutp_ent, D.ent_loc, D.ent_patch, ne, foff, full, prm.cut_mode, e_lo,
                                k0)));
            CF_LAUNCHED();
            k_batched_inverse<<<nk, 256, smb, st>>>(D.cutp_ent + k0, foff, full, nk);
            CF_LAUNCHED();
            if (mmax > mfit) {
              k_batched_inverse_gmem<<<nk, 512, 2 * mmax * sizeof(double), st>>>(D.cutp_ent + k0, foff, full, nk,
                                                                                   mfit + 1);
              CF_LAUNCHED();
            }
            if (packed) {
              k_pack_sym<<<nk, dim3(32, 8), 0, st>>>(D.cutp_ent + k0, foff, full, D.cutp_inv + k0, D.inv, nk);
              CF_LAUNCHED();
            }
          }
          sync();   // foff / full are reused by the next chunk
        }
        for (void* q : {packed ? (void*)full : nullptr, (void*)foff}) {
          if (!q) continue;
          cudaFree(q);
          allocs.erase(std::remove(allocs.begin(), allocs.end(), q), allocs.end());
        }
      }
      D.desc = alloc<CutDesc3>(ncp);
      if (ncp) {
        CF_DISPATCH3(p, (k_cut_desc3<P><<<ceil_div(ncp, 128), 128, 0, st>>>(L, D.cutp_list, ncp, D.cutp_ent, D.ent_loc,
                                                                            D.cutp_inv, (CutDesc3*)D.desc)));
        CF_LAUNCHED();
      }
      if (ncp) method_bytes3(D, ncp);
      D.act_desc = D.desc;
      D.act_cart = D.cart_list;
      D.act_ent = D.ent_node;
      for (int c = 0; c < 9; ++c) {
        D.act_off[c] = D.cutp_off[c];
        D.act_cart_off[c] = D.cart_off[c];
        D.act_ent_off[c] = D.ent_col_off[c];
      }
      sync();
    }
    build_coarse();
    const int64_t nvf = vsize(prm.n_levels - 1);
    cg_x = alloc<double>(nvf);
    cg_r = alloc<double>(nvf);
    cg_z = alloc<double>(nvf);
    cg_p = alloc<double>(nvf);
    cg_q = alloc<double>(nvf);
    part = alloc<double>(DOT_BLOCKS);
    sc = alloc<double>(8);
    if (!sc_host) CF_CUDA(cudaMallocHost(&sc_host, 8 * sizeof(double)));
    for (double* v : {cg_x, cg_r, cg_z, cg_p, cg_q}) CF_CUDA(cudaMemsetAsync(v, 0, nvf * 8, st));
    sync();
    built = true;
  }

  void apply3(int l, const double* x, double* y, const double* b) {
    const LevelData& D = lv[l];
    const LevelArgs& L = D.a;
    BandRange3 R;
    if (D.part) {
      R = BandRange3{D.band3[0], D.band3[1], {D.band3[2], D.band3[3], D.band3[4]}, {D.band3[5], D.band3[6], D.band3[7]}};
    } else {
      // the full ghost list, split by axis is not needed: one range covers it
      R = BandRange3{0, L.n_cut, {0, 0, 0}, {L.n_ghost, 0, 0}};
    }
    const int warps = R.cut_n + ceil_div(R.g_n[0] + R.g_n[1] + R.g_n[2], 32);
    if (warps) {
      CF_DISPATCH3(prm.p, (k_band3<P><<<ceil_div(warps, 4), 128, 0, st>>>(L, x, R)));
      CF_LAUNCHED();
    }
    // under the partition: the lattice planes of the cell planes [c0 - 2, c1 + 2)
    const int64_t ps = (int64_t)L.nl * L.ld;
    const int64_t o0 = D.part ? std::max(0, (D.c0 - 2) * L.p) * ps : 0;
    const int64_t o1 = D.part ? std::min(L.nl, (D.c1 + 2) * L.p + 1) * ps : vsize(l);
    CF_DISPATCH3(prm.p, (k_node_apply3<P><<<ceil_div(o1 - o0, 256), 256, 0, st>>>(L, x, b, y, o0, o1)));
    CF_LAUNCHED();
  }

  void cart_step3(int l, int c, double* x, const double* b) {
    LevelData& D = lv[l];
    const int np = D.act_cart_off[c + 1] - D.act_cart_off[c];
    if (!np) return;
    CF_DISPATCH3(prm.p, (launch(k_cart_colour3<P>, dim3(ceil_div(ceil_div(np, 8), CartMMA3<P>::NW)),
                                dim3(32 * CartMMA3<P>::NW), 0, D.a, (const int*)(D.act_cart + D.act_cart_off[c]), np,
                                host::cart_map3(P), x, b)));
    CF_LAUNCHED();
  }

  void cut_step3(int l, int c, double* x, const double* b) {
    LevelData& D = lv[l];
    const int np = D.act_off[c + 1] - D.act_off[c];
    if (!np) return;
    const int base = D.act_off[c];
    require(!D.part || (prm.cut_mode == 0 && cut3_v >= 2), ERR_STATE, "partitioned 3D levels need the descriptor cut kernels");
    if (prm.cut_mode == 0) {
      if (cut3_v >= 3) {
        CF_DISPATCH3(prm.p, {
          const bool tma3 = use_tma && P == 2;
          CUtensorMap tm;
          std::memset(&tm, 0, sizeof(tm));
          if (tma3) tm = host::lattice_tmap3(x, D.a.nl, D.a.ld, Cut3SmemV3<P, true>::RS, 4 * P + 1, 4 * P + 1);
          static const char attr3_key = 0;   // per-device attribute (dev_once)
          dev_once(&attr3_key, [&] {
            CF_CUDA(cudaFuncSetAttribute(k_cut_colour3v3<P, 128, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
            CF_CUDA(cudaFuncSetAttribute(k_cut_colour3v3<P, 128, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
          });
          if (tma3)
            launch(k_cut_colour3v3<P, 128, true>, dim3(np), dim3(128), Cut3SmemV3<P, true>::bytes, tm, D.a,
                   (const CutDesc3*)D.act_desc + base, np, (const double*)D.inv, (const double*)x, b, D.zbuf);
          else
            launch(k_cut_colour3v3<P, 128, false>, dim3(np), dim3(128), Cut3SmemV3<P, false>::bytes, tm, D.a,
                   (const CutDesc3*)D.act_desc + base, np, (const double*)D.inv, (const double*)x, b, D.zbuf);
        });
      } else
      CF_DISPATCH3(prm.p, {
        const size_t pw = Cut3Smem<P>::per_warp * sizeof(double);
        static const char attr_key = 0;   // per-device attribute (dev_once)
        dev_once(&attr_key, [&] {
          CF_CUDA(cudaFuncSetAttribute(k_cut_colour3v2<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        });
        launch(k_cut_colour3v2<P>, dim3(np), dim3(128), pw, D.a, (const CutDesc3*)D.act_desc + base, np,
               (const double*)D.inv, (const double*)x, b, D.zbuf);
      });
    } else {
      CF_DISPATCH3(prm.p, (launch(k_cut_colour3<P>, dim3(ceil_div(np, 2)), dim3(64), 0, D.a,
                                  (const int*)(D.cutp_list + base), np, base, (const int64_t*)D.cutp_ent,
                                  (const uint16_t*)D.ent_loc, (const int32_t*)D.ent_node, (const int64_t*)D.cutp_inv,
                                  (const double*)D.inv, (const double*)x, b, D.zbuf, prm.cut_mode)));
    }
    CF_LAUNCHED();
    const int64_t e0 = D.act_ent_off[c], e1 = D.act_ent_off[c + 1];
    if (e1 <= e0) return;
    launch(k_cut_apply, dim3(ceil_div(e1 - e0, 256)), dim3(256), 0, (const int32_t*)D.act_ent, (const double*)D.zbuf,
           e0, e1, x);
    CF_LAUNCHED();
  }

  void smooth3(int l, double* x, const double* b, int reverse) {
    std::vector<std::pair<int, int>> seq;
    for (int c = 0; c < 8; ++c) seq.push_back({0, c});
    for (int rep = 0; rep < prm.n_c; ++rep)
      for (int c = 0; c < 8; ++c) seq.push_back({1, c});
    if (reverse) std::reverse(seq.begin(), seq.end());
    for (auto& q : seq) {
      if (q.first == 0) cart_step3(l, q.second, x, b);
      else cut_step3(l, q.second, x, b);
      halo_n(l, x);   // slab partition: one exchange per colour step
    }
  }

  // CG preconditioned by one V-cycle (zero initial guess); x_0 = 0
  void solve_cg(double* x, const double* b, double tol, int max_it, int* iters, double* rel) {
    const int Lf = prm.n_levels - 1;
    LevelData& F = lv[Lf];
    const int64_t nv = vsize(Lf);
    // vector updates and dot products over the owned rows under the slab
    // partition (the dot products are then summed over the ranks)
    const bool dist = comm && F.part;
    const int64_t o = dist ? F.r0 * rowsz(Lf) : 0, no = dist ? (F.r1 - F.r0) * rowsz(Lf) : nv;
    const int grid = 4 * 148;
    k_masked_copy<<<grid, 256, 0, st>>>(cg_r + o, b + o, F.mask + o, no);
    CF_LAUNCHED();
    CF_CUDA(cudaMemsetAsync(cg_x, 0, nv * 8, st));
    dot(cg_r, cg_r, 0, 3);
    CF_CUDA(cudaMemcpyAsync(sc_host, sc, 8 * sizeof(double), cudaMemcpyDeviceToHost, st));
    sync();
    const double r0 = std::sqrt(sc_host[3]);
    int it = 0;
    double rn = r0;
    if (r0 > 0.0) {
      auto precond = [&]() {
        CF_CUDA(cudaMemsetAsync(cg_z, 0, nv * 8, st));
        halo(Lf, cg_r);
        vcycle(Lf, cg_z, cg_r);
      };
      graphed(100, cg_z, cg_r, 0, [&]() {
        precond();
        dot(cg_r, cg_z, 0, 0);
        CF_CUDA(cudaMemcpyAsync(cg_p, cg_z, nv * 8, cudaMemcpyDeviceToDevice, st));
      });
      while (it < max_it) {
        graphed(101, cg_p, cg_q, 0, [&]() {
          halo_n(Lf, cg_p);
          apply(Lf, cg_p, cg_q, nullptr);
          dot(cg_p, cg_q, 1, 0);
          k_cg_update<<<grid, 256, 0, st>>>(cg_x + o, cg_r + o, cg_p + o, cg_q + o, sc, no);
          CF_LAUNCHED();
          dot(cg_r, cg_r, 0, 3);
          CF_CUDA(cudaMemcpyAsync(sc_host, sc, 8 * sizeof(double), cudaMemcpyDeviceToHost, st));
        });
        sync();
        ++it;
        rn = std::sqrt(sc_host[3]);
        if (!(rn > tol * r0)) break;
        graphed(102, cg_z, cg_r, 0, [&]() {
          precond();
          dot(cg_r, cg_z, 2, 0);
          k_cg_direction<<<grid, 256, 0, st>>>(cg_p + o, cg_z + o, sc, no);
          CF_LAUNCHED();
        });
      }
    }
    CF_CUDA(cudaMemcpyAsync(x, cg_x, nv * 8, cudaMemcpyDeviceToDevice, st));
    sync();
    if (iters) *iters = it;
    if (rel) *rel = r0 > 0.0 ? rn / r0 : 0.0;
  }
};

}  // namespace cf
