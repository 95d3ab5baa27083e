// internal.cuh — shared definitions of the CutFEM multigrid CUDA path.
//
// Layout: lattice vectors of a level are NL rows of
// LD doubles, node (a, b) at [b*LD + a]; cells are indexed j*n + i.  The
// per-degree 1D tables live in __constant__ memory (broadcast reads inside
// the sum-factorisation loops); per-level scalars and pointers travel by
// value in LevelArgs.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#define CF_MAXP 4
#define CF_MAXNQ 12

namespace cf {

enum CellType : int8_t { OUTSIDE = 0, INSIDE = 1, CUT = 2 };
enum VertexKind : uint8_t { V_NONE = 0, V_CART = 1, V_CUT = 2 };

// 1D tables of Q_p on the reference interval [0,1] (P l.79), computed on the
// host in tables.cuh and uploaded once per process for p = 1..4.
struct Tab {
  double gll[CF_MAXP + 1];                       // Gauss-Lobatto nodes
  double lc[CF_MAXP + 1][CF_MAXP + 1];           // L_i(xi) = sum_m lc[i][m] xi^m
  double dc[CF_MAXP + 1][CF_MAXP + 1];           // L_i'(xi) = sum_m dc[i][m] xi^m
  double Kref[CF_MAXP + 1][CF_MAXP + 1];         // int_0^1 L_i' L_j'
  double Mref[CF_MAXP + 1][CF_MAXP + 1];         // int_0^1 L_i L_j
  double d0[CF_MAXP + 1][CF_MAXP + 1];           // d0[k][i] = L_i^(k)(0)
  double d1[CF_MAXP + 1][CF_MAXP + 1];           // d1[k][i] = L_i^(k)(1)
  double Kp[2 * CF_MAXP + 1][2 * CF_MAXP + 1];   // two-cell patch stiffness (2p+1 nodes)
  double Mp[2 * CF_MAXP + 1][2 * CF_MAXP + 1];   // two-cell patch mass
  double S[2 * CF_MAXP - 1][2 * CF_MAXP - 1];    // K_int S = M_int S diag(lam), S^T M_int S = I
  double lam[2 * CF_MAXP - 1];
  double tw[CF_MAXP][4 * CF_MAXP + 1];           // restriction: coarse basis of local node m at fine offset d+2p
  double pw[2 * CF_MAXP + 1][CF_MAXP + 1];       // prolongation: L_m at fine offset d in [0,2p] of a coarse cell
};

// single translation unit (capi.cu): the tables are defined here
__constant__ Tab c_tab[CF_MAXP + 1];
__device__ Tab g_tab[CF_MAXP + 1];   // global-memory copy for lane-varying (coalesced) reads
__constant__ double c_gx[CF_MAXNQ + 1][CF_MAXNQ];  // Gauss-Legendre points on [0,1], c_gx[n][i]
__constant__ double c_gw[CF_MAXNQ + 1][CF_MAXNQ];

// PDL: wait until the preceding kernel in the stream has completed (no-op
// when launched without the programmatic-serialization attribute)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
// PDL: allow the next kernel in the stream to be scheduled (its own wait
// still orders it after this kernel's completion)
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// Per-level arguments passed by value to every kernel.
struct LevelArgs {
  int n, p, nl, ld;
  int dim;                           // 2 or 3
  int fitted;                        // fitted box: every cell Inside, no DoF on the box boundary
  int sym_packed;                    // 3D local inverses packed symmetric (k_pack_sym) instead of dense
  int map_one_lane;                  // 2D cut-patch maps summed one lane per row (map_tpr; large levels)
  double h, x0, y0, z0;
  double cx, cy, cz, r;
  double gDh;                        // gamma_D / h
  double gs[CF_MAXP + 1];            // ghost scale gamma_k h^(sigma+1) / (k!)^2 (index k = 1..p)
  const int8_t* ctype;               // n*n
  const uint8_t* mask;               // nl*ld DoF mask
  const int* cut_id;                 // n*n -> cut cell index or -1
  const int* cut_list;               // packed i + n*j
  int n_cut;
  const int* q_off;                  // n_cut+1, volume points
  const double *qx, *qy, *qz, *qw;   // reference coordinates, physical weight
  const int* s_off;                  // n_cut+1, surface points
  const double *sx, *sy, *sz, *sw, *snx, *sny, *snz;
  const int* gx_id;                  // face (i,j)|(i+1,j) -> ghost id or -1, index j*n+i
  const int* gy_id;                  // face (i,j)|(i,j+1)
  const int* gz_id;                  // 3D: face (i,j,k)|(i,j,k+1)
  const uint8_t* ccode;              // 2D: kind | ghost faces left/right/bottom/top << 2..5
  const int* ghost_list;             // packed axis | i << 1 | j << 16... see setup
  int n_ghost;
  double* ycut;                      // n_cut * (p+1)^2 scratch (operator apply)
  double* jm;                        // n_ghost * p * (p+1) scratch (operator apply)
  const double* ecut;                // n_cut * ((p+1)^2)^2 cut-cell matrices (bulk + Nitsche), cut_mode 0
};

// One halo transfer of the slab partition (comm.cuh): rows of a lattice
// vector sent to / received from a neighbouring rank, as double offsets.
struct Xfer {
  int peer;
  int64_t send_off, send_n;   // doubles of my vector sent to `peer` (land at the same offset there)
  int64_t recv_off, recv_n;   // doubles of my vector received from `peer`
};

// Per-level device data owned by the problem.
struct LevelData {
  LevelArgs a;
  int64_t n_dofs = 0;
  int n_inside = 0;
  int8_t* ctype = nullptr;
  uint8_t* mask = nullptr;
  int* cut_id = nullptr;
  int* cut_list = nullptr;
  int* q_off = nullptr;
  double* qbuf = nullptr;            // qx|qy|(qz)|qw
  int* s_off = nullptr;
  double* sbuf = nullptr;            // sx|sy|(sz)|sw|snx|sny|(snz)
  int64_t n_vq = 0, n_sq = 0;
  int* gx_id = nullptr;
  int* gy_id = nullptr;
  int* gz_id = nullptr;
  uint8_t* ccode = nullptr;
  int* ghost_list = nullptr;
  double* ycut = nullptr;
  double* jm = nullptr;
  // patches
  uint8_t* vkind = nullptr;          // (n+1)^dim
  int n_cart[8] = {};
  int* cart_list = nullptr;          // all colours concatenated, packed I + (n+1) J
  int cart_off[9] = {};
  int n_cart_tiles[4] = {0, 0, 0, 0};
  int* cart_tiles = nullptr;         // per colour concatenated, packed ti + 65536 tj
  int cart_tile_off[5] = {0, 0, 0, 0, 0};
  int* fused_tiles = nullptr;        // TC x TC cell tiles for the fused Cartesian sweep
  int n_fused_tiles = 0;
  int tc = 16;                       // cells of the fused tiles of this level in y (rows)
  int tcx = 16;                      // ... and in x
  int* fused_ext = nullptr;          // fused tiles dilated by one tile (split sweep through xs)
  unsigned* tflag = nullptr;         // in-place fused sweep: per-tile "region loaded" counters, (tx+2) x (ty+2)
  int tflag_stride = 0;              //   with a border; tiles not launched hold 0x7fffffff
  int n_fused_ext = 0;
  int* fpl = nullptr;                // in-place fused sweep: precomputed patch lists [dir][tile][4][maxp] (k_fused_plists)
  int* fpc = nullptr;                //   and counts [dir][tile][4], tiles of the tx x ty grid
  int fpl_tx = 0, fpl_nt = 0, fpl_maxp = 0;
  int n_cutp[8] = {};
  int cutp_off[9] = {};
  int* cutp_list = nullptr;          // packed I + (n+1) J
  int64_t* cutp_ent = nullptr;       // n_cutp+1 offsets into entry arrays
  int32_t* ent_node = nullptr;       // lattice index of each interior DoF
  uint16_t* ent_loc = nullptr;       // local index in the (2p+1)^dim block
  int32_t* ent_patch = nullptr;      // owning patch of each entry
  int64_t n_ent = 0;
  int64_t ent_col_off[9] = {};       // host copy of cutp_ent at the colour boundaries
  int64_t* cutp_inv = nullptr;       // n_cutp+1 offsets into inverse storage
  double* inv = nullptr;             // local inverses, m_j^2 each, row-major (symmetric)
  int64_t n_inv = 0;
  double* zbuf = nullptr;            // n_ent corrections (two-phase cut colour step)
  double* ecut = nullptr;            // cut-cell element matrices
  double* gmap = nullptr;            // dense cut-patch maps G_j (k_cut_map), CutDesc::map_off
  int64_t n_gmap = 0;
  int64_t cut_bytes[8] = {};         // algorithmic bytes of one cut colour step (k_cut_step7) per colour
  void* desc = nullptr;              // CutDesc per cut patch (smoother2.cuh)
  double* xs = nullptr;              // shadow lattice vector for the ping-pong cut steps
  long long cut_method_bytes[8] = {};  // method bytes of one cut colour step per colour
  int32_t* copy_lists = nullptr;     // node lists: [prev][cur] = N_prev \ N_cur (prev = 4: read band)
  int copy_off[5][4] = {};           // offsets into copy_lists
  int copy_n[5][4] = {};
  // workspace lattice vectors for the V-cycle
  double *x = nullptr, *b = nullptr, *r = nullptr;
  // slab partition; part = 0: not partitioned (every
  // rank holds and computes the whole level)
  int part = 0;
  int c0 = 0, c1 = 0;                // owned cell rows
  int r0 = 0, r1 = 0;                // owned lattice rows (the last rank also owns the top line)
  int v0 = 0, v1 = 0;                // rows valid after a (level) halo exchange: owned +- hw cells
  int v0n = 0, v1n = 0;              // owned +- HALO cells (the narrow halo)
  int wide = 0, hw = 0;              // wide-halo cut sweeps (hw = 3 * 4 n_c cells), else hw = HALO
  int rc0 = 0, rc1 = 0;              // coarse lattice rows this rank restricts into
  int band[6] = {0, 0, 0, 0, 0, 0};  // k_band range (BandRange): cut cells, two ghost-face ranges
  int at0 = 0, at1 = 0;              // tile rows of the TMA operator (k_apply_tile)
  const void* act_desc = nullptr;    // cut-patch descriptors the sweeps run (this rank's subset)
  int act_off[9] = {};               // ... per colour (4 in 2D, 8 in 3D)
  const int* act_cart = nullptr;     // 3D: Cartesian patches the colour steps run, per colour at act_cart_off
  int act_cart_off[9] = {};
  const int32_t* act_ent = nullptr;  // 3D: interior nodes of the swept cut patches (scatter list), per colour
  int64_t act_ent_off[9] = {};
  int band3[8] = {};                 // 3D k_band ranges (BandRange3)
  std::vector<Xfer> halo;            // transfers of one halo exchange (hw cells)
  std::vector<Xfer> halo_n;          // ... of the narrow halo
  const void* wdesc = nullptr;       // wide-halo cut sweeps: descriptors of step s of direction d
  std::vector<int> wd_off[2];        //   at wdesc + [wd_off[d][s], wd_off[d][s+1])
  int32_t* wcopy = nullptr;          //   copy lists at wcopy + wc_off[d][s], wc_n[d][s] nodes
  std::vector<int> wc_off[2], wc_n[2];
  // DoF span [a0, a1) of every lattice row (host-vector copies, k_copy_spans);
  // built on first use; span_doubles = the doubles they cover
  int* span = nullptr;
  int64_t span_doubles = 0;
  // one-launch cut sweeps (sweep.cuh), per direction (0 forward, 1 reverse);
  // args points at device arrays owned by the problem
  struct Sweep {
    bool ok = false;
    int ncta = 0;
    size_t smem = 0;
    double est_us = 0, redundancy = 0;
    long long map_bytes_total = 0;
    unsigned char args[160];   // SweepArgs (sweep.cuh), stored opaquely here
  } sw[2];
};

struct Params {
  double x0, y0, z0, length, cx, cy, cz, r, gamma_D, gamma_k[CF_MAXP];
  int dim, n_coarse, n_levels, p, sigma, n_q, n_c, symmetric, cut_mode;
  int domain;   // 0: circle / sphere level set; 1: fitted box (strong Dirichlet on its boundary)
};

// launch accounting for the bench's gpu_launches claim
extern int64_t g_launches;

#define CF_CUDA(call)                                                                   \
  do {                                                                                  \
    cudaError_t _e = (call);                                                            \
    if (_e != cudaSuccess)                                                              \
      throw cf::Error(cf::ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
  } while (0)

#define CF_LAUNCHED()                                                                   \
  do {                                                                                  \
    ++cf::g_launches;                                                                   \
    cudaError_t _e = cudaGetLastError();                                                \
    if (_e != cudaSuccess)                                                              \
      throw cf::Error(cf::ERR_CUDA, std::string("kernel launch (") + __FILE__ + ":" + std::to_string(__LINE__) + \
                                        "): " + cudaGetErrorString(_e));                \
  } while (0)

enum { ERR_ARG = 1, ERR_CUDA = 2, ERR_STATE = 3, ERR_GEOMETRY = 4, ERR_SIZE = 5 };

struct Error {
  int code;
  std::string msg;
  Error(int c, std::string m) : code(c), msg(std::move(m)) {}
};

inline void require(bool ok, int code, const std::string& msg) {
  if (!ok) throw Error(code, msg);
}

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// Function attributes, occupancy, __constant__ tables and device-side tables
// belong to a device: host-side caches of them are keyed by (call site, current
// device) and filled under a mutex (the LocalComm ranks are host threads).
inline std::mutex& dev_cache_mutex() {
  static std::mutex m;
  return m;
}
inline std::map<std::pair<const void*, int>, int64_t>& dev_cache_map() {
  static std::map<std::pair<const void*, int>, int64_t> m;
  return m;
}
// value of compute() for (key, current device), computed once
template <class F>
int64_t dev_cached(const void* key, F&& compute) {
  int dev = 0;
  CF_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(dev_cache_mutex());
  auto& m = dev_cache_map();
  auto it = m.find({key, dev});
  if (it != m.end()) return it->second;
  const int64_t v = (int64_t)compute();
  m[{key, dev}] = v;
  return v;
}
// run fn() once per (key, current device)
template <class F>
void dev_once(const void* key, F&& fn) {
  dev_cached(key, [&] {
    fn();
    return 1;
  });
}

}  // namespace cf
