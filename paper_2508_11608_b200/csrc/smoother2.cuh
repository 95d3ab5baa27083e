// smoother2.cuh — latency-optimised smoother kernels (round 1, v2).
//
// Cut patches (P l.193): one warp per patch, one 64-byte descriptor per patch
// (window cell kinds, cut-cell ids, interior-set bit mask, offsets) so that
// after one broadcast load every other load of the patch (x window, b, the
// cut-cell matrices, the local inverse) is issued at once with cp.async into
// shared memory.  The cut-cell operator is either the element matrix of the
// bulk + Nitsche terms precomputed from the cut quadrature at setup
// (cut_mode 0) or the quadrature evaluated on the fly (cut_mode 1).
//
// Cartesian patches (P l.189, l.192): (2p-1) threads per patch (one per
// interior row / column of the fast-diagonalisation passes) so a colour
// keeps ~3x more warps in flight than one thread per patch.
#pragma once
#include <cooperative_groups.h>

#include "kernels.cuh"

#ifdef CF_TIMING
// debug-only phase timestamps (variant builds with -DCF_TIMING): [block][slot]
__device__ unsigned long long g_dbg[8192][8];
#define CF_TSTAMP(slot)                                                                        \
  do {                                                                                         \
    if (threadIdx.x == 0 && blockIdx.x < 8192) {                                               \
      unsigned long long t_;                                                                   \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                   \
      g_dbg[blockIdx.x][slot] = t_;                                                            \
    }                                                                                          \
  } while (0)
#else
#define CF_TSTAMP(slot) \
  do {                  \
  } while (0)
#endif

#ifndef CF_CART_MINB
#define CF_CART_MINB 4   // resident CTAs per SM the fused Cartesian kernel is compiled for
#endif

namespace cf {

struct __align__(16) CutDesc {
  int I, J;
  uint32_t kinds;          // 2 bits per cell of the 4x4 window (I-2..I+1) x (J-2..J+1), index wy*4 + wx
  int e0;                  // first entry (interior DoF) of the patch
  int cid[4];              // cut-cell ids of the patch cells (dx + 2 dy), -1 if not cut
  long long inv_off;       // offset of A_j^{-1}
  unsigned long long mask[2];  // interior set as bits over the (2p+1)^2 block, row-major
  long long map_off;       // patch map G_j: offset (bits 0-47) | exterior columns nnz << 48; -1 if none
};
static_assert(sizeof(CutDesc) == 64, "CutDesc is one 64-byte line");

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }


// patch-map block layout (R13): [int nnz, 0, 8 pad bytes][nnz uint8 window
// indices, padded to 16 bytes][the m x K map, K = m + nnz].  A map row is
// summed by tpr lanes (map_tpr: one lane on levels n >= 256, 4 (2, 1 for
// large m) on coarser ones: V-cycle 601 vs 611 us with one lane everywhere;
// the flushed smoothing step of config1 is the same either way); lane h takes columns
// h, h + 2 tpr, ... into one accumulator and h + tpr, h + 3 tpr, ... into a
// second.  The map is stored in column blocks of B = 2 tpr columns, K padded
// to a multiple of B with zeros: element (i, c), c = B j + h + e tpr (e = 0,
// 1), at (j m + i) B + 2 h + e -- the two columns a lane needs next are one
// 16-byte word, and the 8 rows x B columns that 8 row groups read at once
// are consecutive (no shared-memory bank conflicts).  Blocks start 16-byte
// aligned (bulk copies, k_cut_sweep).
__host__ __device__ constexpr long long map_hdr_d(int nnz) { return 2 + 2 * ((nnz + 15) / 16); }
// lanes per map row: one on levels with one_lane (large levels: many rows per
// step, the instruction count decides), else 4 (2, 1 for larger m: coarse
// levels, where a step's few long rows decide)
__host__ __device__ constexpr int map_tpr(int m, int one_lane) {
  return one_lane ? 1 : (m * 4 <= 128 ? 4 : (m * 2 <= 128 ? 2 : 1));
}
__host__ __device__ constexpr int map_kp(int m, int K, int one_lane) {
  return (K + 2 * map_tpr(m, one_lane) - 1) / (2 * map_tpr(m, one_lane)) * (2 * map_tpr(m, one_lane));
}
__host__ __device__ constexpr long long map_rows_d(int m, int K, int one_lane) {
  return (long long)m * map_kp(m, K, one_lane);
}
__host__ __device__ constexpr long long map_index(int m, int i, int c, int one_lane) {
  return ((long long)(c / (2 * map_tpr(m, one_lane))) * m + i) * (2 * map_tpr(m, one_lane)) +
         2 * ((c % (2 * map_tpr(m, one_lane))) % map_tpr(m, one_lane)) + (c % (2 * map_tpr(m, one_lane))) / map_tpr(m, one_lane);
}
// levels with at least this many cells per side sum a map row with one lane
constexpr int MAP_ONE_LANE_MIN_N = 256;

__device__ __forceinline__ int desc_kind(const CutDesc& d, int wx, int wy) {
  return (d.kinds >> (2 * (wy * 4 + wx))) & 3;
}

// ---- setup: cut-cell element matrices E_c = bulk + Nitsche (P eq. cutfem_nitsche)
// from the cut quadrature (R6); one warp per (cut cell, column).
template <int P>
__global__ void __launch_bounds__(128) k_cut_elem(LevelArgs L, double* E) {
  constexpr int NB = (P + 1) * (P + 1);
  __shared__ double sX[4][NB];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t g = blockIdx.x * 4LL + w;
  if (g >= (int64_t)L.n_cut * NB) return;
  const int cid = (int)(g / NB), col = (int)(g % NB);
  for (int t = lane; t < NB; t += 32) sX[w][t] = t == col ? 1.0 : 0.0;
  __syncwarp();
  double acc[NB];
  cut_cell_warp<P>(L, cid, sX[w], P + 1, acc);
#pragma unroll
  for (int t = 0; t < NB; ++t)
    if (lane == t) E[((int64_t)cid * NB + t) * NB + col] = acc[t];
}

// ---- setup: descriptors of the cut patches (all colours, list order)
template <int P>
__global__ void k_cut_desc(LevelArgs L, const int* plist, int np, const int64_t* ent_off, const uint16_t* ent_loc,
                           const int64_t* inv_off, CutDesc* desc) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= np) return;
  const int n = L.n;
  CutDesc d;
  d.I = plist[k] % (n + 1);
  d.J = plist[k] / (n + 1);
  d.kinds = 0;
  for (int wy = 0; wy < 4; ++wy)
    for (int wx = 0; wx < 4; ++wx)
      d.kinds |= (uint32_t)cell_kind(L, L.ctype, d.I - 2 + wx, d.J - 2 + wy) << (2 * (wy * 4 + wx));
  for (int q = 0; q < 4; ++q) {
    int ci = d.I - 1 + (q & 1), cj = d.J - 1 + (q >> 1);
    d.cid[q] = cell_kind(L, L.ctype, ci, cj) == CUT ? L.cut_id[cj * n + ci] : -1;
  }
  d.e0 = (int)ent_off[k];
  d.inv_off = inv_off[k];
  d.map_off = -1;
  d.mask[0] = d.mask[1] = 0ull;
  for (int64_t e = ent_off[k]; e < ent_off[k + 1]; ++e) {
    int loc = ent_loc[e];
    d.mask[loc >> 6] |= 1ull << (loc & 63);
  }
  desc[k] = d;
}

__device__ __forceinline__ int mask_count(const CutDesc& d) { return __popcll(d.mask[0]) + __popcll(d.mask[1]); }

// i-th set bit of the 128-bit interior mask (block-local index)
__device__ __forceinline__ int mask_select(const CutDesc& d, int i) {
  int c0 = __popcll(d.mask[0]);
  unsigned long long m = i < c0 ? d.mask[0] : d.mask[1];
  int base = i < c0 ? 0 : 64;
  int r = i < c0 ? i : i - c0;
  for (int t = 0; t < r; ++t) m &= m - 1;
  return base + __ffsll((long long)m) - 1;
}

template <int P>
struct CutSmem {
  static constexpr int NB = (P + 1) * (P + 1), BS = 2 * P + 1, WS = 4 * P + 1, MM = BS * BS;
  static constexpr int per_warp = WS * WS + MM + MM + P * (P + 1) + MM * MM + 4 * NB * NB;
};

// Cut-patch colour step, phase 1 (v2): z_j = A_j^{-1} (b - A x)|_{I_j}.
// One warp: z = A_j^{-1} (b - A x)|_{I_j} for the patch of descriptor d,
// written to zbuf[d.e0 ...]; Wp = this warp's CutSmem<P>::per_warp doubles.
template <int P, bool QUAD>
__device__ void cut_patch_z(const LevelArgs& L, const CutDesc& d, const double* ecut, const double* inv,
                            const double* x, const double* b, double* zbuf, const SmTab& T, double* Wp) {
  constexpr int NB = (P + 1) * (P + 1), BS = 2 * P + 1, WS = 4 * P + 1, MM = BS * BS;
  const int lane = threadIdx.x & 31;
  double* Yb = Wp + WS * WS;
  double* Rr = Yb + MM;
  double* Js = Rr + MM;
  double* Ai = Js + P * (P + 1);
  double* Ec = Ai + MM * MM;
  const int m = mask_count(d);
  // ---- issue every load of the patch
  for (int e = lane; e < WS * WS; e += 32) {
    int a = P * (d.I - 2) + e % WS, bb = P * (d.J - 2) + e / WS;
    if (a >= 0 && bb >= 0 && a < L.nl && bb < L.nl) cp_async8(Wp + e, x + (size_t)bb * L.ld + a);
    else Wp[e] = 0.0;
  }
  const double* Ag = inv + d.inv_off;
  for (int e = lane; e < m * m; e += 32) cp_async8(Ai + e, Ag + e);
  if (!QUAD) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (d.cid[q] >= 0)
        for (int e = lane; e < NB * NB; e += 32) cp_async8(Ec + q * NB * NB + e, ecut + (size_t)d.cid[q] * NB * NB + e);
  }
  double bi[(MM + 31) / 32];
#pragma unroll
  for (int t = 0; t < (MM + 31) / 32; ++t) {
    int i = lane + 32 * t;
    bi[t] = 0.0;
    if (i < m) {
      int loc = mask_select(d, i);
      bi[t] = b[(size_t)(P * (d.J - 1) + loc / BS) * L.ld + P * (d.I - 1) + loc % BS];
    }
  }
  for (int e = lane; e < MM; e += 32) Yb[e] = 0.0;
  cp_async_wait_all();
  __syncwarp();
  // ---- (A x) on the block rows: patch cells, then ghost faces
  const int kx = lane % (P + 1), ky = lane / (P + 1);
  for (int q = 0; q < 4; ++q) {
    const int dx = q & 1, dy = q >> 1;
    const int kind = desc_kind(d, dx + 1, dy + 1);
    if (kind == OUTSIDE) continue;
    const double* X = Wp + (P * (dy + 1)) * WS + P * (dx + 1);
    if (kind == INSIDE) {
      if (lane < NB) Yb[(P * dy + ky) * BS + P * dx + kx] += inside_row<P>(T, X, WS, kx, ky);
    } else if (QUAD) {
      double acc[NB];
      cut_cell_warp<P>(L, d.cid[q], X, WS, acc);
#pragma unroll
      for (int t = 0; t < NB; ++t)
        if (lane == t) Yb[(P * dy + ky) * BS + P * dx + kx] += acc[t];
    } else if (lane < NB) {
      const double* Er = Ec + q * NB * NB + lane * NB;
      double s = 0.0;
#pragma unroll
      for (int l = 0; l < NB; ++l) s = fma(Er[l], X[(l / (P + 1)) * WS + l % (P + 1)], s);
      Yb[(P * dy + ky) * BS + P * dx + kx] += s;
    }
    __syncwarp();
  }
  const int I = d.I, J = d.J;
  for (int axis = 0; axis < 2; ++axis)
    for (int s = 0; s < 3; ++s)
      for (int t = 0; t < 2; ++t) {
        int i1, j1, i2, j2;
        if (axis == 0) {
          i1 = I - 2 + s; j1 = J - 1 + t; i2 = i1 + 1; j2 = j1;
        } else {
          i1 = I - 1 + t; j1 = J - 2 + s; i2 = i1; j2 = j1 + 1;
        }
        const int k1 = desc_kind(d, i1 - (I - 2), j1 - (J - 2)), k2 = desc_kind(d, i2 - (I - 2), j2 - (J - 2));
        if (k1 == OUTSIDE || k2 == OUTSIDE || (k1 != CUT && k2 != CUT)) continue;
        const double* X1 = Wp + ((j1 - (J - 2)) * P) * WS + (i1 - (I - 2)) * P;
        const double* X2 = Wp + ((j2 - (J - 2)) * P) * WS + (i2 - (I - 2)) * P;
        double Jm[P + 1][P + 1];
        face_moments<P>(axis, X1, X2, WS, Jm);
        if (lane == 0) {
#pragma unroll
          for (int kk = 1; kk <= P; ++kk)
#pragma unroll
            for (int qq = 0; qq <= P; ++qq) Js[(kk - 1) * (P + 1) + qq] = Jm[kk][qq];
        }
        __syncwarp();
        const bool in1 = i1 >= I - 1 && i1 <= I && j1 >= J - 1 && j1 <= J;
        const bool in2 = i2 >= I - 1 && i2 <= I && j2 >= J - 1 && j2 <= J;
        if (lane < NB) {
          if (in1) Yb[((j1 - (J - 1)) * P + ky) * BS + (i1 - (I - 1)) * P + kx] += face_test<P>(L, T, axis, 1, kx, ky, Js);
          if (in2) Yb[((j2 - (J - 1)) * P + ky) * BS + (i2 - (I - 1)) * P + kx] += face_test<P>(L, T, axis, 2, kx, ky, Js);
        }
        __syncwarp();
      }
  // ---- r = b - A x on the interior set, z = A_j^{-1} r
#pragma unroll
  for (int t = 0; t < (MM + 31) / 32; ++t) {
    int i = lane + 32 * t;
    if (i < m) Rr[i] = bi[t] - Yb[mask_select(d, i)];
  }
  __syncwarp();
  for (int i = lane; i < m; i += 32) {
    double z = 0.0;
    for (int q = 0; q < m; ++q) z = fma(Ai[q * m + i], Rr[q], z);
    zbuf[d.e0 + i] = z;
  }
  __syncwarp();
}

template <int P, bool QUAD>
__global__ void __launch_bounds__(128) k_cut_colour_v2(LevelArgs L, const CutDesc* desc, int np, const double* ecut,
                                                       const double* inv, const double* x, const double* b,
                                                       double* zbuf, int wpb) {
  __shared__ SmTab T;
  extern __shared__ double dsm[];
  load_smtab<P>(T);
  __syncthreads();
  const int w = threadIdx.x >> 5;
  if (w >= wpb) return;
  const int k = blockIdx.x * wpb + w;
  if (k >= np) return;
  const CutDesc d = desc[k];
  cut_patch_z<P, QUAD>(L, d, ecut, inv, x, b, zbuf, T, dsm + (size_t)w * CutSmem<P>::per_warp);
}

// ---- Cartesian colour step (v2): (2p-1) threads per patch -------------------
template <int P, int TP>
struct CartSmem {
  static constexpr int NE = 2 * P + 1, NI = 2 * P - 1, W = 2 * P * TP + 1;
  static constexpr int doubles = 2 * W * W + TP * TP * NE * NI * 2 + TP * TP * NI * NI + 2 * NE * NE + NI * NI + NI;
};

// One tile of TP x TP same-colour Cartesian patches, processed by the first
// NT = TP^2 (2p-1) threads of the block (all threads reach the barriers).
template <int P, int TP>
__device__ void cart_tile(const LevelArgs& L, int tile, int colour, const uint8_t* vk, double* x, const double* b,
                          double* sm) {
  constexpr int NE = 2 * P + 1, NI = 2 * P - 1, W = 2 * P * TP + 1, NT = TP * TP * NI;
  double* Xs = sm;
  double* Bs = Xs + W * W;
  double* T1 = Bs + W * W;                 // [TP*TP][NE][NI]
  double* T2 = T1 + TP * TP * NE * NI;
  double* Ex = T2 + TP * TP * NE * NI;     // [TP*TP][NI][NI]
  double* sK = Ex + TP * TP * NI * NI;     // two-cell matrices, S, lam
  double* sM = sK + NE * NE;
  double* sS = sM + NE * NE;
  double* sL = sS + NI * NI;
  const Tab& Tc = c_tab[P];
  const int tid = threadIdx.x;
  const int nthr = blockDim.x;
  for (int e = tid; e < NE * NE; e += nthr) {
    sK[e] = Tc.Kp[e / NE][e % NE];
    sM[e] = Tc.Mp[e / NE][e % NE];
  }
  for (int e = tid; e < NI * NI; e += nthr) sS[e] = Tc.S[e / NI][e % NI];
  if (tid < NI) sL[tid] = Tc.lam[tid];
  const int ti = tile & 0xffff, tj = tile >> 16;
  const int I0 = (colour & 1) + 2 * ti * TP, J0 = (colour >> 1) + 2 * tj * TP;
  const int a0 = P * (I0 - 1), b0 = P * (J0 - 1);
  for (int e = tid; e < W * W; e += nthr) {
    int a = a0 + e % W, bb = b0 + e / W;
    if (a >= 0 && bb >= 0 && a < L.nl && bb < L.nl) {
      cp_async8(Xs + e, x + (size_t)bb * L.ld + a);
      cp_async8(Bs + e, b + (size_t)bb * L.ld + a);
    } else {
      Xs[e] = 0.0;
      Bs[e] = 0.0;
    }
  }
  cp_async_wait_all();
  __syncthreads();
  const int q = tid / NI, t = tid % NI;
  const int u = q % TP, v = q / TP;
  const int I = I0 + 2 * u, J = J0 + 2 * v, n = L.n;
  const bool cart = tid < NT && I <= n && J <= n && vk[J * (n + 1) + I] == V_CART;
  const double* X = Xs + (2 * P * v) * W + 2 * P * u;
  double* t1 = T1 + q * NE * NI;
  double* t2 = T2 + q * NE * NI;
  double* ex = Ex + q * NI * NI;
  // 1. T1 = X K̄^T, T2 = X M̄^T on the interior columns (rows b' = t, t+NI)
  if (cart) {
    for (int bp = t; bp < NE; bp += NI) {
#pragma unroll
      for (int ia = 0; ia < NI; ++ia) {
        const int a = ia + 1, alo = a <= P ? 0 : P, ahi = a >= P ? 2 * P : P;
        double s1 = 0.0, s2 = 0.0;
#pragma unroll
        for (int ap = alo; ap <= ahi; ++ap) {
          double xv = X[bp * W + ap];
          s1 = fma(Tc.Kp[a][ap], xv, s1);
          s2 = fma(Tc.Mp[a][ap], xv, s2);
        }
        t1[bp * NI + ia] = s1;
        t2[bp * NI + ia] = s2;
      }
    }
  }
  __syncthreads();
  // 2. residual row ib = t, V = R S
  double R[NI];
  if (cart) {
    const int bq = t + 1;
    const double* B = Bs + (2 * P * v) * W + 2 * P * u;
#pragma unroll
    for (int ia = 0; ia < NI; ++ia) R[ia] = B[bq * W + ia + 1];
    for (int bp = 0; bp < NE; ++bp) {
      const double mb = sM[bq * NE + bp], kb = sK[bq * NE + bp];
#pragma unroll
      for (int ia = 0; ia < NI; ++ia) R[ia] = fma(-mb, t1[bp * NI + ia], fma(-kb, t2[bp * NI + ia], R[ia]));
    }
#pragma unroll
    for (int be = 0; be < NI; ++be) {
      double s = 0.0;
#pragma unroll
      for (int ia = 0; ia < NI; ++ia) s = fma(R[ia], Tc.S[ia][be], s);
      ex[t * NI + be] = s;
    }
  }
  __syncthreads();
  // 3. row alpha = t: U = (S^T V) ./ (lam_alpha + lam_beta), Y = U S^T
  double Y[NI];
  if (cart) {
    double U[NI];
#pragma unroll
    for (int be = 0; be < NI; ++be) {
      double s = 0.0;
#pragma unroll
      for (int ib = 0; ib < NI; ++ib) s = fma(sS[ib * NI + t], ex[ib * NI + be], s);
      U[be] = s / (sL[t] + Tc.lam[be]);
    }
#pragma unroll
    for (int ia = 0; ia < NI; ++ia) {
      double s = 0.0;
#pragma unroll
      for (int be = 0; be < NI; ++be) s = fma(U[be], Tc.S[ia][be], s);
      Y[ia] = s;
    }
  }
  __syncthreads();
  if (cart) {
#pragma unroll
    for (int ia = 0; ia < NI; ++ia) ex[t * NI + ia] = Y[ia];
  }
  __syncthreads();
  // 4. row ib = t of Z = S Y, added to the patch interior
  if (cart) {
    double* Xw = Xs + (2 * P * v + t + 1) * W + 2 * P * u + 1;
#pragma unroll
    for (int ia = 0; ia < NI; ++ia) {
      double s = 0.0;
#pragma unroll
      for (int al = 0; al < NI; ++al) s = fma(sS[t * NI + al], ex[al * NI + ia], s);
      Xw[ia] += s;
    }
  }
  __syncthreads();
  for (int e = tid; e < W * W; e += nthr) {
    int c = e % W, r = e / W;
    int lc = c % (2 * P), lr = r % (2 * P);
    if (lc == 0 || lr == 0) continue;
    int uu = c / (2 * P), vv = r / (2 * P);
    int II = I0 + 2 * uu, JJ = J0 + 2 * vv;
    if (II > n || JJ > n || vk[JJ * (n + 1) + II] != V_CART) continue;
    x[(size_t)(b0 + r) * L.ld + a0 + c] = Xs[e];
  }
  __syncthreads();
}

template <int P, int TP>
__global__ void __launch_bounds__(TP* TP*(2 * P - 1)) k_cart_colour_v2(LevelArgs L, const int* tiles, int colour,
                                                                      const uint8_t* vk, double* x, const double* b) {
  extern __shared__ double sm[];
  cart_tile<P, TP>(L, tiles[blockIdx.x], colour, vk, x, b, sm);
}

}  // namespace cf

namespace cf {

// ---- Cartesian sweep, all four colours in one kernel (temporal blocking) ---
// A CTA owns TC x TC cells.  Colour step s (of 4) updates the Cartesian
// patches within 3 - s vertices of the owned vertex range: a colour-c patch
// reads its closed 2x2-cell block, which overlaps the interiors of patches of
// the other colours only within one vertex, so the halo shrinks by one
// vertex per step.  x and b are read once (region of TC + 8 cells), every
// colour is applied in shared memory, the owned nodes are written once.
template <int P, int TC>
struct CartFusedSmem {
  static constexpr int NE = 2 * P + 1, NI = 2 * P - 1, H = 4, RC = TC + 2 * H, RW = RC * P + 1;
  static constexpr int NPR = 256 / NI;
  static constexpr int doubles = 2 * RW * RW + NPR * NE * NI * 2 + NPR * NI * NI + 2 * NE * NE + NI * NI + NI;
};

template <int P, int TC>
__global__ void __launch_bounds__(256) k_cart_fused(LevelArgs L, const int* tiles, const uint8_t* vk, double* x,
                                                    const double* b, int reverse, int gsync) {
  using S = CartFusedSmem<P, TC>;
  constexpr int NE = S::NE, NI = S::NI, H = S::H, RW = S::RW, NPR = S::NPR;
  extern __shared__ double sm[];
  double* Xs = sm;
  double* Bs = Xs + RW * RW;
  double* T1 = Bs + RW * RW;
  double* T2 = T1 + NPR * NE * NI;
  double* Ex = T2 + NPR * NE * NI;
  double* sK = Ex + NPR * NI * NI;
  double* sM = sK + NE * NE;
  double* sS = sM + NE * NE;
  double* sL = sS + NI * NI;
  const Tab& Tc = c_tab[P];
  const int tid = threadIdx.x, n = L.n;
  for (int e = tid; e < NE * NE; e += 256) {
    sK[e] = Tc.Kp[e / NE][e % NE];
    sM[e] = Tc.Mp[e / NE][e % NE];
  }
  for (int e = tid; e < NI * NI; e += 256) sS[e] = Tc.S[e / NI][e % NI];
  if (tid < NI) sL[tid] = Tc.lam[tid];
  pdl_trigger();
  const int tile = tiles[blockIdx.x];
  const int ci0 = (tile & 0xffff) * TC, cj0 = (tile >> 16) * TC;
  const int a0 = P * (ci0 - H), b0 = P * (cj0 - H);
  pdl_wait();
  for (int e = tid; e < RW * RW; e += 256) {
    int a = a0 + e % RW, bb = b0 + e / RW;
    if (a >= 0 && bb >= 0 && a < L.nl && bb < L.nl) {
      cp_async8(Xs + e, x + (size_t)bb * L.ld + a);
      cp_async8(Bs + e, b + (size_t)bb * L.ld + a);
    } else {
      Xs[e] = 0.0;
      Bs[e] = 0.0;
    }
  }
  cp_async_wait_all();
  __syncthreads();
  for (int s = 0; s < 4; ++s) {
    const int c = reverse ? 3 - s : s, rad = 3 - s;
    // colour-c vertices in [ci0 - rad, ci0 + TC + rad]
    const int ilo = ci0 - rad + ((ci0 - rad - (c & 1)) & 1), jlo = cj0 - rad + ((cj0 - rad - (c >> 1)) & 1);
    const int nvx = (ci0 + TC + rad - ilo) / 2 + 1, nvy = (cj0 + TC + rad - jlo) / 2 + 1;
    const int np = nvx * nvy;
    for (int base = 0; base < np; base += NPR) {
      const int q = tid / NI, t = tid % NI, pq = base + q;
      const int I = ilo + 2 * (pq % nvx), J = jlo + 2 * (pq / nvx);
      const bool cart = q < NPR && pq < np && I >= 0 && J >= 0 && I <= n && J <= n && vk[J * (n + 1) + I] == V_CART;
      // patch block origin in the region (cells I-1, J-1)
      const int ox = P * (I - 1 - (ci0 - H)), oy = P * (J - 1 - (cj0 - H));
      const double* X = Xs + oy * RW + ox;
      double* t1 = T1 + q * NE * NI;
      double* t2 = T2 + q * NE * NI;
      double* ex = Ex + q * NI * NI;
      if (cart) {
        for (int bp = t; bp < NE; bp += NI) {
#pragma unroll
          for (int ia = 0; ia < NI; ++ia) {
            const int a = ia + 1, alo = a <= P ? 0 : P, ahi = a >= P ? 2 * P : P;
            double s1 = 0.0, s2 = 0.0;
#pragma unroll
            for (int ap = alo; ap <= ahi; ++ap) {
              double xv = X[bp * RW + ap];
              s1 = fma(Tc.Kp[a][ap], xv, s1);
              s2 = fma(Tc.Mp[a][ap], xv, s2);
            }
            t1[bp * NI + ia] = s1;
            t2[bp * NI + ia] = s2;
          }
        }
      }
      __syncthreads();
      if (cart) {
        const int bq = t + 1;
        const double* B = Bs + oy * RW + ox;
        double R[NI];
#pragma unroll
        for (int ia = 0; ia < NI; ++ia) R[ia] = B[bq * RW + ia + 1];
        for (int bp = 0; bp < NE; ++bp) {
          const double mb = sM[bq * NE + bp], kb = sK[bq * NE + bp];
#pragma unroll
          for (int ia = 0; ia < NI; ++ia) R[ia] = fma(-mb, t1[bp * NI + ia], fma(-kb, t2[bp * NI + ia], R[ia]));
        }
#pragma unroll
        for (int be = 0; be < NI; ++be) {
          double sacc = 0.0;
#pragma unroll
          for (int ia = 0; ia < NI; ++ia) sacc = fma(R[ia], Tc.S[ia][be], sacc);
          ex[t * NI + be] = sacc;
        }
      }
      __syncthreads();
      double Y[NI];
      if (cart) {
        double U[NI];
#pragma unroll
        for (int be = 0; be < NI; ++be) {
          double sacc = 0.0;
#pragma unroll
          for (int ib = 0; ib < NI; ++ib) sacc = fma(sS[ib * NI + t], ex[ib * NI + be], sacc);
          U[be] = sacc / (sL[t] + Tc.lam[be]);
        }
#pragma unroll
        for (int ia = 0; ia < NI; ++ia) {
          double sacc = 0.0;
#pragma unroll
          for (int be = 0; be < NI; ++be) sacc = fma(U[be], Tc.S[ia][be], sacc);
          Y[ia] = sacc;
        }
      }
      __syncthreads();
      if (cart) {
#pragma unroll
        for (int ia = 0; ia < NI; ++ia) ex[t * NI + ia] = Y[ia];
      }
      __syncthreads();
      if (cart) {
        double* Xw = Xs + (oy + t + 1) * RW + ox + 1;
#pragma unroll
        for (int ia = 0; ia < NI; ++ia) {
          double sacc = 0.0;
#pragma unroll
          for (int al = 0; al < NI; ++al) sacc = fma(sS[t * NI + al], ex[al * NI + ia], sacc);
          Xw[ia] += sacc;
        }
      }
      __syncthreads();
    }
  }
  // in place: every CTA of the (cooperative) grid has read its region before any write
  if (gsync) cooperative_groups::this_grid().sync();
  // owned nodes: [P ci0, P (ci0 + TC)) (+ the last lattice line on the mesh boundary)
  const int ahi = (ci0 + TC >= n) ? L.nl : P * (ci0 + TC), bhi = (cj0 + TC >= n) ? L.nl : P * (cj0 + TC);
  const int aw = ahi - P * ci0, bw = bhi - P * cj0;
  for (int e = tid; e < aw * bw; e += 256) {
    const int a = P * ci0 + e % aw, bb = P * cj0 + e / aw;
    x[(size_t)bb * L.ld + a] = Xs[(bb - b0) * RW + (a - a0)];
  }
}

// tiles within one tile of a flagged tile (the tiles whose owned nodes the
// split Cartesian sweep must carry through the shadow buffer)
__global__ void k_dilate_tile_flags(int tx, int ty, const uint8_t* in, uint8_t* out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= tx * ty) return;
  const int ti = t % tx, tj = t / tx;
  uint8_t f = 0;
  for (int dj = -1; dj <= 1; ++dj)
    for (int di = -1; di <= 1; ++di) {
      const int i = ti + di, j = tj + dj;
      if (i >= 0 && j >= 0 && i < tx && j < ty && in[j * tx + i]) f = 1;
    }
  out[t] = f;
}

// tiles of TCX x TCY cells whose owned vertex range holds a Cartesian patch
__global__ void k_fused_tile_flags(int n, const uint8_t* vk, int TCX, int TCY, int tx, uint8_t* flag, int ntiles) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntiles) return;
  const int ci0 = (t % tx) * TCX, cj0 = (t / tx) * TCY;
  uint8_t f = 0;
  for (int J = cj0; J <= min(cj0 + TCY, n) && !f; ++J)
    for (int I = ci0; I <= min(ci0 + TCX, n); ++I)
      if (vk[J * (n + 1) + I] == V_CART) {
        f = 1;
        break;
      }
  flag[t] = f;
}

}  // namespace cf

namespace cf {

template <int P>
struct CutSmem3 {
  static constexpr int NB = (P + 1) * (P + 1), BS = 2 * P + 1, WS = 4 * P + 1, MM = BS * BS, NJ = 12 * P * (P + 1);
  static constexpr int per_warp = WS * WS + 2 * NJ + MM + MM * MM + 4 * NB * NB + MM;
};

// face f of the 12 faces touching the patch cells: axis 0 (x-faces) f = 2 s + t
// between cells (I-2+s, J-1+t) | (I-1+s, J-1+t); axis 1 f = 6 + 2 s + t between
// (I-1+t, J-2+s) | (I-1+t, J-1+s).  Window cell coordinates of both sides:
__device__ __forceinline__ void face_cells(int f, int& axis, int& w1x, int& w1y, int& w2x, int& w2y) {
  axis = f >= 6;
  const int g = f - 6 * axis, s = g >> 1, t = g & 1;
  if (!axis) {
    w1x = s; w1y = 1 + t; w2x = s + 1; w2y = 1 + t;
  } else {
    w1x = 1 + t; w1y = s; w2x = 1 + t; w2y = s + 1;
  }
}

// v3 cut-patch colour step: lanes work on ghost-face jump moments in
// parallel, then one lane per row of the (2p+1)^2 block gathers the cell and
// face contributions (no serial loop over cells and faces).
template <int P, bool QUAD>
__device__ void cut_patch_z3(const LevelArgs& L, const CutDesc& d, const double* ecut, const double* inv,
                             const double* x, const double* b, double* zbuf, const SmTab& T, double* Wp) {
  using S = CutSmem3<P>;
  constexpr int NB = S::NB, BS = S::BS, WS = S::WS, MM = S::MM, NJ = S::NJ, PP = P * (P + 1);
  constexpr int RPL = (MM + 31) / 32;  // block rows per lane
  const int lane = threadIdx.x & 31;
  double* Jt = Wp + WS * WS;   // [12][P][P+1] jumps, then Ycut for QUAD
  double* Jm = Jt + NJ;        // [12][P][P+1] moments
  double* Rr = Jm + NJ;
  double* Ai = Rr + MM;
  double* Ec = Ai + MM * MM;
  const int m = mask_count(d);
  // ---- loads independent of the previous kernel
  const double* Ag = inv + d.inv_off;
  for (int e = lane; e < m * m; e += 32) cp_async8(Ai + e, Ag + e);
  if (!QUAD) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (d.cid[q] >= 0)
        for (int e = lane; e < NB * NB; e += 32) cp_async8(Ec + q * NB * NB + e, ecut + (size_t)d.cid[q] * NB * NB + e);
  }
  pdl_wait();
  // ---- x window and b on the interior rows
  for (int e = lane; e < WS * WS; e += 32) {
    const int r = e / WS, c = e - r * WS;
    const int a = P * (d.I - 2) + c, bb = P * (d.J - 2) + r;
    if (a >= 0 && bb >= 0 && a < L.nl && bb < L.nl) cp_async8(Wp + e, x + (size_t)bb * L.ld + a);
    else Wp[e] = 0.0;
  }
  double bv[RPL];
  bool inm[RPL];
  int iidx[RPL];
#pragma unroll
  for (int t = 0; t < RPL; ++t) {
    const int loc = lane + 32 * t;
    const unsigned long long word = d.mask[loc >> 6];
    inm[t] = loc < MM && ((word >> (loc & 63)) & 1ull);
    iidx[t] = (loc >> 6 ? __popcll(d.mask[0]) : 0) + __popcll(word & ((1ull << (loc & 63)) - 1ull));
    bv[t] = inm[t] ? b[(size_t)(P * (d.J - 1) + loc / BS) * L.ld + P * (d.I - 1) + loc % BS] : 0.0;
  }
  cp_async_wait_all();
  __syncwarp();
  // ---- ghost faces: jumps J[f][k][l] (lane-parallel), then moments M J
  const Tab& Tc = c_tab[P];
  for (int job = lane; job < NJ; job += 32) {
    const int f = job / PP, rem = job - f * PP, k = rem / (P + 1) + 1, l = rem % (P + 1);
    int axis, w1x, w1y, w2x, w2y;
    face_cells(f, axis, w1x, w1y, w2x, w2y);
    const int k1 = desc_kind(d, w1x, w1y), k2 = desc_kind(d, w2x, w2y);
    double s = 0.0;
    if (k1 != OUTSIDE && k2 != OUTSIDE && (k1 == CUT || k2 == CUT)) {
      const double* X1 = Wp + (P * w1y) * WS + P * w1x;
      const double* X2 = Wp + (P * w2y) * WS + P * w2x;
#pragma unroll
      for (int nn = 0; nn <= P; ++nn) {
        const double v1 = axis == 0 ? X1[l * WS + nn] : X1[nn * WS + l];
        const double v2 = axis == 0 ? X2[l * WS + nn] : X2[nn * WS + l];
        s = fma(T.d1[k][nn], v1, fma(-T.d0[k][nn], v2, s));
      }
    }
    Jt[job] = s;
  }
  __syncwarp();
  for (int job = lane; job < NJ; job += 32) {
    const int base = job - job % (P + 1), q = job % (P + 1);
    double s = 0.0;
#pragma unroll
    for (int l = 0; l <= P; ++l) s = fma(T.M[q][l], Jt[base + l], s);
    Jm[job] = s;
  }
  __syncwarp();
  // ---- cut cells by quadrature (warp-cooperative) into Jt (reused as Ycut)
  if (QUAD) {
    for (int q = 0; q < 4; ++q) {
      if (d.cid[q] < 0) continue;
      const int dx = q & 1, dy = q >> 1;
      double acc[NB];
      cut_cell_warp<P>(L, d.cid[q], Wp + (P * (dy + 1)) * WS + P * (dx + 1), WS, acc);
#pragma unroll
      for (int t = 0; t < NB; ++t)
        if (lane == t) Jt[q * NB + t] = acc[t];
    }
    __syncwarp();
  }
  // ---- one lane per block row: (A x) on the row, residual
#pragma unroll
  for (int t = 0; t < RPL; ++t) {
    const int loc = lane + 32 * t;
    if (!inm[t]) continue;
    const int ra = loc % BS, rb = loc / BS;
    double y = 0.0;
    for (int dy = 0; dy < 2; ++dy) {
      const int ky = rb - P * dy;
      if (ky < 0 || ky > P) continue;
      for (int dx = 0; dx < 2; ++dx) {
        const int kx = ra - P * dx;
        if (kx < 0 || kx > P) continue;
        const int kind = desc_kind(d, dx + 1, dy + 1);
        if (kind == OUTSIDE) continue;
        const int q = dx + 2 * dy;
        const double* X = Wp + (P * (dy + 1)) * WS + P * (dx + 1);
        if (kind == INSIDE) {
          y += inside_row<P>(T, X, WS, kx, ky);
        } else if (QUAD) {
          y += Jt[q * NB + ky * (P + 1) + kx];
        } else {
          const double* Er = Ec + q * NB * NB + (ky * (P + 1) + kx) * NB;
#pragma unroll
          for (int l = 0; l < NB; ++l) y = fma(Er[l], X[(l / (P + 1)) * WS + l % (P + 1)], y);
        }
        // ghost faces of this cell: left (side 2), right (side 1), bottom (side 2), top (side 1)
        const int fl = 2 * dx + dy, fr = 2 * (dx + 1) + dy, fb = 6 + 2 * dy + dx, ft = 6 + 2 * (dy + 1) + dx;
#pragma unroll
        for (int kk = 1; kk <= P; ++kk) {
          const double g = L.gs[kk];
          y = fma(-g * T.d0[kk][kx], Jm[fl * PP + (kk - 1) * (P + 1) + ky], y);
          y = fma(g * T.d1[kk][kx], Jm[fr * PP + (kk - 1) * (P + 1) + ky], y);
          y = fma(-g * T.d0[kk][ky], Jm[fb * PP + (kk - 1) * (P + 1) + kx], y);
          y = fma(g * T.d1[kk][ky], Jm[ft * PP + (kk - 1) * (P + 1) + kx], y);
        }
      }
    }
    Rr[iidx[t]] = bv[t] - y;
  }
  __syncwarp();
  for (int i = lane; i < m; i += 32) {
    double z = 0.0;
    for (int q = 0; q < m; ++q) z = fma(Ai[q * m + i], Rr[q], z);
    zbuf[d.e0 + i] = z;
  }
  __syncwarp();
  (void)Tc;
}

template <int P, bool QUAD>
__global__ void __launch_bounds__(128) k_cut_colour_v3(LevelArgs L, const CutDesc* desc, int np, const double* ecut,
                                                       const double* inv, const double* x, const double* b,
                                                       double* zbuf, int wpb) {
  __shared__ SmTab T;
  extern __shared__ double dsm[];
  pdl_trigger();
  load_smtab<P>(T);
  __syncthreads();
  const int w = threadIdx.x >> 5;
  if (w >= wpb) return;
  const int k = blockIdx.x * wpb + w;
  if (k >= np) return;
  const CutDesc d = desc[k];
  cut_patch_z3<P, QUAD>(L, d, ecut, inv, x, b, zbuf, T, dsm + (size_t)w * CutSmem3<P>::per_warp);
}

__global__ void k_cut_apply(const int32_t* ent_node, const double* zbuf, int64_t e0, int64_t e1, double* x) {
  pdl_trigger();
  const int64_t e = e0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int32_t node = e < e1 ? ent_node[e] : 0;
  pdl_wait();
  if (e < e1) x[node] += zbuf[e];
}

}  // namespace cf

namespace cf {

// fp64 tensor-core MMA: D(8x8) = A(8x4, row) B(4x8, col) + C.  Fragments per
// lane: A[lane>>2][lane&3], B[lane&3][lane>>2], C/D[lane>>2][2(lane&3)+{0,1}].
__device__ __forceinline__ void dmma(double a, double b, double& c0, double& c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int P>
struct CartMMA {
  static constexpr int NE = 2 * P + 1, NI = 2 * P - 1, NINT = NI * NI, NEXT = NE * NE, K = NINT + NEXT;
  static constexpr int KS = (K + 3) / 4, MT = (NINT + 7) / 8, COLS = 4 * KS, ROWS = 8 * MT;
};

template <int P, int TC>
struct CartMMASmem {
  static constexpr int H = 4, RC = TC + 2 * H, RW = RC * P + 1;
  static constexpr int doubles = 2 * RW * RW;
  static constexpr int ints = CartMMA<P>::COLS + CartMMA<P>::ROWS;
};

// All four Cartesian colours of one smoothing step (temporal blocking as in
// k_cart_fused); every colour pass is the batched dense contraction
// x_int_new = G [b_int; x_ext] over groups of 8 patches per warp on the fp64
// tensor cores (mma.sync m8n8k4 .f64), G from host::cart_affine_map.
template <int P, int TC>
__global__ void __launch_bounds__(256) k_cart_fused_mma(LevelArgs L, const int* tiles, const uint8_t* vk,
                                                        const double* G, double* x, const double* b, int reverse,
                                                        int gsync) {
  using C = CartMMA<P>;
  using S = CartMMASmem<P, TC>;
  constexpr int NE = C::NE, NI = C::NI, NINT = C::NINT, K = C::K, KS = C::KS, MT = C::MT, H = S::H, RW = S::RW;
  extern __shared__ double sm[];
  double* Xs = sm;
  double* Bs = Xs + RW * RW;
  int* koff = (int*)(Bs + RW * RW);   // operand k: offset in the region (+ (1 << 30) for b)
  int* roff = koff + C::COLS;          // interior row r: offset in the region
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, n = L.n;
  pdl_trigger();
  for (int k = tid; k < C::COLS; k += 256) {
    int v = -1;
    if (k < NINT) v = (1 << 30) + (k / NI + 1) * RW + k % NI + 1;
    else if (k < K) v = ((k - NINT) / NE) * RW + (k - NINT) % NE;
    koff[k] = v;
  }
  for (int r = tid; r < C::ROWS; r += 256) roff[r] = r < NINT ? (r / NI + 1) * RW + r % NI + 1 : -1;
  double af[MT][KS];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int s = 0; s < KS; ++s) af[mt][s] = G[(8 * mt + (lane >> 2)) * C::COLS + 4 * s + (lane & 3)];
  const int tile = tiles[blockIdx.x];
  const int ci0 = (tile & 0xffff) * TC, cj0 = (tile >> 16) * TC;
  const int a0 = P * (ci0 - H), b0 = P * (cj0 - H);
  pdl_wait();
  for (int e = tid; e < RW * RW; e += 256) {
    const int r = e / RW, c = e - r * RW;
    const int a = a0 + c, bb = b0 + r;
    if (a >= 0 && bb >= 0 && a < L.nl && bb < L.nl) {
      cp_async8(Xs + e, x + (size_t)bb * L.ld + a);
      cp_async8(Bs + e, b + (size_t)bb * L.ld + a);
    } else {
      Xs[e] = 0.0;
      Bs[e] = 0.0;
    }
  }
  cp_async_wait_all();
  __syncthreads();
  for (int s = 0; s < 4; ++s) {
    const int c = reverse ? 3 - s : s, rad = 3 - s;
    const int ilo = ci0 - rad + ((ci0 - rad - (c & 1)) & 1), jlo = cj0 - rad + ((cj0 - rad - (c >> 1)) & 1);
    const int nvx = (ci0 + TC + rad - ilo) / 2 + 1, nvy = (cj0 + TC + rad - jlo) / 2 + 1;
    const int np = nvx * nvy, ng = (np + 7) / 8;
    for (int g = warp; g < ng; g += 8) {
      // this lane's patch in the B fragment: n = lane >> 2
      const int pq = 8 * g + (lane >> 2);
      const int I = ilo + 2 * (pq % nvx), J = jlo + 2 * (pq / nvx);
      const bool cart = pq < np && I >= 0 && J >= 0 && I <= n && J <= n && vk[J * (n + 1) + I] == V_CART;
      const int base = cart ? P * (J - 1 - (cj0 - H)) * RW + P * (I - 1 - (ci0 - H)) : -1;
      double acc[MT][2];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) acc[mt][0] = acc[mt][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int ko = koff[4 * ks + (lane & 3)];
        double v = 0.0;
        if (base >= 0 && ko >= 0) v = ko >= (1 << 30) ? Bs[base + ko - (1 << 30)] : Xs[base + ko];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) dmma(af[mt][ks], v, acc[mt][0], acc[mt][1]);
      }
      // D[r][n'] with r = 8 mt + (lane >> 2), n' = 2 (lane & 3) + i
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int bo = __shfl_sync(0xffffffffu, base, 4 * (2 * (lane & 3) + i));
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const int r = 8 * mt + (lane >> 2);
          if (bo >= 0 && r < NINT) Xs[bo + roff[r]] = acc[mt][i];
        }
      }
    }
    __syncthreads();
  }
  if (gsync) cooperative_groups::this_grid().sync();
  const int ahi = (ci0 + TC >= n) ? L.nl : P * (ci0 + TC), bhi = (cj0 + TC >= n) ? L.nl : P * (cj0 + TC);
  const int aw = ahi - P * ci0, bw = bhi - P * cj0;
  for (int e = tid; e < aw * bw; e += 256) {
    const int rr = e / aw, cc = e - rr * aw;
    const int a = P * ci0 + cc, bb = P * cj0 + rr;
    x[(size_t)bb * L.ld + a] = Xs[(bb - b0) * RW + (a - a0)];
  }
}

}  // namespace cf

namespace cf {

// ---- cut colour step without a separate scatter (ping-pong buffers) --------
// Step s reads R (the current state) and writes W, which before the step holds
// the state two steps back, i.e. differs from R exactly on N_{s-1} (the
// interior nodes of the previous step).  The kernel writes
//   W[node] = R[node] + z   for node in N_s (this colour's interior sets)
//   W[node] = R[node]       for node in N_{s-1} \ N_s   (copy list)
// so that afterwards W holds the state after step s and R differs from it
// exactly on N_s; R and W then swap.  No node is read and written in the same
// launch, so the colour-start snapshot semantics (R9) hold without a second
// kernel.  The first cut step of a sweep copies the whole read band instead.
template <int P, bool QUAD>
__global__ void __launch_bounds__(128) k_cut_step(LevelArgs L, const CutDesc* desc, int np, int wpb, int patch_blocks,
                                                  const double* ecut, const double* inv, const double* R, double* W,
                                                  const double* b, const int32_t* copy, int ncopy) {
  using S = CutSmem3<P>;
  constexpr int BS = S::BS, WS = S::WS, MM = S::MM, RPL = (MM + 31) / 32;
  __shared__ SmTab T;
  extern __shared__ double dsm[];
  pdl_trigger();
  if ((int)blockIdx.x >= patch_blocks) {
    const int e = (blockIdx.x - patch_blocks) * blockDim.x + threadIdx.x;
    const int32_t node = e < ncopy ? copy[e] : 0;
    pdl_wait();
    if (e < ncopy) W[node] = R[node];
    return;
  }
  load_smtab<P>(T);
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w >= wpb) return;
  const int k = blockIdx.x * wpb + w;
  if (k >= np) return;
  const CutDesc d = desc[k];
  double* Wp = dsm + (size_t)w * S::per_warp;
  double* zs = Wp + WS * WS + 2 * S::NJ + MM + MM * MM + 4 * S::NB * S::NB;  // per-warp tail: MM doubles
  CutDesc dl = d;
  dl.e0 = 0;
  cut_patch_z3<P, QUAD>(L, dl, ecut, inv, R, b, zs, T, Wp);   // z_i -> zs[i]
#pragma unroll
  for (int t = 0; t < RPL; ++t) {
    const int loc = lane + 32 * t;
    if (loc >= MM) continue;
    const unsigned long long word = d.mask[loc >> 6];
    if (!((word >> (loc & 63)) & 1ull)) continue;
    const int i = (loc >> 6 ? __popcll(d.mask[0]) : 0) + __popcll(word & ((1ull << (loc & 63)) - 1ull));
    const int ra = loc % BS, rb = loc / BS;
    const double xr = Wp[(P + rb) * WS + P + ra];   // R at the node (window origin p(I-2), p(J-2))
    W[(size_t)(P * (d.J - 1) + rb) * L.ld + P * (d.I - 1) + ra] = xr + zs[i];
  }
}

// marks of the interior nodes of one colour's cut patches / of the read band
__global__ void k_mark_entries(const int32_t* ent_node, int64_t e0, int64_t e1, uint8_t* mark) {
  const int64_t e = e0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < e1) mark[ent_node[e]] = 1;
}
__global__ void k_mark_band(const CutDesc* desc, int np, LevelArgs L, uint8_t* mark) {
  constexpr int MAXW = 4 * CF_MAXP + 1;
  const int k = blockIdx.x;
  if (k >= np) return;
  const CutDesc d = desc[k];
  const int WS = 4 * L.p + 1;
  for (int e = threadIdx.x; e < WS * WS; e += blockDim.x) {
    const int a = L.p * (d.I - 2) + e % WS, bb = L.p * (d.J - 2) + e / WS;
    if (a >= 0 && bb >= 0 && a < L.nl && bb < L.nl) mark[(size_t)bb * L.ld + a] = 1;
  }
  (void)MAXW;
}
__global__ void k_andnot_flags(const uint8_t* a, const uint8_t* b, int64_t n, uint8_t* out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = a[i] && !b[i];
}

}  // namespace cf

#include "tma.cuh"

namespace cf {

// ---- fused Cartesian sweep, v2: TMA tile loads, hoisted operand offsets ----
// grid-wide barrier of a cooperative (co-resident) launch: one arrival per
// CTA on a monotonic 64-bit counter owned by the caller (one per launch
// configuration, never reset: the target is the next multiple of the grid
// size).  Control only -- the CTAs' region loads have completed (TMA
// mbarrier) before they arrive, which is all the in-place sweep needs.
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void grid_barrier(unsigned long long* ctr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long nb = gridDim.x, t = atomicAdd(ctr, 1ull);
    const unsigned long long target = (t / nb + 1) * nb;
    while (*(volatile unsigned long long*)ctr < target) __nanosleep(20);
  }
  __syncthreads();
}

// setup: the compacted Cartesian patch lists of every (direction, tile of the
// fused grid, pass) of the in-place fused sweep (passes 0..3, radius 3 - s),
// as k_cart_fused_tma would compact them, in vertex order: lists
// [dir][tile][4][maxp] (block origins in the region), counts [dir][tile][4]
__global__ void k_fused_plists(int n, int P, int TC, int TCX, int H, int RWP, int maxp, const uint8_t* vk, int tx,
                               int ty, int* lists, int* counts) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  const int nt = tx * ty;
  if (q >= 2 * nt * 4) return;
  const int s = q % 4, t = (q / 4) % nt, dir = q / (4 * nt);
  const int ci0 = (t % tx) * TCX, cj0 = (t / tx) * TC;
  const int c = dir ? 3 - s : s, rad = 3 - s;
  const int ilo = ci0 - rad + ((ci0 - rad - (c & 1)) & 1), jlo = cj0 - rad + ((cj0 - rad - (c >> 1)) & 1);
  const int nvx = (ci0 + TCX + rad - ilo) / 2 + 1, nvy = (cj0 + TC + rad - jlo) / 2 + 1;
  int* out = lists + ((size_t)(dir * nt + t) * 4 + s) * maxp;
  int cnt = 0;
  for (int pj = 0; pj < nvy; ++pj)
    for (int pi = 0; pi < nvx; ++pi) {
      const int I = ilo + 2 * pi, J = jlo + 2 * pj;
      if (I >= 0 && J >= 0 && I <= n && J <= n && vk[J * (n + 1) + I] == V_CART)
        out[cnt++] = P * (J - 1 - (cj0 - H)) * RWP + P * (I - 1 - (ci0 - H));
    }
  counts[(dir * nt + t) * 4 + s] = cnt;
}

template <int P, int TC, int TCX = TC>
struct CartTmaSmem {
  // TC = cells per tile in y (rows: the partitioned direction), TCX in x
  static constexpr int H = 4, RW = (TC + 2 * H) * P + 1, RWX = (TCX + 2 * H) * P + 1, RWP = (RWX + 1) & ~1;
  static constexpr int tile_doubles = (RW * RWP + 15) & ~15;   // 128-byte aligned tiles (TMA destination)
  static constexpr int maxp = ((TCX + 7) / 2 + 1) * ((TC + 7) / 2 + 1);
  static constexpr int VW = TCX + 7, VH = TC + 7;   // vertex kinds of the region (widest pass: radius 3)
  static constexpr int vk_off = 32 + 4 * 4 * maxp;
  static constexpr int head = ((vk_off + VW * VH) + 127) & ~127;   // mbarrier, 4 counts, 4 pass patch lists, vertex kinds
  static constexpr size_t bytes = head + 2 * tile_doubles * sizeof(double);
};

// Passes s0..s1-1 of the four colour passes (halo radius s1-1-s).  The tile
// region is read from the tensor map `tmx` and the owned nodes are written to
// `xout`.  In place (xout = the source of tmx) only with tile flags in a
// cooperative (co-resident) launch: a CTA publishes "my region is loaded" on
// its tile's counter (st.release after the TMA load completed) and writes its
// owned nodes back only after its 8 neighbour tiles -- the only ones whose
// aprons (H = 4 < tile width) hold them -- have published (ld.acquire poll).
// Counters advance by one per in-place launch on every launched tile, so a
// launch reads its own counter as the base; tiles not in the launch hold
// 0x7fffffff.  Otherwise the sweep is split into two launches through the
// shadow buffer (passes 0-1 x -> xs, 2-3 xs -> x).
template <int P, int TC, int NT = 256, int TCX = TC>
__global__ void __launch_bounds__(NT, (TC >= 32 || P >= 3) ? 2 : CF_CART_MINB) k_cart_fused_tma(const __grid_constant__ CUtensorMap tmx,
                                                        const __grid_constant__ CUtensorMap tmb, LevelArgs L,
                                                        const int* tiles, const uint8_t* vk, const double* G,
                                                        double* xout, int reverse, int s0, int s1,
                                                        unsigned* tflag, int tstride, const unsigned char* pf,
                                                        unsigned long long pf_bytes, const int* gpl,
                                                        const int* gpc, int gtx) {
  using C = CartMMA<P>;
  using S = CartTmaSmem<P, TC, TCX>;
  constexpr int NE = C::NE, NI = C::NI, NINT = C::NINT, K = C::K, KS = C::KS;
  constexpr int MF = NINT / 8;                 // full 8-row tiles on the tensor cores
  constexpr int RR = NINT - 8 * MF;            // remainder rows on the FMA pipe (p = 1: 1, p = 2: 1, p = 3: 1)
  constexpr int H = S::H, RW = S::RW, RWP = S::RWP, TD = S::tile_doubles;
  constexpr int MAXP = S::maxp;   // candidate patches of the widest pass
  extern __shared__ __align__(128) unsigned char smraw[];
  uint64_t* bar = (uint64_t*)smraw;
  int* pcount = (int*)(smraw + 8);             // [4] patches per pass
  int* plists = (int*)(smraw + 32);            // [4][MAXP] compacted Cartesian patches of each pass (block origins)
  double* Xs = (double*)(smraw + S::head);     // x tile [RW][RWP]; the b tile follows at Xs + TD
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, n = L.n;
  pdl_trigger();
  if (tid == 0 && pf_bytes) {   // this CTA's slice of [pf, pf + pf_bytes) towards L2 (the next kernel's data)
    const unsigned long long sl = ((pf_bytes + gridDim.x - 1) / gridDim.x + 15) & ~15ull, a = sl * blockIdx.x;
    if (a < pf_bytes) prefetch_l2(pf + a, (size_t)(pf_bytes - a < sl ? pf_bytes - a : sl));
  }
  int ko[KS];
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) {
    const int k = 4 * ks + (lane & 3);
    int v = -1;
    if (k < NINT) v = TD + (k / NI + 1) * RWP + k % NI + 1;
    else if (k < K) v = ((k - NINT) / NE) * RWP + (k - NINT) % NE;
    ko[ks] = v;
  }
  double af[MF > 0 ? MF : 1][KS];
  double gr[RR > 0 ? RR : 1][KS];
#pragma unroll
  for (int mt = 0; mt < MF; ++mt)
#pragma unroll
    for (int s = 0; s < KS; ++s) af[mt][s] = G[(8 * mt + (lane >> 2)) * C::COLS + 4 * s + (lane & 3)];
#pragma unroll
  for (int rr = 0; rr < RR; ++rr)
#pragma unroll
    for (int s = 0; s < KS; ++s) gr[rr][s] = G[(8 * MF + rr) * C::COLS + 4 * s + (lane & 3)];
  const int tile = tiles[blockIdx.x];
  const int ci0 = (tile & 0xffff) * TCX, cj0 = (tile >> 16) * TC;
  const int a0 = P * (ci0 - H), b0 = P * (cj0 - H);
  CF_TSTAMP(0);
  unsigned* myflag = tflag ? tflag + ((tile >> 16) + 1) * tstride + (tile & 0xffff) + 1 : nullptr;
  unsigned fbase = 0;
  if (gpl && s0 == 0 && s1 == 4) {
    // x and b regions by TMA right away (after the predecessor completed) while
    // every thread loads the tile's patch lists, precomputed at setup
    // (k_fused_plists) in one round of independent loads
    if (tid == 0) {
      mbar_init(bar, 1);
      pdl_wait();
      mbar_expect_tx(bar, 2u * RW * RWP * sizeof(double));
      tma_load_2d(Xs, &tmx, a0, b0, bar);
      tma_load_2d(Xs + TD, &tmb, a0, b0, bar);
      if (myflag) fbase = *(volatile unsigned*)myflag;
    }
    const int gt = (tile >> 16) * gtx + (tile & 0xffff);
    const int* src = gpl + (size_t)gt * 4 * MAXP;
    constexpr int NL = (4 * MAXP + NT - 1) / NT;
    int r[NL];
#pragma unroll
    for (int u = 0; u < NL; ++u) r[u] = (tid + u * NT < 4 * MAXP) ? __ldg(src + tid + u * NT) : 0;
    const int cn = tid < 4 ? __ldg(gpc + gt * 4 + tid) : 0;
#pragma unroll
    for (int u = 0; u < NL; ++u)
      if (tid + u * NT < 4 * MAXP) plists[tid + u * NT] = r[u];
    if (tid < 4) pcount[tid] = cn;
    __syncthreads();
    CF_TSTAMP(1);
  } else {
    if (tid < 4) pcount[tid] = 0;
    if (tid == 0) mbar_init(bar, 1);
    uint8_t* vks = smraw + S::vk_off;   // vertex kinds of [ci0 - 3, ci0 + TCX + 3] x [cj0 - 3, cj0 + TC + 3]
    // the region's vertex kinds (setup data: before the PDL wait; outside the mesh: none)
    constexpr int NVK = (S::VW * S::VH + NT - 1) / NT;
    uint8_t r[NVK];
#pragma unroll
    for (int u = 0; u < NVK; ++u) {
      const int q = tid + u * NT, I = ci0 - 3 + q % S::VW, J = cj0 - 3 + q / S::VW;
      r[u] = (q < S::VW * S::VH && I >= 0 && J >= 0 && I <= n && J <= n) ? __ldg(vk + J * (n + 1) + I) : (uint8_t)V_NONE;
    }
#pragma unroll
    for (int u = 0; u < NVK; ++u)
      if (tid + u * NT < S::VW * S::VH) vks[tid + u * NT] = r[u];
    __syncthreads();
    CF_TSTAMP(1);
    if (tid == 0) {   // x and b regions by TMA (after the predecessor completed); the patch lists are compacted meanwhile
      pdl_wait();
      mbar_expect_tx(bar, 2u * RW * RWP * sizeof(double));
      tma_load_2d(Xs, &tmx, a0, b0, bar);
      tma_load_2d(Xs + TD, &tmb, a0, b0, bar);
      if (myflag) fbase = *(volatile unsigned*)myflag;
    }
    // compact the Cartesian patches of every pass
    for (int s = s0; s < s1; ++s) {
      const int c = reverse ? 3 - s : s, rad = s1 - 1 - s;
      const int ilo = ci0 - rad + ((ci0 - rad - (c & 1)) & 1), jlo = cj0 - rad + ((cj0 - rad - (c >> 1)) & 1);
      const int nvx = (ci0 + TCX + rad - ilo) / 2 + 1, nvy = (cj0 + TC + rad - jlo) / 2 + 1;
      for (int q = tid; q < nvx * nvy; q += NT) {
        const int pj = q / nvx, pi = q - pj * nvx;
        const int I = ilo + 2 * pi, J = jlo + 2 * pj;
        if (vks[(J - cj0 + 3) * S::VW + I - ci0 + 3] == V_CART)
          plists[s * MAXP + atomicAdd(pcount + s, 1)] = P * (J - 1 - (cj0 - H)) * RWP + P * (I - 1 - (ci0 - H));
      }
    }
  }
  pdl_wait();
  CF_TSTAMP(2);
  for (int s = s0; s < s1; ++s) {
    const int* plist = plists + s * MAXP;
    if (s == s0) {
      mbar_wait(bar, 0);
      CF_TSTAMP(3);
      if (myflag && tid == 0) st_release_u32(myflag, fbase + 1u);   // region loaded: neighbours may write
    }
    __syncthreads();
    if (s == s0 + 2) CF_TSTAMP(4);
    const int np = pcount[s], ng = (np + 7) / 8;
#ifndef CF_CART_GPW
#define CF_CART_GPW 1   // groups of 8 patches per warp iteration (2: measured no faster, spills at 16-cell tiles)
#endif
    constexpr int GW = CF_CART_GPW;
    for (int g = warp; g < ng; g += GW * (NT / 32)) {
      int base[GW];
      double acc[GW][MF > 0 ? MF : 1][2][2];
      double rs[GW][RR > 0 ? RR : 1];
#pragma unroll
      for (int u = 0; u < GW; ++u) {
        const int gu = g + u * (NT / 32), pq = 8 * gu + (lane >> 2);
        base[u] = (gu < ng && pq < np) ? plist[pq] : -1;
#pragma unroll
        for (int mt = 0; mt < MF; ++mt) acc[u][mt][0][0] = acc[u][mt][0][1] = acc[u][mt][1][0] = acc[u][mt][1][1] = 0.0;
#pragma unroll
        for (int rr = 0; rr < RR; ++rr) rs[u][rr] = 0.0;
      }
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
#pragma unroll
        for (int u = 0; u < GW; ++u) {
          const double v = (base[u] >= 0 && ko[ks] >= 0) ? Xs[base[u] + ko[ks]] : 0.0;
#pragma unroll
          for (int mt = 0; mt < MF; ++mt) dmma(af[mt][ks], v, acc[u][mt][ks & 1][0], acc[u][mt][ks & 1][1]);
#pragma unroll
          for (int rr = 0; rr < RR; ++rr) rs[u][rr] = fma(gr[rr][ks], v, rs[u][rr]);
        }
      }
#pragma unroll
      for (int u = 0; u < GW; ++u) {
#pragma unroll
        for (int rr = 0; rr < RR; ++rr) {
          double t = rs[u][rr];
          t += __shfl_xor_sync(0xffffffffu, t, 1);
          t += __shfl_xor_sync(0xffffffffu, t, 2);
          const int r = 8 * MF + rr;
          if ((lane & 3) == 0 && base[u] >= 0) Xs[base[u] + (r / NI + 1) * RWP + r % NI + 1] = t;
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int bo = __shfl_sync(0xffffffffu, base[u], 4 * (2 * (lane & 3) + i));
#pragma unroll
          for (int mt = 0; mt < MF; ++mt) {
            const int r = 8 * mt + (lane >> 2);
            if (bo >= 0) Xs[bo + (r / NI + 1) * RWP + r % NI + 1] = acc[u][mt][0][i] + acc[u][mt][1][i];
          }
        }
      }
    }
    __syncthreads();
  }
  if (s1 == s0) {
    mbar_wait(bar, 0);
    if (myflag && tid == 0) st_release_u32(myflag, fbase + 1u);
  }
  CF_TSTAMP(5);
  if (myflag) {   // the 8 neighbours have loaded their aprons (which hold our owned nodes)
    const unsigned want = __shfl_sync(0xffffffffu, fbase, 0) + 1u;   // (warp 0: thread 0's base)
    if (tid < 9 && tid != 4) {
      const unsigned* f = myflag + (tid / 3 - 1) * tstride + (tid % 3 - 1);
      while (ld_acquire_u32(f) < want) {
      }
    }
    __syncthreads();
  }
  CF_TSTAMP(6);
  // owned nodes [P ci0, P (ci0 + TC)) (+ the last lattice line), warp per row
  const int ahi = (ci0 + TCX >= n) ? L.nl : P * (ci0 + TCX), bhi = (cj0 + TC >= n) ? L.nl : P * (cj0 + TC);
  for (int bb = P * cj0 + warp; bb < bhi; bb += NT / 32) {
    const double* src = Xs + (bb - b0) * RWP - a0;
    double* dst = xout + (size_t)bb * L.ld;
    for (int a = P * ci0 + lane; a < ahi; a += 32) dst[a] = src[a];
  }
  CF_TSTAMP(7);
}

}  // namespace cf

namespace cf {

// ---- operator A x (or b - A x) on a TMA-staged tile ------------------------
// CTA per TX x TX cells; the x tile with a one-cell halo is loaded by TMA
// (zero-filled outside the lattice); one thread per owned lattice node sums
// the cell rows of its (up to 4) cells from shared memory, the cut-cell
// outputs (ycut) and the ghost-face moments (jm) of k_band.
template <int P, int TX>
struct ApplySmem {
  // the box starts at an even column (16-byte aligned inner coordinate), so
  // it is one column wider than the region when P (i0 - 1) is odd
  static constexpr int RW = (TX + 2) * P + 1, RWP = (RW + 2) & ~1;
  static constexpr int tile = (RW * RWP + 15) & ~15;
  static constexpr size_t bytes = 128 + tile * sizeof(double) + sizeof(SmTab) + (TX + 2) * (TX + 2);
};

template <int P, int TX>
__global__ void __launch_bounds__(256) k_apply_tile(const __grid_constant__ CUtensorMap tmx, LevelArgs L,
                                                    const double* b, double* y, int ty0) {
  using S = ApplySmem<P, TX>;
  constexpr int NB = (P + 1) * (P + 1), RWP = S::RWP, RW = S::RW;
  extern __shared__ __align__(128) unsigned char smraw[];   // no static shared memory: keeps the TMA tile 128-byte aligned
  uint64_t* bar = (uint64_t*)smraw;
  double* Xs = (double*)(smraw + 128);
  SmTab& T = *(SmTab*)(smraw + 128 + S::tile * sizeof(double));
  uint8_t* Cs = smraw + 128 + S::tile * sizeof(double) + sizeof(SmTab);   // cell codes of the tile + halo
  const int tid = threadIdx.x, n = L.n;
  const int tx = blockIdx.x, ty = ty0 + blockIdx.y;
  const int i0 = tx * TX, j0 = ty * TX;
  const int a0 = (P * (i0 - 1)) & ~1, b0 = P * (j0 - 1), sh = P * (i0 - 1) - a0;   // sh = 0 or 1
  pdl_trigger();
  load_smtab<P>(T);
  for (int e = tid; e < (TX + 2) * (TX + 2); e += 256) {
    const int ci = i0 - 1 + e % (TX + 2), cj = j0 - 1 + e / (TX + 2);
    Cs[e] = (ci >= 0 && cj >= 0 && ci < n && cj < n) ? L.ccode[cj * n + ci] : 0;
  }
  if (tid == 0) mbar_init(bar, 1);
  __syncthreads();
  pdl_wait();
  if (tid == 0) {
    mbar_expect_tx(bar, (unsigned)(RW * RWP * sizeof(double)));
    tma_load_2d(Xs, &tmx, a0, b0, bar);
  }
  mbar_wait(bar, 0);
  // owned nodes [P i0, P (i0 + TX)) (+ the last lattice line)
  const int ahi = min(P * (i0 + TX), L.nl - 1) + ((i0 + TX >= n) ? 1 : 0);
  const int bhi = min(P * (j0 + TX), L.nl - 1) + ((j0 + TX >= n) ? 1 : 0);
  const int aw = ahi - P * i0, bw = bhi - P * j0;
  for (int e = tid; e < aw * bw; e += 256) {
    const int a = P * i0 + e % aw, bb = P * j0 + e / aw;
    const size_t o = (size_t)bb * L.ld + a;
    if (!L.mask[o]) {
      y[o] = 0.0;
      continue;
    }
    const int ci0 = (a % P == 0) ? a / P - 1 : a / P, ci1 = min(a / P, n - 1);
    const int cj0 = (bb % P == 0) ? bb / P - 1 : bb / P, cj1 = min(bb / P, n - 1);
    double acc = 0.0;
    for (int j = max(cj0, 0); j <= cj1; ++j)
      for (int i = max(ci0, 0); i <= ci1; ++i) {
        const int code = Cs[(j - j0 + 1) * (TX + 2) + i - i0 + 1];
        const int kind = code & 3;
        if (kind == OUTSIDE) continue;
        const int kx = a - i * P, ky = bb - j * P;
        if (kind == INSIDE) acc += inside_row<P>(T, Xs + (P * (j - j0 + 1)) * RWP + sh + P * (i - i0 + 1), RWP, kx, ky);
        else acc += L.ycut[(size_t)L.cut_id[j * n + i] * NB + ky * (P + 1) + kx];
        if (code & 60) {
          if (code & 4) acc += face_test<P>(L, T, 0, 2, kx, ky, L.jm + (size_t)L.gx_id[j * n + i - 1] * P * (P + 1));
          if (code & 8) acc += face_test<P>(L, T, 0, 1, kx, ky, L.jm + (size_t)L.gx_id[j * n + i] * P * (P + 1));
          if (code & 16) acc += face_test<P>(L, T, 1, 2, kx, ky, L.jm + (size_t)L.gy_id[(j - 1) * n + i] * P * (P + 1));
          if (code & 32) acc += face_test<P>(L, T, 1, 1, kx, ky, L.jm + (size_t)L.gy_id[j * n + i] * P * (P + 1));
        }
      }
    y[o] = b ? b[o] - acc : acc;
  }
  // zero the padding columns of the owned rows
  if (i0 + TX >= n)
    for (int bb = P * j0 + tid; bb < bhi; bb += 256)
      for (int a = L.nl; a < L.ld; ++a) y[(size_t)bb * L.ld + a] = 0.0;
}


// ---- v6: one cut-patch step as a device routine for a group of NT threads
// (a whole CTA, or one of several groups of a cluster-resident CTA, with its
// own named barrier `bar`).  Four barriers: (1) ghost-face jumps + moments
// (registers) and the cell parts of the (cell, row) outputs; (2) the ghost
// terms of each (cell, row) output; (3) gather of the interior rows and the
// residual; (4) z = A_j^{-1} r written to the interior nodes of W.
template <int P>
struct CutGroup6 {
  static constexpr int NB = (P + 1) * (P + 1), BS = 2 * P + 1, WS = 4 * P + 1, MM = BS * BS, PP = P * (P + 1);
  // doubles: window, face moments, cell outputs, residual, inverse, element matrices
  static constexpr int doubles = WS * WS + 12 * PP + 4 * NB + MM + MM * MM + 4 * NB * NB;
  static constexpr int bytes = doubles * 8 + 128 + 2 * MM + 8;   // + descriptor, interior locations, ghost mask
};

__device__ __forceinline__ void group_sync(int bar, int nt) { asm volatile("bar.sync %0, %1;\n" ::"r"(bar), "r"(nt) : "memory"); }

// prologue (independent of the previous step): descriptor, inverse and
// element matrices by cp.async.  Returns after the descriptor is visible.
template <int P, int NT>
__device__ __forceinline__ void cut6_prologue(const CutDesc* desc, int k, const double* ecut, const double* inv,
                                              unsigned char* gsm, int gt, int bar) {
  using S = CutGroup6<P>;
  constexpr int NB = S::NB, WS = S::WS, MM = S::MM, PP = S::PP;
  CutDesc& d = *(CutDesc*)gsm;
  double* Wp = (double*)(gsm + 128);
  double* Ai = Wp + WS * WS + 12 * PP + 4 * NB + MM;
  double* Ec = Ai + MM * MM;
  if (gt < (int)(sizeof(CutDesc) / 16)) ((int4*)&d)[gt] = ((const int4*)(desc + k))[gt];
  group_sync(bar, NT);
  const int m = mask_count(d);
  const double* Ag = inv + d.inv_off;
  for (int e = gt; e < m * m; e += NT) cp_async8(Ai + e, Ag + e);
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (d.cid[q] >= 0)
      for (int e = gt; e < NB * NB; e += NT) cp_async8(Ec + q * NB * NB + e, ecut + (size_t)d.cid[q] * NB * NB + e);
}

template <int P, int NT>
__device__ __forceinline__ void cut6_resid(const LevelArgs& L, const SmTab& T, unsigned char* gsm, int gt, int bar);

// main part (after the previous step's W is visible).  LDCG: read the window
// through L2 only (ld.global.cg) -- inside one launch whose earlier steps
// wrote R from other SMs, where an L1-cached (cp.async.ca) line could be stale
template <int P, int NT, bool LDCG = false>
__device__ __forceinline__ void cut6_main(const LevelArgs& L, const SmTab& T, const double* R, double* W,
                                          const double* b, unsigned char* gsm, int gt, int bar) {
  using S = CutGroup6<P>;
  constexpr int NB = S::NB, BS = S::BS, WS = S::WS, MM = S::MM, PP = S::PP, N1 = P + 1;
  const CutDesc& d = *(const CutDesc*)gsm;
  double* Wp = (double*)(gsm + 128);
  double* Jm = Wp + WS * WS;
  double* Yc = Jm + 12 * PP;
  double* Rr = Yc + 4 * NB;
  double* Ai = Rr + MM;
  double* Ec = Ai + MM * MM;
  short* Lc = (short*)(Ec + 4 * NB * NB);
  unsigned* gmask = (unsigned*)(Lc + MM + (MM & 1));
  const int m = mask_count(d);
  if (gt == 0) *gmask = 0u;
  for (int e = gt; e < WS * WS; e += NT) {
    const int r = e / WS, c = e - r * WS;
    const int a = P * (d.I - 2) + c, bb = P * (d.J - 2) + r;
    if (a >= 0 && bb >= 0 && a < L.nl && bb < L.nl) {
      if (LDCG) Wp[e] = __ldcg(R + (size_t)bb * L.ld + a);
      else cp_async8(Wp + e, R + (size_t)bb * L.ld + a);
    } else {
      Wp[e] = 0.0;
    }
  }
  for (int loc = gt; loc < MM; loc += NT) {
    const unsigned long long word = d.mask[loc >> 6];
    if ((word >> (loc & 63)) & 1ull) {
      const int i = (loc >> 6 ? __popcll(d.mask[0]) : 0) + __popcll(word & ((1ull << (loc & 63)) - 1ull));
      Lc[i] = (short)loc;
      Rr[i] = b[(size_t)(P * (d.J - 1) + loc / BS) * L.ld + P * (d.I - 1) + loc % BS];
    }
  }
  cp_async_wait_all();
  group_sync(bar, NT);
  cut6_resid<P, NT>(L, T, gsm, gt, bar);
  // (4) z = A_j^{-1} r on the interior nodes
  for (int i = gt; i < m; i += NT) {
    double z0 = 0.0, z1 = 0.0, z2 = 0.0, z3 = 0.0;
    int q = 0;
    for (; q + 3 < m; q += 4) {
      z0 = fma(Ai[q * m + i], Rr[q], z0);
      z1 = fma(Ai[(q + 1) * m + i], Rr[q + 1], z1);
      z2 = fma(Ai[(q + 2) * m + i], Rr[q + 2], z2);
      z3 = fma(Ai[(q + 3) * m + i], Rr[q + 3], z3);
    }
    for (; q < m; ++q) z0 = fma(Ai[q * m + i], Rr[q], z0);
    const int loc = Lc[i], ra = loc % BS, rb = loc / BS;
    W[(size_t)(P * (d.J - 1) + rb) * L.ld + P * (d.I - 1) + ra] = Wp[(P + rb) * WS + P + ra] + ((z0 + z1) + (z2 + z3));
  }
}

// phases (1)-(3) of the group routine on the shared-memory window Wp and the
// interior b values in Rr (Lc: interior locations): Rr <- b - A_{I,W} x_W
// (cell terms by sum factorisation / cut-cell matrices, ghost-face terms);
// ends with a group barrier
template <int P, int NT>
__device__ __forceinline__ void cut6_resid(const LevelArgs& L, const SmTab& T, unsigned char* gsm, int gt, int bar) {
  using S = CutGroup6<P>;
  constexpr int NB = S::NB, BS = S::BS, WS = S::WS, MM = S::MM, PP = S::PP, N1 = P + 1;
  const CutDesc& d = *(const CutDesc*)gsm;
  double* Wp = (double*)(gsm + 128);
  double* Jm = Wp + WS * WS;
  double* Yc = Jm + 12 * PP;
  double* Rr = Yc + 4 * NB;
  double* Ai = Rr + MM;
  double* Ec = Ai + MM * MM;
  short* Lc = (short*)(Ec + 4 * NB * NB);
  unsigned* gmask = (unsigned*)(Lc + MM + (MM & 1));
  const int m = mask_count(d);
  // (1) cell parts (jobs < 4 NB) and ghost-face moments
  for (int job = gt; job < 4 * NB + 12 * P; job += NT) {
    if (job < 4 * NB) {
      const int q = job / NB, t = job - q * NB;
      const int dx = q & 1, dy = q >> 1, kx = t % N1, ky = t / N1;
      const int kind = desc_kind(d, dx + 1, dy + 1);
      double y = 0.0;
      if (kind != OUTSIDE) {
        const double* X = Wp + (P * (dy + 1)) * WS + P * (dx + 1);
        if (kind == INSIDE) {
          y = inside_row<P>(T, X, WS, kx, ky);
        } else {
          const double* Er = Ec + q * NB * NB + t * NB;
          double y1 = 0.0, y2 = 0.0;
#pragma unroll
          for (int l = 0; l < NB; l += 3) {
            y = fma(Er[l], X[(l / N1) * WS + l % N1], y);
            if (l + 1 < NB) y1 = fma(Er[l + 1], X[((l + 1) / N1) * WS + (l + 1) % N1], y1);
            if (l + 2 < NB) y2 = fma(Er[l + 2], X[((l + 2) / N1) * WS + (l + 2) % N1], y2);
          }
          y += y1 + y2;
        }
      }
      Yc[job] = y;
      continue;
    }
    const int jf = job - 4 * NB, f = jf / P, k = jf - f * P + 1;
    int axis, w1x, w1y, w2x, w2y;
    face_cells(f, axis, w1x, w1y, w2x, w2y);
    const int k1 = desc_kind(d, w1x, w1y), k2 = desc_kind(d, w2x, w2y);
    if (!(k1 != OUTSIDE && k2 != OUTSIDE && (k1 == CUT || k2 == CUT))) continue;
    if (k == 1) atomicOr(gmask, 1u << f);
    const double* X1 = Wp + (P * w1y) * WS + P * w1x;
    const double* X2 = Wp + (P * w2y) * WS + P * w2x;
    const int sn = axis == 0 ? 1 : WS, st = axis == 0 ? WS : 1;
    double J[N1];
#pragma unroll
    for (int l = 0; l < N1; ++l) {
      double a1 = 0.0, a2 = 0.0;
#pragma unroll
      for (int nn = 0; nn <= P; ++nn) {
        a1 = fma(T.d1[k][nn], X1[l * st + nn * sn], a1);
        a2 = fma(T.d0[k][nn], X2[l * st + nn * sn], a2);
      }
      J[l] = a1 - a2;
    }
#pragma unroll
    for (int q = 0; q < N1; ++q) {
      double a = 0.0;
#pragma unroll
      for (int l = 0; l < N1; ++l) a = fma(T.M[q][l], J[l], a);
      Jm[f * PP + (k - 1) * N1 + q] = a;
    }
  }
  group_sync(bar, NT);
  // (2) ghost terms of the (cell, row) outputs
  const unsigned gm = *gmask;
  if (gm)
    for (int job = gt; job < 4 * NB; job += NT) {
      const int q = job / NB, t = job - q * NB;
      const int dx = q & 1, dy = q >> 1, kx = t % N1, ky = t / N1;
      const int fl = 2 * dx + dy, fr = 2 * (dx + 1) + dy, fb = 6 + 2 * dy + dx, ft = 6 + 2 * (dy + 1) + dx;
      if (!(gm & ((1u << fl) | (1u << fr) | (1u << fb) | (1u << ft)))) continue;
      double y0 = 0.0, y1 = 0.0;
#pragma unroll
      for (int kk = 1; kk <= P; ++kk) {
        const double gk = L.gs[kk];
        if ((gm >> fl) & 1u) y0 = fma(-gk * T.d0[kk][kx], Jm[fl * PP + (kk - 1) * N1 + ky], y0);
        if ((gm >> fr) & 1u) y1 = fma(gk * T.d1[kk][kx], Jm[fr * PP + (kk - 1) * N1 + ky], y1);
        if ((gm >> fb) & 1u) y0 = fma(-gk * T.d0[kk][ky], Jm[fb * PP + (kk - 1) * N1 + kx], y0);
        if ((gm >> ft) & 1u) y1 = fma(gk * T.d1[kk][ky], Jm[ft * PP + (kk - 1) * N1 + kx], y1);
      }
      Yc[job] += y0 + y1;
    }
  group_sync(bar, NT);
  // (3) residual on the interior rows
  for (int i = gt; i < m; i += NT) {
    const int loc = Lc[i], ra = loc % BS, rb = loc / BS;
    double y = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int kx = ra - P * (q & 1), ky = rb - P * (q >> 1);
      if (kx >= 0 && kx <= P && ky >= 0 && ky <= P) y += Yc[q * NB + ky * N1 + kx];
    }
    Rr[i] -= y;
  }
  group_sync(bar, NT);
}

template <int P, int NT>
__global__ void __launch_bounds__(NT) k_cut_step6(LevelArgs L, const CutDesc* desc, int np, const double* ecut,
                                                  const double* inv, const double* R, double* W, const double* b,
                                                  const int32_t* copy, int ncopy) {
  __shared__ SmTab T;
  extern __shared__ __align__(128) unsigned char sm6[];
  const int tid = threadIdx.x;
  CF_TSTAMP(0);
  pdl_trigger();
  if ((int)blockIdx.x >= np) {
    const int e = (blockIdx.x - np) * NT + tid;
    if (e < ncopy) {
      const int32_t node = copy[e];
      pdl_wait();
      W[node] = R[node];
    }
    return;
  }
  load_smtab<P>(T);
  cut6_prologue<P, NT>(desc, blockIdx.x, ecut, inv, sm6, tid, 0);
  CF_TSTAMP(1);
  pdl_wait();
  CF_TSTAMP(2);
  cut6_main<P, NT>(L, T, R, W, b, sm6, tid, 0);
  CF_TSTAMP(3);
}

}  // namespace cf

namespace cf {

// ---- cut patches as dense affine maps (v7) ----------------------------------
// The cut-patch update of eq. (smoother) is affine in (b, x):
//   z_j = A_j^{-1} (b_I - A_{I,W} x_W) = G_j [b_I ; x_W],
//   G_j = [A_j^{-1} | -A_j^{-1} A_{I,W}]   (m_j x (m_j + (4p+1)^2), row-major),
// with W the (4p+1)^2 window of the patch, so it is precomputed at setup --
// the cut-patch analogue of the Cartesian patch map -- and a colour step is
// one gather and one small dense matvec per patch.  Column w of the right
// block is obtained by running the residual phases of the group routine on
// the unit window e_w (b = 0) and applying A_j^{-1}: the same arithmetic the
// matrix-free step performs, so G_j [b; x] equals it up to summation order.

// setup: one CTA per (patch, column); column block y = WS^2 copies A_j^{-1}
template <int P, int NT>
__global__ void __launch_bounds__(NT) k_cut_map(LevelArgs L, const CutDesc* desc, const double* ecut,
                                                const double* inv, double* G) {
  using S = CutGroup6<P>;
  constexpr int NB = S::NB, WS = S::WS, MM = S::MM, PP = S::PP, WW = WS * WS;
  __shared__ SmTab T;
  extern __shared__ __align__(128) unsigned char smm[];
  const int tid = threadIdx.x, k = blockIdx.x, w = blockIdx.y;
  load_smtab<P>(T);
  cut6_prologue<P, NT>(desc, k, ecut, inv, smm, tid, 0);
  const CutDesc& d = *(const CutDesc*)smm;
  double* Wp = (double*)(smm + 128);
  double* Rr = Wp + WW + 12 * PP + 4 * NB;
  double* Ai = Rr + MM;
  short* Lc = (short*)(Ai + MM * MM + 4 * NB * NB);
  unsigned* gmask = (unsigned*)(Lc + MM + (MM & 1));
  const int m = mask_count(d), K = m + WW;
  double* Gj = G + d.map_off;
  if (tid == 0) *gmask = 0u;
  for (int e = tid; e < WW; e += NT) Wp[e] = e == w ? 1.0 : 0.0;
  for (int loc = tid; loc < MM; loc += NT) {
    const unsigned long long word = d.mask[loc >> 6];
    if ((word >> (loc & 63)) & 1ull) {
      const int i = (loc >> 6 ? __popcll(d.mask[0]) : 0) + __popcll(word & ((1ull << (loc & 63)) - 1ull));
      Lc[i] = (short)loc;
      Rr[i] = 0.0;
    }
  }
  cp_async_wait_all();
  __syncthreads();
  if (w == WW) {   // A_j^{-1} (stored [q][i], symmetric)
    for (int e = tid; e < m * m; e += NT) Gj[(size_t)(e / m) * K + e % m] = Ai[(e % m) * m + e / m];
    return;
  }
  cut6_resid<P, NT>(L, T, smm, tid, 0);
  for (int i = tid; i < m; i += NT) {
    double z = 0.0;
    for (int q = 0; q < m; ++q) z = fma(Ai[q * m + i], Rr[q], z);
    Gj[(size_t)i * K + m + w] = z;
  }
}

// Compression of the maps: the interior columns of -A_j^{-1} A_{I,W} are -I
// (A_{I,I} = A_j), so x_I^new = x_I + z_j = A_j^{-1} (b_I - A_{I,E} x_E) over
// the exterior window nodes E; of those only the columns with a nonzero entry
// (nodes coupled to the interior through a patch cell or a ghost face) are
// kept.  Compressed block of patch j at map_off:
//   [int32 nnz, pad][nnz uint8 window indices, padded to 8 bytes]
//   [m_j x (m_j + nnz) rows: A_j^{-1} | -A_j^{-1} A_{I,E'}]
template <int P>
__device__ __forceinline__ bool window_interior(const CutDesc& d, int w) {
  constexpr int WS = 4 * P + 1, BS = 2 * P + 1;
  const int r = w / WS - P, c = w % WS - P;
  if (r < 0 || c < 0 || r >= BS || c >= BS) return false;
  const int loc = r * BS + c;
  return (d.mask[loc >> 6] >> (loc & 63)) & 1ull;
}

// nonzero exterior columns of the dense map (one CTA per patch)
template <int P>
__global__ void k_map_nnz(const CutDesc* desc, const int64_t* dense_off, const double* Gd, int* nnz) {
  constexpr int WW = (4 * P + 1) * (4 * P + 1);
  const CutDesc d = desc[blockIdx.x];
  const int m = mask_count(d), K = m + WW;
  const double* g = Gd + dense_off[blockIdx.x];
  __shared__ int cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  for (int w = threadIdx.x; w < WW; w += blockDim.x) {
    if (window_interior<P>(d, w)) continue;
    bool nz = false;
    for (int i = 0; i < m && !nz; ++i) nz = g[(size_t)i * K + m + w] != 0.0;
    if (nz) atomicAdd(&cnt, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) nnz[blockIdx.x] = cnt;
}

template <int P>
__global__ void k_map_compact(const CutDesc* desc, const int64_t* dense_off, const double* Gd, double* Gc, int one_lane) {
  constexpr int WW = (4 * P + 1) * (4 * P + 1);
  const CutDesc d = desc[blockIdx.x];
  const int m = mask_count(d), K = m + WW;
  const double* g = Gd + dense_off[blockIdx.x];
  double* out = Gc + (d.map_off & ((1ll << 48) - 1));
  __shared__ uint8_t keep[WW];
  __shared__ uint8_t idx[WW];
  __shared__ int nnz;
  for (int w = threadIdx.x; w < WW; w += blockDim.x) {
    bool nz = false;
    if (!window_interior<P>(d, w))
      for (int i = 0; i < m && !nz; ++i) nz = g[(size_t)i * K + m + w] != 0.0;
    keep[w] = nz;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int c = 0;
    for (int w = 0; w < WW; ++w)
      if (keep[w]) idx[c++] = (uint8_t)w;
    nnz = c;
    ((int*)out)[0] = c;
    ((int*)out)[1] = 0;
    out[1] = 0.0;
    uint8_t* ob = (uint8_t*)(out + 2);
    for (int q = 0; q < ((c + 15) & ~15); ++q) ob[q] = q < c ? idx[q] : 0;
  }
  __syncthreads();
  const int Kc = m + nnz, Kp = map_kp(m, Kc, one_lane), tpr = map_tpr(m, one_lane), B = 2 * tpr;
  double* rows = out + map_hdr_d(nnz);
  for (int e = threadIdx.x; e < m * Kp; e += blockDim.x) {
    const int j = e / (B * m), rem = e - j * B * m, i = rem / B, pos = rem % B;
    const int c = B * j + pos / 2 + (pos % 2) * tpr;
    rows[e] = c >= Kc ? 0.0 : (c < m ? g[(size_t)i * K + c] : g[(size_t)i * K + m + idx[c - m]]);
  }
}

template <int P>
struct CutMapSmem {
  static constexpr int BS = 2 * P + 1, WS = 4 * P + 1, MM = BS * BS, WW = WS * WS;
  static constexpr int maxK = MM + WW + 7;   // K padded to a multiple of 2 tpr <= 8 (map_kp)
  // descriptor | v[maxK] | G_j [MM x maxK] | Lc[MM] shorts | exterior indices, window mask
  static constexpr size_t gs_off = 64 + (((size_t)maxK * 8 + 15) & ~(size_t)15);
  static constexpr size_t bytes = gs_off + (size_t)MM * maxK * 8 + 2 * MM + 2 * WW + 16;
};

// the cut-step-7 routine for a group of NT threads with named barrier `bar`:
// prologue (setup data only: descriptor, map block by cp.async, interior
// locations, exterior window indices), then main (after the previous step's
// writes are visible): gather b_I and x_E, x_I^new = G_j [b_I ; x_E], store.
// LDCG: read x through L2 only (previous step written by other SMs of the
// same launch).
template <int P, int NT>
__device__ __forceinline__ void cut7_prologue(const CutDesc* desc, int k, const double* G, unsigned char* gsm, int gt,
                                              int bar, int one_lane) {
  using S = CutMapSmem<P>;
  constexpr int MM = S::MM;
  CutDesc& d = *(CutDesc*)gsm;
  double* Gs = (double*)(gsm + S::gs_off);
  short* Lc = (short*)(Gs + (size_t)MM * S::maxK);
  uint8_t* ix = (uint8_t*)(Lc + MM);
  if (gt < 4) ((int4*)&d)[gt] = ((const int4*)(desc + k))[gt];
  group_sync(bar, NT);
  const int m = mask_count(d);
  // the kept exterior columns are DoF nodes inside the lattice (a column is
  // nonzero only if its node shares an active cell or a ghost face with the
  // interior), so the gather needs no mask
  const double* blk = G + (d.map_off & ((1ll << 48) - 1));
  const int nnz = (int)(d.map_off >> 48), K = m + nnz;
  const double* rows = blk + map_hdr_d(nnz);
  for (int e = gt; e < m * map_kp(m, K, one_lane); e += NT) cp_async8(Gs + e, rows + e);
  for (int loc = gt; loc < MM; loc += NT) {
    const unsigned long long word = d.mask[loc >> 6];
    if ((word >> (loc & 63)) & 1ull)
      Lc[(loc >> 6 ? __popcll(d.mask[0]) : 0) + __popcll(word & ((1ull << (loc & 63)) - 1ull))] = (short)loc;
  }
  for (int j = gt; j < nnz; j += NT) ix[j] = ((const uint8_t*)(blk + 2))[j];
  group_sync(bar, NT);   // Lc, ix visible (in k_cut_step7: before griddepcontrol.wait)
}

template <int P, int NT, bool LDCG>
__device__ __forceinline__ void cut7_main(const LevelArgs& L, const double* R, double* W, const double* b,
                                          unsigned char* gsm, int gt, int bar) {
  using S = CutMapSmem<P>;
  constexpr int BS = S::BS, WS = S::WS, MM = S::MM;
  const CutDesc& d = *(const CutDesc*)gsm;
  double* v = (double*)(gsm + 64);
  double* Gs = (double*)(gsm + S::gs_off);
  short* Lc = (short*)(Gs + (size_t)MM * S::maxK);
  uint8_t* ix = (uint8_t*)(Lc + MM);
  const int m = mask_count(d), nnz = (int)(d.map_off >> 48), K = m + nnz;
  const int a0 = P * (d.I - 2), b0 = P * (d.J - 2);
  for (int i = gt; i < m; i += NT) {
    const int loc = Lc[i];
    v[i] = b[(size_t)(P * (d.J - 1) + loc / BS) * L.ld + P * (d.I - 1) + loc % BS];
  }
  for (int j = gt; j < nnz; j += NT) {
    const int w = ix[j];
    const double* src = R + (size_t)(b0 + w / WS) * L.ld + a0 + w % WS;
    v[m + j] = LDCG ? __ldcg(src) : *src;
  }
  cp_async_wait_all();
  group_sync(bar, NT);
  // x_I^new = G_j v: TPR threads per row (power of two), shuffle-reduced; lane
  // h sums columns h + 2 tpr j (a0c) and h + tpr + 2 tpr j (a1c), j = 0, 1, ...
  // (the map's column-block layout, map_index; the order k_cut_sweep repeats)
  const int tpr = map_tpr(m, L.map_one_lane);
  static_assert(NT >= 128, "the map layout assumes 128-thread row groups (map_tpr)");
  for (int r0 = 0; r0 < m; r0 += NT / tpr) {
    const int i = r0 + gt / tpr, h = gt % tpr;
    double a0c = 0.0, a1c = 0.0;
    if (i < m) {
      const double* g = Gs + 2 * tpr * i + 2 * h;
      int c = h;
      for (; c + tpr < K; c += 2 * tpr, g += 2 * tpr * m) {
        a0c = fma(g[0], v[c], a0c);
        a1c = fma(g[1], v[c + tpr], a1c);
      }
      if (c < K) a0c = fma(g[0], v[c], a0c);
    }
    double z = a0c + a1c;
    for (int o = tpr >> 1; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
    if (i < m && h == 0) {
      const int loc = Lc[i];
      W[(size_t)(P * (d.J - 1) + loc / BS) * L.ld + P * (d.I - 1) + loc % BS] = z;
    }
  }
}

// hot path: one cut colour step with the precomputed maps (ping-pong as
// k_cut_step6): the prologue before griddepcontrol.wait, the main part after
template <int P, int NT>
__global__ void __launch_bounds__(NT) k_cut_step7(LevelArgs L, const CutDesc* desc, int np, const double* G,
                                                  const double* R, double* W, const double* b, const int32_t* copy,
                                                  int ncopy) {
  extern __shared__ __align__(128) unsigned char sm7[];
  const int tid = threadIdx.x;
  pdl_trigger();
  if ((int)blockIdx.x >= np) {
    const int e = (blockIdx.x - np) * NT + tid;
    if (e < ncopy) {
      const int32_t node = copy[e];
      pdl_wait();
      W[node] = R[node];
    }
    return;
  }
  cut7_prologue<P, NT>(desc, blockIdx.x, G, sm7, tid, 0, L.map_one_lane);
  pdl_wait();
  cut7_main<P, NT, false>(L, R, W, b, sm7, tid, 0);
}

}  // namespace cf
