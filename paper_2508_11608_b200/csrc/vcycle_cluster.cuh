// vcycle_cluster.cuh — the coarse end of the V-cycle (levels lmax .. 0) in ONE
// launch of one thread-block cluster (DESIGN.md row n3).
//
// Below ~64^2 cells every step of the V-cycle (P l.124) is a few hundred
// patches or nodes of work, and a launch per step costs more than the work:
// the launch-per-step V-cycle spends ~35 us per smoothing step on every
// coarse level (9 dependent kernels).  Here the same steps run as phases of
// one cluster-resident kernel separated by cluster barriers
// (barrier.cluster.arrive.release / wait.acquire orders the global-memory
// writes of a phase before the reads of the next):
//   down  l = lmax..1: Cartesian colours (dense patch map, in place), the
//         4 n_c ping-pong cut steps (precomputed cut-patch maps), residual
//         (cut cells / ghost faces, then the node gather), restriction;
//   level 0: exact coarse solve;
//   up    l = 1..lmax: prolongation, reverse smoothing step.
// The arithmetic of every item is the one of the per-step kernels (same
// operands, same order), so the result is bit-identical to the launch path.
#pragma once
#include "smoother2.cuh"

namespace cf {

constexpr int VC_MAXL = 12;

struct CoarseLevel {
  LevelArgs L;
  const int* cart_list;      // Cartesian patches (packed I + (n+1) J) per colour
  int cart_off[5];
  const CutDesc* desc;       // cut patches per colour (maps in L / gmap)
  int cut_off[5];
  const double* gmap;
  const int32_t* copy;       // ping-pong copy lists [prev][cur]
  int copy_off[5][4], copy_n[5][4];
  double *x, *b, *r, *xs;    // workspaces (x, b of level lmax are the kernel arguments)
};

struct CoarseArgs {
  const CoarseLevel* lv;     // device array, levels 0..lmax
  int lmax, n_c, symmetric;
  const double* Gc;          // Cartesian patch map (host::cart_map)
  const double* c_inv;       // coarse inverse
  const int* c_nodes;
  int n0;
  double* x;                 // level lmax
  const double* b;
};

struct VcCtx {
  int gt, gs;                // cluster-wide thread index and count
  int lane, gw, nw;          // lane, cluster-wide warp index and count
};

// ---- phases --------------------------------------------------------------

template <int P>
__device__ void vc_cart_colour(const CoarseLevel& V, const double* Gc, int c, double* x, const double* b,
                               const VcCtx& t) {
  using C = CartMMA<P>;
  constexpr int NE = C::NE, NI = C::NI, NINT = C::NINT, K = C::K, COLS = C::COLS;
  const LevelArgs& L = V.L;
  const int p0 = V.cart_off[c], np = V.cart_off[c + 1] - p0;
  for (int q = t.gt; q < np; q += t.gs) {
    const int v = V.cart_list[p0 + q], I = v % (L.n + 1), J = v / (L.n + 1);
    const size_t o = (size_t)(P * (J - 1)) * L.ld + P * (I - 1);
    double op[K];
#pragma unroll
    for (int k = 0; k < NINT; ++k) op[k] = b[o + (size_t)(k / NI + 1) * L.ld + k % NI + 1];
#pragma unroll
    for (int k = 0; k < NE * NE; ++k) op[NINT + k] = x[o + (size_t)(k / NE) * L.ld + k % NE];
    double out[NINT];
#pragma unroll
    for (int r = 0; r < NINT; ++r) {
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int k = 0; k < K; k += 2) {
        s0 = fma(Gc[r * COLS + k], op[k], s0);
        if (k + 1 < K) s1 = fma(Gc[r * COLS + k + 1], op[k + 1], s1);
      }
      out[r] = s0 + s1;
    }
#pragma unroll
    for (int r = 0; r < NINT; ++r) x[o + (size_t)(r / NI + 1) * L.ld + r % NI + 1] = out[r];
  }
}

// one ping-pong cut step (as k_cut_step7): warp per patch, v gathered in shared memory
template <int P>
__device__ void vc_cut_step(const CoarseLevel& V, int c, int prev, const double* R, double* W, const double* b,
                            double* vsm, const VcCtx& t) {
  constexpr int BS = 2 * P + 1, WS = 4 * P + 1, MM = BS * BS;
  const LevelArgs& L = V.L;
  const int nco = prev < 0 ? 0 : V.copy_n[prev][c];
  const int32_t* cl = V.copy + (prev < 0 ? 0 : V.copy_off[prev][c]);
  for (int e = t.gt; e < nco; e += t.gs) W[cl[e]] = R[cl[e]];
  const int p0 = V.cut_off[c], np = V.cut_off[c + 1] - p0;
  short* Lc = (short*)(vsm + MM + WS * WS);
  for (int k = t.gw; k < np; k += t.nw) {
    const CutDesc d = V.desc[p0 + k];
    const int m = mask_count(d);
    const double* blk = V.gmap + (d.map_off & ((1ll << 48) - 1));
    const int nnz = (int)(d.map_off >> 48), K = m + nnz;
    const uint8_t* ix = (const uint8_t*)(blk + 1);
    const double* rows = blk + 1 + (nnz + 7) / 8;
    for (int loc = t.lane; loc < MM; loc += 32) {
      const unsigned long long word = d.mask[loc >> 6];
      if ((word >> (loc & 63)) & 1ull)
        Lc[(loc >> 6 ? __popcll(d.mask[0]) : 0) + __popcll(word & ((1ull << (loc & 63)) - 1ull))] = (short)loc;
    }
    __syncwarp();
    for (int i = t.lane; i < m; i += 32) {
      const int loc = Lc[i];
      vsm[i] = b[(size_t)(P * (d.J - 1) + loc / BS) * L.ld + P * (d.I - 1) + loc % BS];
    }
    const int a0 = P * (d.I - 2), b0 = P * (d.J - 2);
    for (int j = t.lane; j < nnz; j += 32) {
      const int w = ix[j];
      vsm[m + j] = R[(size_t)(b0 + w / WS) * L.ld + a0 + w % WS];
    }
    __syncwarp();
    for (int i = t.lane; i < m; i += 32) {
      const double* g = rows + (size_t)i * K;
      double s0 = 0.0, s1 = 0.0;
      int cc = 0;
      for (; cc + 1 < K; cc += 2) {
        s0 = fma(g[cc], vsm[cc], s0);
        s1 = fma(g[cc + 1], vsm[cc + 1], s1);
      }
      if (cc < K) s0 = fma(g[cc], vsm[cc], s0);
      const int loc = Lc[i];
      W[(size_t)(P * (d.J - 1) + loc / BS) * L.ld + P * (d.I - 1) + loc % BS] = s0 + s1;
    }
    __syncwarp();
  }
}

// residual pass 1 (k_band, element-matrix mode): cut cells (thread per
// (cell, test function)) and ghost faces (thread per face)
template <int P>
__device__ void vc_band(const LevelArgs& L, const double* x, const VcCtx& t) {
  constexpr int NB = (P + 1) * (P + 1);
  const int ncell = L.n_cut * NB;
  for (int it = t.gt; it < ncell + L.n_ghost; it += t.gs) {
    if (it < ncell) {
      const int gw = it / NB, tt = it - gw * NB;
      const int cidx = L.cut_list[gw], i = cidx % L.n, j = cidx / L.n;
      const double* Er = L.ecut + ((size_t)gw * NB + tt) * NB;
      double s = 0.0;
#pragma unroll
      for (int l = 0; l < NB; ++l) s = fma(Er[l], x[(size_t)(j * P + l / (P + 1)) * L.ld + i * P + l % (P + 1)], s);
      L.ycut[(size_t)gw * NB + tt] = s;
      continue;
    }
    const int g = it - ncell;
    const int f = L.ghost_list[g], n = L.n;
    const int axis = f >= n * n, cc = f - axis * n * n, i = cc % n, j = cc / n;
    const double* X1 = x + (size_t)(j * P) * L.ld + i * P;
    const double* X2 = axis == 0 ? X1 + P : X1 + (size_t)P * L.ld;
    double Jm[P + 1][P + 1];
    face_moments<P>(axis, X1, X2, L.ld, Jm);
#pragma unroll
    for (int k = 1; k <= P; ++k)
#pragma unroll
      for (int q = 0; q <= P; ++q) L.jm[((size_t)g * P + k - 1) * (P + 1) + q] = Jm[k][q];
  }
}

// residual pass 2 (k_node_apply): y = b - A x at every lattice node
template <int P>
__device__ void vc_node_apply(const LevelArgs& L, const SmTab& T, const double* x, const double* b, double* y,
                              const VcCtx& t) {
  constexpr int NB = (P + 1) * (P + 1);
  const int n = L.n;
  const int total = L.nl * L.ld;
  for (int o = t.gt; o < total; o += t.gs) {
    const int bb = o / L.ld, a = o - bb * L.ld;
    if (a >= L.nl || !L.mask[o]) {
      y[o] = 0.0;
      continue;
    }
    const int i0 = (a % P == 0) ? a / P - 1 : a / P, i1 = min(a / P, n - 1);
    const int j0 = (bb % P == 0) ? bb / P - 1 : bb / P, j1 = min(bb / P, n - 1);
    double acc = 0.0;
    for (int j = max(j0, 0); j <= j1; ++j)
      for (int i = max(i0, 0); i <= i1; ++i) {
        const int kind = L.ctype[j * n + i];
        if (kind == OUTSIDE) continue;
        const int kx = a - i * P, ky = bb - j * P;
        if (kind == INSIDE) acc += inside_row<P>(T, x + (size_t)(j * P) * L.ld + i * P, L.ld, kx, ky);
        else acc += L.ycut[(size_t)L.cut_id[j * n + i] * NB + ky * (P + 1) + kx];
        int g;
        if (i >= 1 && (g = L.gx_id[j * n + i - 1]) >= 0) acc += face_test<P>(L, T, 0, 2, kx, ky, L.jm + (size_t)g * P * (P + 1));
        if ((g = L.gx_id[j * n + i]) >= 0) acc += face_test<P>(L, T, 0, 1, kx, ky, L.jm + (size_t)g * P * (P + 1));
        if (j >= 1 && (g = L.gy_id[(j - 1) * n + i]) >= 0) acc += face_test<P>(L, T, 1, 2, kx, ky, L.jm + (size_t)g * P * (P + 1));
        if ((g = L.gy_id[j * n + i]) >= 0) acc += face_test<P>(L, T, 1, 1, kx, ky, L.jm + (size_t)g * P * (P + 1));
      }
    y[o] = b[o] - acc;
  }
}

// b_c = P^T r_f (k_restrict) and x_c = 0
template <int P>
__device__ void vc_restrict(const LevelArgs& Lf, const LevelArgs& Lc, const double* rf, double* bc, double* xc,
                            const VcCtx& t) {
  const Tab& Tb = c_tab[P];
  const int total = Lc.nl * Lc.ld;
  for (int o = t.gt; o < total; o += t.gs) {
    xc[o] = 0.0;
    const int B = o / Lc.ld, A = o - B * Lc.ld;
    if (A >= Lc.nl || !Lc.mask[o]) {
      bc[o] = 0.0;
      continue;
    }
    const int mA = A % P, IA = A / P, mB = B % P, IB = B / P;
    const int dalo = mA == 0 ? -2 * P : 0, dblo = mB == 0 ? -2 * P : 0;
    double s = 0.0;
    for (int db = dblo; db <= 2 * P; ++db) {
      const int fb = 2 * P * IB + db;
      if (fb < 0 || fb >= Lf.nl) continue;
      const double wb = Tb.tw[mB][db + 2 * P];
      if (wb == 0.0) continue;
      double tt = 0.0;
      for (int da = dalo; da <= 2 * P; ++da) {
        const int fa = 2 * P * IA + da;
        if (fa < 0 || fa >= Lf.nl) continue;
        tt = fma(Tb.tw[mA][da + 2 * P], rf[(size_t)fb * Lf.ld + fa], tt);
      }
      s = fma(wb, tt, s);
    }
    bc[o] = s;
  }
}

// x_f += P x_c (k_prolongate_add)
template <int P>
__device__ void vc_prolongate(const LevelArgs& Lf, const LevelArgs& Lc, const double* xc, double* xf, const VcCtx& t) {
  const Tab& Tb = c_tab[P];
  const int total = Lf.nl * Lf.nl;
  for (int e = t.gt; e < total; e += t.gs) {
    const int bb = e / Lf.nl, a = e - bb * Lf.nl;
    const size_t o = (size_t)bb * Lf.ld + a;
    if (!Lf.mask[o]) continue;
    const int Ia = min(min(a / P, Lf.n - 1) / 2, Lc.n - 1), Ib = min(min(bb / P, Lf.n - 1) / 2, Lc.n - 1);
    const int da = a - 2 * P * Ia, db = bb - 2 * P * Ib;
    double s = 0.0;
#pragma unroll
    for (int nn = 0; nn <= P; ++nn) {
      double tt = 0.0;
#pragma unroll
      for (int m = 0; m <= P; ++m) tt = fma(Tb.pw[da][m], xc[(size_t)(Ib * P + nn) * Lc.ld + Ia * P + m], tt);
      s = fma(Tb.pw[db][nn], tt, s);
    }
    xf[o] += s;
  }
}

template <int P>
__device__ void vc_smooth(const CoarseLevel& V, const CoarseArgs& A, double* x, const double* b, int reverse,
                          double* vsm, const VcCtx& t) {
  if (!reverse)
    for (int c = 0; c < 4; ++c) {
      vc_cart_colour<P>(V, A.Gc, c, x, b, t);
      cluster_sync_all();
    }
  double* bufs[2] = {x, V.xs};
  int prev = 4, s = 0;
  for (int rep = 0; rep < A.n_c; ++rep)
    for (int cc = 0; cc < 4; ++cc, ++s) {
      const int c = reverse ? 3 - cc : cc;
      vc_cut_step<P>(V, c, prev, bufs[s & 1], bufs[(s + 1) & 1], b, vsm, t);
      cluster_sync_all();
      prev = c;
    }
  if (reverse)
    for (int c = 3; c >= 0; --c) {
      vc_cart_colour<P>(V, A.Gc, c, x, b, t);
      cluster_sync_all();
    }
}

template <int P>
__global__ void __launch_bounds__(256) k_vcycle_cluster(CoarseArgs A) {
  constexpr int BS = 2 * P + 1, WS = 4 * P + 1, MM = BS * BS;
  constexpr int VW = MM + WS * WS + MM;   // per warp: v (<= MM + WS^2 doubles) + interior locations
  __shared__ SmTab T;
  __shared__ double vsm_all[8][VW];
  const int tid = threadIdx.x;
  VcCtx t;
  const int cr = (int)cluster_rank(), cs = (int)cluster_nctas();
  t.gt = cr * blockDim.x + tid;
  t.gs = cs * blockDim.x;
  t.lane = tid & 31;
  t.gw = cr * (blockDim.x >> 5) + (tid >> 5);
  t.nw = cs * (blockDim.x >> 5);
  double* vsm = vsm_all[tid >> 5];
  pdl_trigger();
  load_smtab<P>(T);
  __syncthreads();
  pdl_wait();
  cluster_sync_all();
  // down
  for (int l = A.lmax; l >= 1; --l) {
    const CoarseLevel& V = A.lv[l];
    double* x = l == A.lmax ? A.x : V.x;
    const double* b = l == A.lmax ? A.b : V.b;
    vc_smooth<P>(V, A, x, b, 0, vsm, t);
    vc_band<P>(V.L, x, t);
    cluster_sync_all();
    vc_node_apply<P>(V.L, T, x, b, V.r, t);
    cluster_sync_all();
    vc_restrict<P>(V.L, A.lv[l - 1].L, V.r, A.lv[l - 1].b, A.lv[l - 1].x, t);
    cluster_sync_all();
  }
  // exact coarse solve (P l.124)
  {
    const CoarseLevel& V = A.lv[0];
    for (int i = t.gt; i < A.n0; i += t.gs) {
      double s = 0.0;
      for (int q = 0; q < A.n0; ++q) s = fma(A.c_inv[(size_t)i * A.n0 + q], V.b[A.c_nodes[q]], s);
      V.x[A.c_nodes[i]] = s;
    }
    cluster_sync_all();
  }
  // up
  for (int l = 1; l <= A.lmax; ++l) {
    const CoarseLevel& V = A.lv[l];
    double* x = l == A.lmax ? A.x : V.x;
    const double* b = l == A.lmax ? A.b : V.b;
    vc_prolongate<P>(V.L, A.lv[l - 1].L, A.lv[l - 1].x, x, t);
    cluster_sync_all();
    vc_smooth<P>(V, A, x, b, A.symmetric ? 1 : 0, vsm, t);
  }
}

}  // namespace cf
