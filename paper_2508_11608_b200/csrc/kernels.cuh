// kernels.cuh — hot-path kernels of the CutFEM vertex-patch multigrid.
//
//  * k_cart_colour   Cartesian-patch colour sweep (P l.189 sum factorisation,
//                    l.192 fast diagonalisation, eq. smoother-split l.200-201)
//  * k_cut_colour_p1 cut-patch colour sweep, phase 1: residual from cell
//                    quadrature + Nitsche (P eq. cutfem_nitsche l.81-86),
//                    tensor cells, ghost faces (l.104-108); z = A_j^{-1} r
//                    (l.193); phase 2 (k_cut_colour_p2) scatters x += z.
//  * k_band / k_node_apply   matrix-free A x (P l.187-190)
//  * k_prolongate_add / k_restrict   transfer (P l.126-137)
//  * vector kernels for CG (deterministic two-stage reductions)
#pragma once
#include "internal.cuh"
#include "setup.cuh"

namespace cf {

// host <-> device copy of the DoF span of every lattice row (host pointers of
// pinned, mapped memory are read / written directly over PCIe): block per
// row, span [a0, a1) of row b from span[2 b], span[2 b + 1]; rows of LD doubles
__global__ void k_copy_spans(const double* __restrict__ src, double* __restrict__ dst, const int* __restrict__ span,
                             int ld, int row0, const double* __restrict__ src2, double* __restrict__ dst2) {
  const int b = row0 + blockIdx.x;
  const int a0 = span[2 * b], a1 = span[2 * b + 1];
  const size_t o = (size_t)b * ld;
  if (blockIdx.y) {   // a second vector in the same launch (x and b together)
    src = src2;
    dst = dst2;
  }
  for (int a = a0 + threadIdx.x; a < a1; a += blockDim.x) dst[o + a] = src[o + a];
}


// 1D tables staged in shared memory where lanes index them with different
// (runtime) indices; constant memory serialises divergent addresses.
struct SmTab {
  double K[CF_MAXP + 1][CF_MAXP + 1];
  double M[CF_MAXP + 1][CF_MAXP + 1];
  double d0[CF_MAXP + 1][CF_MAXP + 1];
  double d1[CF_MAXP + 1][CF_MAXP + 1];
};

template <int P>
__device__ __forceinline__ void load_smtab(SmTab& s) {
  const Tab& T = g_tab[P];   // global copy: lane-varying indices would serialise constant-bank reads
  for (int e = threadIdx.x + blockDim.x * threadIdx.y; e < (CF_MAXP + 1) * (CF_MAXP + 1);
       e += blockDim.x * blockDim.y) {
    int i = e / (CF_MAXP + 1), j = e % (CF_MAXP + 1);
    s.K[i][j] = T.Kref[i][j];
    s.M[i][j] = T.Mref[i][j];
    s.d0[i][j] = T.d0[i][j];
    s.d1[i][j] = T.d1[i][j];
  }
}

// Lagrange values and first derivatives on [0,1] at xi (Horner, uniform
// constant-memory reads)
template <int P>
__device__ __forceinline__ void eval1d(double xi, double (&v)[P + 1], double (&d)[P + 1]) {
  const Tab& T = c_tab[P];
#pragma unroll
  for (int i = 0; i <= P; ++i) {
    double a = T.lc[i][P];
#pragma unroll
    for (int m = P - 1; m >= 0; --m) a = fma(a, xi, T.lc[i][m]);
    double b = T.dc[i][P - 1];
#pragma unroll
    for (int m = P - 2; m >= 0; --m) b = fma(b, xi, T.dc[i][m]);
    v[i] = a;
    d[i] = b;
  }
}

// one row (kx, ky) of the uncut cell matrix K⊗M + M⊗K applied to the cell
// values X (row stride xs); P l.189 (tensor-product cell, exact quadrature)
template <int P>
__device__ __forceinline__ double inside_row(const SmTab& T, const double* X, int xs, int kx, int ky) {
  double y = 0.0;
#pragma unroll
  for (int ly = 0; ly <= P; ++ly) {
    double sK = 0.0, sM = 0.0;
#pragma unroll
    for (int lx = 0; lx <= P; ++lx) {
      double v = X[ly * xs + lx];
      sK = fma(T.K[kx][lx], v, sK);
      sM = fma(T.M[kx][lx], v, sM);
    }
    y = fma(T.M[ky][ly], sK, fma(T.K[ky][ly], sM, y));
  }
  return y;
}

// Cut cell: bulk (grad u, grad v)_{T∩Omega} and Nitsche terms on Gamma∩T
// (P eq. cutfem_nitsche) by quadrature (R6).  Lanes stride over the points;
// the (p+1)^2 test-function sums are reduced across the warp, every lane
// returns the totals in acc.
template <int P>
__device__ __forceinline__ void cut_cell_warp(const LevelArgs& L, int cid, const double* X, int xs,
                                              double (&acc)[(P + 1) * (P + 1)]) {
  constexpr int NB = (P + 1) * (P + 1);
  const int lane = threadIdx.x & 31;
  const double hinv = 1.0 / L.h;
#pragma unroll
  for (int t = 0; t < NB; ++t) acc[t] = 0.0;
  double Xr[NB];
#pragma unroll
  for (int ky = 0; ky <= P; ++ky)
#pragma unroll
    for (int kx = 0; kx <= P; ++kx) Xr[ky * (P + 1) + kx] = X[ky * xs + kx];
  const int q0 = L.q_off[cid], q1 = L.q_off[cid + 1];
  for (int q = q0 + lane; q < q1; q += 32) {
    double Lx[P + 1], Dx[P + 1], Ly[P + 1], Dy[P + 1];
    eval1d<P>(L.qx[q], Lx, Dx);
    eval1d<P>(L.qy[q], Ly, Dy);
    double ux = 0.0, uy = 0.0;
#pragma unroll
    for (int ky = 0; ky <= P; ++ky) {
      double sd = 0.0, sv = 0.0;
#pragma unroll
      for (int kx = 0; kx <= P; ++kx) {
        sd = fma(Dx[kx], Xr[ky * (P + 1) + kx], sd);
        sv = fma(Lx[kx], Xr[ky * (P + 1) + kx], sv);
      }
      ux = fma(Ly[ky], sd, ux);
      uy = fma(Dy[ky], sv, uy);
    }
    const double wq = L.qw[q] * hinv * hinv;
    ux *= wq;
    uy *= wq;
#pragma unroll
    for (int ky = 0; ky <= P; ++ky)
#pragma unroll
      for (int kx = 0; kx <= P; ++kx)
        acc[ky * (P + 1) + kx] = fma(ux, Dx[kx] * Ly[ky], fma(uy, Lx[kx] * Dy[ky], acc[ky * (P + 1) + kx]));
  }
  const int s0 = L.s_off[cid], s1 = L.s_off[cid + 1];
  for (int q = s0 + lane; q < s1; q += 32) {
    double Lx[P + 1], Dx[P + 1], Ly[P + 1], Dy[P + 1];
    eval1d<P>(L.sx[q], Lx, Dx);
    eval1d<P>(L.sy[q], Ly, Dy);
    const double nx = L.snx[q] * hinv, ny = L.sny[q] * hinv, w = L.sw[q];
    double u = 0.0, ux = 0.0, uy = 0.0;
#pragma unroll
    for (int ky = 0; ky <= P; ++ky) {
      double sd = 0.0, sv = 0.0;
#pragma unroll
      for (int kx = 0; kx <= P; ++kx) {
        sd = fma(Dx[kx], Xr[ky * (P + 1) + kx], sd);
        sv = fma(Lx[kx], Xr[ky * (P + 1) + kx], sv);
      }
      ux = fma(Ly[ky], sd, ux);
      uy = fma(Dy[ky], sv, uy);
      u = fma(Ly[ky], sv, u);
    }
    const double un = nx * ux + ny * uy;          // d_n u
    const double cu = w * (L.gDh * u - un);       // coefficient of v
    const double cd = -w * u;                     // coefficient of d_n v
#pragma unroll
    for (int ky = 0; ky <= P; ++ky)
#pragma unroll
      for (int kx = 0; kx <= P; ++kx) {
        double v = Lx[kx] * Ly[ky];
        double dn = nx * Dx[kx] * Ly[ky] + ny * Lx[kx] * Dy[ky];
        acc[ky * (P + 1) + kx] = fma(cu, v, fma(cd, dn, acc[ky * (P + 1) + kx]));
      }
  }
#pragma unroll
  for (int t = 0; t < NB; ++t) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc[t] += __shfl_xor_sync(0xffffffffu, acc[t], off);
  }
}

// Ghost-penalty face (P l.104-108): moments Jm[k][q] = sum_l Mref[q][l] J_k[l]
// of the jumps J_k = d^k_n u|_T1 - d^k_n u|_T2 (reference derivatives) in the
// tangential basis.  axis 0: T1 = (i,j), T2 = (i+1,j); axis 1: T2 = (i,j+1).
template <int P>
__device__ __forceinline__ void face_moments(int axis, const double* X1, const double* X2, int xs,
                                             double (&Jm)[P + 1][P + 1]) {
  const Tab& T = c_tab[P];
#pragma unroll
  for (int k = 1; k <= P; ++k) {
    double J[P + 1];
#pragma unroll
    for (int l = 0; l <= P; ++l) {
      double s = 0.0;
#pragma unroll
      for (int nn = 0; nn <= P; ++nn) {
        double v1 = axis == 0 ? X1[l * xs + nn] : X1[nn * xs + l];
        double v2 = axis == 0 ? X2[l * xs + nn] : X2[nn * xs + l];
        s = fma(T.d1[k][nn], v1, fma(-T.d0[k][nn], v2, s));
      }
      J[l] = s;
    }
#pragma unroll
    for (int q = 0; q <= P; ++q) {
      double s = 0.0;
#pragma unroll
      for (int l = 0; l <= P; ++l) s = fma(T.Mref[q][l], J[l], s);
      Jm[k][q] = s;
    }
  }
}

// contribution of a ghost face to test function (kx, ky) of one of its cells;
// side 1 = T1 (derivatives at xi = 1, sign +), side 2 = T2 (xi = 0, sign -)
template <int P>
__device__ __forceinline__ double face_test(const LevelArgs& L, const SmTab& T, int axis, int side, int kx, int ky,
                                            const double* Jm /* [k][q] with stride P+1, k from 1 */) {
  double s = 0.0;
  int nn = axis == 0 ? kx : ky, tt = axis == 0 ? ky : kx;
#pragma unroll
  for (int k = 1; k <= P; ++k) {
    double d = side == 1 ? T.d1[k][nn] : -T.d0[k][nn];
    s = fma(L.gs[k] * d, Jm[(k - 1) * (P + 1) + tt], s);
  }
  return s;
}

// (A x) on the (2p+1)^2 block rows of the patch at vertex (I, J), from the
// (4p+1)^2 window W of x around it (origin lattice (p(I-2), p(J-2))).  Adds
// the patch cells (tensor or quadrature) and every ghost face with a patch
// cell on one side.  Complete for the rows whose support lies in the patch
// (the interior set).  One warp.
template <int P>
__device__ void local_block_apply(const LevelArgs& L, int I, int J, const double* W, double* Yb, const SmTab& T,
                                  double* Jsm /* per-warp P*(P+1) scratch */) {
  constexpr int NB = (P + 1) * (P + 1), BS = 2 * P + 1, WS = 4 * P + 1;
  const int lane = threadIdx.x & 31;
  const int kx = lane % (P + 1), ky = lane / (P + 1);
  for (int dy = 0; dy < 2; ++dy)
    for (int dx = 0; dx < 2; ++dx) {
      int ci = I - 1 + dx, cj = J - 1 + dy;
      int kind = cell_kind(L, L.ctype, ci, cj);
      if (kind == OUTSIDE) continue;
      const double* X = W + (P * (dy + 1)) * WS + P * (dx + 1);
      if (kind == INSIDE) {
        if (lane < NB) Yb[(P * dy + ky) * BS + P * dx + kx] += inside_row<P>(T, X, WS, kx, ky);
      } else {
        double acc[NB];
        cut_cell_warp<P>(L, L.cut_id[cj * L.n + ci], X, WS, acc);
#pragma unroll
        for (int t = 0; t < NB; ++t)
          if (lane == t) Yb[(P * dy + ky) * BS + P * dx + kx] += acc[t];
      }
      __syncwarp();
    }
  for (int axis = 0; axis < 2; ++axis)
    for (int s = 0; s < 3; ++s)
      for (int t = 0; t < 2; ++t) {
        int i1, j1, i2, j2;
        if (axis == 0) {
          i1 = I - 2 + s; j1 = J - 1 + t; i2 = i1 + 1; j2 = j1;
        } else {
          i1 = I - 1 + t; j1 = J - 2 + s; i2 = i1; j2 = j1 + 1;
        }
        int k1 = cell_kind(L, L.ctype, i1, j1), k2 = cell_kind(L, L.ctype, i2, j2);
        if (k1 == OUTSIDE || k2 == OUTSIDE || (k1 != CUT && k2 != CUT)) continue;
        const double* X1 = W + ((j1 - (J - 2)) * P) * WS + (i1 - (I - 2)) * P;
        const double* X2 = W + ((j2 - (J - 2)) * P) * WS + (i2 - (I - 2)) * P;
        double Jm[P + 1][P + 1];
        face_moments<P>(axis, X1, X2, WS, Jm);
        if (lane == 0) {
#pragma unroll
          for (int k = 1; k <= P; ++k)
#pragma unroll
            for (int q = 0; q <= P; ++q) Jsm[(k - 1) * (P + 1) + q] = Jm[k][q];
        }
        __syncwarp();
        bool in1 = i1 >= I - 1 && i1 <= I && j1 >= J - 1 && j1 <= J;
        bool in2 = i2 >= I - 1 && i2 <= I && j2 >= J - 1 && j2 <= J;
        if (lane < NB) {
          if (in1) Yb[((j1 - (J - 1)) * P + ky) * BS + (i1 - (I - 1)) * P + kx] += face_test<P>(L, T, axis, 1, kx, ky, Jsm);
          if (in2) Yb[((j2 - (J - 1)) * P + ky) * BS + (i2 - (I - 1)) * P + kx] += face_test<P>(L, T, axis, 2, kx, ky, Jsm);
        }
        __syncwarp();
      }
}

// ---------------------------------------------------------------------------
// Cut-patch colour step, phase 1: one warp per patch of the colour.
// z_j = A_j^{-1} (b - A x)|_{I_j} with x read before any update of this colour
// (R9); the corrections go to zbuf and are applied by phase 2.
template <int P, int WPB>
__global__ void __launch_bounds__(32 * WPB) k_cut_colour_p1(LevelArgs L, const int* plist, int np, int pbase,
                                                           const int64_t* ent_off, const uint16_t* ent_loc,
                                                           const int32_t* ent_node, const int64_t* inv_off,
                                                           const double* inv, const double* x, const double* b,
                                                           double* zbuf) {
  constexpr int BS = 2 * P + 1, WS = 4 * P + 1;
  __shared__ SmTab T;
  __shared__ double sW[WPB][WS * WS];
  __shared__ double sY[WPB][BS * BS];
  __shared__ double sR[WPB][BS * BS];
  __shared__ double sJ[WPB][P * (P + 1)];
  load_smtab<P>(T);
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k = blockIdx.x * WPB + w;
  if (k >= np) return;
  const int j = pbase + k;
  const int I = plist[k] % (L.n + 1), J = plist[k] / (L.n + 1);
  double* Wp = sW[w];
  double* Yb = sY[w];
  for (int e = lane; e < WS * WS; e += 32) {
    int a = P * (I - 2) + e % WS, bb = P * (J - 2) + e / WS;
    Wp[e] = (a >= 0 && bb >= 0 && a < L.nl && bb < L.nl) ? x[(size_t)bb * L.ld + a] : 0.0;
  }
  for (int e = lane; e < BS * BS; e += 32) Yb[e] = 0.0;
  __syncwarp();
  local_block_apply<P>(L, I, J, Wp, Yb, T, sJ[w]);
  __syncwarp();
  const int64_t e0 = ent_off[j];
  const int m = (int)(ent_off[j + 1] - e0);
  for (int i = lane; i < m; i += 32) sR[w][i] = b[ent_node[e0 + i]] - Yb[ent_loc[e0 + i]];
  __syncwarp();
  const double* A = inv + inv_off[j];
  for (int i = lane; i < m; i += 32) {
    double z = 0.0;
    for (int q = 0; q < m; ++q) z = fma(A[q * m + i], sR[w][q], z);
    zbuf[e0 + i] = z;
  }
}

// phase 2: x[node] += z for the entries of one colour
__global__ void k_cut_colour_p2(const int32_t* ent_node, const double* zbuf, int64_t e0, int64_t e1, double* x) {
  int64_t e = e0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < e1) x[ent_node[e]] += zbuf[e];
}

// local matrix column k of cut patch j: A_j e_k (setup, P l.156/l.193)
template <int P, int WPB>
__global__ void __launch_bounds__(32 * WPB) k_local_matrix(LevelArgs L, const int* plist_all, const int64_t* ent_off,
                                                          const uint16_t* ent_loc, const int32_t* ent_patch,
                                                          int64_t n_ent, const int64_t* inv_off, double* inv) {
  constexpr int BS = 2 * P + 1, WS = 4 * P + 1;
  __shared__ SmTab T;
  __shared__ double sW[WPB][WS * WS];
  __shared__ double sY[WPB][BS * BS];
  __shared__ double sJ[WPB][P * (P + 1)];
  load_smtab<P>(T);
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t e = blockIdx.x * (int64_t)WPB + w;
  if (e >= n_ent) return;
  const int j = ent_patch[e];
  const int I = plist_all[j] % (L.n + 1), J = plist_all[j] / (L.n + 1);
  const int64_t e0 = ent_off[j];
  const int m = (int)(ent_off[j + 1] - e0), kcol = (int)(e - e0);
  for (int q = lane; q < WS * WS; q += 32) sW[w][q] = 0.0;
  for (int q = lane; q < BS * BS; q += 32) sY[w][q] = 0.0;
  __syncwarp();
  if (lane == 0) {
    int loc = ent_loc[e];
    sW[w][(P + loc / BS) * WS + P + loc % BS] = 1.0;
  }
  __syncwarp();
  local_block_apply<P>(L, I, J, sW[w], sY[w], T, sJ[w]);
  __syncwarp();
  double* A = inv + inv_off[j];
  for (int i = lane; i < m; i += 32) A[i * m + kcol] = sY[w][ent_loc[e0 + i]];
}

// ---------------------------------------------------------------------------
// Cartesian-patch colour step: one CTA per tile of TP x TP same-colour
// patches; the (2p TP + 1)^2 lattice region of x and b is staged in shared
// memory with coalesced loads; one thread per patch computes the residual on
// the (2p-1)^2 interior by sum factorisation with the two-cell 1D matrices
// (K̄⊗M̄ + M̄⊗K̄) and applies the fast-diagonalisation inverse
// S (S^T R S ./ (lam_a + lam_b)) S^T (P l.192); interior nodes of Cartesian
// patches are written back coalesced.
template <int P, int TP>
__global__ void __launch_bounds__(TP* TP) k_cart_colour(LevelArgs L, const int* tiles, int colour, const uint8_t* vk,
                                                        double* x, const double* b) {
  constexpr int W = 2 * P * TP + 1, NE = 2 * P + 1, NI = 2 * P - 1;
  extern __shared__ double smem[];
  double* Xs = smem;
  double* Bs = smem + W * W;
  const Tab& T = c_tab[P];
  const int tile = tiles[blockIdx.x];
  const int ti = tile & 0xffff, tj = tile >> 16;
  const int I0 = (colour & 1) + 2 * ti * TP, J0 = (colour >> 1) + 2 * tj * TP;
  const int a0 = P * (I0 - 1), b0 = P * (J0 - 1);
  const int tid = threadIdx.x;
  for (int e = tid; e < W * W; e += TP * TP) {
    int a = a0 + e % W, bb = b0 + e / W;
    bool in = a >= 0 && bb >= 0 && a < L.nl && bb < L.nl;
    Xs[e] = in ? x[(size_t)bb * L.ld + a] : 0.0;
    Bs[e] = in ? b[(size_t)bb * L.ld + a] : 0.0;
  }
  __syncthreads();
  const int u = tid % TP, v = tid / TP;
  const int I = I0 + 2 * u, J = J0 + 2 * v, n = L.n;
  const bool cart = I <= n && J <= n && vk[J * (n + 1) + I] == V_CART;
  if (cart) {
    const double* X = Xs + (2 * P * v) * W + 2 * P * u;
    const double* B = Bs + (2 * P * v) * W + 2 * P * u;
    double R[NI][NI];
#pragma unroll
    for (int ia = 0; ia < NI; ++ia) {
      const int a = ia + 1;
      const int alo = a <= P ? 0 : P, ahi = a >= P ? 2 * P : P;  // band of the two-cell matrices
      double t1[NE], t2[NE];
#pragma unroll
      for (int bp = 0; bp < NE; ++bp) {
        double s1 = 0.0, s2 = 0.0;
#pragma unroll
        for (int ap = alo; ap <= ahi; ++ap) {
          double xv = X[bp * W + ap];
          s1 = fma(T.Kp[a][ap], xv, s1);
          s2 = fma(T.Mp[a][ap], xv, s2);
        }
        t1[bp] = s1;
        t2[bp] = s2;
      }
#pragma unroll
      for (int ib = 0; ib < NI; ++ib) {
        const int bq = ib + 1;
        const int blo = bq <= P ? 0 : P, bhi = bq >= P ? 2 * P : P;
        double s = B[bq * W + a];
#pragma unroll
        for (int bp = blo; bp <= bhi; ++bp) s = fma(-T.Mp[bq][bp], t1[bp], fma(-T.Kp[bq][bp], t2[bp], s));
        R[ib][ia] = s;
      }
    }
    // U = S^T R S ./ (lam_a + lam_b)
    double V[NI][NI];
#pragma unroll
    for (int ib = 0; ib < NI; ++ib)
#pragma unroll
      for (int be = 0; be < NI; ++be) {
        double s = 0.0;
#pragma unroll
        for (int ia = 0; ia < NI; ++ia) s = fma(R[ib][ia], T.S[ia][be], s);
        V[ib][be] = s;
      }
#pragma unroll
    for (int al = 0; al < NI; ++al)
#pragma unroll
      for (int be = 0; be < NI; ++be) {
        double s = 0.0;
#pragma unroll
        for (int ib = 0; ib < NI; ++ib) s = fma(T.S[ib][al], V[ib][be], s);
        R[al][be] = s / (T.lam[al] + T.lam[be]);
      }
    // Z = S U S^T, added to the interior of the patch block
#pragma unroll
    for (int al = 0; al < NI; ++al)
#pragma unroll
      for (int ia = 0; ia < NI; ++ia) {
        double s = 0.0;
#pragma unroll
        for (int be = 0; be < NI; ++be) s = fma(R[al][be], T.S[ia][be], s);
        V[al][ia] = s;
      }
    double* Xw = Xs + (2 * P * v) * W + 2 * P * u;
#pragma unroll
    for (int ib = 0; ib < NI; ++ib)
#pragma unroll
      for (int ia = 0; ia < NI; ++ia) {
        double s = 0.0;
#pragma unroll
        for (int al = 0; al < NI; ++al) s = fma(T.S[ib][al], V[al][ia], s);
        Xw[(ib + 1) * W + ia + 1] += s;
      }
  }
  __syncthreads();
  for (int e = tid; e < W * W; e += TP * TP) {
    int c = e % W, r = e / W;
    int lc = c % (2 * P), lr = r % (2 * P);
    if (lc == 0 || lr == 0) continue;
    int uu = c / (2 * P), vv = r / (2 * P);
    int II = I0 + 2 * uu, JJ = J0 + 2 * vv;
    if (II > n || JJ > n || vk[JJ * (n + 1) + II] != V_CART) continue;
    x[(size_t)(b0 + r) * L.ld + a0 + c] = Xs[e];
  }
}

// ---------------------------------------------------------------------------
// Operator A x, pass 1: cut cells (warp each, quadrature) and ghost faces
// (thread each, jump moments) into the level's scratch buffers.
// BandRange selects the cut cells [cut_lo, cut_lo + cut_n) and the ghost
// faces [g_lo0, g_lo0 + g_n0) U [g_lo1, g_lo1 + g_n1) (a rank's rows under the
// slab partition; everything otherwise).
struct BandRange {
  int cut_lo, cut_n, g_lo0, g_n0, g_lo1, g_n1;
};

template <int P, bool QUAD>
__global__ void __launch_bounds__(128) k_band(LevelArgs L, const double* x, BandRange R) {
  constexpr int NB = (P + 1) * (P + 1);
  __shared__ double sX[4][NB];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw0 = blockIdx.x * 4 + w;
  pdl_trigger();
  pdl_wait();
  if (gw0 < R.cut_n) {
    const int gw = R.cut_lo + gw0;
    const int c = L.cut_list[gw], i = c % L.n, j = c / L.n;
    for (int t = lane; t < NB; t += 32)
      sX[w][t] = x[(size_t)(j * P + t / (P + 1)) * L.ld + i * P + t % (P + 1)];
    __syncwarp();
    if (QUAD) {
      double acc[NB];
      cut_cell_warp<P>(L, gw, sX[w], P + 1, acc);
#pragma unroll
      for (int t = 0; t < NB; ++t)
        if (lane == t) L.ycut[(size_t)gw * NB + t] = acc[t];
    } else if (lane < NB) {
      const double* Er = L.ecut + ((size_t)gw * NB + lane) * NB;
      double s = 0.0;
#pragma unroll
      for (int l = 0; l < NB; ++l) s = fma(Er[l], sX[w][l], s);
      L.ycut[(size_t)gw * NB + lane] = s;
    }
    return;
  }
  const int k = (gw0 - R.cut_n) * 32 + lane;
  if (k >= R.g_n0 + R.g_n1) return;
  const int g = k < R.g_n0 ? R.g_lo0 + k : R.g_lo1 + (k - R.g_n0);
  const int f = L.ghost_list[g], n = L.n;
  const int axis = f >= n * n, c = f - axis * n * n, i = c % n, j = c / n;
  const double* X1 = x + (size_t)(j * P) * L.ld + i * P;
  const double* X2 = axis == 0 ? X1 + P : X1 + (size_t)P * L.ld;
  double Jm[P + 1][P + 1];
  face_moments<P>(axis, X1, X2, L.ld, Jm);
#pragma unroll
  for (int k = 1; k <= P; ++k)
#pragma unroll
    for (int q = 0; q <= P; ++q) L.jm[((size_t)g * P + k - 1) * (P + 1) + q] = Jm[k][q];
}

// Operator pass 2: one thread per lattice node gathers the contributions of
// the cells containing it (tensor rows on uncut cells, the cut-cell buffer)
// and of the ghost faces of those cells.  y = A x, or y = b - A x if b != 0.
template <int P>
__global__ void __launch_bounds__(256) k_node_apply(LevelArgs L, const double* x, const double* b, double* y, int row0,
                                                    int row1) {
  constexpr int NB = (P + 1) * (P + 1);
  __shared__ SmTab T;
  pdl_trigger();
  load_smtab<P>(T);
  __syncthreads();
  pdl_wait();
  const int a = blockIdx.x * blockDim.x + threadIdx.x, bb = row0 + blockIdx.y * blockDim.y + threadIdx.y;
  if (a >= L.ld || bb >= row1) return;
  const size_t o = (size_t)bb * L.ld + a;
  if (!L.mask[o]) {
    y[o] = 0.0;
    return;
  }
  const int n = L.n;
  const int i0 = (a % P == 0) ? a / P - 1 : a / P, i1 = min(a / P, n - 1);
  const int j0 = (bb % P == 0) ? bb / P - 1 : bb / P, j1 = min(bb / P, n - 1);
  double acc = 0.0;
  for (int j = max(j0, 0); j <= j1; ++j)
    for (int i = max(i0, 0); i <= i1; ++i) {
      const int kind = L.ctype[j * n + i];
      if (kind == OUTSIDE) continue;
      const int kx = a - i * P, ky = bb - j * P;
      if (kind == INSIDE) {
        acc += inside_row<P>(T, x + (size_t)(j * P) * L.ld + i * P, L.ld, kx, ky);
      } else {
        acc += L.ycut[(size_t)L.cut_id[j * n + i] * NB + ky * (P + 1) + kx];
      }
      int g;
      if (i >= 1 && (g = L.gx_id[j * n + i - 1]) >= 0) acc += face_test<P>(L, T, 0, 2, kx, ky, L.jm + (size_t)g * P * (P + 1));
      if ((g = L.gx_id[j * n + i]) >= 0) acc += face_test<P>(L, T, 0, 1, kx, ky, L.jm + (size_t)g * P * (P + 1));
      if (j >= 1 && (g = L.gy_id[(j - 1) * n + i]) >= 0) acc += face_test<P>(L, T, 1, 2, kx, ky, L.jm + (size_t)g * P * (P + 1));
      if ((g = L.gy_id[j * n + i]) >= 0) acc += face_test<P>(L, T, 1, 1, kx, ky, L.jm + (size_t)g * P * (P + 1));
    }
  y[o] = b ? b[o] - acc : acc;
}

// ---------------------------------------------------------------------------
// Transfer (P l.126-137).  x_f += P x_c: one thread per fine node; the
// coarse cell is the parent of the fine cell min(a/p, n_f-1); weights
// L_m((child + xi_k)/2).
template <int P>
__global__ void k_prolongate_add(LevelArgs Lf, LevelArgs Lc, const double* xc, double* xf, int row0, int row1) {
  __shared__ double pw[2 * P + 1][P + 1];
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  pdl_trigger();
  if (tid < (2 * P + 1) * (P + 1)) pw[tid / (P + 1)][tid % (P + 1)] = c_tab[P].pw[tid / (P + 1)][tid % (P + 1)];
  __syncthreads();
  pdl_wait();
  const int a = blockIdx.x * blockDim.x + threadIdx.x, bb = row0 + blockIdx.y * blockDim.y + threadIdx.y;
  if (a >= Lf.nl || bb >= row1) return;
  const size_t o = (size_t)bb * Lf.ld + a;
  if (!Lf.mask[o]) return;
  const int Ia = min(min(a / P, Lf.n - 1) / 2, Lc.n - 1), Ib = min(min(bb / P, Lf.n - 1) / 2, Lc.n - 1);
  const int da = a - 2 * P * Ia, db = bb - 2 * P * Ib;
  double s = 0.0;
#pragma unroll
  for (int nn = 0; nn <= P; ++nn) {
    double t = 0.0;
#pragma unroll
    for (int m = 0; m <= P; ++m) t = fma(pw[da][m], xc[(size_t)(Ib * P + nn) * Lc.ld + Ia * P + m], t);
    s = fma(pw[db][nn], t, s);
  }
  xf[o] += s;
}

// b_c = P^T r_f: one thread per coarse node gathers the fine nodes of the
// support of its basis function with weights phi^c(x_f) (tensor of 1D).
template <int P>
__global__ void k_restrict(LevelArgs Lf, LevelArgs Lc, const double* rf, double* bc, int row0, int row1,
                           double* xz /* optional: zeroed at the same entries (the coarse initial guess) */) {
  __shared__ double tw[P][4 * P + 1];
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  pdl_trigger();
  if (tid < P * (4 * P + 1)) tw[tid / (4 * P + 1)][tid % (4 * P + 1)] = c_tab[P].tw[tid / (4 * P + 1)][tid % (4 * P + 1)];
  __syncthreads();
  pdl_wait();
  const int A = blockIdx.x * blockDim.x + threadIdx.x, B = row0 + blockIdx.y * blockDim.y + threadIdx.y;
  if (A >= Lc.ld || B >= row1) return;
  const size_t o = (size_t)B * Lc.ld + A;
  if (xz) xz[o] = 0.0;
  if (A >= Lc.nl || !Lc.mask[o]) {
    bc[o] = 0.0;
    return;
  }
  const int mA = A % P, IA = A / P, mB = B % P, IB = B / P;
  const int dalo = mA == 0 ? -2 * P : 0, dblo = mB == 0 ? -2 * P : 0;
  // fully unrolled with predicated (zero-weight) terms so that all (4p+1)^2
  // loads are in flight at once; a zero-weight term adds fma(0, v, t) = t
  // (v is finite: residual entries of non-DoF nodes are 0)
  double s = 0.0;
#pragma unroll
  for (int db = -2 * P; db <= 2 * P; ++db) {
    const int fb = 2 * P * IB + db;
    const bool rb = db >= dblo && fb >= 0 && fb < Lf.nl;
    const double wb = rb ? tw[mB][db + 2 * P] : 0.0;
    double t = 0.0;
#pragma unroll
    for (int da = -2 * P; da <= 2 * P; ++da) {
      const int fa = 2 * P * IA + da;
      const bool ok = rb && wb != 0.0 && da >= dalo && fa >= 0 && fa < Lf.nl;
      const double v = ok ? rf[(size_t)fb * Lf.ld + fa] : 0.0;
      t = fma(ok ? tw[mA][da + 2 * P] : 0.0, v, t);
    }
    s = fma(wb, t, s);
  }
  bc[o] = s;
}

// ---------------------------------------------------------------------------
// exact coarse solve x_0 = A_0^{-1} b_0 (P l.124); one CTA
__global__ void k_coarse_solve(const double* Ainv, const int* nodes, int n0, const double* b, double* x) {
  extern __shared__ double bv[];
  for (int i = threadIdx.x; i < n0; i += blockDim.x) bv[i] = b[nodes[i]];
  __syncthreads();
  for (int i = threadIdx.x; i < n0; i += blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < n0; ++q) s = fma(Ainv[(size_t)i * n0 + q], bv[q], s);
    x[nodes[i]] = s;
  }
}

__global__ void k_gather_column(const double* y, const int* nodes, int n0, double* col) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n0) col[i] = y[nodes[i]];
}

__global__ void k_set_entry(double* v, int64_t idx, double val) { v[idx] = val; }

// ---------------------------------------------------------------------------
// vector kernels (CG); deterministic two-stage dot product with a fixed grid
constexpr int DOT_BLOCKS = 296, DOT_THREADS = 256;

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double ws[32];
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) ws[w] = v;
  __syncthreads();
  v = (threadIdx.x < blockDim.x / 32) ? ws[threadIdx.x] : 0.0;
  if (w == 0)
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

__global__ void __launch_bounds__(DOT_THREADS) k_dot_partial(const double* a, const double* b, int64_t n, double* part) {
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)DOT_THREADS + threadIdx.x; i < n; i += (int64_t)DOT_BLOCKS * DOT_THREADS)
    s = fma(a[i], b[i], s);
  s = block_sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// mode 0: sc[slot] = sum; mode 1 (alpha): sc[2] = sc[0] / sum, sc[1] = sum;
// mode 2 (beta): sc[5] = sum / sc[0], sc[0] = sum, sc[4] = sum
__global__ void __launch_bounds__(DOT_THREADS) k_dot_final(const double* part, double* sc, int mode, int slot) {
  double s = 0.0;
  for (int i = threadIdx.x; i < DOT_BLOCKS; i += DOT_THREADS) s += part[i];
  s = block_sum(s);
  if (threadIdx.x == 0) {
    if (mode == 0) sc[slot] = s;
    else if (mode == 1) { sc[1] = s; sc[2] = sc[0] / s; }
    else { sc[4] = s; sc[5] = s / sc[0]; sc[0] = s; }
  }
}

// the mode logic of k_dot_final applied to an all-reduced sum sc[7] (slab partition)
__global__ void k_dot_mode(double* sc, int mode, int slot) {
  const double s = sc[7];
  if (mode == 0) sc[slot] = s;
  else if (mode == 1) { sc[1] = s; sc[2] = sc[0] / s; }
  else { sc[4] = s; sc[5] = s / sc[0]; sc[0] = s; }
}

// x += alpha p, r -= alpha q
__global__ void k_cg_update(double* x, double* r, const double* p, const double* q, const double* sc, int64_t n) {
  const double al = sc[2];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = fma(al, p[i], x[i]);
    r[i] = fma(-al, q[i], r[i]);
  }
}

// p = z + beta p
__global__ void k_cg_direction(double* p, const double* z, const double* sc, int64_t n) {
  const double be = sc[5];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = fma(be, p[i], z[i]);
}

// dst = mask ? src : 0
// fitted box: zero the lattice nodes on the box boundary (no DoF, u = 0
// strongly), which the cell kernels read as part of their cells: 2D the 4
// boundary lines (4 nl threads), 3D the 6 boundary faces (6 nl^2 threads)
__global__ void k_zero_boundary(LevelArgs L, double* v) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int nl = L.nl, ld = L.ld;
  if (L.dim == 3) {
    if (t >= 6 * (int64_t)nl * nl) return;
    const int f = (int)(t / ((int64_t)nl * nl)), r = (int)(t % ((int64_t)nl * nl)), u = r % nl, w = r / nl;
    const int e = (f & 1) ? nl - 1 : 0;
    int a, b, c;
    if (f < 2) a = e, b = u, c = w;
    else if (f < 4) a = u, b = e, c = w;
    else a = u, b = w, c = e;
    v[((size_t)c * nl + b) * ld + a] = 0.0;
    return;
  }
  if (t >= 4 * (int64_t)nl) return;
  const int f = (int)(t / nl), u = (int)(t % nl), e = (f & 1) ? nl - 1 : 0;
  const int a = f < 2 ? e : u, b = f < 2 ? u : e;
  v[(size_t)b * ld + a] = 0.0;
}

__global__ void k_masked_copy(double* dst, const double* src, const uint8_t* mask, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = mask[i] ? src[i] : 0.0;
}

}  // namespace cf
