// dim3.cuh — 3D (sphere) kernels: the same method as the 2D path with
// hexahedral Q_p cells (p = 1, 2), 2x2x2 vertex patches and 8 colours
// (BASELINE.json configs[2..4]; oracle/dim3.py is the reference).
//
// Layout: lattice vectors NL x NL rows of LD doubles, node (a, b, c) at
// (c NL + b) LD + a; cells (k n + j) n + i; vertices (K (n+1) + J) (n+1) + I.
#pragma once
#include "kernels.cuh"
#include "smoother2.cuh"

namespace cf {

__device__ __forceinline__ int cell_kind3(const LevelArgs& L, int i, int j, int k) {
  const int n = L.n;
  return (i >= 0 && j >= 0 && k >= 0 && i < n && j < n && k < n) ? L.ctype[((size_t)k * n + j) * n + i] : OUTSIDE;
}

__device__ __forceinline__ void cell_bounds3(const LevelArgs& L, int i, int j, int k, double* lo, double* hi) {
  lo[0] = __dadd_rn(L.x0, __dmul_rn((double)i, L.h));
  hi[0] = __dadd_rn(L.x0, __dmul_rn((double)(i + 1), L.h));
  lo[1] = __dadd_rn(L.y0, __dmul_rn((double)j, L.h));
  hi[1] = __dadd_rn(L.y0, __dmul_rn((double)(j + 1), L.h));
  lo[2] = __dadd_rn(L.z0, __dmul_rn((double)k, L.h));
  hi[2] = __dadd_rn(L.z0, __dmul_rn((double)(k + 1), L.h));
}

// classification (reading R2 in 3D: sums in the order x, y, z)
__global__ void k_classify3(LevelArgs L, int8_t* ct) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int n = L.n;
  if (c >= (int64_t)n * n * n) return;
  const int i = c % n, j = (c / n) % n, k = c / ((int64_t)n * n);
  if (L.fitted) {   // fitted box: every cell is Inside
    ct[c] = INSIDE;
    return;
  }
  double lo[3], hi[3];
  cell_bounds3(L, i, j, k, lo, hi);
  const double cc[3] = {L.cx, L.cy, L.cz};
  double dmin2 = 0.0, dmax2 = 0.0;
  for (int d = 0; d < 3; ++d) {
    const double q = __dsub_rn(fmin(fmax(cc[d], lo[d]), hi[d]), cc[d]);
    const double f = fmax(fabs(__dsub_rn(lo[d], cc[d])), fabs(__dsub_rn(hi[d], cc[d])));
    dmin2 = d == 0 ? __dmul_rn(q, q) : __dadd_rn(dmin2, __dmul_rn(q, q));
    dmax2 = d == 0 ? __dmul_rn(f, f) : __dadd_rn(dmax2, __dmul_rn(f, f));
  }
  const double r2 = __dmul_rn(L.r, L.r);
  int8_t t = CUT;
  if (dmax2 <= r2) t = INSIDE;
  if (dmin2 >= r2) t = OUTSIDE;
  ct[c] = t;
}

__global__ void k_mask3(LevelArgs L, const int8_t* ct, uint8_t* mask, int* count) {
  const int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int nl = L.nl, ld = L.ld, p = L.p;
  if (o >= (int64_t)nl * nl * ld) return;
  const int a = o % ld, b = (o / ld) % nl, c = o / ((int64_t)ld * nl);
  uint8_t m = 0;
  if (a < nl) {
    const int i0 = (a % p == 0) ? a / p - 1 : a / p, i1 = a / p;
    const int j0 = (b % p == 0) ? b / p - 1 : b / p, j1 = b / p;
    const int k0 = (c % p == 0) ? c / p - 1 : c / p, k1 = c / p;
    for (int k = k0; k <= k1; ++k)
      for (int j = j0; j <= j1; ++j)
        for (int i = i0; i <= i1; ++i)
          if (cell_kind3(L, i, j, k) != OUTSIDE) m = 1;
    if (L.fitted && (a == 0 || b == 0 || c == 0 || a == nl - 1 || b == nl - 1 || c == nl - 1)) m = 0;
  }
  mask[o] = m;
  if (m) atomicAdd(count, 1);
}

__global__ void k_parent_check3(LevelArgs Lf, LevelArgs Lc, int* bad) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int n = Lf.n;
  if (c >= (int64_t)n * n * n) return;
  const int i = c % n, j = (c / n) % n, k = c / ((int64_t)n * n);
  if (Lf.ctype[c] != OUTSIDE && cell_kind3(Lc, i / 2, j / 2, k / 2) == OUTSIDE) atomicAdd(bad, 1);
}

__global__ void k_cell_flags(int64_t ncell, const int8_t* ct, int8_t want, uint8_t* flag) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c < ncell) flag[c] = ct[c] == want;
}

// ghost faces F_G in 3D: f = axis n^3 + cell, face between cell and its + neighbour
__global__ void k_ghost_flags3(LevelArgs L, uint8_t* flag) {
  const int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int n = L.n;
  const int64_t n3 = (int64_t)n * n * n;
  if (f >= 3 * n3) return;
  const int axis = (int)(f / n3);
  const int64_t c = f - axis * n3;
  const int i = c % n, j = (c / n) % n, k = c / ((int64_t)n * n);
  const int k1 = cell_kind3(L, i, j, k), k2 = cell_kind3(L, i + (axis == 0), j + (axis == 1), k + (axis == 2));
  flag[f] = k1 != OUTSIDE && k2 != OUTSIDE && (k1 == CUT || k2 == CUT);
}

__global__ void k_ghost_maps3(const int* list, int ng, int n, int* gx, int* gy, int* gz) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= ng) return;
  const int64_t n3 = (int64_t)n * n * n, f = list[g];
  const int axis = (int)(f / n3);
  int* m = axis == 0 ? gx : (axis == 1 ? gy : gz);
  m[f - axis * n3] = g;
}

// ---- cut-cell quadrature in 3D (reading R12, oracle.dim3.cut_cell_rules3) ----
__device__ __forceinline__ int sort_unique(double* v, int nv, double lo, double hi, double* out) {
  int np = 0;
  for (int k = 0; k < nv; ++k)
    if (lo <= v[k] && v[k] <= hi) out[np++] = v[k];
  for (int a = 1; a < np; ++a) {
    const double x = out[a];
    int b = a - 1;
    while (b >= 0 && out[b] > x) {
      out[b + 1] = out[b];
      --b;
    }
    out[b + 1] = x;
  }
  int nu = 0;
  for (int k = 0; k < np; ++k)
    if (nu == 0 || out[k] != out[nu - 1]) out[nu++] = out[k];
  return nu;
}

template <bool WRITE>
__device__ void cut_rule3(const LevelArgs& L, int i, int j, int k, int nq, int& nv, int& ns, int64_t vo, int64_t so,
                          double* const* q, double* const* s) {
  double lo[3], hi[3];
  cell_bounds3(L, i, j, k, lo, hi);
  const double c[3] = {L.cx, L.cy, L.cz};
  const double r = L.r, r2 = __dmul_rn(r, r), h = L.h;
  double dist[3];
  for (int d = 0; d < 3; ++d) dist[d] = fabs(__dsub_rn(__dmul_rn(0.5, __dadd_rn(lo[d], hi[d])), c[d]));
  int hax = 0;
  for (int d = 1; d < 3; ++d)
    if (dist[d] >= dist[hax]) hax = d;
  const int b0 = hax == 0 ? 1 : 0, b1 = hax == 2 ? 1 : 2;
  const int vax = dist[b1] >= dist[b0] ? b1 : b0, uax = vax == b1 ? b0 : b1;
  double radii2[3];
  int nr = 0;
  radii2[nr++] = r2;
  const double faces[2] = {lo[hax], hi[hax]};
  for (int f = 0; f < 2; ++f) {
    const double dd = __dsub_rn(faces[f], c[hax]);
    const double D = __dsub_rn(r2, __dmul_rn(dd, dd));
    if (D > 0.0) radii2[nr++] = D;
  }
  double br[20], ub[20];
  int nb = 0;
  br[nb++] = lo[uax];
  br[nb++] = hi[uax];
  for (int t = 0; t < nr; ++t) {
    const double vf[2] = {lo[vax], hi[vax]};
    for (int f = 0; f < 2; ++f) {
      const double dv = __dsub_rn(vf[f], c[vax]);
      const double D = __dsub_rn(radii2[t], __dmul_rn(dv, dv));
      if (D > 0.0) {
        const double qq = sqrt(D);
        br[nb++] = __dsub_rn(c[uax], qq);
        br[nb++] = __dadd_rn(c[uax], qq);
      }
    }
    const double R = sqrt(radii2[t]);
    br[nb++] = __dsub_rn(c[uax], R);
    br[nb++] = __dadd_rn(c[uax], R);
  }
  const int nub = sort_unique(br, nb, lo[uax], hi[uax], ub);
  const double* g = c_gx[nq];
  const double* w = c_gw[nq];
  nv = 0;
  ns = 0;
  for (int iu = 0; iu + 1 < nub; ++iu) {
    const double ua = ub[iu], ubb = ub[iu + 1];
    if (!(ubb > ua)) continue;
    for (int gi = 0; gi < nq; ++gi) {
      const double u = __dadd_rn(ua, __dmul_rn(__dsub_rn(ubb, ua), g[gi]));
      const double wu = w[gi] * (ubb - ua);
      const double du = __dsub_rn(u, c[uax]);
      double vbr[8], vb[8];
      int nvb = 0;
      vbr[nvb++] = lo[vax];
      vbr[nvb++] = hi[vax];
      for (int t = 0; t < nr; ++t) {
        const double D = __dsub_rn(radii2[t], __dmul_rn(du, du));
        if (D > 0.0) {
          const double qq = sqrt(D);
          vbr[nvb++] = __dsub_rn(c[vax], qq);
          vbr[nvb++] = __dadd_rn(c[vax], qq);
        }
      }
      const int nvu = sort_unique(vbr, nvb, lo[vax], hi[vax], vb);
      for (int iv = 0; iv + 1 < nvu; ++iv) {
        const double va = vb[iv], vbb = vb[iv + 1];
        if (!(vbb > va)) continue;
        for (int gj = 0; gj < nq; ++gj) {
          const double v = __dadd_rn(va, __dmul_rn(__dsub_rn(vbb, va), g[gj]));
          const double wuv = wu * (w[gj] * (vbb - va));
          const double dv = __dsub_rn(v, c[vax]);
          const double D = __dsub_rn(r2, __dadd_rn(__dmul_rn(du, du), __dmul_rn(dv, dv)));
          if (!(D > 0.0)) continue;
          const double S = sqrt(D);
          const double hl = fmax(lo[hax], __dsub_rn(c[hax], S)), hh = fmin(hi[hax], __dadd_rn(c[hax], S));
          double pt[3];
          pt[uax] = u;
          pt[vax] = v;
          if (hh > hl) {
            for (int gk = 0; gk < nq; ++gk) {
              if (WRITE) {
                pt[hax] = hl + (hh - hl) * g[gk];
                for (int d = 0; d < 3; ++d) q[d][vo + nv] = (pt[d] - lo[d]) / h;
                q[3][vo + nv] = wuv * (w[gk] * (hh - hl));
              }
              ++nv;
            }
          }
          const double sv[2] = {__dsub_rn(c[hax], S), __dadd_rn(c[hax], S)};
          for (int e = 0; e < 2; ++e) {
            if (lo[hax] < sv[e] && sv[e] < hi[hax]) {
              if (WRITE) {
                pt[hax] = sv[e];
                for (int d = 0; d < 3; ++d) {
                  s[d][so + ns] = (pt[d] - lo[d]) / h;
                  s[4 + d][so + ns] = (pt[d] - c[d]) / r;
                }
                s[3][so + ns] = wuv * r / S;
              }
              ++ns;
            }
          }
        }
      }
    }
  }
}

__global__ void k_cut_count3(LevelArgs L, int nq, int* vc, int* sc) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= L.n_cut) return;
  const int64_t c = L.cut_list[t];
  const int n = L.n;
  int nv, ns;
  cut_rule3<false>(L, c % n, (c / n) % n, c / ((int64_t)n * n), nq, nv, ns, 0, 0, nullptr, nullptr);
  vc[t] = nv;
  sc[t] = ns;
}

struct QPtrs3 {
  double* q[4];  // qx qy qz qw
  double* s[7];  // sx sy sz sw snx sny snz
};

__global__ void k_cut_fill3(LevelArgs L, int nq, QPtrs3 P) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= L.n_cut) return;
  const int64_t c = L.cut_list[t];
  const int n = L.n;
  int nv, ns;
  cut_rule3<true>(L, c % n, (c / n) % n, c / ((int64_t)n * n), nq, nv, ns, L.q_off[t], L.s_off[t], P.q, P.s);
}

// ---- cut-cell operator by quadrature (setup: element matrices) -------------
template <int P>
__device__ void cut_cell_warp3(const LevelArgs& L, int cid, const double* X /*(P+1)^3 contiguous*/,
                               double (&acc)[(P + 1) * (P + 1) * (P + 1)]) {
  constexpr int N1 = P + 1, NB = N1 * N1 * N1;
  const int lane = threadIdx.x & 31;
  const double hinv = 1.0 / L.h;
#pragma unroll
  for (int t = 0; t < NB; ++t) acc[t] = 0.0;
  for (int q = L.q_off[cid] + lane; q < L.q_off[cid + 1]; q += 32) {
    double Lx[N1], Dx[N1], Ly[N1], Dy[N1], Lz[N1], Dz[N1];
    eval1d<P>(L.qx[q], Lx, Dx);
    eval1d<P>(L.qy[q], Ly, Dy);
    eval1d<P>(L.qz[q], Lz, Dz);
    double ux = 0.0, uy = 0.0, uz = 0.0;
#pragma unroll
    for (int t = 0; t < NB; ++t) {
      const int kx = t % N1, ky = (t / N1) % N1, kz = t / (N1 * N1);
      ux = fma(Dx[kx] * Ly[ky] * Lz[kz], X[t], ux);
      uy = fma(Lx[kx] * Dy[ky] * Lz[kz], X[t], uy);
      uz = fma(Lx[kx] * Ly[ky] * Dz[kz], X[t], uz);
    }
    const double wq = L.qw[q] * hinv * hinv;
#pragma unroll
    for (int t = 0; t < NB; ++t) {
      const int kx = t % N1, ky = (t / N1) % N1, kz = t / (N1 * N1);
      acc[t] = fma(wq, ux * Dx[kx] * Ly[ky] * Lz[kz] + uy * Lx[kx] * Dy[ky] * Lz[kz] + uz * Lx[kx] * Ly[ky] * Dz[kz],
                   acc[t]);
    }
  }
  for (int q = L.s_off[cid] + lane; q < L.s_off[cid + 1]; q += 32) {
    double Lx[N1], Dx[N1], Ly[N1], Dy[N1], Lz[N1], Dz[N1];
    eval1d<P>(L.sx[q], Lx, Dx);
    eval1d<P>(L.sy[q], Ly, Dy);
    eval1d<P>(L.sz[q], Lz, Dz);
    const double nx = L.snx[q] * hinv, ny = L.sny[q] * hinv, nz = L.snz[q] * hinv, w = L.sw[q];
    double u = 0.0, un = 0.0;
#pragma unroll
    for (int t = 0; t < NB; ++t) {
      const int kx = t % N1, ky = (t / N1) % N1, kz = t / (N1 * N1);
      const double v = Lx[kx] * Ly[ky] * Lz[kz];
      const double dn = nx * Dx[kx] * Ly[ky] * Lz[kz] + ny * Lx[kx] * Dy[ky] * Lz[kz] + nz * Lx[kx] * Ly[ky] * Dz[kz];
      u = fma(v, X[t], u);
      un = fma(dn, X[t], un);
    }
    const double cu = w * (L.gDh * u - un), cd = -w * u;
#pragma unroll
    for (int t = 0; t < NB; ++t) {
      const int kx = t % N1, ky = (t / N1) % N1, kz = t / (N1 * N1);
      const double v = Lx[kx] * Ly[ky] * Lz[kz];
      const double dn = nx * Dx[kx] * Ly[ky] * Lz[kz] + ny * Lx[kx] * Dy[ky] * Lz[kz] + nz * Lx[kx] * Ly[ky] * Dz[kz];
      acc[t] = fma(cu, v, fma(cd, dn, acc[t]));
    }
  }
#pragma unroll
  for (int t = 0; t < NB; ++t)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc[t] += __shfl_xor_sync(0xffffffffu, acc[t], off);
}

template <int P>
__global__ void __launch_bounds__(128) k_cut_elem3(LevelArgs L, double* E) {
  constexpr int NB = (P + 1) * (P + 1) * (P + 1);
  __shared__ double sX[4][NB];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t g = blockIdx.x * 4LL + w;
  if (g >= (int64_t)L.n_cut * NB) return;
  const int cid = (int)(g / NB), col = (int)(g % NB);
  for (int t = lane; t < NB; t += 32) sX[w][t] = t == col ? 1.0 : 0.0;
  __syncwarp();
  double acc[NB];
  cut_cell_warp3<P>(L, cid, sX[w], acc);
#pragma unroll
  for (int t = 0; t < NB; ++t)
    if (lane == (t & 31)) E[((int64_t)cid * NB + t) * NB + col] = acc[t];   // (all lanes hold the sums; NB > 32 for Q3)
}

// ---- element pieces shared by the patch kernels and the operator ------------
// row (kx,ky,kz) of the uncut hex matrix h (K⊗M⊗M + M⊗K⊗M + M⊗M⊗K) applied
// to the cell values X (strides sy, sz)
template <int P>
__device__ __forceinline__ double inside_row3(const SmTab& T, const double* X, int sy, int sz, int kx, int ky, int kz,
                                              double h) {
  double y = 0.0;
#pragma unroll
  for (int lz = 0; lz <= P; ++lz)
#pragma unroll
    for (int ly = 0; ly <= P; ++ly) {
      double sK = 0.0, sM = 0.0;
#pragma unroll
      for (int lx = 0; lx <= P; ++lx) {
        const double v = X[lz * sz + ly * sy + lx];
        sK = fma(T.K[kx][lx], v, sK);
        sM = fma(T.M[kx][lx], v, sM);
      }
      y = fma(T.M[ky][ly] * T.M[kz][lz], sK, y);
      y = fma(T.K[ky][ly] * T.M[kz][lz] + T.M[ky][ly] * T.K[kz][lz], sM, y);
    }
  return y * h;
}

// ghost face moments in 3D: Jm[k][q1][q2] = sum (M⊗M) J_k over the
// tangential (t1 < t2) indices; X1, X2 = cell value arrays (strides sy, sz)
template <int P>
__device__ __forceinline__ void face_moments3(int axis, const double* X1, const double* X2, int sy, int sz,
                                              double* Jm /* [P][(P+1)^2] */) {
  const Tab& T = c_tab[P];
  constexpr int N1 = P + 1;
  const int st[3] = {1, sy, sz};
  const int t1 = axis == 0 ? 1 : 0, t2 = axis == 2 ? 1 : 2;
  for (int k = 1; k <= P; ++k) {
    double J[N1][N1];
#pragma unroll
    for (int l1 = 0; l1 < N1; ++l1)
#pragma unroll
      for (int l2 = 0; l2 < N1; ++l2) {
        double s = 0.0;
#pragma unroll
        for (int nn = 0; nn < N1; ++nn) {
          const int o = nn * st[axis] + l1 * st[t1] + l2 * st[t2];
          s = fma(T.d1[k][nn], X1[o], fma(-T.d0[k][nn], X2[o], s));
        }
        J[l1][l2] = s;
      }
#pragma unroll
    for (int q1 = 0; q1 < N1; ++q1)
#pragma unroll
      for (int q2 = 0; q2 < N1; ++q2) {
        double s = 0.0;
#pragma unroll
        for (int l1 = 0; l1 < N1; ++l1)
#pragma unroll
          for (int l2 = 0; l2 < N1; ++l2) s = fma(T.Mref[q1][l1] * T.Mref[q2][l2], J[l1][l2], s);
        Jm[(k - 1) * N1 * N1 + q1 * N1 + q2] = s;
      }
  }
}

// contribution of a ghost face (moments Jm) to test (kx,ky,kz) of side 1 (+d1) or 2 (-d0)
template <int P>
__device__ __forceinline__ double face_test3(const LevelArgs& L, const SmTab& T, int axis, int side, int kx, int ky,
                                             int kz, const double* Jm) {
  constexpr int N1 = P + 1;
  const int kk[3] = {kx, ky, kz};
  const int t1 = axis == 0 ? 1 : 0, t2 = axis == 2 ? 1 : 2;
  double s = 0.0;
#pragma unroll
  for (int k = 1; k <= P; ++k) {
    const double d = side == 1 ? T.d1[k][kk[axis]] : -T.d0[k][kk[axis]];
    s = fma(L.gs[k] * d, Jm[(k - 1) * N1 * N1 + kk[t1] * N1 + kk[t2]], s);
  }
  return s;
}

// (A x) on the (2p+1)^3 block rows of the patch at vertex (I,J,K) from the
// (4p+1)^3 window W (origin p(I-2), p(J-2), p(K-2)); one warp; Yb (2p+1)^3.
// Cut cells use the precomputed element matrices E (cut_mode 0) or quadrature.
template <int P>
__device__ void local_block_apply3(const LevelArgs& L, int I, int J, int K, const double* W, double* Yb, const SmTab& T,
                                   double* Js, bool quad) {
  constexpr int N1 = P + 1, NB = N1 * N1 * N1, BS = 2 * P + 1, WS = 4 * P + 1;
  const int lane = threadIdx.x & 31;
  for (int q = 0; q < 8; ++q) {
    const int dx = q & 1, dy = (q >> 1) & 1, dz = q >> 2;
    const int ci = I - 1 + dx, cj = J - 1 + dy, ck = K - 1 + dz;
    const int kind = cell_kind3(L, ci, cj, ck);
    if (kind == OUTSIDE) continue;
    const double* X = W + (P * (dz + 1) * WS + P * (dy + 1)) * WS + P * (dx + 1);
    if (kind == INSIDE) {
      for (int t = lane; t < NB; t += 32) {
        const int kx = t % N1, ky = (t / N1) % N1, kz = t / (N1 * N1);
        Yb[((P * dz + kz) * BS + P * dy + ky) * BS + P * dx + kx] += inside_row3<P>(T, X, WS, WS * WS, kx, ky, kz, L.h);
      }
    } else {
      const int cid = L.cut_id[((size_t)ck * L.n + cj) * L.n + ci];
      if (quad) {
        double xc[NB];
#pragma unroll
        for (int t = 0; t < NB; ++t) xc[t] = X[((t / (N1 * N1)) * WS + (t / N1) % N1) * WS + t % N1];
        // stage the cell values contiguously for cut_cell_warp3 (Js as scratch)
        __syncwarp();
        if (lane == 0)
          for (int t = 0; t < NB; ++t) Js[t] = xc[t];
        __syncwarp();
        double acc[NB];
        cut_cell_warp3<P>(L, cid, Js, acc);
#pragma unroll
        for (int t = 0; t < NB; ++t)
          if (lane == (t & 31)) {
            const int kx = t % N1, ky = (t / N1) % N1, kz = t / (N1 * N1);
            Yb[((P * dz + kz) * BS + P * dy + ky) * BS + P * dx + kx] += acc[t];
          }
      } else {
        const double* E = L.ecut + (size_t)cid * NB * NB;
        for (int t = lane; t < NB; t += 32) {
          double s = 0.0;
          for (int l = 0; l < NB; ++l) s = fma(E[t * NB + l], X[((l / (N1 * N1)) * WS + (l / N1) % N1) * WS + l % N1], s);
          const int kx = t % N1, ky = (t / N1) % N1, kz = t / (N1 * N1);
          Yb[((P * dz + kz) * BS + P * dy + ky) * BS + P * dx + kx] += s;
        }
      }
    }
    __syncwarp();
  }
  // faces with a patch cell on one side: axis a, cells c1 | c1 + e_a with the
  // normal coordinate s in {-2..0} + 1 (i.e. I-2..I relative) and the 2x2
  // tangential positions of the block
  for (int axis = 0; axis < 3; ++axis)
    for (int s = 0; s < 3; ++s)
      for (int t = 0; t < 4; ++t) {
        int c1[3];
        const int t1 = axis == 0 ? 1 : 0, t2 = axis == 2 ? 1 : 2;
        const int base[3] = {I - 1, J - 1, K - 1};
        c1[axis] = base[axis] - 1 + s;
        c1[t1] = base[t1] + (t & 1);
        c1[t2] = base[t2] + (t >> 1);
        int c2[3] = {c1[0], c1[1], c1[2]};
        c2[axis] += 1;
        const int k1 = cell_kind3(L, c1[0], c1[1], c1[2]), k2 = cell_kind3(L, c2[0], c2[1], c2[2]);
        if (k1 == OUTSIDE || k2 == OUTSIDE || (k1 != CUT && k2 != CUT)) continue;
        const double* X1 = W + (P * (c1[2] - K + 2) * WS + P * (c1[1] - J + 2)) * WS + P * (c1[0] - I + 2);
        const double* X2 = W + (P * (c2[2] - K + 2) * WS + P * (c2[1] - J + 2)) * WS + P * (c2[0] - I + 2);
        __syncwarp();
        if (lane == 0) face_moments3<P>(axis, X1, X2, WS, WS * WS, Js);
        __syncwarp();
        for (int side = 1; side <= 2; ++side) {
          const int* cc = side == 1 ? c1 : c2;
          if (cc[0] < I - 1 || cc[0] > I || cc[1] < J - 1 || cc[1] > J || cc[2] < K - 1 || cc[2] > K) continue;
          for (int tt = lane; tt < NB; tt += 32) {
            const int kx = tt % N1, ky = (tt / N1) % N1, kz = tt / (N1 * N1);
            Yb[((P * (cc[2] - K + 1) + kz) * BS + P * (cc[1] - J + 1) + ky) * BS + P * (cc[0] - I + 1) + kx] +=
                face_test3<P>(L, T, axis, side, kx, ky, kz, Js);
          }
        }
        __syncwarp();
      }
}

// interior sets of the 3D cut patches (count / fill)
template <bool WRITE>
__global__ void k_cut_interior3(LevelArgs L, const int* plist, int np, int* count, const int64_t* off, int32_t* node,
                                uint16_t* loc, int32_t* owner) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= np) return;
  const int n = L.n, p = L.p, nv = n + 1;
  const int I = plist[k] % nv, J = (plist[k] / nv) % nv, K = plist[k] / (nv * nv);
  int m = 0;
  const int64_t o = WRITE ? off[k] : 0;
  for (int dc = 0; dc <= 2 * p; ++dc)
    for (int db = 0; db <= 2 * p; ++db)
      for (int da = 0; da <= 2 * p; ++da) {
        const int a = p * (I - 1) + da, b = p * (J - 1) + db, c = p * (K - 1) + dc;
        if (a < 0 || b < 0 || c < 0 || a >= L.nl || b >= L.nl || c >= L.nl) continue;
        const int64_t idx = ((int64_t)c * L.nl + b) * L.ld + a;
        if (!L.mask[idx]) continue;
        const int i0 = (a % p == 0) ? a / p - 1 : a / p, i1 = a / p;
        const int j0 = (b % p == 0) ? b / p - 1 : b / p, j1 = b / p;
        const int k0 = (c % p == 0) ? c / p - 1 : c / p, k1 = c / p;
        bool inside = true;
        for (int kk = k0; kk <= k1; ++kk)
          for (int jj = j0; jj <= j1; ++jj)
            for (int ii = i0; ii <= i1; ++ii)
              if (cell_kind3(L, ii, jj, kk) != OUTSIDE &&
                  !(ii >= I - 1 && ii <= I && jj >= J - 1 && jj <= J && kk >= K - 1 && kk <= K))
                inside = false;
        if (!inside) continue;
        if (WRITE) {
          node[o + m] = (int32_t)idx;
          loc[o + m] = (uint16_t)((dc * (2 * p + 1) + db) * (2 * p + 1) + da);
          owner[o + m] = k;
        }
        ++m;
      }
  if (!WRITE) count[k] = m;
}

__global__ void k_vertex_kind3(LevelArgs L, uint8_t* vk) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int n = L.n, nv = n + 1;
  if (v >= (int64_t)nv * nv * nv) return;
  const int I = v % nv, J = (v / nv) % nv, K = v / ((int64_t)nv * nv);
  int nact = 0, ninside = 0;
  for (int dz = -1; dz <= 0; ++dz)
    for (int dy = -1; dy <= 0; ++dy)
      for (int dx = -1; dx <= 0; ++dx) {
        const int k = cell_kind3(L, I + dx, J + dy, K + dz);
        nact += k != OUTSIDE;
        ninside += k == INSIDE;
      }
  uint8_t r = V_NONE;
  if (nact > 0 && !(L.fitted && (I == 0 || J == 0 || K == 0 || I == n || J == n || K == n))) {
    bool cart = ninside == 8;
    for (int axis = 0; axis < 3 && cart; ++axis)
      for (int side = 0; side < 2 && cart; ++side)
        for (int s1 = -1; s1 <= 0 && cart; ++s1)
          for (int s2 = -1; s2 <= 0 && cart; ++s2) {
            int o[3] = {I, J, K};
            const int t1 = axis == 0 ? 1 : 0, t2 = axis == 2 ? 1 : 2;
            o[axis] += side == 0 ? -2 : 1;
            o[t1] += s1;
            o[t2] += s2;
            if (cell_kind3(L, o[0], o[1], o[2]) == CUT) cart = false;
          }
    r = cart ? V_CART : V_CUT;
  }
  vk[v] = r;
}

__global__ void k_vertex_flags3(int n, const uint8_t* vk, uint8_t kind, int colour, uint8_t* flag) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int nv = n + 1;
  if (v >= (int64_t)nv * nv * nv) return;
  const int I = v % nv, J = (v / nv) % nv, K = v / ((int64_t)nv * nv);
  flag[v] = vk[v] == kind && ((I & 1) + 2 * (J & 1) + 4 * (K & 1)) == colour;
}

// local matrix column of a 3D cut patch (setup)
// (entries [e_lo, e_lo + n_ent) of the patches [j0, ...); column kcol of
// patch j goes to the chunk buffer inv at inv_off[j - j0], m x m row-major)
template <int P>
__global__ void __launch_bounds__(64) k_local_matrix3(LevelArgs L, const int* plist_all, const int64_t* ent_off,
                                                     const uint16_t* ent_loc, const int32_t* ent_patch, int64_t n_ent,
                                                     const int64_t* inv_off, double* inv, int quad, int64_t e_lo,
                                                     int j0) {
  constexpr int BS = 2 * P + 1, WS = 4 * P + 1, N1 = P + 1;
  __shared__ SmTab T;
  __shared__ double sW[2][WS * WS * WS];
  __shared__ double sY[2][BS * BS * BS];
  __shared__ double sJ[2][P * N1 * N1 > N1 * N1 * N1 ? P * N1 * N1 : N1 * N1 * N1];
  load_smtab<P>(T);
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t e = e_lo + blockIdx.x * 2LL + w;
  if (e >= e_lo + n_ent) return;
  const int j = ent_patch[e], nv = L.n + 1;
  const int I = plist_all[j] % nv, J = (plist_all[j] / nv) % nv, K = plist_all[j] / (nv * nv);
  const int64_t e0 = ent_off[j];
  const int m = (int)(ent_off[j + 1] - e0), kcol = (int)(e - e0);
  for (int q = lane; q < WS * WS * WS; q += 32) sW[w][q] = 0.0;
  for (int q = lane; q < BS * BS * BS; q += 32) sY[w][q] = 0.0;
  __syncwarp();
  if (lane == 0) {
    const int loc = ent_loc[e];
    const int la = loc % BS, lb = (loc / BS) % BS, lc = loc / (BS * BS);
    sW[w][((P + lc) * WS + P + lb) * WS + P + la] = 1.0;
  }
  __syncwarp();
  local_block_apply3<P>(L, I, J, K, sW[w], sY[w], T, sJ[w], quad != 0);
  __syncwarp();
  double* A = inv + inv_off[j - j0];
  for (int i = lane; i < m; i += 32) A[(int64_t)i * m + kcol] = sY[w][ent_loc[e0 + i]];
}

// Symmetric local inverses in PACKED mode (large problems, e.g. 3D Q3 at
// 256^3 where the dense inverses would not fit): the lower triangle by rows,
// row i at i (i+1) / 2, m (m+1) / 2 doubles per patch (half the dense
// storage).  Packing of a chunk of full Gauss-Jordan inverses (symmetric up to
// rounding): A(i, q) = F[i m + q], q <= i.
__global__ void k_pack_sym(const int64_t* ent_off, const int64_t* full_off, const double* full,
                           const int64_t* pack_off, double* pack, int np) {
  const int k = blockIdx.x;
  if (k >= np) return;
  const int m = (int)(ent_off[k + 1] - ent_off[k]);
  const double* F = full + full_off[k];
  double* Pk = pack + pack_off[k];
  for (int i = threadIdx.y; i < m; i += blockDim.y)
    for (int q = threadIdx.x; q <= i; q += blockDim.x) Pk[(int64_t)i * (i + 1) / 2 + q] = F[(int64_t)i * m + q];
}

// z_i = sum_q A(i, q) r_q, A packed as above: for each q the lanes i < q read
// A(q, i) = row q (consecutive i: coalesced), the lanes i >= q their own row i
// (sequential per lane, sector reuse in L1)
__device__ __forceinline__ double packed_sym_row(const double* A, const double* r, int m, int i) {
  const int64_t ri = (int64_t)i * (i + 1) / 2;
  double z0 = 0.0, z1 = 0.0;
  int q = 0;
  for (; q + 1 < m; q += 2) {
    const int64_t a0 = i < q ? (int64_t)q * (q + 1) / 2 + i : ri + q;
    const int64_t a1 = i < q + 1 ? (int64_t)(q + 1) * (q + 2) / 2 + i : ri + q + 1;
    z0 = fma(__ldg(A + a0), r[q], z0);
    z1 = fma(__ldg(A + a1), r[q + 1], z1);
  }
  if (q < m) z0 = fma(__ldg(A + (i < q ? (int64_t)q * (q + 1) / 2 + i : ri + q)), r[q], z0);
  return z0 + z1;
}

// z_i = sum_q A[q m + i] r_q, A dense (default): coalesced over i for every q
__device__ __forceinline__ double dense_col_dot(const double* A, const double* r, int m, int i) {
  double z0 = 0.0, z1 = 0.0;
  int q = 0;
  for (; q + 1 < m; q += 2) {
    z0 = fma(__ldg(A + (int64_t)q * m + i), r[q], z0);
    z1 = fma(__ldg(A + (int64_t)(q + 1) * m + i), r[q + 1], z1);
  }
  if (q < m) z0 = fma(__ldg(A + (int64_t)q * m + i), r[q], z0);
  return z0 + z1;
}

// ---- 3D smoother kernels ----------------------------------------------------
// cut patch colour step, phase 1: z_j = A_j^{-1} (b - A x)|_{I_j} (warp per patch)
template <int P>
__global__ void __launch_bounds__(64) k_cut_colour3(LevelArgs L, const int* plist, int np, int pbase,
                                                   const int64_t* ent_off, const uint16_t* ent_loc,
                                                   const int32_t* ent_node, const int64_t* inv_off, const double* inv,
                                                   const double* x, const double* b, double* zbuf, int quad) {
  constexpr int BS = 2 * P + 1, WS = 4 * P + 1, N1 = P + 1, MM = BS * BS * BS;
  __shared__ SmTab T;
  __shared__ double sW[2][WS * WS * WS];
  __shared__ double sY[2][MM];
  __shared__ double sR[2][MM];
  __shared__ double sJ[2][P * N1 * N1 > N1 * N1 * N1 ? P * N1 * N1 : N1 * N1 * N1];
  pdl_trigger();
  load_smtab<P>(T);
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k = blockIdx.x * 2 + w;
  if (k >= np) return;
  const int j = pbase + k, nv = L.n + 1;
  const int I = plist[k] % nv, J = (plist[k] / nv) % nv, K = plist[k] / (nv * nv);
  pdl_wait();
  for (int e = lane; e < WS * WS * WS; e += 32) {
    const int a = P * (I - 2) + e % WS, bb = P * (J - 2) + (e / WS) % WS, c = P * (K - 2) + e / (WS * WS);
    sW[w][e] = (a >= 0 && bb >= 0 && c >= 0 && a < L.nl && bb < L.nl && c < L.nl)
                   ? x[((size_t)c * L.nl + bb) * L.ld + a] : 0.0;
  }
  for (int e = lane; e < MM; e += 32) sY[w][e] = 0.0;
  __syncwarp();
  local_block_apply3<P>(L, I, J, K, sW[w], sY[w], T, sJ[w], quad != 0);
  __syncwarp();
  const int64_t e0 = ent_off[j];
  const int m = (int)(ent_off[j + 1] - e0);
  for (int i = lane; i < m; i += 32) sR[w][i] = b[ent_node[e0 + i]] - sY[w][ent_loc[e0 + i]];
  __syncwarp();
  const double* A = inv + inv_off[j];
  for (int i = lane; i < m; i += 32) zbuf[e0 + i] = L.sym_packed ? packed_sym_row(A, sR[w], m, i) : dense_col_dot(A, sR[w], m, i);
}

// Cartesian colour step in 3D: x_int_new = G [b_int; x_ext] for groups of 8
// patches per warp on the fp64 tensor cores, operands gathered from global
// memory (L1/L2) and the map G (27 x 152 for Q2) streamed from L1.
template <int P>
struct CartMMA3 {
  static constexpr int NE = 2 * P + 1, NI = 2 * P - 1, NINT = NI * NI * NI, NEXT = NE * NE * NE, K = NINT + NEXT;
  static constexpr int KS = (K + 3) / 4, COLS = 4 * KS, MF = NINT / 8, RR = NINT - 8 * MF, ROWS = 8 * ((NINT + 7) / 8);
  // Q3 (G = 128 x 468 doubles, 468 KB): G is staged through shared memory in
  // chunks of KC k-steps shared by the CTA's NW warps (one L2 read of G per
  // CTA instead of per warp); Q1 / Q2 read G (<= 38 KB) through L1
  static constexpr bool STAGE = P >= 3;
  static constexpr int NW = STAGE ? 8 : 4, KC = 8, GS = 4 * KC + 4;   // GS: padded row stride (2 wavefronts)
};

template <int P>
__global__ void __launch_bounds__(32 * CartMMA3<P>::NW) k_cart_colour3(LevelArgs L, const int* plist, int np,
                                                                      const double* G, double* x, const double* b) {
  using C = CartMMA3<P>;
  constexpr int NE = C::NE, NI = C::NI, NINT = C::NINT, K = C::K, KS = C::KS, MF = C::MF, RR = C::RR, NW = C::NW;
  __shared__ int koff[C::COLS];
  __shared__ int roff[NINT];
  __shared__ double gs[C::STAGE ? C::ROWS * C::GS : 1];
  const int tid = threadIdx.x, lane = tid & 31, nl = L.nl, ld = L.ld;
  pdl_trigger();
  for (int k = tid; k < C::COLS; k += blockDim.x) {
    int v = -1;
    if (k < NINT) {
      const int ia = k % NI, ib = (k / NI) % NI, ic = k / (NI * NI);
      v = (1 << 30) + ((ic + 1) * nl + ib + 1) * ld + ia + 1;
    } else if (k < K) {
      const int e = k - NINT, aa = e % NE, bb = (e / NE) % NE, cc = e / (NE * NE);
      v = (cc * nl + bb) * ld + aa;
    }
    koff[k] = v;
  }
  for (int r = tid; r < NINT; r += blockDim.x) {
    const int ia = r % NI, ib = (r / NI) % NI, ic = r / (NI * NI);
    roff[r] = ((ic + 1) * nl + ib + 1) * ld + ia + 1;
  }
  __syncthreads();
  const int g = blockIdx.x * NW + (tid >> 5);
  if (!C::STAGE && 8 * g >= np) return;   // (staged: every warp takes part in the chunk loads)
  const int pq = 8 * g + (lane >> 2), nv = L.n + 1;
  const double hinv = 1.0 / L.h;   // G holds the h = 1 map; A scales with h in 3D
  int64_t base = -1;
  if (pq < np) {
    const int v = plist[pq];
    const int I = v % nv, J = (v / nv) % nv, Kv = v / (nv * nv);
    base = ((int64_t)(P * (Kv - 1)) * nl + P * (J - 1)) * ld + P * (I - 1);
  }
  pdl_wait();
  double acc[MF > 0 ? MF : 1][2];
  double rs[RR > 0 ? RR : 1];
#pragma unroll
  for (int mt = 0; mt < MF; ++mt) acc[mt][0] = acc[mt][1] = 0.0;
#pragma unroll
  for (int rr = 0; rr < RR; ++rr) rs[rr] = 0.0;
  if constexpr (C::STAGE) {
    for (int ks0 = 0; ks0 < KS; ks0 += C::KC) {
      const int nk = KS - ks0 < C::KC ? KS - ks0 : C::KC;
      __syncthreads();
      for (int e = tid; e < C::ROWS * 4 * nk; e += blockDim.x) {
        const int r = e / (4 * nk), c = e - r * 4 * nk;
        gs[r * C::GS + c] = __ldg(G + r * C::COLS + 4 * ks0 + c);
      }
      __syncthreads();
      for (int kk = 0; kk < nk; ++kk) {
        const int ks = ks0 + kk;
        const int ko = koff[4 * ks + (lane & 3)];
        double v = 0.0;
        if (base >= 0 && ko >= 0) v = ko >= (1 << 30) ? b[base + ko - (1 << 30)] * hinv : x[base + ko];
#pragma unroll
        for (int mt = 0; mt < MF; ++mt)
          dmma(gs[(8 * mt + (lane >> 2)) * C::GS + 4 * kk + (lane & 3)], v, acc[mt][0], acc[mt][1]);
#pragma unroll
        for (int rr = 0; rr < RR; ++rr) rs[rr] = fma(gs[(8 * MF + rr) * C::GS + 4 * kk + (lane & 3)], v, rs[rr]);
      }
    }
    if (8 * g >= np) return;
  } else {
    for (int ks = 0; ks < KS; ++ks) {
      const int ko = koff[4 * ks + (lane & 3)];
      double v = 0.0;
      if (base >= 0 && ko >= 0) v = ko >= (1 << 30) ? b[base + ko - (1 << 30)] * hinv : x[base + ko];
#pragma unroll
      for (int mt = 0; mt < MF; ++mt)
        dmma(__ldg(G + (8 * mt + (lane >> 2)) * C::COLS + 4 * ks + (lane & 3)), v, acc[mt][0], acc[mt][1]);
#pragma unroll
      for (int rr = 0; rr < RR; ++rr) rs[rr] = fma(__ldg(G + (8 * MF + rr) * C::COLS + 4 * ks + (lane & 3)), v, rs[rr]);
    }
  }
  // all reads of this warp's patches are done before any write (each patch's
  // reads are its own block; same-colour blocks do not contain other interiors)
#pragma unroll
  for (int rr = 0; rr < RR; ++rr) {
    rs[rr] += __shfl_xor_sync(0xffffffffu, rs[rr], 1);
    rs[rr] += __shfl_xor_sync(0xffffffffu, rs[rr], 2);
    if ((lane & 3) == 0 && base >= 0) x[base + roff[8 * MF + rr]] = rs[rr];
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int64_t bo = __shfl_sync(0xffffffffu, base, 4 * (2 * (lane & 3) + i));
#pragma unroll
    for (int mt = 0; mt < MF; ++mt)
      if (bo >= 0) x[bo + roff[8 * mt + (lane >> 2)]] = acc[mt][i];
  }
}

// ---- operator: band (cut cells + ghost faces) and node gather ---------------
// R: cut cells [cut_lo, cut_lo + cut_n) and ghost faces of the three axes
// [g_lo[a], g_lo[a] + g_n[a]) (a rank's planes under the slab partition)
struct BandRange3 {
  int cut_lo, cut_n, g_lo[3], g_n[3];
};

template <int P>
__global__ void __launch_bounds__(128) k_band3(LevelArgs L, const double* x, BandRange3 R) {
  constexpr int N1 = P + 1, NB = N1 * N1 * N1;
  __shared__ double sX[4][NB];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw0 = blockIdx.x * 4 + w;
  const int n = L.n, nl = L.nl, ld = L.ld;
  if (gw0 < R.cut_n) {
    const int gw = R.cut_lo + gw0;
    const int64_t c = L.cut_list[gw];
    const int i = c % n, j = (c / n) % n, k = c / ((int64_t)n * n);
    for (int t = lane; t < NB; t += 32)
      sX[w][t] = x[((size_t)(k * P + t / (N1 * N1)) * nl + j * P + (t / N1) % N1) * ld + i * P + t % N1];
    __syncwarp();
    for (int t = lane; t < NB; t += 32) {
      const double* Er = L.ecut + ((size_t)gw * NB + t) * NB;
      double s = 0.0;
      for (int l = 0; l < NB; ++l) s = fma(Er[l], sX[w][l], s);
      L.ycut[(size_t)gw * NB + t] = s;
    }
    return;
  }
  int kk = (gw0 - R.cut_n) * 32 + lane, g = -1;
  for (int a = 0; a < 3 && g < 0; ++a) {
    if (kk < R.g_n[a]) g = R.g_lo[a] + kk;
    else kk -= R.g_n[a];
  }
  if (g < 0) return;
  const int64_t n3 = (int64_t)n * n * n, f = L.ghost_list[g];
  const int axis = (int)(f / n3);
  const int64_t c = f - axis * n3;
  const int i = c % n, j = (c / n) % n, k = c / ((int64_t)n * n);
  const double* X1 = x + ((size_t)(k * P) * nl + j * P) * ld + i * P;
  const size_t step = axis == 0 ? P : (axis == 1 ? (size_t)P * ld : (size_t)P * nl * ld);
  face_moments3<P>(axis, X1, X1 + step, ld, nl * ld, L.jm + (size_t)g * P * N1 * N1);
}

template <int P>
__global__ void __launch_bounds__(256) k_node_apply3(LevelArgs L, const double* x, const double* b, double* y,
                                                     int64_t o0, int64_t o1) {
  constexpr int N1 = P + 1, NB = N1 * N1 * N1;
  __shared__ SmTab T;
  load_smtab<P>(T);
  __syncthreads();
  const int64_t o = o0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int nl = L.nl, ld = L.ld, n = L.n;
  if (o >= o1) return;
  if (!L.mask[o]) {
    y[o] = 0.0;
    return;
  }
  const int a = o % ld, bb = (o / ld) % nl, cc = o / ((int64_t)ld * nl);
  const int i0 = max((a % P == 0) ? a / P - 1 : a / P, 0), i1 = min(a / P, n - 1);
  const int j0 = max((bb % P == 0) ? bb / P - 1 : bb / P, 0), j1 = min(bb / P, n - 1);
  const int k0 = max((cc % P == 0) ? cc / P - 1 : cc / P, 0), k1 = min(cc / P, n - 1);
  const int64_t n3 = (int64_t)n * n;
  double acc = 0.0;
  for (int k = k0; k <= k1; ++k)
    for (int j = j0; j <= j1; ++j)
      for (int i = i0; i <= i1; ++i) {
        const int64_t cell = (k * n3) + (int64_t)j * n + i;
        const int kind = L.ctype[cell];
        if (kind == OUTSIDE) continue;
        const int kx = a - i * P, ky = bb - j * P, kz = cc - k * P;
        if (kind == INSIDE)
          acc += inside_row3<P>(T, x + ((size_t)(k * P) * nl + j * P) * ld + i * P, ld, nl * ld, kx, ky, kz, L.h);
        else
          acc += L.ycut[(size_t)L.cut_id[cell] * NB + (kz * N1 + ky) * N1 + kx];
        const int* maps[3] = {L.gx_id, L.gy_id, L.gz_id};
        const int64_t prev[3] = {1, n, n3};
        const int pos[3] = {i, j, k};
        for (int axis = 0; axis < 3; ++axis) {
          int g;
          if (pos[axis] >= 1 && (g = maps[axis][cell - prev[axis]]) >= 0)
            acc += face_test3<P>(L, T, axis, 2, kx, ky, kz, L.jm + (size_t)g * P * N1 * N1);
          if ((g = maps[axis][cell]) >= 0) acc += face_test3<P>(L, T, axis, 1, kx, ky, kz, L.jm + (size_t)g * P * N1 * N1);
        }
      }
  y[o] = b ? b[o] - acc : acc;
}

// ---- transfer in 3D ---------------------------------------------------------
template <int P>
__global__ void k_prolongate_add3(LevelArgs Lf, LevelArgs Lc, const double* xc, double* xf, int64_t o0, int64_t o1) {
  __shared__ double pw[2 * P + 1][P + 1];
  if (threadIdx.x < (2 * P + 1) * (P + 1)) pw[threadIdx.x / (P + 1)][threadIdx.x % (P + 1)] = g_tab[P].pw[threadIdx.x / (P + 1)][threadIdx.x % (P + 1)];
  __syncthreads();
  const int64_t o = o0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int nl = Lf.nl, ld = Lf.ld;
  if (o >= o1) return;
  if (!Lf.mask[o]) return;
  const int a = o % ld, bb = (o / ld) % nl, cc = o / ((int64_t)ld * nl);
  const int Ia = min(min(a / P, Lf.n - 1) / 2, Lc.n - 1), Ib = min(min(bb / P, Lf.n - 1) / 2, Lc.n - 1),
            Ic = min(min(cc / P, Lf.n - 1) / 2, Lc.n - 1);
  const int da = a - 2 * P * Ia, db = bb - 2 * P * Ib, dc = cc - 2 * P * Ic;
  double s = 0.0;
  for (int nz = 0; nz <= P; ++nz) {
    const double wz = pw[dc][nz];
    if (wz == 0.0) continue;
    for (int ny = 0; ny <= P; ++ny) {
      const double wyz = wz * pw[db][ny];
      if (wyz == 0.0) continue;
      for (int nx = 0; nx <= P; ++nx)
        s = fma(wyz * pw[da][nx], xc[((size_t)(Ic * P + nz) * Lc.nl + Ib * P + ny) * Lc.ld + Ia * P + nx], s);
    }
  }
  xf[o] += s;
}

template <int P>
__global__ void k_restrict3(LevelArgs Lf, LevelArgs Lc, const double* rf, double* bc, int64_t o0, int64_t o1) {
  __shared__ double tw[P][4 * P + 1];
  if (threadIdx.x < P * (4 * P + 1)) tw[threadIdx.x / (4 * P + 1)][threadIdx.x % (4 * P + 1)] = g_tab[P].tw[threadIdx.x / (4 * P + 1)][threadIdx.x % (4 * P + 1)];
  __syncthreads();
  const int64_t o = o0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int nl = Lc.nl, ld = Lc.ld;
  if (o >= o1) return;
  const int A = o % ld, B = (o / ld) % nl, Cc = o / ((int64_t)ld * nl);
  if (A >= nl || !Lc.mask[o]) {
    bc[o] = 0.0;
    return;
  }
  const int mA = A % P, mB = B % P, mC = Cc % P;
  const int dal = mA == 0 ? -2 * P : 0, dbl = mB == 0 ? -2 * P : 0, dcl = mC == 0 ? -2 * P : 0;
  double s = 0.0;
  for (int dc = dcl; dc <= 2 * P; ++dc) {
    const int fc = 2 * P * (Cc / P) + dc;
    if (fc < 0 || fc >= Lf.nl) continue;
    const double wc = tw[mC][dc + 2 * P];
    if (wc == 0.0) continue;
    for (int db = dbl; db <= 2 * P; ++db) {
      const int fb = 2 * P * (B / P) + db;
      if (fb < 0 || fb >= Lf.nl) continue;
      const double wbc = wc * tw[mB][db + 2 * P];
      if (wbc == 0.0) continue;
      double t = 0.0;
      for (int da = dal; da <= 2 * P; ++da) {
        const int fa = 2 * P * (A / P) + da;
        if (fa < 0 || fa >= Lf.nl) continue;
        t = fma(tw[mA][da + 2 * P], rf[((size_t)fc * Lf.nl + fb) * Lf.ld + fa], t);
      }
      s = fma(wbc, t, s);
    }
  }
  bc[o] = s;
}

}  // namespace cf

namespace cf {

// ---- 3D cut patches, v2: descriptor + lane-parallel faces and cells --------
struct __align__(16) CutDesc3 {
  int I, J, K, e0;
  unsigned long long kinds[2];   // 2 bits per cell of the 4x4x4 window, index (wz*4 + wy)*4 + wx
  int cid[8];                    // cut ids of the patch cells q = dx + 2 dy + 4 dz (-1 if not cut)
  long long inv_off;
  unsigned long long mask[6];    // interior set over the (2p+1)^3 block (p <= 3: <= 343 bits)
};
static_assert(sizeof(CutDesc3) == 128, "CutDesc3 is two 64-byte lines");

// interior-set bit mask of a 3D cut patch: count, membership, rank (index of
// the interior DoF in A_j's order = number of set bits below it); words beyond
// (2p+1)^3 bits are zero
template <int P>
__device__ __forceinline__ int mask_count3(const CutDesc3& d) {
  constexpr int NW = ((2 * P + 1) * (2 * P + 1) * (2 * P + 1) + 63) / 64;
  int s = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) s += __popcll(d.mask[w]);
  return s;
}
__device__ __forceinline__ bool mask_bit3(const CutDesc3& d, int loc) { return (d.mask[loc >> 6] >> (loc & 63)) & 1ull; }
template <int P>
__device__ __forceinline__ int mask_rank3(const CutDesc3& d, int loc) {
  constexpr int NW = ((2 * P + 1) * (2 * P + 1) * (2 * P + 1) + 63) / 64;
  const int w = loc >> 6;
  int s = __popcll(d.mask[w] & ((1ull << (loc & 63)) - 1ull));
#pragma unroll
  for (int q = 0; q < NW; ++q)
    if (q < w) s += __popcll(d.mask[q]);
  return s;
}

__device__ __forceinline__ int dkind3(const CutDesc3& d, int wx, int wy, int wz) {
  const int idx = (wz * 4 + wy) * 4 + wx;
  return (int)((d.kinds[idx >> 5] >> (2 * (idx & 31))) & 3ull);
}

template <int P>
__global__ void k_cut_desc3(LevelArgs L, const int* plist, int np, const int64_t* ent_off, const uint16_t* ent_loc,
                            const int64_t* inv_off, CutDesc3* desc) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= np) return;
  const int nv = L.n + 1;
  CutDesc3 d;
  d.I = plist[k] % nv;
  d.J = (plist[k] / nv) % nv;
  d.K = plist[k] / (nv * nv);
  d.kinds[0] = d.kinds[1] = 0ull;
  for (int wz = 0; wz < 4; ++wz)
    for (int wy = 0; wy < 4; ++wy)
      for (int wx = 0; wx < 4; ++wx) {
        const int idx = (wz * 4 + wy) * 4 + wx;
        d.kinds[idx >> 5] |= (unsigned long long)cell_kind3(L, d.I - 2 + wx, d.J - 2 + wy, d.K - 2 + wz) << (2 * (idx & 31));
      }
  for (int q = 0; q < 8; ++q) {
    const int ci = d.I - 1 + (q & 1), cj = d.J - 1 + ((q >> 1) & 1), ck = d.K - 1 + (q >> 2);
    d.cid[q] = cell_kind3(L, ci, cj, ck) == CUT ? L.cut_id[((size_t)ck * L.n + cj) * L.n + ci] : -1;
  }
  d.e0 = (int)ent_off[k];
  d.inv_off = inv_off[k];
  for (int w = 0; w < 6; ++w) d.mask[w] = 0ull;
  for (int64_t e = ent_off[k]; e < ent_off[k + 1]; ++e) d.mask[ent_loc[e] >> 6] |= 1ull << (ent_loc[e] & 63);
  desc[k] = d;
}

template <int P>
struct Cut3Smem {
  static constexpr int N1 = P + 1, NB = N1 * N1 * N1, BS = 2 * P + 1, WS = 4 * P + 1, MM = BS * BS * BS;
  static constexpr int NJ = 36 * P * N1 * N1;
  static constexpr int per_warp = WS * WS * WS + 2 * NJ + 8 * NB + 2 * MM;
};

// one CTA of NT threads per patch: z = A_j^{-1} (b - A x)|_{I_j} -> zbuf[d.e0 + i]
template <int P, int NT>
__device__ void cut_patch_z3d(const LevelArgs& L, const CutDesc3& d, const double* inv, const double* x,
                              const double* b, double* zbuf, const SmTab& T, double* Wp) {
  using S = Cut3Smem<P>;
  constexpr int N1 = S::N1, NB = S::NB, BS = S::BS, WS = S::WS, MM = S::MM, NJ = S::NJ, FJ = P * N1 * N1;
  const int lane = threadIdx.x;   // thread index within the patch group of NT threads
  double* Jt = Wp + WS * WS * WS;
  double* Jm = Jt + NJ;
  double* Yc = Jm + NJ;        // [8][NB] per-cell outputs
  double* Rr = Yc + 8 * NB;    // [MM]
  const int m = mask_count3<P>(d);
  pdl_wait();
  for (int e = lane; e < WS * WS * WS; e += NT) {
    const int a = P * (d.I - 2) + e % WS, bb = P * (d.J - 2) + (e / WS) % WS, c = P * (d.K - 2) + e / (WS * WS);
    if (a >= 0 && bb >= 0 && c >= 0 && a < L.nl && bb < L.nl && c < L.nl)
      cp_async8(Wp + e, x + ((size_t)c * L.nl + bb) * L.ld + a);
    else Wp[e] = 0.0;
  }
  cp_async_wait_all();
  __syncthreads();
  // ghost faces: jumps (face f = (axis*3 + s)*4 + t), then (M⊗M) moments
  for (int job = lane; job < NJ; job += NT) {
    const int f = job / FJ, rem = job - f * FJ;
    const int k = rem / (N1 * N1) + 1, l1 = (rem / N1) % N1, l2 = rem % N1;
    const int axis = f / 12, s = (f / 4) % 3, t = f % 4;
    // window cell of side 1 (w1x, w1y, w1z) and the strides of the normal / tangential axes
    const int ta = 1 + (t & 1), tb = 1 + (t >> 1);
    const int w1x = axis == 0 ? s : ta, w1y = axis == 1 ? s : (axis == 0 ? ta : tb), w1z = axis == 2 ? s : tb;
    const int w2x = w1x + (axis == 0), w2y = w1y + (axis == 1), w2z = w1z + (axis == 2);
    const int sn = axis == 0 ? 1 : (axis == 1 ? WS : WS * WS);
    const int s1 = axis == 0 ? WS : 1, s2 = axis == 2 ? WS : WS * WS;
    const int k1 = dkind3(d, w1x, w1y, w1z), k2 = dkind3(d, w2x, w2y, w2z);
    double sacc = 0.0;
    if (k1 != OUTSIDE && k2 != OUTSIDE && (k1 == CUT || k2 == CUT)) {
      const double* X1 = Wp + (P * w1z * WS + P * w1y) * WS + P * w1x + l1 * s1 + l2 * s2;
      const double* X2 = X1 + P * sn;
#pragma unroll
      for (int nn = 0; nn < N1; ++nn) sacc = fma(T.d1[k][nn], X1[nn * sn], fma(-T.d0[k][nn], X2[nn * sn], sacc));
    }
    Jt[job] = sacc;
  }
  __syncthreads();
  for (int job = lane; job < NJ; job += NT) {
    const int base = job - job % (N1 * N1), q1 = (job / N1) % N1, q2 = job % N1;
    double sacc = 0.0;
#pragma unroll
    for (int l1 = 0; l1 < N1; ++l1)
#pragma unroll
      for (int l2 = 0; l2 < N1; ++l2) sacc = fma(T.M[q1][l1] * T.M[q2][l2], Jt[base + l1 * N1 + l2], sacc);
    Jm[job] = sacc;
  }
  __syncthreads();
  // per (cell, local row): cell term + the ghost faces of that cell
  for (int job = lane; job < 8 * NB; job += NT) {
    const int q = job / NB, t = job % NB;
    const int dx = q & 1, dy = (q >> 1) & 1, dz = q >> 2;
    const int kind = dkind3(d, dx + 1, dy + 1, dz + 1);
    double y = 0.0;
    if (kind != OUTSIDE) {
      const int kx = t % N1, ky = (t / N1) % N1, kz = t / (N1 * N1);
      const double* X = Wp + (P * (dz + 1) * WS + P * (dy + 1)) * WS + P * (dx + 1);
      if (kind == INSIDE) {
        y = inside_row3<P>(T, X, WS, WS * WS, kx, ky, kz, L.h);
      } else {
        const double* Er = L.ecut + ((size_t)d.cid[q] * NB + t) * NB;
#pragma unroll
        for (int l = 0; l < NB; ++l) y = fma(__ldg(Er + l), X[((l / (N1 * N1)) * WS + (l / N1) % N1) * WS + l % N1], y);
      }
#pragma unroll
      for (int axis = 0; axis < 3; ++axis) {
        const int ka = axis == 0 ? kx : (axis == 1 ? ky : kz);
        const int kt1 = axis == 0 ? ky : kx, kt2 = axis == 2 ? ky : kz;
        const int da = axis == 0 ? dx : (axis == 1 ? dy : dz);
        const int tt = axis == 0 ? dy + 2 * dz : (axis == 1 ? dx + 2 * dz : dx + 2 * dy);
        const int flo = (axis * 3 + da) * 4 + tt, fhi = flo + 4;
#pragma unroll
        for (int k = 1; k <= P; ++k) {
          const int o = (k - 1) * N1 * N1 + kt1 * N1 + kt2;
          y = fma(-L.gs[k] * T.d0[k][ka], Jm[flo * FJ + o], y);
          y = fma(L.gs[k] * T.d1[k][ka], Jm[fhi * FJ + o], y);
        }
      }
    }
    Yc[job] = y;
  }
  __syncthreads();
  // gather the interior rows (fixed cell order), residual
  for (int loc = lane; loc < MM; loc += NT) {
    if (!mask_bit3(d, loc)) continue;
    const int i = mask_rank3<P>(d, loc);
    const int ra = loc % BS, rb = (loc / BS) % BS, rc = loc / (BS * BS);
    double y = 0.0;
    for (int q = 0; q < 8; ++q) {
      const int dx = q & 1, dy = (q >> 1) & 1, dz = q >> 2;
      const int kx = ra - P * dx, ky = rb - P * dy, kz = rc - P * dz;
      if (kx < 0 || kx > P || ky < 0 || ky > P || kz < 0 || kz > P) continue;
      y += Yc[q * NB + (kz * N1 + ky) * N1 + kx];
    }
    const double bv = b[((size_t)(P * (d.K - 1) + rc) * L.nl + P * (d.J - 1) + rb) * L.ld + P * (d.I - 1) + ra];
    Rr[i] = bv - y;
  }
  __syncthreads();
  const double* A = inv + d.inv_off;
  for (int i = lane; i < m; i += NT) zbuf[d.e0 + i] = L.sym_packed ? packed_sym_row(A, Rr, m, i) : dense_col_dot(A, Rr, m, i);
}

template <int P>
__global__ void __launch_bounds__(128) k_cut_colour3v2(LevelArgs L, const CutDesc3* desc, int np, const double* inv,
                                                       const double* x, const double* b, double* zbuf) {
  __shared__ SmTab T;
  extern __shared__ double dsm[];
  pdl_trigger();
  load_smtab<P>(T);
  __syncthreads();
  const int k = blockIdx.x;
  if (k >= np) return;
  const CutDesc3 d = desc[k];
  cut_patch_z3d<P, 128>(L, d, inv, x, b, zbuf, T, dsm);
}

// v3: one thread per (ghost face, derivative order) computes the face jumps in
// registers and their (M x M) moments (no jump array in shared memory), a
// 36-bit ghost-face mask lets the cell rows skip non-ghost faces, and the
// cut-cell rows read column t of the symmetric element matrix (a warp's loads
// of one cell are coalesced).  TMA = true: the (4p+1)^3 window arrives as one
// 3D TMA box with rows padded to RS = 4p+2 doubles (16-byte box rows; the
// hardware zero-fills coordinates outside the lattice).
template <int P, bool TMA>
struct Cut3SmemV3 {
  static constexpr int N1 = P + 1, NB = N1 * N1 * N1, BS = 2 * P + 1, WS = 4 * P + 1, MM = BS * BS * BS;
  static constexpr int RS = TMA ? ((WS + 1) & ~1) : WS, PS = RS * WS;   // row / plane stride of the window
  static constexpr int FJ = P * N1 * N1;
  static constexpr int doubles = WS * PS + 36 * FJ + 8 * NB + MM + 1;
  static constexpr size_t bytes = 128 + doubles * sizeof(double);
};

template <int P, int NT, bool TMA>
__global__ void __launch_bounds__(NT) k_cut_colour3v3(const __grid_constant__ CUtensorMap tmx, LevelArgs L,
                                                      const CutDesc3* desc, int np, const double* inv,
                                                      const double* x, const double* b, double* zbuf) {
  using S = Cut3SmemV3<P, TMA>;
  constexpr int N1 = S::N1, NB = S::NB, BS = S::BS, WS = S::WS, MM = S::MM, FJ = S::FJ, RS = S::RS, PS = S::PS;
  __shared__ SmTab T;
  __shared__ CutDesc3 d;
  __shared__ unsigned long long gmask;
  extern __shared__ __align__(128) unsigned char smraw3[];
  uint64_t* bar = (uint64_t*)smraw3;
  double* Wp = (double*)(smraw3 + 128);
  double* Jm = Wp + WS * PS;        // [36 faces][P][N1][N1]
  double* Yc = Jm + 36 * FJ;        // [8][NB]
  double* Rr = Yc + 8 * NB;         // [MM]
  const int lane = threadIdx.x;
  pdl_trigger();
  if ((int)blockIdx.x >= np) return;
  load_smtab<P>(T);
  if (lane == 0) {
    d = desc[blockIdx.x];
    gmask = 0ull;
    if (TMA) mbar_init(bar, 1);
  }
  __syncthreads();
  const int m = mask_count3<P>(d);
  // setup-time data (element matrices of the cut cells, local inverse): start
  // streaming it into L2 now, overlapping the previous kernel's tail (PDL)
  if (lane < 8) {
    if (d.cid[lane] >= 0) prefetch_l2(L.ecut + (size_t)d.cid[lane] * NB * NB, NB * NB * sizeof(double));
  } else if (lane == 8) {
    prefetch_l2(inv + d.inv_off, (size_t)(L.sym_packed ? m * (m + 1) / 2 : m * m) * sizeof(double));
  }
  pdl_wait();
  if (TMA) {
    if (lane == 0) {
      mbar_expect_tx(bar, (unsigned)(RS * WS * WS * sizeof(double)));
      tma_load_3d(Wp, &tmx, P * (d.I - 2), P * (d.J - 2), P * (d.K - 2), bar);
    }
  } else {
    for (int e = lane; e < WS * WS * WS; e += NT) {
      const int a = P * (d.I - 2) + e % WS, bb = P * (d.J - 2) + (e / WS) % WS, c = P * (d.K - 2) + e / (WS * WS);
      const int o = (e / (WS * WS)) * PS + ((e / WS) % WS) * RS + e % WS;
      if (a >= 0 && bb >= 0 && c >= 0 && a < L.nl && bb < L.nl && c < L.nl)
        cp_async8(Wp + o, x + ((size_t)c * L.nl + bb) * L.ld + a);
      else Wp[o] = 0.0;
    }
    cp_async_wait_all();
  }
  // residual rhs of the interior rows (independent of the window)
  for (int loc = lane; loc < MM; loc += NT) {
    if (!mask_bit3(d, loc)) continue;
    const int i = mask_rank3<P>(d, loc);
    const int ra = loc % BS, rb = (loc / BS) % BS, rc = loc / (BS * BS);
    Rr[i] = b[((size_t)(P * (d.K - 1) + rc) * L.nl + P * (d.J - 1) + rb) * L.ld + P * (d.I - 1) + ra];
  }
  if (TMA) mbar_wait(bar, 0);
  __syncthreads();
  // phase A: ghost-face moments (jobs < 36 P) and the cell parts of the
  // per-(cell, row) outputs (the element-matrix loads overlap the face math)
  for (int job = lane; job < 36 * P + 8 * NB; job += NT) {
    if (job >= 36 * P) {
      const int jr = job - 36 * P;
      const int q = jr / NB, t = jr - q * NB;
      const int dx = q & 1, dy = (q >> 1) & 1, dz = q >> 2;
      const int kind = dkind3(d, dx + 1, dy + 1, dz + 1);
      double y = 0.0;
      if (kind != OUTSIDE) {
        const int kx = t % N1, ky = (t / N1) % N1, kz = t / (N1 * N1);
        const double* X = Wp + P * (dz + 1) * PS + P * (dy + 1) * RS + P * (dx + 1);
        if (kind == INSIDE) {
          y = inside_row3<P>(T, X, RS, PS, kx, ky, kz, L.h);
        } else {
          const double* Ec = L.ecut + (size_t)d.cid[q] * NB * NB + t;   // column t = row t (symmetric)
#pragma unroll
          for (int l = 0; l < NB; ++l) y = fma(__ldg(Ec + l * NB), X[(l / (N1 * N1)) * PS + ((l / N1) % N1) * RS + l % N1], y);
        }
      }
      Yc[jr] = y;
      continue;
    }
    const int f = job / P, k = job - f * P + 1;
    const int axis = f / 12, s = (f / 4) % 3, t = f % 4;
    const int ta = 1 + (t & 1), tb = 1 + (t >> 1);
    const int w1x = axis == 0 ? s : ta, w1y = axis == 1 ? s : (axis == 0 ? ta : tb), w1z = axis == 2 ? s : tb;
    const int w2x = w1x + (axis == 0), w2y = w1y + (axis == 1), w2z = w1z + (axis == 2);
    const int k1 = dkind3(d, w1x, w1y, w1z), k2 = dkind3(d, w2x, w2y, w2z);
    if (!(k1 != OUTSIDE && k2 != OUTSIDE && (k1 == CUT || k2 == CUT))) continue;
    if (k == 1) atomicOr(&gmask, 1ull << f);
    double* out = Jm + f * FJ + (k - 1) * N1 * N1;
    const int sn = axis == 0 ? 1 : (axis == 1 ? RS : PS);
    const int s1 = axis == 0 ? RS : 1, s2 = axis == 2 ? RS : PS;
    const double* X1 = Wp + P * w1z * PS + P * w1y * RS + P * w1x;
    const double* X2 = X1 + P * sn;
    double H[N1][N1];   // H[l1][q2] = sum_l2 M[q2][l2] J[l1][l2]
#pragma unroll
    for (int l1 = 0; l1 < N1; ++l1) {
      double J[N1];
#pragma unroll
      for (int l2 = 0; l2 < N1; ++l2) {
        double a = 0.0;
        const int o = l1 * s1 + l2 * s2;
#pragma unroll
        for (int nn = 0; nn < N1; ++nn) a = fma(T.d1[k][nn], X1[o + nn * sn], fma(-T.d0[k][nn], X2[o + nn * sn], a));
        J[l2] = a;
      }
#pragma unroll
      for (int q2 = 0; q2 < N1; ++q2) {
        double a = 0.0;
#pragma unroll
        for (int l2 = 0; l2 < N1; ++l2) a = fma(T.M[q2][l2], J[l2], a);
        H[l1][q2] = a;
      }
    }
#pragma unroll
    for (int q1 = 0; q1 < N1; ++q1)
#pragma unroll
      for (int q2 = 0; q2 < N1; ++q2) {
        double a = 0.0;
#pragma unroll
        for (int l1 = 0; l1 < N1; ++l1) a = fma(T.M[q1][l1], H[l1][q2], a);
        out[q1 * N1 + q2] = a;
      }
  }
  __syncthreads();
  // phase B: interior rows gather the cell parts of their cells plus those
  // cells' ghost-face terms; residual = b - A x on the interior
  const unsigned long long gm = gmask;
  for (int loc = lane; loc < MM; loc += NT) {
    if (!mask_bit3(d, loc)) continue;
    const int i = mask_rank3<P>(d, loc);
    const int ra = loc % BS, rb = (loc / BS) % BS, rc = loc / (BS * BS);
    double y = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int dx = q & 1, dy = (q >> 1) & 1, dz = q >> 2;
      const int kx = ra - P * dx, ky = rb - P * dy, kz = rc - P * dz;
      if (kx < 0 || kx > P || ky < 0 || ky > P || kz < 0 || kz > P) continue;
      double yq = Yc[q * NB + (kz * N1 + ky) * N1 + kx];
#pragma unroll
      for (int axis = 0; axis < 3; ++axis) {
        const int ka = axis == 0 ? kx : (axis == 1 ? ky : kz);
        const int kt1 = axis == 0 ? ky : kx, kt2 = axis == 2 ? ky : kz;
        const int da = axis == 0 ? dx : (axis == 1 ? dy : dz);
        const int tt = axis == 0 ? dy + 2 * dz : (axis == 1 ? dx + 2 * dz : dx + 2 * dy);
        const int flo = (axis * 3 + da) * 4 + tt, fhi = flo + 4;
        if ((gm >> flo) & 1ull) {
#pragma unroll
          for (int k = 1; k <= P; ++k)
            yq = fma(-L.gs[k] * T.d0[k][ka], Jm[flo * FJ + (k - 1) * N1 * N1 + kt1 * N1 + kt2], yq);
        }
        if ((gm >> fhi) & 1ull) {
#pragma unroll
          for (int k = 1; k <= P; ++k)
            yq = fma(L.gs[k] * T.d1[k][ka], Jm[fhi * FJ + (k - 1) * N1 * N1 + kt1 * N1 + kt2], yq);
        }
      }
      y += yq;
    }
    Rr[i] -= y;
  }
  __syncthreads();
  const double* A = inv + d.inv_off;
  for (int i = lane; i < m; i += NT) zbuf[d.e0 + i] = L.sym_packed ? packed_sym_row(A, Rr, m, i) : dense_col_dot(A, Rr, m, i);
}

}  // namespace cf
