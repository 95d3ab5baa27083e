// setup.cuh — device kernels that build the level geometry and the patch
// data (P l.65-69 mesh + classification, l.97-101 ghost faces, l.190 cut
// quadrature, l.141-156 + l.179 patches and colouring, l.193 cut-patch local
// matrices).  Setup-time only; the hot path is in kernels.cuh.
#pragma once
#include "internal.cuh"

namespace cf {

// cell bounds x0 + i*h, x0 + (i+1)*h with round-to-nearest product then sum
// (reading R2: both sides evaluate the same fp64 expressions, no FMA)
__device__ __forceinline__ void cell_bounds(const LevelArgs& L, int i, int j, double& xl, double& xh, double& yl,
                                            double& yh) {
  xl = __dadd_rn(L.x0, __dmul_rn((double)i, L.h));
  xh = __dadd_rn(L.x0, __dmul_rn((double)(i + 1), L.h));
  yl = __dadd_rn(L.y0, __dmul_rn((double)j, L.h));
  yh = __dadd_rn(L.y0, __dmul_rn((double)(j + 1), L.h));
}

// Inside / Cut / Outside (P l.69, reading R2)
__global__ void k_classify(LevelArgs L, int8_t* ct) {
  int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= L.n || j >= L.n) return;
  if (L.fitted) {   // fitted box: Omega is the background box, every cell is Inside
    ct[j * L.n + i] = INSIDE;
    return;
  }
  double xl, xh, yl, yh;
  cell_bounds(L, i, j, xl, xh, yl, yh);
  double r2 = __dmul_rn(L.r, L.r);
  double qx = __dsub_rn(fmin(fmax(L.cx, xl), xh), L.cx);
  double qy = __dsub_rn(fmin(fmax(L.cy, yl), yh), L.cy);
  double fx = fmax(fabs(__dsub_rn(xl, L.cx)), fabs(__dsub_rn(xh, L.cx)));
  double fy = fmax(fabs(__dsub_rn(yl, L.cy)), fabs(__dsub_rn(yh, L.cy)));
  double dmin2 = __dadd_rn(__dmul_rn(qx, qx), __dmul_rn(qy, qy));
  double dmax2 = __dadd_rn(__dmul_rn(fx, fx), __dmul_rn(fy, fy));
  int8_t t = CUT;
  if (dmax2 <= r2) t = INSIDE;
  if (dmin2 >= r2) t = OUTSIDE;
  ct[j * L.n + i] = t;
}

__device__ __forceinline__ bool cell_active(const LevelArgs& L, const int8_t* ct, int i, int j) {
  return i >= 0 && j >= 0 && i < L.n && j < L.n && ct[j * L.n + i] != OUTSIDE;
}
__device__ __forceinline__ int cell_kind(const LevelArgs& L, const int8_t* ct, int i, int j) {
  return (i >= 0 && j >= 0 && i < L.n && j < L.n) ? ct[j * L.n + i] : OUTSIDE;
}

// DoF nodes: nodes of active cells (P l.121)
__global__ void k_mask(LevelArgs L, const int8_t* ct, uint8_t* mask, int* count) {
  int a = blockIdx.x * blockDim.x + threadIdx.x, b = blockIdx.y * blockDim.y + threadIdx.y;
  if (a >= L.ld || b >= L.nl) return;
  uint8_t m = 0;
  if (a < L.nl) {
    int p = L.p;
    int i0 = (a % p == 0) ? a / p - 1 : a / p, i1 = a / p;
    int j0 = (b % p == 0) ? b / p - 1 : b / p, j1 = b / p;
    for (int j = j0; j <= j1; ++j)
      for (int i = i0; i <= i1; ++i)
        if (cell_active(L, ct, i, j)) m = 1;
    // fitted box: strong Dirichlet, no DoF on the box boundary
    if (L.fitted && (a == 0 || b == 0 || a == L.nl - 1 || b == L.nl - 1)) m = 0;
  }
  mask[(size_t)b * L.ld + a] = m;
  if (m) atomicAdd(count, 1);
}

// Omega_l ⊆ Omega_{l-1} (P l.128-129): fine active cell with inactive parent
__global__ void k_parent_check(LevelArgs Lf, const int8_t* ctf, int nc, const int8_t* ctc, int* bad) {
  int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= Lf.n || j >= Lf.n) return;
  if (ctf[j * Lf.n + i] != OUTSIDE && ctc[(j / 2) * nc + i / 2] == OUTSIDE) atomicAdd(bad, 1);
}

__global__ void k_iota_flags_cells(int n, const int8_t* ct, int8_t want, uint8_t* flag) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < n * n) flag[c] = ct[c] == want;
}

__global__ void k_fill(int* a, int64_t n, int v) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) a[i] = v;
}

__global__ void k_scatter_id(const int* list, int n, int* map) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) map[list[k]] = k;
}

// ghost faces F_G (P l.97-101): index j*n+i for the face (i,j)|(i+1,j), n*n + j*n+i for (i,j)|(i,j+1)
__global__ void k_ghost_flags(LevelArgs L, const int8_t* ct, uint8_t* flag) {
  int f = blockIdx.x * blockDim.x + threadIdx.x;
  int n = L.n;
  if (f >= 2 * n * n) return;
  int axis = f >= n * n, c = f - axis * n * n, i = c % n, j = c / n;
  int i2 = i + (axis == 0), j2 = j + (axis == 1);
  bool g = cell_active(L, ct, i, j) && cell_active(L, ct, i2, j2) &&
           (cell_kind(L, ct, i, j) == CUT || cell_kind(L, ct, i2, j2) == CUT);
  flag[f] = g;
}

__global__ void k_ghost_maps(const int* list, int ng, int n, int* gx, int* gy) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= ng) return;
  int f = list[k];
  if (f < n * n) gx[f] = k;
  else gy[f - n * n] = k;
}

// compact per-cell code: bits 0-1 kind, bit 2..5 = ghost face on the left,
// right, bottom, top (one byte per cell instead of five integer loads)
__global__ void k_cell_codes(LevelArgs L, uint8_t* code) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = L.n;
  if (c >= n * n) return;
  const int i = c % n, j = c / n;
  uint8_t v = (uint8_t)L.ctype[c];
  if (i >= 1 && L.gx_id[c - 1] >= 0) v |= 4;
  if (L.gx_id[c] >= 0) v |= 8;
  if (j >= 1 && L.gy_id[c - n] >= 0) v |= 16;
  if (L.gy_id[c] >= 0) v |= 32;
  code[c] = v;
}

// ---- cut-cell quadrature (P l.190, reading R6) -----------------------------
// One thread per cut cell.  WRITE = false counts the points.
template <bool WRITE>
__device__ void cut_rule(const LevelArgs& L, int i, int j, int nq, int& nv, int& ns, int vo, int so, double* qx,
                         double* qy, double* qw, double* sx, double* sy, double* sw, double* snx, double* sny) {
  double xl, xh, yl, yh;
  cell_bounds(L, i, j, xl, xh, yl, yh);
  const double cx = L.cx, cy = L.cy, r = L.r, h = L.h;
  double xc = __dmul_rn(0.5, __dadd_rn(xl, xh)), yc = __dmul_rn(0.5, __dadd_rn(yl, yh));
  bool swap = !(fabs(__dsub_rn(yc, cy)) >= fabs(__dsub_rn(xc, cx)));
  double t_lo = swap ? yl : xl, t_hi = swap ? yh : xh, s_lo = swap ? xl : yl, s_hi = swap ? xh : yh;
  double ct = swap ? cy : cx, cs = swap ? cx : cy;
  double r2 = __dmul_rn(r, r);
  double brk[8];
  int nb = 0;
  brk[nb++] = t_lo;
  brk[nb++] = t_hi;
  double faces[2] = {s_lo, s_hi};
  for (int f = 0; f < 2; ++f) {
    double df = __dsub_rn(faces[f], cs);
    double D = __dsub_rn(r2, __dmul_rn(df, df));
    if (D > 0.0) {
      double q = sqrt(D);
      brk[nb++] = __dsub_rn(ct, q);
      brk[nb++] = __dadd_rn(ct, q);
    }
  }
  brk[nb++] = __dsub_rn(ct, r);
  brk[nb++] = __dadd_rn(ct, r);
  // keep points in [t_lo, t_hi], sort, unique
  double pts[8];
  int np = 0;
  for (int k = 0; k < nb; ++k)
    if (t_lo <= brk[k] && brk[k] <= t_hi) pts[np++] = brk[k];
  for (int a = 1; a < np; ++a) {
    double v = pts[a];
    int b = a - 1;
    while (b >= 0 && pts[b] > v) {
      pts[b + 1] = pts[b];
      --b;
    }
    pts[b + 1] = v;
  }
  int nu = 0;
  for (int k = 0; k < np; ++k)
    if (nu == 0 || pts[k] != pts[nu - 1]) pts[nu++] = pts[k];
  nv = 0;
  ns = 0;
  const double* g = c_gx[nq];
  const double* w = c_gw[nq];
  for (int k = 0; k + 1 < nu; ++k) {
    double ta = pts[k], tb = pts[k + 1];
    if (!(tb > ta)) continue;
    for (int a = 0; a < nq; ++a) {
      double t = __dadd_rn(ta, __dmul_rn(__dsub_rn(tb, ta), g[a]));
      double wt = w[a] * (tb - ta);
      double dt = __dsub_rn(t, ct);
      double D = __dsub_rn(r2, __dmul_rn(dt, dt));
      if (!(D > 0.0)) continue;
      double S = sqrt(D);
      double lo = fmax(s_lo, __dsub_rn(cs, S)), hi = fmin(s_hi, __dadd_rn(cs, S));
      if (hi > lo) {
        for (int m = 0; m < nq; ++m) {
          if (WRITE) {
            double s = lo + (hi - lo) * g[m];
            double x = swap ? s : t, y = swap ? t : s;
            qx[vo + nv] = (x - xl) / h;
            qy[vo + nv] = (y - yl) / h;
            qw[vo + nv] = wt * w[m] * (hi - lo);
          }
          ++nv;
        }
      }
      double sv[2] = {__dsub_rn(cs, S), __dadd_rn(cs, S)};
      for (int e = 0; e < 2; ++e) {
        double s = sv[e];
        if (s_lo < s && s < s_hi) {
          if (WRITE) {
            double x = swap ? s : t, y = swap ? t : s;
            sx[so + ns] = (x - xl) / h;
            sy[so + ns] = (y - yl) / h;
            sw[so + ns] = wt * r / S;
            snx[so + ns] = (x - cx) / r;
            sny[so + ns] = (y - cy) / r;
          }
          ++ns;
        }
      }
    }
  }
}

__global__ void k_cut_count(LevelArgs L, int nq, int* vcount, int* scount) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= L.n_cut) return;
  int c = L.cut_list[k];
  int nv, ns;
  cut_rule<false>(L, c % L.n, c / L.n, nq, nv, ns, 0, 0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                  nullptr, nullptr);
  vcount[k] = nv;
  scount[k] = ns;
}

__global__ void k_cut_fill(LevelArgs L, int nq, double* qx, double* qy, double* qw, double* sx, double* sy, double* sw,
                           double* snx, double* sny) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= L.n_cut) return;
  int c = L.cut_list[k];
  int nv, ns;
  cut_rule<true>(L, c % L.n, c / L.n, nq, nv, ns, L.q_off[k], L.s_off[k], qx, qy, qw, sx, sy, sw, snx, sny);
}

// ---- vertex patches (P l.141-156, l.179; readings R3, R4) -----------------
__global__ void k_vertex_kind(LevelArgs L, const int8_t* ct, uint8_t* vk) {
  int I = blockIdx.x * blockDim.x + threadIdx.x, J = blockIdx.y * blockDim.y + threadIdx.y;
  int n = L.n;
  if (I > n || J > n) return;
  int nact = 0, ninside = 0;
  for (int dy = -1; dy <= 0; ++dy)
    for (int dx = -1; dx <= 0; ++dx) {
      int k = cell_kind(L, ct, I + dx, J + dy);
      nact += k != OUTSIDE;
      ninside += k == INSIDE;
    }
  uint8_t v = V_NONE;
  // fitted box: patches at the vertices contained in the open box (P l.143)
  if (nact > 0 && !(L.fitted && (I == 0 || J == 0 || I == n || J == n))) {
    bool cart = ninside == 4;
    const int nb[8][2] = {{-2, -1}, {-2, 0}, {1, -1}, {1, 0}, {-1, -2}, {0, -2}, {-1, 1}, {0, 1}};
    for (int q = 0; q < 8 && cart; ++q)
      if (cell_kind(L, ct, I + nb[q][0], J + nb[q][1]) == CUT) cart = false;
    v = cart ? V_CART : V_CUT;
  }
  vk[J * (n + 1) + I] = v;
}

__global__ void k_vertex_flags(int n, const uint8_t* vk, uint8_t kind, int colour, uint8_t* flag) {
  int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= (n + 1) * (n + 1)) return;
  int I = v % (n + 1), J = v / (n + 1);
  flag[v] = vk[v] == kind && ((I & 1) + 2 * (J & 1)) == colour;
}

// Cartesian tiles of TP x TP same-colour patches containing at least one Cartesian patch
__global__ void k_tile_flags(int n, const uint8_t* vk, int colour, int TP, int tx, int ty, uint8_t* flag) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= tx * ty) return;
  int ti = t % tx, tj = t / tx;
  int cxo = colour & 1, cyo = colour >> 1;
  uint8_t f = 0;
  for (int v = 0; v < TP && !f; ++v)
    for (int u = 0; u < TP; ++u) {
      int I = cxo + 2 * (ti * TP + u), J = cyo + 2 * (tj * TP + v);
      if (I <= n && J <= n && vk[J * (n + 1) + I] == V_CART) {
        f = 1;
        break;
      }
    }
  flag[t] = f;
}

__global__ void k_pack_tiles(const int* sel, int nsel, int tx, int* out) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nsel) out[k] = (sel[k] % tx) | ((sel[k] / tx) << 16);
}

// interior DoF set of a cut patch: DoF nodes of the block whose active support
// lies in the patch (P l.153, reading R3).  WRITE = false counts.
template <bool WRITE>
__global__ void k_cut_interior(LevelArgs L, const int8_t* ct, const int* plist, int np, int* count,
                               const int64_t* off, int32_t* node, uint16_t* loc, int32_t* owner) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= np) return;
  int n = L.n, p = L.p;
  int I = plist[k] % (n + 1), J = plist[k] / (n + 1);
  int m = 0;
  int64_t o = WRITE ? off[k] : 0;
  for (int db = 0; db <= 2 * p; ++db)
    for (int da = 0; da <= 2 * p; ++da) {
      int a = p * (I - 1) + da, b = p * (J - 1) + db;
      if (a < 0 || b < 0 || a >= L.nl || b >= L.nl) continue;
      if (!L.mask[(size_t)b * L.ld + a]) continue;
      int i0 = (a % p == 0) ? a / p - 1 : a / p, i1 = a / p;
      int j0 = (b % p == 0) ? b / p - 1 : b / p, j1 = b / p;
      bool inside = true;
      for (int j = j0; j <= j1; ++j)
        for (int i = i0; i <= i1; ++i)
          if (cell_active(L, ct, i, j) && !(i >= I - 1 && i <= I && j >= J - 1 && j <= J)) inside = false;
      if (!inside) continue;
      if (WRITE) {
        node[o + m] = b * L.ld + a;
        loc[o + m] = (uint16_t)(db * (2 * p + 1) + da);
        owner[o + m] = k;
      }
      ++m;
    }
  if (!WRITE) count[k] = m;
}

__global__ void k_widen(const int* in, int n, int64_t* out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) out[k] = in[k];
}

__global__ void k_square(const int* m, int n, int* out) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) out[k] = m[k] * m[k];
}

// In-place Gauss-Jordan inverse of SPD matrices (no pivoting needed for SPD).
// One CTA per matrix; matrix plus pivot row/column staged in dynamic shared
// memory ((m*m + 2m) doubles).
// the same Gauss-Jordan elimination in place in global memory, for local
// matrices too large for shared memory (3D Q3 cut patches, m up to 343): one
// CTA per patch, the pivot row / column staged in shared memory (2 m doubles)
__global__ void k_batched_inverse_gmem(const int64_t* ent_off, const int64_t* inv_off, double* inv, int np,
                                       int mmin) {
  extern __shared__ double rc[];
  const int k = blockIdx.x;
  if (k >= np) return;
  const int m = (int)(ent_off[k + 1] - ent_off[k]);
  if (m < mmin) return;   // done by k_batched_inverse
  double* A = inv + inv_off[k];
  double* rowk = rc;
  double* colk = rc + m;
  for (int c = 0; c < m; ++c) {
    const double piv = A[(int64_t)c * m + c];
    for (int e = threadIdx.x; e < m; e += blockDim.x) {
      rowk[e] = (e == c ? 1.0 : A[(int64_t)c * m + e]) / piv;
      colk[e] = A[(int64_t)e * m + c];
    }
    __syncthreads();
    for (int64_t e = threadIdx.x; e < (int64_t)m * m; e += blockDim.x) {
      const int i = (int)(e / m), jj = (int)(e % m);
      A[e] = (i == c) ? rowk[jj] : ((jj == c ? 0.0 : A[e]) - colk[i] * rowk[jj]);
    }
    __syncthreads();
  }
}

__global__ void k_batched_inverse(const int64_t* ent_off, const int64_t* inv_off, double* inv, int np) {
  extern __shared__ double sm[];
  int k = blockIdx.x;
  if (k >= np) return;
  int m = (int)(ent_off[k + 1] - ent_off[k]);
  if ((size_t)(m * m + 2 * m) * sizeof(double) > 200 * 1024) return;   // k_batched_inverse_gmem
  double* A = inv + inv_off[k];
  double* rowk = sm + m * m;
  double* colk = rowk + m;
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) sm[e] = A[e];
  __syncthreads();
  for (int c = 0; c < m; ++c) {
    double piv = sm[c * m + c];
    for (int e = threadIdx.x; e < m; e += blockDim.x) {
      rowk[e] = (e == c ? 1.0 : sm[c * m + e]) / piv;
      colk[e] = sm[e * m + c];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
      int i = e / m, jj = e % m;
      sm[e] = (i == c) ? rowk[jj] : ((jj == c ? 0.0 : sm[e]) - colk[i] * rowk[jj]);
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) A[e] = sm[e];
}

}  // namespace cf
