// tables.cuh — host computation of the per-degree 1D tables (P l.79: Q_p
// with Gauss-Lobatto nodal basis) and of Gauss-Legendre rules, uploaded to
// __constant__ memory.  Plain C++ on the host, independent of the oracle.
#pragma once
#include <cmath>
#include <cstring>
#include <vector>

#include "internal.cuh"

namespace cf {

namespace host {

// n-point Gauss-Legendre rule on [0,1] by Newton iteration on P_n.
inline void gauss_legendre(int n, double* x, double* w) {
  for (int i = 0; i < n; ++i) {
    double z = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    double dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = 0.0;
      for (int j = 1; j <= n; ++j) {
        double p2 = p1;
        p1 = p0;
        p0 = ((2.0 * j - 1.0) * z * p1 - (j - 1.0) * p2) / j;
      }
      dp = n * (z * p0 - p1) / (z * z - 1.0);
      double dz = p0 / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-16) break;
    }
    // recompute derivative at the converged root
    double p0 = 1.0, p1 = 0.0;
    for (int j = 1; j <= n; ++j) {
      double p2 = p1;
      p1 = p0;
      p0 = ((2.0 * j - 1.0) * z * p1 - (j - 1.0) * p2) / j;
    }
    dp = n * (z * p0 - p1) / (z * z - 1.0);
    x[n - 1 - i] = 0.5 * (z + 1.0);
    w[n - 1 - i] = 1.0 / ((1.0 - z * z) * dp * dp);  // 2/((1-z^2)P'^2) on [-1,1], halved
  }
}

// Gauss-Lobatto nodes on [0,1] in closed form for p <= 4.
inline void gauss_lobatto(int p, double* xi) {
  xi[0] = 0.0;
  xi[p] = 1.0;
  if (p == 2) xi[1] = 0.5;
  if (p == 3) {
    double s = 1.0 / std::sqrt(5.0);
    xi[1] = 0.5 * (1.0 - s);
    xi[2] = 0.5 * (1.0 + s);
  }
  if (p == 4) {
    double s = std::sqrt(3.0 / 7.0);
    xi[1] = 0.5 * (1.0 - s);
    xi[2] = 0.5;
    xi[3] = 0.5 * (1.0 + s);
  }
}

// L_m(x) by the product formula (exact 0 / 1 at the nodes).
inline double lagrange(int p, const double* xi, int m, double x) {
  double v = 1.0;
  for (int j = 0; j <= p; ++j)
    if (j != m) v *= (x - xi[j]) / (xi[m] - xi[j]);
  return v;
}

// symmetric eigen-decomposition by cyclic Jacobi rotations: A = Q diag(d) Q^T
inline void jacobi_eigen(int n, std::vector<double> A, std::vector<double>& Q, std::vector<double>& d) {
  Q.assign(n * n, 0.0);
  for (int i = 0; i < n; ++i) Q[i * n + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = i + 1; j < n; ++j) off += A[i * n + j] * A[i * n + j];
    if (off < 1e-32) break;
    for (int pp = 0; pp < n; ++pp)
      for (int q = pp + 1; q < n; ++q) {
        double apq = A[pp * n + q];
        if (std::fabs(apq) < 1e-300) continue;
        double theta = (A[q * n + q] - A[pp * n + pp]) / (2.0 * apq);
        double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {  // A <- J^T A J
          double akp = A[k * n + pp], akq = A[k * n + q];
          A[k * n + pp] = c * akp - s * akq;
          A[k * n + q] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          double apk = A[pp * n + k], aqk = A[q * n + k];
          A[pp * n + k] = c * apk - s * aqk;
          A[q * n + k] = s * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {
          double qkp = Q[k * n + pp], qkq = Q[k * n + q];
          Q[k * n + pp] = c * qkp - s * qkq;
          Q[k * n + q] = s * qkp + c * qkq;
        }
      }
  }
  d.resize(n);
  for (int i = 0; i < n; ++i) d[i] = A[i * n + i];
}

inline void build_tab(int p, Tab& t) {
  std::memset(&t, 0, sizeof(Tab));
  gauss_lobatto(p, t.gll);
  // power coefficients of L_i by expanding prod_{j != i} (x - xi_j) / (xi_i - xi_j)
  for (int i = 0; i <= p; ++i) {
    double c[CF_MAXP + 1] = {1.0};
    int deg = 0;
    double den = 1.0;
    for (int j = 0; j <= p; ++j) {
      if (j == i) continue;
      double nc[CF_MAXP + 1] = {0};
      for (int m = 0; m <= deg; ++m) {
        nc[m + 1] += c[m];
        nc[m] -= t.gll[j] * c[m];
      }
      ++deg;
      std::memcpy(c, nc, sizeof(c));
      den *= t.gll[i] - t.gll[j];
    }
    for (int m = 0; m <= p; ++m) t.lc[i][m] = c[m] / den;
    for (int m = 1; m <= p; ++m) t.dc[i][m - 1] = m * t.lc[i][m];
  }
  // derivatives of order k at 0 and 1
  for (int k = 0; k <= p; ++k)
    for (int i = 0; i <= p; ++i) {
      double v0 = 0.0, v1 = 0.0;
      for (int m = k; m <= p; ++m) {
        double f = 1.0;
        for (int q = 0; q < k; ++q) f *= (m - q);
        if (m == k) v0 = f * t.lc[i][m];
        v1 += f * t.lc[i][m];
      }
      t.d0[k][i] = v0;
      t.d1[k][i] = v1;
    }
  // exact reference matrices: int_0^1 x^m = 1/(m+1)
  for (int i = 0; i <= p; ++i)
    for (int j = 0; j <= p; ++j) {
      double kk = 0.0, mm = 0.0;
      for (int a = 0; a <= p; ++a)
        for (int b = 0; b <= p; ++b) mm += t.lc[i][a] * t.lc[j][b] / (a + b + 1.0);
      for (int a = 0; a < p; ++a)
        for (int b = 0; b < p; ++b) kk += t.dc[i][a] * t.dc[j][b] / (a + b + 1.0);
      t.Kref[i][j] = kk;
      t.Mref[i][j] = mm;
    }
  // two-cell patch matrices
  for (int c = 0; c < 2; ++c)
    for (int i = 0; i <= p; ++i)
      for (int j = 0; j <= p; ++j) {
        t.Kp[c * p + i][c * p + j] += t.Kref[i][j];
        t.Mp[c * p + i][c * p + j] += t.Mref[i][j];
      }
  // fast diagonalisation of the interior block (rows/cols 1..2p-1)
  int ni = 2 * p - 1;
  std::vector<double> K(ni * ni), M(ni * ni), Lc(ni * ni, 0.0), Li(ni * ni, 0.0);
  for (int i = 0; i < ni; ++i)
    for (int j = 0; j < ni; ++j) {
      K[i * ni + j] = t.Kp[i + 1][j + 1];
      M[i * ni + j] = t.Mp[i + 1][j + 1];
    }
  for (int j = 0; j < ni; ++j) {  // Cholesky M = Lc Lc^T
    double s = M[j * ni + j];
    for (int k = 0; k < j; ++k) s -= Lc[j * ni + k] * Lc[j * ni + k];
    Lc[j * ni + j] = std::sqrt(s);
    for (int i = j + 1; i < ni; ++i) {
      double v = M[i * ni + j];
      for (int k = 0; k < j; ++k) v -= Lc[i * ni + k] * Lc[j * ni + k];
      Lc[i * ni + j] = v / Lc[j * ni + j];
    }
  }
  for (int c = 0; c < ni; ++c)  // Li = Lc^{-1} by forward substitution
    for (int i = 0; i < ni; ++i) {
      double v = (i == c) ? 1.0 : 0.0;
      for (int k = 0; k < i; ++k) v -= Lc[i * ni + k] * Li[k * ni + c];
      Li[i * ni + c] = v / Lc[i * ni + i];
    }
  std::vector<double> C(ni * ni, 0.0), Q, d;
  for (int i = 0; i < ni; ++i)
    for (int j = 0; j < ni; ++j) {
      double v = 0.0;
      for (int a = 0; a < ni; ++a)
        for (int b = 0; b < ni; ++b) v += Li[i * ni + a] * K[a * ni + b] * Li[j * ni + b];
      C[i * ni + j] = v;
    }
  jacobi_eigen(ni, C, Q, d);
  for (int i = 0; i < ni; ++i)  // S = Li^T Q
    for (int j = 0; j < ni; ++j) {
      double v = 0.0;
      for (int a = 0; a < ni; ++a) v += Li[a * ni + i] * Q[a * ni + j];
      t.S[i][j] = v;
    }
  for (int i = 0; i < ni; ++i) t.lam[i] = d[i];
  // transfer weights
  for (int d2 = 0; d2 <= 2 * p; ++d2) {
    int child = d2 / p, k = d2 - child * p;
    if (child == 2) child = 1, k = p;
    double xc = (child + t.gll[k]) / 2.0;
    for (int m = 0; m <= p; ++m) t.pw[d2][m] = lagrange(p, t.gll, m, xc);
  }
  for (int m = 0; m < p; ++m)
    for (int d = -2 * p; d <= 2 * p; ++d) {
      double v = 0.0;
      if (d >= 0) v = t.pw[d][m];
      else if (m == 0) v = t.pw[d + 2 * p][p];
      t.tw[m][d + 2 * p] = v;
    }
}

inline void upload_tables() {   // __constant__ / __device__ tables: once per device
  static const char key = 0;
  dev_once(&key, [] {
  Tab tabs[CF_MAXP + 1];
  std::memset(&tabs[0], 0, sizeof(Tab));
  for (int p = 1; p <= CF_MAXP; ++p) build_tab(p, tabs[p]);
  CF_CUDA(cudaMemcpyToSymbol(c_tab, tabs, sizeof(tabs)));
  CF_CUDA(cudaMemcpyToSymbol(g_tab, tabs, sizeof(tabs)));
  double gx[CF_MAXNQ + 1][CF_MAXNQ] = {}, gw[CF_MAXNQ + 1][CF_MAXNQ] = {};
  for (int n = 1; n <= CF_MAXNQ; ++n) gauss_legendre(n, gx[n], gw[n]);
  CF_CUDA(cudaMemcpyToSymbol(c_gx, gx, sizeof(gx)));
  CF_CUDA(cudaMemcpyToSymbol(c_gw, gw, sizeof(gw)));
  });
}

}  // namespace host
}  // namespace cf

namespace cf {
namespace host {

// Dense affine map of one Cartesian patch solve (P l.192 fast diagonalisation,
// written out): x_int_new = A_int^{-1} b_int + (E - A_int^{-1} Ā) x_ext with
// A = K̄⊗M̄ + M̄⊗K̄ on the two-cell patch (h-free in 2D), rows = interior
// nodes (ib*NI + ia), columns = [b_int (NI^2) | x_ext (NE^2)], padded to
// (8*MT) x (4*KS) for the fp64 tensor-core (DMMA m8n8k4) fragments.
inline std::vector<double> cart_affine_map(int p, const Tab& t, int& rows_pad, int& cols_pad) {
  const int NE = 2 * p + 1, NI = 2 * p - 1, NINT = NI * NI, NEXT = NE * NE, K = NINT + NEXT;
  rows_pad = 8 * ((NINT + 7) / 8);
  cols_pad = 4 * ((K + 3) / 4);
  std::vector<double> Aext(NINT * NEXT), Ai(NINT * NINT);
  for (int ib = 0; ib < NI; ++ib)
    for (int ia = 0; ia < NI; ++ia)
      for (int bb = 0; bb < NE; ++bb)
        for (int aa = 0; aa < NE; ++aa) {
          const int r = ib * NI + ia, c = bb * NE + aa, a = ia + 1, b = ib + 1;
          Aext[r * NEXT + c] = t.Kp[a][aa] * t.Mp[b][bb] + t.Mp[a][aa] * t.Kp[b][bb];
        }
  for (int r = 0; r < NINT; ++r)
    for (int q = 0; q < NINT; ++q) {
      const int ib = q / NI, ia = q % NI;
      Ai[r * NINT + q] = Aext[r * NEXT + (ib + 1) * NE + ia + 1];
    }
  // Gauss-Jordan inverse with partial pivoting
  std::vector<double> inv(NINT * NINT, 0.0);
  for (int i = 0; i < NINT; ++i) inv[i * NINT + i] = 1.0;
  for (int c = 0; c < NINT; ++c) {
    int pr = c;
    for (int r = c + 1; r < NINT; ++r)
      if (std::fabs(Ai[r * NINT + c]) > std::fabs(Ai[pr * NINT + c])) pr = r;
    for (int q = 0; q < NINT; ++q) {
      std::swap(Ai[c * NINT + q], Ai[pr * NINT + q]);
      std::swap(inv[c * NINT + q], inv[pr * NINT + q]);
    }
    const double piv = Ai[c * NINT + c];
    for (int q = 0; q < NINT; ++q) {
      Ai[c * NINT + q] /= piv;
      inv[c * NINT + q] /= piv;
    }
    for (int r = 0; r < NINT; ++r) {
      if (r == c) continue;
      const double f = Ai[r * NINT + c];
      if (f == 0.0) continue;
      for (int q = 0; q < NINT; ++q) {
        Ai[r * NINT + q] -= f * Ai[c * NINT + q];
        inv[r * NINT + q] -= f * inv[c * NINT + q];
      }
    }
  }
  std::vector<double> G((size_t)rows_pad * cols_pad, 0.0);
  for (int r = 0; r < NINT; ++r) {
    for (int q = 0; q < NINT; ++q) G[r * cols_pad + q] = inv[r * NINT + q];
    for (int c = 0; c < NEXT; ++c) {
      double s = 0.0;
      for (int q = 0; q < NINT; ++q) s += inv[r * NINT + q] * Aext[q * NEXT + c];
      const int ib = r / NI, ia = r % NI;
      const double e = (c == (ib + 1) * NE + ia + 1) ? 1.0 : 0.0;
      G[r * cols_pad + NINT + c] = e - s;
    }
  }
  return G;
}

}  // namespace host
}  // namespace cf

namespace cf {
namespace host {
// per-degree dense patch maps in global memory (p = 1..3), built once per process
inline const double* cart_map(int p) {
  static const char keys[CF_MAXP + 1] = {};   // device pointer per (degree, device)
  if (p < 1 || p > 3) return nullptr;
  return (const double*)dev_cached(&keys[p], [&] {
    Tab t;
    build_tab(p, t);
    int rp = 0, cp = 0;
    std::vector<double> G = cart_affine_map(p, t, rp, cp);
    void* d = nullptr;
    CF_CUDA(cudaMalloc(&d, G.size() * sizeof(double)));
    CF_CUDA(cudaMemcpy(d, G.data(), G.size() * sizeof(double), cudaMemcpyHostToDevice));
    return (int64_t)d;
  });
}
}  // namespace host
}  // namespace cf

namespace cf {
namespace host {
// 3D dense patch map for h = 1 (A scales with h in 3D; the kernel divides
// the b operands by h): rows = interior nodes (ic, ib, ia), columns =
// [b_int | x_ext]
inline std::vector<double> cart_affine_map3(int p, const Tab& t, int& cols_pad) {
  const int NE = 2 * p + 1, NI = 2 * p - 1, NINT = NI * NI * NI, NEXT = NE * NE * NE, K = NINT + NEXT;
  cols_pad = 4 * ((K + 3) / 4);
  const int rows_pad = 8 * ((NINT + 7) / 8);
  std::vector<double> Aext((size_t)NINT * NEXT), Ai((size_t)NINT * NINT);
  for (int r = 0; r < NINT; ++r) {
    const int a = r % NI + 1, b = (r / NI) % NI + 1, c = r / (NI * NI) + 1;
    for (int q = 0; q < NEXT; ++q) {
      const int aa = q % NE, bb = (q / NE) % NE, cc = q / (NE * NE);
      Aext[(size_t)r * NEXT + q] = t.Kp[a][aa] * t.Mp[b][bb] * t.Mp[c][cc] + t.Mp[a][aa] * t.Kp[b][bb] * t.Mp[c][cc] +
                                   t.Mp[a][aa] * t.Mp[b][bb] * t.Kp[c][cc];
    }
  }
  for (int r = 0; r < NINT; ++r)
    for (int q = 0; q < NINT; ++q) {
      const int a = q % NI + 1, b = (q / NI) % NI + 1, c = q / (NI * NI) + 1;
      Ai[(size_t)r * NINT + q] = Aext[(size_t)r * NEXT + (c * NE + b) * NE + a];
    }
  std::vector<double> inv((size_t)NINT * NINT, 0.0);
  for (int i = 0; i < NINT; ++i) inv[(size_t)i * NINT + i] = 1.0;
  for (int c = 0; c < NINT; ++c) {
    int pr = c;
    for (int r = c + 1; r < NINT; ++r)
      if (std::fabs(Ai[(size_t)r * NINT + c]) > std::fabs(Ai[(size_t)pr * NINT + c])) pr = r;
    for (int q = 0; q < NINT; ++q) {
      std::swap(Ai[(size_t)c * NINT + q], Ai[(size_t)pr * NINT + q]);
      std::swap(inv[(size_t)c * NINT + q], inv[(size_t)pr * NINT + q]);
    }
    const double piv = Ai[(size_t)c * NINT + c];
    for (int q = 0; q < NINT; ++q) {
      Ai[(size_t)c * NINT + q] /= piv;
      inv[(size_t)c * NINT + q] /= piv;
    }
    for (int r = 0; r < NINT; ++r) {
      if (r == c) continue;
      const double f = Ai[(size_t)r * NINT + c];
      if (f == 0.0) continue;
      for (int q = 0; q < NINT; ++q) {
        Ai[(size_t)r * NINT + q] -= f * Ai[(size_t)c * NINT + q];
        inv[(size_t)r * NINT + q] -= f * inv[(size_t)c * NINT + q];
      }
    }
  }
  std::vector<double> G((size_t)rows_pad * cols_pad, 0.0);
  for (int r = 0; r < NINT; ++r) {
    for (int q = 0; q < NINT; ++q) G[(size_t)r * cols_pad + q] = inv[(size_t)r * NINT + q];
    const int a = r % NI + 1, b = (r / NI) % NI + 1, c = r / (NI * NI) + 1;
    for (int qe = 0; qe < NEXT; ++qe) {
      double s = 0.0;
      for (int q = 0; q < NINT; ++q) s += inv[(size_t)r * NINT + q] * Aext[(size_t)q * NEXT + qe];
      G[(size_t)r * cols_pad + NINT + qe] = (qe == (c * NE + b) * NE + a ? 1.0 : 0.0) - s;
    }
  }
  return G;
}

inline const double* cart_map3(int p) {
  static const char keys[CF_MAXP + 1] = {};   // device pointer per (degree, device)
  if (p < 1 || p > 3) return nullptr;
  return (const double*)dev_cached(&keys[p], [&] {
    Tab t;
    build_tab(p, t);
    int cp = 0;
    std::vector<double> G = cart_affine_map3(p, t, cp);
    void* d = nullptr;
    CF_CUDA(cudaMalloc(&d, G.size() * sizeof(double)));
    CF_CUDA(cudaMemcpy(d, G.data(), G.size() * sizeof(double), cudaMemcpyHostToDevice));
    return (int64_t)d;
  });
}
}  // namespace host
}  // namespace cf
