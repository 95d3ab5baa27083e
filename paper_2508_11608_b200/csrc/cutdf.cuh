// cutdf.cuh — all 4 n_c cut colour steps of one smoothing step (P eq.
// smoother-split, l.203-205: "repeat n_c times ... j in J_c", coloured as
// l.212) in ONE launch, synchronised by dataflow flags instead of kernel
// boundaries or a grid barrier.
//
// Each cut patch is the affine map x_I <- G_j [b_I ; x_E] of reading R13
// (G_j = [A_j^{-1} | -A_j^{-1} A_{I,E}], built by k_cut_map).  The patches are
// grouped into spatially compact SEGMENTS (tiles of T x T vertices, split to a
// shared-memory budget); one CTA owns one segment for the whole sweep and
// keeps every map of its segment resident in shared memory: the segment's
// blob (header, row table, maps, gather and copy lists) arrives with a few
// cp.async.bulk copies on one mbarrier, before griddepcontrol.wait, so it
// overlaps the predecessor kernel and is read from HBM once per smoothing step
// although each patch is applied n_c times.
//
// Step s (colour c_s) reads buffer R = B_{s-1} and writes W = B_s (ping-pong
// between x and xs, as k_cut_step7): W = R + update on the interiors N_s and
// W = R on N_{s-1} \ N_s (copy lists; at s = 0 the read band \ N_0).  A patch
// reads its window (vertex distance <= 2) and writes its interior (distance
// <= 1), and the copy of a node is done by the segment of the step-(s-1)
// patch that owns it (at s = 0: of the first patch whose window holds it), so
// every read-after-write and write-after-read hazard of step s is between
// patches at vertex (Chebyshev) distance <= 4.  Segment A therefore starts
// step s after every segment with a patch within distance 4 of one of A's
// patches has published step s-1 on its flag (ld.acquire spin), and
// publishes its own step s with a release store after its writes.  Flags
// count completed steps and are never reset: a launch reads its own flag as
// the base (every flag equals it at launch start: the previous launch ran all
// 4 n_c steps on every segment), so CUDA-graph replays need no memset.  All
// segments are co-resident (cooperative launch; the builder checks the
// occupancy), so the spin waits cannot deadlock.
//
// The update rows are evaluated exactly as k_cut_step7 does (tpr lanes per
// row, two accumulators, xor-shuffle reduction), so the two kernels are
// bit-identical.
#pragma once
#include <algorithm>
#include <cstring>
#include <unordered_map>
#include <vector>

#include "internal.cuh"
#include "tma.cuh"

namespace cf {

constexpr int DF_MAXDEP = 64;
constexpr int DF_FLAG_STRIDE = 32;   // flags 128 bytes apart: one L2 line (and slice hash) per segment

// per-segment blob header (256 bytes); offsets in bytes from the blob start
struct DfHdr {
  int blob_bytes;     // size of the blob (the v area follows it in shared memory)
  int v_doubles;      // size of the gathered-operand area
  int nrow[4], row_off[4];   // update rows per colour
  int nx[4], x_off[4];       // x_E gathers per colour: int2 {lattice node, v index}
  int nb, b_off;             // b_I gathers of every colour (once per launch): int2 {node, v index}
  int ncp[20], cp_off[20];   // copy lists per (prev, cur), prev = 4: read band of step 0
  int pad[4];
};
static_assert(sizeof(DfHdr) == 256, "DfHdr is 256 bytes");

struct DfRow {
  int g;       // first double of the row of G_j (index from the blob start)
  int v;       // first double of the patch operand [b_I ; x_E] in the v area
  int out;     // lattice node of the interior DoF the row updates
  short K;     // m_j + nnz_j
  short tpr;   // lanes per row (as k_cut_step7 with 128 threads)
};
static_assert(sizeof(DfRow) == 16, "DfRow is 16 bytes");

struct DfArgs {
  const unsigned char* blob;
  const long long* seg_off;   // nseg + 1 byte offsets into blob
  const int* dep_off;         // nseg + 1
  const int* deps;
  unsigned* flags;            // nseg completed-step counters, DF_FLAG_STRIDE apart
  double* x;
  double* xs;
  const double* b;
  int S;                      // 4 n_c steps (even)
  int reverse;                // colours 3..0 (adjoint sweep, R9)
  unsigned long long* trace;  // debug (CUTFEM_DF_TRACE): globaltimer stamps per CTA, else nullptr
  unsigned spin_ns;           // back-off of the flag polls
};
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          (unsigned)__cvta_generic_to_shared(dst)),
      "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
      : "memory");
}

// v[dst] = src[node] over an int2 {node, dst} list; U loads in flight per
// thread before the stores (the loop is latency bound: one L2 round trip per
// batch instead of one per entry)
template <int NT, int U, bool CG>
__device__ __forceinline__ void df_gather(const int2* lst, int n, const double* __restrict__ src, double* v) {
  for (int e0 = threadIdx.x; e0 < n; e0 += NT * U) {
    double val[U];
    int dst[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * NT;
      dst[u] = -1;
      if (e < n) {
        const int2 q = lst[e];
        dst[u] = q.y;
        val[u] = CG ? __ldcg(src + q.x) : __ldg(src + q.x);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (dst[u] >= 0) v[dst[u]] = val[u];
  }
}
// W[node] = R[node] over a node list, U loads in flight per thread
template <int NT, int U>
__device__ __forceinline__ void df_copy(const int* lst, int n, const double* R, double* W) {
  for (int e0 = threadIdx.x; e0 < n; e0 += NT * U) {
    double val[U];
    int nd[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * NT;
      nd[u] = e < n ? lst[e] : -1;
      if (nd[u] >= 0) val[u] = __ldcg(R + nd[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (nd[u] >= 0) W[nd[u]] = val[u];
  }
}

template <int NT>
__global__ void __launch_bounds__(NT) k_cut_df(DfArgs A) {
  extern __shared__ __align__(128) unsigned char sdf[];
  __shared__ uint64_t bar;
  __shared__ int sdeps[DF_MAXDEP];
  __shared__ unsigned sbase;
  const int seg = blockIdx.x, tid = threadIdx.x;
  unsigned long long* tr = A.trace ? A.trace + (size_t)seg * 64 : nullptr;
  if (tr && tid == 0) tr[0] = gtimer();
  const long long o0 = A.seg_off[seg];
  const unsigned nbytes = (unsigned)(A.seg_off[seg + 1] - o0);
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_expect_tx(&bar, nbytes);
    constexpr unsigned CH = 32768;
    for (unsigned off = 0; off < nbytes; off += CH)
      bulk_g2s(sdf + off, A.blob + o0 + off, nbytes - off < CH ? nbytes - off : CH, &bar);
  }
  const int d0 = A.dep_off[seg], nd = A.dep_off[seg + 1] - d0;
  for (int i = tid; i < nd; i += NT) sdeps[i] = A.deps[d0 + i];
  pdl_trigger();
  __syncthreads();   // mbarrier initialised before anyone waits on it
  mbar_wait(&bar, 0);
  if (tr && tid == 0) tr[1] = gtimer();
  pdl_wait();        // x, xs, b of the predecessor are final from here on
  if (tr && tid == 0) tr[2] = gtimer();
  const DfHdr& H = *(const DfHdr*)sdf;
  const double* G = (const double*)sdf;
  double* v = (double*)(sdf + H.blob_bytes);
  df_gather<NT, 4, false>((const int2*)(sdf + H.b_off), H.nb, A.b, v);
  if (tid == 0) sbase = *(volatile unsigned*)(A.flags + (size_t)seg * DF_FLAG_STRIDE);
  __syncthreads();
  if (tr && tid == 0) tr[3] = gtimer();
  const unsigned base = sbase;
  for (int s = 0; s < A.S; ++s) {
    const int c = A.reverse ? 3 - (s & 3) : (s & 3);
    const int prev = s == 0 ? 4 : (A.reverse ? 3 - ((s - 1) & 3) : ((s - 1) & 3));
    const double* R = (s & 1) ? A.xs : A.x;
    double* W = (s & 1) ? A.x : A.xs;
    if (s > 0) {
      if (tid < nd) {
        const unsigned* f = A.flags + (size_t)sdeps[tid] * DF_FLAG_STRIDE;
        const unsigned want = base + (unsigned)s;
        while ((int)(ld_acquire_u32(f) - want) < 0) __nanosleep(A.spin_ns);
      }
      __syncthreads();
    }
    if (tr && tid == 0) tr[4 + 4 * s] = gtimer();
    // copy loads W = R on N_prev \ N_cur (this segment's share) in flight with
    // the x_E gathers of this colour; their stores follow the update rows
    const int pc = prev * 4 + c;
    const int* cl = (const int*)(sdf + H.cp_off[pc]);
    const int ncp = H.ncp[pc];
    constexpr int UC = 4;
    double cv[UC];
    int cn[UC];
#pragma unroll
    for (int u = 0; u < UC; ++u) {
      const int e = tid + u * NT;
      cn[u] = e < ncp ? cl[e] : -1;
      if (cn[u] >= 0) cv[u] = __ldcg(R + cn[u]);
    }
    df_gather<NT, 4, true>((const int2*)(sdf + H.x_off[c]), H.nx[c], R, v);   // x_E of this colour
    __syncthreads();
    if (tr && tid == 0) tr[5 + 4 * s] = gtimer();
    const DfRow* rows = (const DfRow*)(sdf + H.row_off[c]);
    const int nr = H.nrow[c];
    for (int t0 = 0; t0 < 4 * nr; t0 += NT) {
      const int t = t0 + tid, r = t >> 2, h = t & 3;
      double a0 = 0.0, a1 = 0.0;
      int out = 0;
      if (r < nr) {
        const DfRow w = rows[r];
        const int K = w.K, tpr = w.tpr;
        out = w.out;
        if (h < tpr) {
          const double* g = G + w.g;
          const double* vv = v + w.v;
          int cc = h;
          for (; cc + tpr < K; cc += 2 * tpr) {
            a0 = fma(g[cc], vv[cc], a0);
            a1 = fma(g[cc + tpr], vv[cc + tpr], a1);
          }
          if (cc < K) a0 = fma(g[cc], vv[cc], a0);
        }
      }
      double z = a0 + a1;
      z += __shfl_xor_sync(0xffffffffu, z, 2);
      z += __shfl_xor_sync(0xffffffffu, z, 1);
      if (r < nr && h == 0) W[out] = z;
    }
#pragma unroll
    for (int u = 0; u < UC; ++u)
      if (cn[u] >= 0) W[cn[u]] = cv[u];
    if (ncp > UC * NT) df_copy<NT, 4>(cl + UC * NT, ncp - UC * NT, R, W);
    __syncthreads();
    if (tr && tid == 0) tr[6 + 4 * s] = gtimer();
    if (tid == 0) {   // release: orders the CTA's writes (bar.sync above) before the flag at gpu scope
      st_release_u32(A.flags + (size_t)seg * DF_FLAG_STRIDE, base + (unsigned)s + 1u);
      if (tr) tr[7 + 4 * s] = gtimer();
    }
  }
}

namespace host {

// host plan of the dataflow cut sweep of one level
struct DfPlan {
  std::vector<unsigned char> blob;
  std::vector<long long> seg_off;
  std::vector<int> dep_off, deps;
  size_t smem = 0;     // dynamic shared memory of the launch (max blob + v area)
  int nseg = 0;
  int max_dep = 0;
  long long map_bytes = 0;   // the G_j blocks streamed from HBM per launch
};

// desc: the level's cut-patch descriptors (host copy; cut_off[c]..cut_off[c+1]
// = colour c), gmap: host copy of the compressed maps (build_cut_maps),
// L: level geometry.  budget: max bytes of one segment's shared memory,
// tile: segment tile in vertices.  Returns false if a segment needs more
// dependencies than DF_MAXDEP (caller keeps the per-step launches).
template <class Desc>
inline bool df_build(const std::vector<Desc>& desc, const int cut_off[5], const std::vector<double>& gmap,
                     const LevelArgs& L, size_t budget, int tile, DfPlan& out) {
  const int P = L.p, BS = 2 * P + 1, WS = 4 * P + 1, NTC = 128;
  const int np = (int)desc.size();
  if (np == 0) return false;
  struct HP {
    int I, J, c, m, nnz;
    long long g;              // first double of the G rows in gmap
    std::vector<int> nI, nE;  // lattice nodes of the interior / kept exterior columns
  };
  std::vector<HP> hp(np);
  for (int c = 0; c < 4; ++c)
    for (int k = cut_off[c]; k < cut_off[c + 1]; ++k) {
      const Desc& d = desc[k];
      HP& q = hp[k];
      q.I = d.I;
      q.J = d.J;
      q.c = c;
      const long long off = d.map_off & ((1ll << 48) - 1);
      q.nnz = (int)(d.map_off >> 48);
      for (int loc = 0; loc < BS * BS; ++loc)
        if ((d.mask[loc >> 6] >> (loc & 63)) & 1ull)
          q.nI.push_back((P * (d.J - 1) + loc / BS) * L.ld + P * (d.I - 1) + loc % BS);
      q.m = (int)q.nI.size();
      const unsigned char* ix = (const unsigned char*)(gmap.data() + off + 1);
      for (int j = 0; j < q.nnz; ++j) {
        const int w = ix[j];
        q.nE.push_back((P * (d.J - 2) + w / WS) * L.ld + P * (d.I - 2) + w % WS);
      }
      q.g = off + 1 + (q.nnz + 7) / 8;
    }
  // bytes of one patch in the blob (+ its operands in the v area) and the
  // copy-list reserve (interior nodes in two lists, window band)
  auto pbytes = [&](const HP& q) {
    const long long K = q.m + q.nnz;
    return (long long)16 * q.m + 8 * q.m * K + 8 * K + 8 * K + 4 * (2 * q.m + 2 * WS * WS);
  };
  // segments: patches in Morton order of their tile x tile vertex tiles,
  // packed greedily up to the budget (compact groups of neighbouring tiles;
  // the dependencies below are exact for any grouping)
  auto morton = [](unsigned x, unsigned y) {
    unsigned long long m = 0;
    for (int b = 0; b < 16; ++b) m |= ((unsigned long long)((x >> b) & 1) << (2 * b)) | ((unsigned long long)((y >> b) & 1) << (2 * b + 1));
    return m;
  };
  std::vector<int> order(np);
  std::vector<unsigned long long> key(np);
  for (int k = 0; k < np; ++k) {
    order[k] = k;
    key[k] = morton(hp[k].I / tile, hp[k].J / tile);
  }
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return key[a] < key[b]; });
  std::vector<int> seg_of(np, -1);
  std::vector<std::vector<int>> segs;
  {
    long long used = 0;
    for (int k : order) {
      const long long pb = pbytes(hp[k]);
      if (segs.empty() || used + pb > (long long)budget - 512) {
        segs.emplace_back();
        used = 0;
      }
      segs.back().push_back(k);
      seg_of[k] = (int)segs.size() - 1;
      used += pb;
    }
  }
  const int nseg = (int)segs.size();
  // dependencies: segments with a patch within vertex distance 4
  const int NV = L.n + 1;
  std::vector<int> at((size_t)NV * NV, -1);
  for (int k = 0; k < np; ++k) at[(size_t)hp[k].J * NV + hp[k].I] = k;
  out.dep_off.assign(nseg + 1, 0);
  out.deps.clear();
  out.max_dep = 0;
  for (int s = 0; s < nseg; ++s) {
    std::vector<int> ds;
    for (int k : segs[s])
      for (int dj = -4; dj <= 4; ++dj)
        for (int di = -4; di <= 4; ++di) {
          const int I = hp[k].I + di, J = hp[k].J + dj;
          if (I < 0 || J < 0 || I >= NV || J >= NV) continue;
          const int q = at[(size_t)J * NV + I];
          if (q >= 0 && seg_of[q] != s) ds.push_back(seg_of[q]);
        }
    std::sort(ds.begin(), ds.end());
    ds.erase(std::unique(ds.begin(), ds.end()), ds.end());
    if ((int)ds.size() > DF_MAXDEP) return false;
    out.max_dep = std::max(out.max_dep, (int)ds.size());
    out.deps.insert(out.deps.end(), ds.begin(), ds.end());
    out.dep_off[s + 1] = (int)out.deps.size();
  }
  // copy lists: N_prev \ N_cur by the owner of the prev patch; band \ N_cur
  // (prev = 4) by the first patch whose window holds the node
  std::unordered_map<int, int> owner[4];   // interior node -> segment, per colour
  for (int k = 0; k < np; ++k)
    for (int n : hp[k].nI) owner[hp[k].c][n] = seg_of[k];
  std::vector<std::vector<int>> cps((size_t)nseg * 20);
  // only the (prev, cur) pairs of the forward (c = prev + 1) and reverse
  // (c = prev - 1) colour orders occur
  for (int pv = 0; pv < 4; ++pv)
    for (int c = 0; c < 4; ++c) {
      if (c != (pv + 1) % 4 && c != (pv + 3) % 4) continue;
      for (int k = cut_off[pv]; k < cut_off[pv + 1]; ++k)
        for (int n : hp[k].nI)
          if (!owner[c].count(n)) cps[(size_t)seg_of[k] * 20 + pv * 4 + c].push_back(n);
    }
  {
    std::unordered_map<int, int> band;
    std::vector<int> band_nodes;
    for (int k = 0; k < np; ++k)
      for (int w = 0; w < WS * WS; ++w) {
        const int a = P * (hp[k].I - 2) + w % WS, bb = P * (hp[k].J - 2) + w / WS;
        if (a < 0 || bb < 0 || a >= L.nl || bb >= L.nl) continue;
        const int n = bb * L.ld + a;
        if (band.emplace(n, seg_of[k]).second) band_nodes.push_back(n);
      }
    for (int n : band_nodes)
      for (int c : {0, 3})   // first colour of the forward / reverse sweep
        if (!owner[c].count(n)) cps[(size_t)band[n] * 20 + 16 + c].push_back(n);
  }
  // blobs
  out.blob.clear();
  out.seg_off.assign(nseg + 1, 0);
  out.smem = 0;
  out.map_bytes = 0;
  auto align16 = [](size_t x) { return (x + 15) & ~(size_t)15; };
  for (int s = 0; s < nseg; ++s) {
    std::vector<int> byc[4];
    for (int k : segs[s]) byc[hp[k].c].push_back(k);
    DfHdr H;
    std::memset(&H, 0, sizeof(H));
    size_t off = sizeof(DfHdr);
    int vo = 0;
    int vofc[4];
    for (int c = 0; c < 4; ++c) {
      int nr = 0, nx = 0, ng = 0;
      for (int k : byc[c]) {
        nr += hp[k].m;
        nx += hp[k].nnz;
        ng += hp[k].m + hp[k].nnz;
      }
      H.nrow[c] = nr;
      H.row_off[c] = (int)off;
      off = align16(off + 16 * (size_t)nr);
      H.nx[c] = nx;
      H.x_off[c] = (int)off;
      off = align16(off + 8 * (size_t)nx);
      H.nb += nr;
      vofc[c] = vo;
      vo += ng;
    }
    H.b_off = (int)off;
    off = align16(off + 8 * (size_t)H.nb);
    for (int pc = 0; pc < 20; ++pc) {
      H.ncp[pc] = (int)cps[(size_t)s * 20 + pc].size();
      H.cp_off[pc] = (int)off;
      off = align16(off + 4 * (size_t)H.ncp[pc]);
    }
    const size_t gstart = off;
    size_t gsz = 0;
    for (int k : segs[s]) gsz += 8 * (size_t)hp[k].m * (hp[k].m + hp[k].nnz);
    off = align16(gstart + gsz);
    H.blob_bytes = (int)off;
    H.v_doubles = vo;
    const size_t b0 = out.blob.size();
    out.blob.resize(b0 + off, 0);
    unsigned char* B = out.blob.data() + b0;
    size_t gp = gstart;   // byte cursor in the G area
    int2* bl = (int2*)(B + H.b_off);
    int eb = 0;
    for (int c = 0; c < 4; ++c) {
      DfRow* rows = (DfRow*)(B + H.row_off[c]);
      int2* xl = (int2*)(B + H.x_off[c]);
      int r = 0, ex = 0, vbase = vofc[c];
      for (int k : byc[c]) {
        const HP& q = hp[k];
        const int K = q.m + q.nnz;
        const int tpr = q.m * 4 <= NTC ? 4 : (q.m * 2 <= NTC ? 2 : 1);
        if (tpr < 2) return false;   // not reachable for p <= 3
        for (int i = 0; i < q.m; ++i) {
          DfRow& w = rows[r++];
          w.g = (int)(gp / 8) + i * K;
          w.v = vbase;
          w.out = q.nI[i];
          w.K = (short)K;
          w.tpr = (short)tpr;
        }
        // operand [b_I ; x_E] of the patch at v[vbase ..)
        for (int i = 0; i < q.m; ++i) bl[eb++] = make_int2(q.nI[i], vbase + i);
        for (int j = 0; j < q.nnz; ++j) xl[ex++] = make_int2(q.nE[j], vbase + q.m + j);
        vbase += K;
        std::memcpy(B + gp, gmap.data() + q.g, 8 * (size_t)q.m * K);
        gp += 8 * (size_t)q.m * K;
        out.map_bytes += 8 * (long long)q.m * K;
      }
    }
    for (int pc = 0; pc < 20; ++pc)
      if (H.ncp[pc]) std::memcpy(B + H.cp_off[pc], cps[(size_t)s * 20 + pc].data(), 4 * (size_t)H.ncp[pc]);
    std::memcpy(B, &H, sizeof(H));
    out.seg_off[s + 1] = (long long)out.blob.size();
    out.smem = std::max(out.smem, off + 8 * (size_t)vo);
  }
  out.nseg = nseg;
  return true;
}

}  // namespace host
}  // namespace cf
