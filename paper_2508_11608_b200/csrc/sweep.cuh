// sweep.cuh — the cut sweep of one smoothing step in ONE launch (2D, p <= 3).
//
// The cut part of S(x, b) (P eq. smoother-split l.196-210) is S = 4 n_c
// colour steps over the cut patches; each step reads the state its colour
// starts from (R9) and overwrites the interiors of its patches with the affine
// patch map x_I <- G_j [b_I ; x_E] (R13).  Launching one kernel per step makes
// the sweep a chain of 8 grid-wide dependencies (~3.5 us each at config1).
//
// Here every CTA owns a disjoint set of the "dynamic" nodes (nodes in some
// cut-patch interior) and computes their final values alone: at step s it
// runs the step-s patches of its backward dependency cone (built on the host,
// build_sweep below: the patches whose interior meets the nodes it still needs,
// which need the coupled window nodes after step s-1, ...), on a private copy
// of those nodes in shared memory.  No CTA waits for another between steps;
// patches near an ownership boundary are computed redundantly by both sides
// from identical inputs.  The per-patch arithmetic is k_cut_step7's
// (cut7_main: same row split, accumulation order and shuffle tree), so the
// result is bit-identical to the launch-per-step chain.
//
// Data movement: the CTA's chunk and run lists are bulk-copied into shared
// memory before griddepcontrol.wait (setup data).  A producer warp streams the
// "chunks" through a ring of NCH shared-memory slots with cp.async.bulk (full
// / empty mbarriers): a chunk is the maps of consecutive tasks of one step (as
// 1-2 "runs" of adjacent map blocks: the maps of a colour are stored in angle
// order, and one bulk copy costs ~130 cycles of issue however small), their
// row jobs (one 8-byte record per matrix row: where its map row and input
// vector are, its length and output slot) and, for the first chunk of a step,
// the step's gather list (the slot of every entry of the step's input
// vectors).  The 16 consumer warps: load the slots of x and b (after the
// wait); per step wait for its first chunk, gather v = [b_I ; x_E] of every
// task from the slots, barrier, then the step's rows round-robin over 4-lane
// groups, barrier.  At the end the owned slots are stored to x -- after a
// grid-wide ticket counter says every CTA has read its initial slots (a CTA
// must not overwrite a node another CTA has not loaded yet; the launch is
// cooperative, at most one CTA per SM, so all CTAs are resident).  The
// forward Cartesian sweep before it prefetches the level's maps towards L2.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "smoother2.cuh"
#include "tma.cuh"

namespace cf {

constexpr int SW_MAXS = 16;    // steps per sweep (4 n_c, n_c <= 4)
constexpr int SW_MAXNCH = 8;   // ring slots
constexpr int SW_NW = 16;      // consumer warps per CTA (+ 1 producer warp)

struct SweepRun {         // one bulk copy of adjacent map blocks into a ring slot
  long long src;          // byte offset into gmap (16-byte aligned)
  unsigned dst, bytes;    // slot-relative byte offset, size (multiple of 16)
};
static_assert(sizeof(SweepRun) == 16, "SweepRun is 16 bytes");

struct SweepChunk {       // one ring fill: consecutive tasks of one step
  unsigned run0;          // CTA-relative first run
  unsigned short nrun, nrows;
  unsigned short ngat;    // gather entries (first chunk of a step), else 0
  unsigned short row0;    // rows of the step's earlier chunks (round-robin row assignment)
  unsigned bytes;         // bytes landing in the slot (runs + row jobs + gather list)
  unsigned rj_soff;       // slot-relative offset of [row jobs | gather list] (the aux copy)
  unsigned gat_soff;      // slot-relative offset of the gather list
  long long aux_src;      // byte offset of [row jobs | gather list] in the aux array
};
static_assert(sizeof(SweepChunk) == 32, "SweepChunk is 32 bytes");

// row job (8 bytes): bits 0-15 map row i of a task (the task's map base +
// B i, B = 2 tpr, in doubles from the ring base; layout of map_index), 16-31
// the task's input vector offset (doubles; the vector is stored in the map's
// column-block order, so a lane's two next entries are one 16-byte word),
// 32-39 K, 40-45 m, 46-47 log2 tpr, 48-62 output slot
__host__ __device__ constexpr unsigned long long sweep_rowjob(unsigned goff, unsigned voff, unsigned K, unsigned m,
                                                            unsigned ltpr, unsigned oslot) {
  return (unsigned long long)goff | ((unsigned long long)voff << 16) | ((unsigned long long)K << 32) |
         ((unsigned long long)m << 40) | ((unsigned long long)ltpr << 46) | ((unsigned long long)oslot << 48);
}

struct SweepCta {
  int chunk0, nchunk;     // into the chunk array
  int run0, nrun;         // into the run array
  int slot0, nslot;       // into slot_node
  int own0, nown;         // into own: (slot, lattice node)
  // chunk 0 repeated here, so the producer can issue it before the chunk and
  // run lists have arrived (f_nrun < 0: more runs than fit, issue it later)
  int f_nrun, f_bytes, f_rj_soff, f_pad;
  long long f_aux_src;
  SweepRun f_run[4];
  long long f_pad2;
};
static_assert(sizeof(SweepCta) == 128, "SweepCta is 128 bytes");

struct SweepArgs {
  const SweepCta* cta;
  const SweepChunk* chunk;
  const SweepRun* run;
  const unsigned char* aux;      // per chunk: row jobs (8 B each), then the gather list (u16: slot | 0x8000 if b)
  const int32_t* slot_node;
  const int2* own;
  const double* gmap;
  unsigned long long* gbar;   // launch counter (tickets; all launches of one program have the same grid)
  int S, nch, cb;             // steps, ring slots, ring slot bytes
  int one_lane;               // maps summed one lane per row (map_tpr), else 4-lane groups
  unsigned off_chunk, off_run, off_xs, off_bs, off_v, off_ring;   // shared-memory byte offsets
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}
// bytes (multiple of 16, 16-byte aligned ends) global -> shared, completing on bar
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          (unsigned)__cvta_generic_to_shared(smem)),
      "l"(gmem), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
      : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}

#ifdef CF_TIMING
#define SW_TSTAMP(slot)                                                    \
  do {                                                                     \
    if (threadIdx.x == 0 && blockIdx.x < 8192) {                           \
      unsigned long long t_;                                               \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));               \
      g_dbg[blockIdx.x][slot] = t_;                                        \
    }                                                                      \
  } while (0)
#else
#define SW_TSTAMP(slot) \
  do {                  \
  } while (0)
#endif

// chunk k of the CTA into ring slot k % nch (its runs of adjacent map
// blocks, then its row jobs and gather list), completing on full[k % nch].
// Executed by the whole producer warp: one bulk copy costs ~130 cycles of
// issue even when small, so the copies of a chunk go out from different lanes
// (lane 0 expects the bytes first; lanes 0.. the runs, lane 31 the aux copy)
__device__ __forceinline__ void sweep_fill(const SweepArgs& A, const SweepChunk* CH, const SweepRun* RU, int k,
                                           unsigned char* ring, uint64_t* full, int lane) {
  const SweepChunk& ch = CH[k];
  const int sl = k % A.nch;
  unsigned char* slot = ring + (size_t)sl * A.cb;
  if (lane == 0) mbar_expect_tx(&full[sl], ch.bytes);
  __syncwarp();
  const unsigned char* gm = (const unsigned char*)A.gmap;
  for (int q = lane; q < (int)ch.nrun && lane < 31; q += 31) {
    const SweepRun& r = RU[ch.run0 + q];
    bulk_g2s(slot + r.dst, gm + r.src, r.bytes, &full[sl]);
  }
  if (lane == 31) bulk_g2s(slot + ch.rj_soff, A.aux + ch.aux_src, ch.bytes - ch.rj_soff, &full[sl]);
}

__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;\n" ::"n"(32 * SW_NW) : "memory"); }

// SW_NW consumer warps + one producer warp (the ring fills: bulk copies stall
// the issuing thread, so they do not run on a consumer)
__global__ void __launch_bounds__(32 * (SW_NW + 1), 1) k_cut_sweep(SweepArgs A, double* __restrict__ x,
                                                                   const double* __restrict__ b) {
  extern __shared__ __align__(128) unsigned char swm[];
  uint64_t* full = (uint64_t*)swm;
  uint64_t* empty = full + SW_MAXNCH;
  uint64_t* pbar = empty + SW_MAXNCH;
  __shared__ __align__(16) SweepCta C;
  __shared__ unsigned long long ticket;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int NT = 32 * SW_NW;
  if (tid < (int)(sizeof(SweepCta) / 16)) ((int4*)&C)[tid] = ((const int4*)(A.cta + blockIdx.x))[tid];
  if (tid == 0) {
    for (int k = 0; k < A.nch; ++k) {
      mbar_init(&full[k], 1);
      mbar_init(&empty[k], SW_NW);
    }
    mbar_init(pbar, 1);
  }
  __syncthreads();
  pdl_trigger();
  SweepChunk* CH = (SweepChunk*)(swm + A.off_chunk);
  SweepRun* RU = (SweepRun*)(swm + A.off_run);
  unsigned char* ring = swm + A.off_ring;
  SW_TSTAMP(0);
  if (warp == SW_NW) {   // producer: the program, then every chunk as its ring slot frees up
    const bool early = C.nchunk > 0 && C.f_nrun >= 0;
    if (lane == 0) {
      const unsigned chb = 32u * C.nchunk, rub = 16u * C.nrun;
      mbar_expect_tx(pbar, chb + rub);
      if (chb) bulk_g2s(CH, A.chunk + C.chunk0, chb, pbar);
      if (rub) bulk_g2s(RU, A.run + C.run0, rub, pbar);
      if (early) {   // chunk 0 from the CTA record, without waiting for the lists
        mbar_expect_tx(&full[0], (unsigned)C.f_bytes);
        const unsigned char* gm = (const unsigned char*)A.gmap;
        for (int q = 0; q < C.f_nrun; ++q) bulk_g2s(ring + C.f_run[q].dst, gm + C.f_run[q].src, C.f_run[q].bytes, &full[0]);
        bulk_g2s(ring + C.f_rj_soff, A.aux + C.f_aux_src, (unsigned)(C.f_bytes - C.f_rj_soff), &full[0]);
      }
    }
    mbar_wait(pbar, 0);
    for (int k = early ? 1 : 0; k < C.nchunk; ++k) {
      if (k >= A.nch) mbar_wait(&empty[k % A.nch], ((k / A.nch) - 1) & 1);
#ifdef CF_TIMING
      if (lane == 0 && blockIdx.x == 0 && k < 32) g_dbg[5000 + k / 8][k % 8] = clock64();
#endif
      sweep_fill(A, CH, RU, k, ring, full, lane);
    }
    return;
  }
  double* xs = (double*)(swm + A.off_xs);
  double* bs = (double*)(swm + A.off_bs);
  double* v = (double*)(swm + A.off_v);
  const double* ringd = (const double*)ring;
  pdl_wait();
  for (int i = tid; i < C.nslot; i += NT) {
    const int n = A.slot_node[C.slot0 + i];
    xs[i] = x[n];
    bs[i] = b[n];
  }
  mbar_wait(pbar, 0);
  consumer_sync();
  SW_TSTAMP(1);
  if (tid == 0) {
    __threadfence();
    ticket = atomicAdd(A.gbar, 1ull);
  }
  int s = -1, sl = 0;
  unsigned par = 0;
#ifdef CF_TIMING
  long long tacc[4] = {0, 0, 0, 0}, tq = clock64();
#define SW_LAP(i)                      \
  do {                                 \
    const long long tn_ = clock64();   \
    tacc[i] += tn_ - tq;               \
    tq = tn_;                          \
  } while (0)
#else
#define SW_LAP(i) \
  do {            \
  } while (0)
#endif
  for (int k = 0; k < C.nchunk; ++k) {
    SW_LAP(3);
    mbar_wait(&full[sl], par);
    SW_LAP(0);
#ifdef CF_TIMING
    if (blockIdx.x == 0 && tid == 0 && k < 32) g_dbg[5004 + k / 8][k % 8] = clock64();
#endif
    const SweepChunk& ch = CH[k];
    const unsigned char* slot = ring + (size_t)sl * A.cb;
    if (ch.ngat) {   // first chunk of a step: v = [b_I ; x_E] of its tasks, from the state after the previous step
      ++s;
      if (s == 1) SW_TSTAMP(2);
      if (s == A.S / 2) SW_TSTAMP(3);
      if (k) consumer_sync();   // the previous step's rows are done (they read v, write xs)
      const uint16_t* gl = (const uint16_t*)(slot + ch.gat_soff);
      const int ng = ch.ngat;
      // four independent entries per thread and round (loads before stores:
      // the smem latency is paid once per round, not per entry)
      for (int e0 = tid; e0 < ng; e0 += 4 * NT) {
        unsigned src[4];
        double val[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) src[u] = e0 + u * NT < ng ? gl[e0 + u * NT] : 0u;
#pragma unroll
        for (int u = 0; u < 4; ++u) val[u] = (src[u] & 0x8000u) ? bs[src[u] & 0x7fffu] : xs[src[u]];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (e0 + u * NT < ng) v[e0 + u * NT] = val[u];
      }
      consumer_sync();
    }
    SW_LAP(1);
    const unsigned long long* rj = (const unsigned long long*)(slot + ch.rj_soff);
    const int nrows = ch.nrows, row0 = ch.row0;
    if (A.one_lane) {
      // one lane per row (large levels), round-robin over the step: thread t
      // takes the step's rows congruent to t mod NT (columns 2j into a0c,
      // 2j + 1 into a1c, one 16-byte read of the map pair and of v per pair)
      const int first = row0 - ((row0 - tid) % NT + NT) % NT;
      for (int R = first - row0; R < nrows; R += NT) {
        if (R < 0) continue;
        const unsigned long long job = rj[R];
        const int K = (int)((job >> 32) & 0xffu), m = (int)((job >> 40) & 0x3fu);
        const double* g = ringd + (unsigned)(job & 0xffffu);
        const double* q = v + (unsigned)((job >> 16) & 0xffffu);
        double a0c = 0.0, a1c = 0.0;
        int c = 0;
#pragma unroll 4
        for (; c + 1 < K; c += 2, g += 2 * m, q += 2) {
          const double2 gg = *(const double2*)g, vv = *(const double2*)q;
          a0c = fma(gg.x, vv.x, a0c);
          a1c = fma(gg.y, vv.y, a1c);
        }
        if (c < K) a0c = fma(g[0], q[0], a0c);
        xs[(unsigned)(job >> 48)] = a0c + a1c;
      }
    } else {
      // rows over 4-lane groups, round-robin over the step (group warp*8 + lane/4
      // takes the step's rows congruent to it mod NT/4; warp-uniform trip count:
      // every lane reaches the shuffles).  x_I^new[i] = G_j[i,:] v in cut7_main's
      // order (lane h: columns h + 2 tpr j into a0c, h + tpr + 2 tpr j into a1c)
      // and shuffle tree: bit-identical to k_cut_step7
      const int first = row0 - ((row0 - warp * 8) % (NT / 4) + (NT / 4)) % (NT / 4);
      for (int Rb = first; Rb < row0 + nrows; Rb += NT / 4) {
        const int R = Rb + (lane >> 2) - row0;
        const bool act = R >= 0 && R < nrows;
        const unsigned long long job = act ? rj[R] : 0ull;
        const int K = (int)((job >> 32) & 0xffu), m = (int)((job >> 40) & 0x3fu);
        const int tpr = 1 << (int)((job >> 46) & 3u), h = lane & 3, B = 2 * tpr;
        const double* g = ringd + (unsigned)(job & 0xffffu) + 2 * h;
        const double* q = v + (unsigned)((job >> 16) & 0xffffu) + 2 * h;
        double a0c = 0.0, a1c = 0.0;
        if (act && h < tpr) {
          int c = h;
#pragma unroll 4
          for (; c + tpr < K; c += B, g += B * m, q += B) {
            const double2 gg = *(const double2*)g, vv = *(const double2*)q;
            a0c = fma(gg.x, vv.x, a0c);
            a1c = fma(gg.y, vv.y, a1c);
          }
          if (c < K) a0c = fma(g[0], q[0], a0c);
        }
        double z = a0c + a1c;
        const double z2 = __shfl_xor_sync(0xffffffffu, z, 2, 4);
        if (tpr == 4) z += z2;
        const double z1 = __shfl_xor_sync(0xffffffffu, z, 1, 4);
        if (tpr >= 2) z += z1;
        if (act && h == 0) xs[(unsigned)(job >> 48)] = z;
      }
    }
    SW_LAP(2);
    __syncwarp();
#ifdef CF_TIMING
    if (blockIdx.x == 0 && tid == 0 && k < 32) g_dbg[5008 + k / 8][k % 8] = clock64();
#endif
    if (lane == 0) mbar_arrive(&empty[sl]);
    if (++sl == A.nch) {
      sl = 0;
      par ^= 1u;
    }
  }
  consumer_sync();
#ifdef CF_TIMING
  if (tid == 0 && blockIdx.x < 4096) {
    for (int i = 0; i < 4; ++i) g_dbg[4096 + blockIdx.x][i] = tacc[i];
    g_dbg[4096 + blockIdx.x][4] = C.nchunk;
    g_dbg[4096 + blockIdx.x][5] = C.nrun;
    unsigned tot = 0;
    for (int k = 0; k < C.nchunk; ++k) tot += CH[k].bytes;
    g_dbg[4096 + blockIdx.x][6] = tot;
  }
#endif
  SW_TSTAMP(4);
  // every CTA has read its initial slots before any owned node is stored
  if (tid == 0) {
    const unsigned long long G = gridDim.x, target = (ticket / G + 1) * G;
    while (ld_acquire_u64(A.gbar) < target) __nanosleep(64);
  }
  consumer_sync();
  SW_TSTAMP(5);
  for (int i = tid; i < C.nown; i += NT) {
    const int2 o = A.own[C.own0 + i];
    x[o.y] = xs[o.x];
  }
  SW_TSTAMP(6);
}

// setup: the exterior window indices of every patch map (header of the block), WW bytes per patch
__global__ void k_map_idx(const CutDesc* desc, int np, const double* gmap, int WW, uint8_t* out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= np) return;
  const CutDesc d = desc[k];
  if (d.map_off < 0) return;
  const int nnz = (int)(d.map_off >> 48);
  const uint8_t* ix = (const uint8_t*)(gmap + (d.map_off & ((1ll << 48) - 1)) + 2);
  for (int j = 0; j < nnz && j < WW; ++j) out[(size_t)k * WW + j] = ix[j];
}

// ------------------------------------------------------------------ host
namespace host {

// One cut patch as the sweep builder sees it (2D, lattice node indices).
struct SweepPatch {
  int I, J, colour;
  std::vector<int> in;    // interior nodes, in map row order
  std::vector<int> ex;    // coupled exterior window nodes, in map column order
  long long blk0, rows, blk1;   // map block [blk0, blk1) in gmap (doubles), its rows at `rows`
};

// The built program of one level and direction (host arrays, uploaded by the caller).
struct SweepProgram {
  bool ok = false;
  std::string why;
  int S = 0, nch = 0, cb = 0, ncta = 0;
  size_t smem = 0;
  std::vector<SweepCta> cta;
  std::vector<SweepChunk> chunk;
  std::vector<SweepRun> run;
  std::vector<unsigned char> aux;
  std::vector<int32_t> slot_node;
  std::vector<int2> own;
  unsigned off_chunk = 0, off_run = 0, off_xs = 0, off_bs = 0, off_v = 0, off_ring = 0;
  double est_us = 0, redundancy = 0;
  long long map_bytes_total = 0, map_bytes_max = 0;
};

inline unsigned long long hilbert_d(unsigned nside, unsigned x, unsigned y) {
  unsigned long long d = 0;
  for (unsigned s = nside / 2; s > 0; s /= 2) {
    const unsigned rx = (x & s) > 0, ry = (y & s) > 0;
    d += (unsigned long long)s * s * ((3 * rx) ^ ry);
    if (ry == 0) {
      if (rx == 1) {
        x = s - 1 - x;
        y = s - 1 - y;
      }
      std::swap(x, y);
    }
  }
  return d;
}

// Cone of one CTA: owned dynamic nodes -> per step the patch ids (sorted).
// need_{S} = owned; T_s = patches of colour c_s whose interior meets need_{s+1};
// need_s = (need_{s+1} \ interiors(T_s)) u (exterior nodes of T_s that are dynamic).
inline std::vector<std::vector<int>> sweep_cone(const std::vector<SweepPatch>& P,
                                                const std::unordered_map<int, std::vector<int>>& node_patches,
                                                const std::vector<int>& owned, int S, int reverse) {
  std::vector<std::vector<int>> steps(S);
  std::unordered_map<int, char> need;
  for (int n : owned) need[n] = 1;
  for (int s = S - 1; s >= 0; --s) {
    const int c = reverse ? 3 - (s & 3) : (s & 3);
    std::vector<int>& Ts = steps[s];
    for (auto& kv : need) {
      auto it = node_patches.find(kv.first);
      if (it == node_patches.end()) continue;
      for (int k : it->second)
        if (P[k].colour == c) Ts.push_back(k);
    }
    std::sort(Ts.begin(), Ts.end());
    Ts.erase(std::unique(Ts.begin(), Ts.end()), Ts.end());
    for (int k : Ts)
      for (int n : P[k].in) need.erase(n);
    for (int k : Ts)
      for (int n : P[k].ex)
        if (node_patches.count(n)) need[n] = 1;
  }
  return steps;
}

// Build the one-launch sweep program of one level and direction.
//   P: the cut patches with maps (nodes = b * ld + a); n, p, ld: the level;
//   S = 4 n_c; nsm: SMs; smem_max: opt-in shared memory per block;
//   force_ng > 0 forces the CTA count; (ca, cb): the level-set centre in
//   lattice coordinates; [own_b0, own_b1): the owned lattice rows of a slab
//   partition (the CTAs own the dynamic nodes there; their cones reach into
//   the wide halo, which the exchange before the launch makes valid).
// Ownership: the dynamic nodes are ordered by their angle about the level-set
// centre and cut into contiguous runs of equal work (the map doubles of their
// patches, shared among the patch interior's nodes); a run is one CTA.  The
// cut band is a closed curve around the centre, so these are arcs of it, the
// split with the smallest dependency cones (scripts/cone_study.py: x2.0 map
// bytes at 139 CTAs on config1, x2.5 for Hilbert-ordered 4x4-cell atoms).
// The CTA count minimises an estimate of the sweep time: the largest cone's
// map bytes / per-SM shared-memory throughput + all cones' bytes / L2 bandwidth.
// The chosen split: per CTA its owned dynamic nodes and, per step, the
// patches of its dependency cone.
struct SweepPlan {
  int ng = 0;
  std::vector<std::vector<int>> owned;
  std::vector<std::vector<std::vector<int>>> cones;
  long long tot = 0, mx = 0;
  double est = 1e30;
};

inline SweepProgram build_sweep(const std::vector<SweepPatch>& P, int n, int p, int ld, int S, int reverse,
                                int nsm, size_t smem_max, int force_ng, bool verbose, double ca, double cb,
                                int own_b0 = -1, int own_b1 = -1, int one_lane = 0, SweepPlan* plan_out = nullptr) {
  SweepProgram R;
  R.S = S;
  if (S > SW_MAXS) {
    R.why = "n_c > 4";
    return R;
  }
  std::unordered_map<int, std::vector<int>> node_patches;   // dynamic node -> patches with it in their interior
  for (int k = 0; k < (int)P.size(); ++k)
    for (int nd : P[k].in) node_patches[nd].push_back(k);
  if (node_patches.empty()) {
    R.why = "no cut patch interiors";
    return R;
  }
  auto map_d = [&](int k) { return map_rows_d((int)P[k].in.size(), (int)(P[k].in.size() + P[k].ex.size()), one_lane); };
  auto kp_of = [&](int k) {
    return (long long)map_kp((int)P[k].in.size(), (int)(P[k].in.size() + P[k].ex.size()), one_lane);
  };
  // dynamic nodes by angle, with their work
  std::vector<std::pair<double, int>> byang;
  std::unordered_map<int, double> work;
  for (int k = 0; k < (int)P.size(); ++k)
    for (int nd : P[k].in) work[nd] += (double)map_d(k) / P[k].in.size();
  for (auto& kv : node_patches)   // (slab partition: only the nodes of the owned lattice rows)
    if (own_b0 < 0 || (kv.first / ld >= own_b0 && kv.first / ld < own_b1))
      byang.push_back({std::atan2((kv.first / ld) - cb, (kv.first % ld) - ca), kv.first});
  if (byang.empty()) {
    R.why = "no owned cut-patch interior nodes";
    return R;
  }
  std::sort(byang.begin(), byang.end());

  using Plan = SweepPlan;
  // split the angle-ordered nodes into ng arcs of equal weight (wt: per-node
  // weights, indexed like byang)
  auto make_plan = [&](int ng, const std::vector<double>& wt) {
    Plan pl;
    pl.owned.assign(ng, {});
    double acc = 0, tot = 0;
    for (double w : wt) tot += w;
    for (size_t i = 0; i < byang.size(); ++i) {
      const double w = wt[i];
      const int g = (int)std::min<double>(ng - 1, std::floor((acc + 0.5 * w) / tot * ng));
      acc += w;
      pl.owned[g].push_back(byang[i].second);
    }
    pl.owned.erase(std::remove_if(pl.owned.begin(), pl.owned.end(), [](const std::vector<int>& v) { return v.empty(); }),
                   pl.owned.end());
    pl.ng = (int)pl.owned.size();
    for (auto& o : pl.owned) {
      pl.cones.push_back(sweep_cone(P, node_patches, o, S, reverse));
      long long b = 0;
      for (auto& st : pl.cones.back())
        for (int k : st) b += 8 * map_d(k);
      pl.tot += b;
      pl.mx = std::max(pl.mx, b);
    }
    // the largest cone passes through one SM's shared memory twice (bulk copy in,
    // row reads out): per-SM bound; the sum over CTAs is L2 traffic (measured on
    // config1: 148 CTAs (x2.1) 30.7 us beat 92 CTAs (x1.7) 34.8 us)
    pl.est = (pl.mx / 60e9 + pl.tot / 40e12) * 1e6;
    return pl;
  };
  std::vector<double> wt0(byang.size());
  for (size_t i = 0; i < byang.size(); ++i) wt0[i] = work[byang[i].second];
  // equal own work leaves the cones unequal (an arc's cone also covers its
  // neighbourhood); rebalance: scale each arc's node weights by its cone bytes
  // over the mean and split again, keeping the plan with the smallest largest cone
  auto balanced_plan = [&](int ng) {
    std::vector<double> wt = wt0;
    Plan bestp = make_plan(ng, wt);
    for (int it = 0; it < 3 && bestp.ng > 1; ++it) {
      const Plan& cur = bestp;
      const double mean = (double)cur.tot / cur.ng;
      std::unordered_map<int, double> f;
      for (int g = 0; g < cur.ng; ++g) {
        long long b = 0;
        for (auto& st : cur.cones[g])
          for (int k : st) b += 8 * map_d(k);
        for (int nd : cur.owned[g]) f[nd] = std::sqrt(b / mean);   // damped
      }
      for (size_t i = 0; i < byang.size(); ++i) wt[i] *= f[byang[i].second];
      Plan pl = make_plan(ng, wt);
      if (pl.mx < bestp.mx) bestp = std::move(pl);
      else break;
    }
    return bestp;
  };
  Plan best;
  std::vector<int> cands;
  if (force_ng > 0) cands.push_back(std::min(force_ng, nsm));
  else {
    // (large levels: few CTAs are never competitive -- every level with more
    // than 10 nsm patches chose >= 92 of 148 -- and their cones are the costliest
    // to build, so the search starts at nsm / 4)
    const int g0 = P.size() > 10 * (size_t)nsm ? std::max(1, nsm / 4) : 1;
    for (int g = g0; g < nsm; g = g * 3 / 2 + 1) cands.push_back(g);
    cands.push_back(nsm);
  }
  long long once = 0;
  for (int k = 0; k < (int)P.size(); ++k) once += 8 * map_d(k) * (S / 4);
  std::vector<std::pair<double, int>> ranked;   // (estimate, CTA count) of the plain splits
  for (int g : cands) {
    if (g > (int)byang.size() && g != cands.front()) continue;
    Plan pl = make_plan(g, wt0);
    if (verbose)
      std::fprintf(stderr, "[cutfem] sweep plan n=%d dir=%d: %d CTAs, cone map bytes max %.0f KB total %.1f MB (x%.2f), est %.2f us\n",
                   n, reverse, pl.ng, pl.mx / 1e3, pl.tot / 1e6, (double)pl.tot / std::max(1ll, once), pl.est);
    ranked.push_back({pl.est, g});
    if (pl.est < best.est) best = std::move(pl);
  }
  // the two best CTA counts and the full device with their arcs rebalanced;
  // the best of them is kept
  std::sort(ranked.begin(), ranked.end());
  std::vector<int> tryb;
  for (size_t r = 0; r < ranked.size() && r < 2; ++r) tryb.push_back(ranked[r].second);
  if (force_ng <= 0 && std::find(tryb.begin(), tryb.end(), nsm) == tryb.end() && nsm <= (int)byang.size())
    tryb.push_back(nsm);
  // (within 3 % of the best estimate and at most 15 % more map bytes, the plan
  // with more CTAs is taken: measured faster than the model says, e.g. config1
  // 148 vs 128 CTAs: 26.6 vs 28.7 us)
  for (int gb : tryb) {
    Plan pl = balanced_plan(gb);
    if (verbose)
      std::fprintf(stderr, "[cutfem] sweep plan n=%d dir=%d: %d CTAs rebalanced, cone max %.0f KB, est %.2f us\n", n,
                   reverse, pl.ng, pl.mx / 1e3, pl.est);
    if (pl.est < 0.97 * best.est || (pl.est <= 1.03 * best.est && pl.ng > best.ng && pl.tot <= 1.15 * best.tot))
      best = std::move(pl);
  }
  if (plan_out) *plan_out = best;
  const int ng = best.ng;
  R.ncta = ng;
  R.est_us = best.est;
  R.map_bytes_total = best.tot;
  R.map_bytes_max = best.mx;
  R.redundancy = (double)best.tot / std::max(1ll, once);
  auto r16 = [](long long v) { return (v + 15) & ~15ll; };
  const long long GAP = 2048;   // bridge gaps of up to this many bytes between map blocks of one run

  // per CTA: tasks per step sorted by map position, slots (owned nodes first)
  struct Tmp {
    std::vector<std::vector<int>> steps;
    std::vector<int> slots;
    std::unordered_map<int, int> slot_of;
  };
  std::vector<Tmp> tmp(ng);
  size_t mx_slot = 0, mx_v = 0;
  long long mx_gat = 0, mx_one = 0;
  for (int g = 0; g < ng; ++g) {
    Tmp& t = tmp[g];
    auto slot = [&](int nd) {
      auto it = t.slot_of.find(nd);
      if (it != t.slot_of.end()) return it->second;
      const int sl = (int)t.slots.size();
      t.slot_of[nd] = sl;
      t.slots.push_back(nd);
      return sl;
    };
    for (int nd : best.owned[g]) slot(nd);
    t.steps = best.cones[g];
    for (int s = 0; s < S; ++s) {
      std::sort(t.steps[s].begin(), t.steps[s].end(), [&](int a2, int b2) { return P[a2].blk0 < P[b2].blk0; });
      size_t nv = 0;
      for (int k : t.steps[s]) {
        nv += (size_t)kp_of(k);
        for (int nd : P[k].in) slot(nd);
        for (int nd : P[k].ex) slot(nd);
        mx_one = std::max<long long>(mx_one, 8 * (P[k].blk1 - P[k].blk0) + r16(8 * (long long)P[k].in.size()));
      }
      mx_v = std::max(mx_v, nv);
      mx_gat = std::max<long long>(mx_gat, r16(2ll * nv));
    }
    if (t.slots.size() > 32767 || mx_v > 65535) {
      R.why = "a CTA needs more than 32767 slots or 65535 vector entries";
      return R;
    }
    mx_slot = std::max(mx_slot, t.slots.size());
  }
  // ring slots: the largest of 96, 80, 64, 48, 32 KB for which two slots fit
  // (large slots: about one chunk per step, the fewest fills; config1 cut sweep
  // 24.7 us with 6 x 32 KB, 21.8 us with 2 x 96 KB; env CUTFEM_SWEEP_CB_KB fixes it)
  const long long need = (mx_one + mx_gat + 127) & ~127ll;
  std::vector<long long> cb_try = {96 * 1024, 80 * 1024, 64 * 1024, 48 * 1024, 32 * 1024};
  if (const char* e = std::getenv("CUTFEM_SWEEP_CB_KB")) cb_try = {std::max(8, std::atoi(e)) * 1024ll};
  // chunks: consecutive tasks of one step whose runs, row jobs and (first chunk)
  // gather list fit one ring slot; runs: adjacent map blocks (gaps <= GAP bridged)
  struct TmpRun {
    long long b0, b1;   // doubles
  };
  struct TmpChunk {
    int step, t0, nt;   // tasks t0.. of the step's sorted list
    std::vector<TmpRun> runs;
    long long run_bytes = 0, rows = 0;
    bool first = false;
  };
  std::vector<std::vector<TmpChunk>> chunks;
  auto al = [](size_t v, size_t a2) { return (v + a2 - 1) / a2 * a2; };
  const size_t static_smem = 1024;   // __shared__ SweepCta + ticket, margin
  size_t o = 0, mx_chunk = 0, mx_run = 0;
  bool fits = false;
  for (long long cbt : cb_try) {
    R.cb = (int)std::max<long long>(cbt, need);
    chunks.assign(ng, {});
    mx_chunk = 0;
    mx_run = 0;
    for (int g = 0; g < ng; ++g) {
      Tmp& t = tmp[g];
      size_t nrun = 0;
      for (int s = 0; s < S; ++s) {
        const std::vector<int>& st = t.steps[s];
        long long nv = 0;
        for (int k : st) nv += kp_of(k);
        const long long gb = r16(2 * nv);
        TmpChunk cur;
        cur.step = s;
        cur.t0 = 0;
        cur.nt = 0;
        cur.first = true;
        for (int i = 0; i < (int)st.size(); ++i) {
          const int k = st[i];
          const long long kb0 = P[k].blk0, kb1 = P[k].blk1;
          // bytes if appended: extend the last run or open a new one
          const bool extend = !cur.runs.empty() && kb0 >= cur.runs.back().b1 && 8 * (kb0 - cur.runs.back().b1) <= GAP;
          const long long add = extend ? 8 * (kb1 - cur.runs.back().b1) : 8 * (kb1 - kb0);
          const long long used = cur.run_bytes + add + r16(8 * (cur.rows + (long long)P[k].in.size())) + (cur.first ? gb : 0);
          if (cur.nt && used > R.cb) {
            nrun += cur.runs.size();
            chunks[g].push_back(cur);
            TmpChunk nx;
            nx.step = s;
            nx.t0 = i;
            nx.nt = 0;
            cur = nx;
          }
          const bool ext2 = !cur.runs.empty() && kb0 >= cur.runs.back().b1 && 8 * (kb0 - cur.runs.back().b1) <= GAP;
          if (ext2) {
            cur.run_bytes += 8 * (kb1 - cur.runs.back().b1);
            cur.runs.back().b1 = kb1;
          } else {
            cur.runs.push_back({kb0, kb1});
            cur.run_bytes += 8 * (kb1 - kb0);
          }
          if (!cur.nt) cur.t0 = i;
          ++cur.nt;
          cur.rows += (long long)P[k].in.size();
        }
        if (cur.nt) {
          nrun += cur.runs.size();
          chunks[g].push_back(cur);
        }
      }
      mx_chunk = std::max(mx_chunk, chunks[g].size());
      mx_run = std::max(mx_run, nrun);
    }
    // shared-memory layout: barriers | chunks | runs | xs | bs | v | ring
    o = 256;
    R.off_chunk = (unsigned)o;
    o = al(o + 32 * mx_chunk, 128);
    R.off_run = (unsigned)o;
    o = al(o + 16 * mx_run, 128);
    R.off_xs = (unsigned)o;
    o = al(o + 8 * mx_slot, 128);
    R.off_bs = (unsigned)o;
    o = al(o + 8 * mx_slot, 128);
    R.off_v = (unsigned)o;
    o = al(o + 8 * mx_v, 128);
    R.off_ring = (unsigned)o;
    if (o + static_smem + 2 * (size_t)R.cb <= smem_max && 2 * (size_t)R.cb / 8 <= 65535) {
      fits = true;
      break;
    }
  }
  if (!fits) {
    R.why = "shared memory: program + two ring slots exceed the per-block limit";
    return R;
  }
  R.nch = (int)std::min<size_t>(SW_MAXNCH, (smem_max - static_smem - o) / R.cb);
  while (R.nch > 2 && (size_t)R.nch * R.cb / 8 > 65535) --R.nch;   // 16-bit row offsets from the ring base
  R.smem = o + (size_t)R.nch * R.cb;
  // emit
  for (int g = 0; g < ng; ++g) {
    Tmp& t = tmp[g];
    SweepCta c = {};
    c.chunk0 = (int)R.chunk.size();
    c.nchunk = (int)chunks[g].size();
    c.run0 = (int)R.run.size();
    c.slot0 = (int)R.slot_node.size();
    c.nslot = (int)t.slots.size();
    c.own0 = (int)R.own.size();
    c.nown = (int)best.owned[g].size();
    std::vector<unsigned> voff;
    size_t step_rows = 0;
    int cur_step = -1;
    for (int ci = 0; ci < (int)chunks[g].size(); ++ci) {
      const TmpChunk& tc = chunks[g][ci];
      const std::vector<int>& st = t.steps[tc.step];
      if (tc.step != cur_step) {   // input-vector offsets of the step's tasks
        cur_step = tc.step;
        voff.assign(st.size(), 0);
        unsigned vo = 0;
        for (int i = 0; i < (int)st.size(); ++i) {
          voff[i] = vo;
          vo += (unsigned)kp_of(st[i]);
        }
      }
      const unsigned slot_base = (unsigned)((size_t)(ci % R.nch) * R.cb);   // from the ring base
      SweepChunk ch = {};
      ch.run0 = (unsigned)(R.run.size() - c.run0);
      ch.nrun = (unsigned short)tc.runs.size();
      unsigned off = 0;
      std::vector<std::pair<long long, unsigned>> run_dst;   // (b0 doubles, slot byte offset)
      for (const TmpRun& r : tc.runs) {
        SweepRun sr;
        sr.src = 8 * r.b0;
        sr.dst = off;
        sr.bytes = (unsigned)(8 * (r.b1 - r.b0));
        run_dst.push_back({r.b0, off});
        R.run.push_back(sr);
        off += sr.bytes;
      }
      // row jobs
      std::vector<unsigned long long> rows;
      for (int i = tc.t0; i < tc.t0 + tc.nt; ++i) {
        const int k = st[i];
        unsigned dst = 0;
        for (size_t q = 0; q < tc.runs.size(); ++q)
          if (P[k].blk0 >= tc.runs[q].b0 && P[k].blk1 <= tc.runs[q].b1)
            dst = run_dst[q].second + (unsigned)(8 * (P[k].rows - tc.runs[q].b0));
        const unsigned m = (unsigned)P[k].in.size(), K = (unsigned)(m + P[k].ex.size());
        const unsigned tpr = (unsigned)map_tpr((int)m, one_lane), ltpr = tpr == 4 ? 2 : (tpr == 2 ? 1 : 0);
        for (unsigned r = 0; r < m; ++r)
          rows.push_back(sweep_rowjob((slot_base + dst) / 8 + 2 * tpr * r, voff[i], K, m, ltpr,
                                      (unsigned)t.slot_of[P[k].in[r]]));
      }
      ch.nrows = (unsigned short)rows.size();
      if (tc.first) step_rows = 0;
      ch.row0 = (unsigned short)step_rows;
      step_rows += rows.size();
      ch.rj_soff = off;
      const size_t aux0 = R.aux.size();
      ch.aux_src = (long long)aux0;
      R.aux.resize(aux0 + r16(8 * (long long)rows.size()), 0);
      std::memcpy(R.aux.data() + aux0, rows.data(), 8 * rows.size());
      off += (unsigned)r16(8 * (long long)rows.size());
      if (tc.first) {
        // each task's v in the map's column-block order (map_index): position
        // B j + 2 h + e holds column B j + h + e tpr; padding positions read slot 0
        std::vector<uint16_t> gl;
        for (int i = 0; i < (int)st.size(); ++i) {
          const int k = st[i];
          const int m = (int)P[k].in.size(), K = m + (int)P[k].ex.size(), tpr = map_tpr(m, one_lane), B = 2 * tpr;
          for (int pos = 0; pos < (int)kp_of(k); ++pos) {
            const int c = B * (pos / B) + (pos % B) / 2 + ((pos % B) % 2) * tpr;
            if (c >= K) gl.push_back(0);
            else if (c < m) gl.push_back((uint16_t)(t.slot_of[P[k].in[c]] | 0x8000));
            else gl.push_back((uint16_t)t.slot_of[P[k].ex[c - m]]);
          }
        }
        if (gl.size() > 65535) {
          R.why = "a step's gather list exceeds 65535 entries";
          return R;
        }
        ch.ngat = (unsigned short)gl.size();
        ch.gat_soff = off;
        const size_t a1 = R.aux.size();
        R.aux.resize(a1 + r16(2ll * gl.size()), 0);
        std::memcpy(R.aux.data() + a1, gl.data(), 2 * gl.size());
        off += (unsigned)r16(2ll * gl.size());
      }
      ch.bytes = off;
      if (off > (unsigned)R.cb || ch.nrows != rows.size()) {
        R.why = "internal: chunk exceeds the ring slot";
        return R;
      }
      R.chunk.push_back(ch);
    }
    c.nrun = (int)(R.run.size() - c.run0);
    c.f_nrun = -1;
    if (c.nchunk) {
      const SweepChunk& f0 = R.chunk[c.chunk0];
      if (f0.nrun <= 4) {
        c.f_nrun = f0.nrun;
        for (int q = 0; q < (int)f0.nrun; ++q) c.f_run[q] = R.run[c.run0 + f0.run0 + q];
        c.f_bytes = (int)f0.bytes;
        c.f_rj_soff = (int)f0.rj_soff;
        c.f_aux_src = f0.aux_src;
      }
    }
    R.slot_node.insert(R.slot_node.end(), t.slots.begin(), t.slots.end());
    for (int i = 0; i < c.nown; ++i) R.own.push_back(make_int2(i, best.owned[g][i]));   // owned nodes are slots 0..nown-1
    R.cta.push_back(c);
  }
  R.aux.resize(R.aux.size() + 16, 0);
  if (verbose)
    std::fprintf(stderr, "[cutfem] sweep n=%d dir=%d: %d CTAs, smem %zu B (ring %d x %d B), chunks max %zu, runs max %zu, "
                 "slots max %zu, redundancy %.2f\n", n, reverse, ng, R.smem, R.nch, R.cb, mx_chunk, mx_run, mx_slot,
                 R.redundancy);
  R.ok = true;
  return R;
}

}  // namespace host
}  // namespace cf
