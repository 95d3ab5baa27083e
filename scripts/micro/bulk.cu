// per-SM throughput of cp.async.bulk global->shared from L2-resident data:
// one thread issues `ncopy` copies of `bytes` each onto one mbarrier; 148 CTAs
// (one per SM) do the same on disjoint-or-shared sources; cycles per round.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("{\n.reg .pred p;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WAIT_%=;\n}\n" ::"r"(a), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(smem)), "l"(gmem), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}

__global__ void k_bulk(const char* src, long long stride_cta, int bytes, int ncopy, int rounds, long long* out, int lanes, int mis) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    if (threadIdx.x == 0) mbar_expect_tx(&bar, (unsigned)bytes * ncopy);
    __syncwarp();
    if (threadIdx.x < lanes)
      for (int c = threadIdx.x; c < ncopy; c += lanes)
        bulk_g2s(sm + (size_t)c * bytes + mis, src + blockIdx.x * stride_cta + (size_t)((c + r * 7) % 64) * bytes + mis, bytes, &bar);
    mbar_wait(&bar, r & 1);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
  char* src; long long* out;
  cudaMalloc(&src, 256 << 20); cudaMemset(src, 1, 256 << 20); cudaMalloc(&out, 8 * 1024);
  cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  long long h[148];
  struct { int bytes, ncopy, lanes, ctas, mis; } cfg[] = {{3072, 40, 1, 1, 0}, {3072, 40, 1, 148, 0}, {3072, 40, 32, 148, 0}, {3072, 10, 1, 148, 0},
                                                    {16384, 8, 1, 148, 0}, {32768, 4, 1, 148, 0}, {1024, 128, 1, 148, 0}, {1024, 128, 32, 148, 0},
                                                    {24576, 6, 1, 148, 0}, {24576, 6, 1, 148, 16}, {24576, 6, 1, 148, 48}, {3072, 40, 1, 148, 16}};
  for (auto c : cfg) {
    const int rounds = 50;
    k_bulk<<<c.ctas, 32, c.bytes * c.ncopy + 128>>>(src, 0, c.bytes, c.ncopy, 2, out, c.lanes, c.mis);   // warm L2 (shared source)
    k_bulk<<<c.ctas, 32, c.bytes * c.ncopy + 128>>>(src, 0, c.bytes, c.ncopy, rounds, out, c.lanes, c.mis);
    cudaDeviceSynchronize();
    cudaMemcpy(h, out, 8 * c.ctas, cudaMemcpyDeviceToHost);
    double mx = 0, sum = 0;
    for (int i = 0; i < c.ctas; ++i) { mx = h[i] > mx ? h[i] : mx; sum += h[i]; }
    const double cyc = mx / rounds, kb = c.bytes * c.ncopy / 1024.0;
    printf("%3d CTAs, %2d lanes issue %3d x %5d B (%6.1f KB, +%2d B misalign) per round: %7.0f cycles/round (max CTA) = %6.1f B/clk/SM, %.2f us\n",
           c.ctas, c.lanes, c.ncopy, c.bytes, kb, c.mis, cyc, c.bytes * c.ncopy / cyc, cyc / 1965.0);
  }
  return 0;
}
