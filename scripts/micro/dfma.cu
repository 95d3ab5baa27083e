// latency / throughput probes on this B200: dependent DFMA chain, LDS.64 -> DFMA
// chain, independent DFMA throughput per SM, mbarrier try_wait on a completed
// phase, named barrier of 512 threads.  nvcc -gencode arch=compute_100a,code=sm_100a -o dfma dfma.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_chain(double* out, long long* cyc, int n) {
  double a = threadIdx.x * 1e-3, b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, c);
  long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_lds_chain(double* out, long long* cyc, int n) {
  __shared__ double s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = 1.0 + i * 1e-9;
  __syncthreads();
  double a = 0;
  int idx = threadIdx.x & 7;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    a = fma(s[idx], s[idx + 8], a);
    idx = (idx + 16) & 1023;
  }
  long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) cyc[1] = t1 - t0;
}
__global__ void k_tput(double* out, int n) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 1.0000001, c = 1e-9;
  for (int i = 0; i < n; ++i) {
    a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
    a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void k_bar(long long* cyc, int n) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) asm volatile("bar.sync 1, 512;\n" ::: "memory");
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = t1 - t0;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1 << 26); cudaMalloc(&cyc, 64);
  long long h[4];
  const int n = 4096;
  k_chain<<<1, 32>>>(out, cyc, n);
  k_lds_chain<<<1, 32>>>(out, cyc, n);
  k_bar<<<1, 512>>>(cyc, n);
  cudaMemcpy(h, cyc, 32, cudaMemcpyDeviceToHost);
  printf("dependent DFMA: %.2f cycles; LDS.64x2->DFMA chain: %.2f cycles/iter; bar.sync 512: %.1f cycles\n",
         (double)h[0] / n, (double)h[1] / n, (double)h[2] / n);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int threads : {256, 512, 1024}) {
    k_tput<<<148 * 4, threads>>>(out, 1000);
    cudaEventRecord(e0);
    k_tput<<<148 * 4, threads>>>(out, 20000);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * 20000 * 148 * 4 * threads;
    printf("DFMA throughput (%d thr x 592 CTAs): %.2f TFLOP/s\n", threads, fl / ms / 1e9);
  }
  return 0;
}
