// Micro-benchmark: dependent-launch latency (graph, with/without PDL) versus
// in-kernel barriers (cluster of 16 CTAs, cooperative grid barrier).
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void k_chain(double* x, int pdl) {
  if (pdl) asm volatile("griddepcontrol.launch_dependents;");
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) x[blockIdx.x] += 1.0;
}

__global__ void __cluster_dims__(16, 1, 1) k_cluster(double* x, int iters) {
  cg::cluster_group cl = cg::this_cluster();
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x == 0) x[blockIdx.x] += 1.0;
    cl.sync();
  }
}

__device__ unsigned g_bar;
__global__ void k_grid(double* x, int iters) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x == 0) x[blockIdx.x] += 1.0;
    g.sync();
  }
}

__global__ void k_cl_chain(double* x, int pdl) {
  if (pdl) asm volatile("griddepcontrol.launch_dependents;");
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) x[blockIdx.x] += 1.0;
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

int main() {
  double* x;
  cudaMalloc(&x, 1 << 20);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int grid : {1, 148, 1184})
    for (int pdl = 0; pdl < 2; ++pdl) {
      cudaGraph_t gr;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
      for (int i = 0; i < 200; ++i) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = 128;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = pdl;
        cudaLaunchKernelEx(&cfg, k_chain, x, pdl);
      }
      cudaStreamEndCapture(s, &gr);
      cudaGraphExec_t ge;
      cudaGraphInstantiate(&ge, gr, 0);
      cudaGraphLaunch(ge, s);
      cudaStreamSynchronize(s);
      cudaEventRecord(a, s);
      for (int r = 0; r < 5; ++r) cudaGraphLaunch(ge, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("chain grid=%d pdl=%d: %.2f us per launch\n", grid, pdl, ms * 1e3 / 1000);
    }
  cudaFuncSetAttribute(k_cl_chain, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(k_cl_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  for (int cs : {8, 16})
    for (int smem : {0, 80 * 1024})
      for (int pdl = 0; pdl < 2; ++pdl) {
        cudaGraph_t gr;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        for (int i = 0; i < 200; ++i) {
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = cs;
          cfg.blockDim = 512;
          cfg.dynamicSmemBytes = smem;
          cfg.stream = s;
          cudaLaunchAttribute at[2];
          at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = cs;
          at[0].val.clusterDim.y = 1;
          at[0].val.clusterDim.z = 1;
          at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[1].val.programmaticStreamSerializationAllowed = 1;
          cfg.attrs = at;
          cfg.numAttrs = 1 + pdl;
          cudaLaunchKernelEx(&cfg, k_cl_chain, x, pdl);
        }
        cudaStreamEndCapture(s, &gr);
        cudaGraphExec_t ge;
        cudaGraphInstantiate(&ge, gr, 0);
        cudaGraphLaunch(ge, s);
        cudaStreamSynchronize(s);
        cudaEventRecord(a, s);
        for (int r = 0; r < 5; ++r) cudaGraphLaunch(ge, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("cluster chain cs=%d smem=%d pdl=%d: %.2f us per launch (%s)\n", cs, smem, pdl, ms * 1e3 / 1000,
               cudaGetErrorString(cudaGetLastError()));
      }
  {
    cudaFuncSetAttribute(k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    k_cluster<<<16, 1024, 0, s>>>(x, 10);
    cudaStreamSynchronize(s);
    cudaEventRecord(a, s);
    k_cluster<<<16, 1024, 0, s>>>(x, 10000);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("cluster16 x1024 barrier: %.3f us; err %s\n", ms * 1e3 / 10000, cudaGetErrorString(cudaGetLastError()));
  }
  for (int grid : {148, 296}) {
    int it = 10000;
    void* args[] = {&x, &it};
    cudaEventRecord(a, s);
    cudaLaunchCooperativeKernel((void*)k_grid, grid, 256, args, 0, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("grid sync %d CTAs: %.3f us; err %s\n", grid, ms * 1e3 / it, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
