#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long gt(){unsigned long long t;asm volatile("mov.u64 %0, %%globaltimer;":"=l"(t));return t;}
__device__ __forceinline__ long long clk(){long long t;asm volatile("mov.u64 %0, %%clock64;":"=l"(t));return t;}
__global__ void k(double* x, unsigned* f, unsigned long long* out, long long* oc){
  // dependent ldcg chain
  int idx = 0; double acc=0;
  unsigned long long t0=gt(); long long c0=clk();
  for(int i=0;i<32;i++){ double v=__ldcg(x+idx); acc+=v; idx = ((int)v + i*4099) & ((1<<20)-1); }
  unsigned long long t1=gt(); long long c1=clk();
  // store + release chain
  for(int i=0;i<32;i++){ x[i*1024]=acc; asm volatile("st.release.gpu.global.u32 [%0], %1;"::"l"(f),"r"(i):"memory"); }
  unsigned long long t2=gt(); long long c2=clk();
  for(int i=0;i<32;i++){ unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];":"=r"(v):"l"(f+32*((i+1)&7)):"memory"); acc+=v; }
  unsigned long long t3=gt(); long long c3=clk();
  for(int i=0;i<32;i++){ x[i*1024]=acc; __threadfence(); }
  unsigned long long t4=gt(); long long c4=clk();
  out[0]=t1-t0; out[1]=t2-t1; out[2]=t3-t2; out[3]=t4-t3; oc[0]=c1-c0; oc[1]=c2-c1; oc[2]=c3-c2; oc[3]=c4-c3; x[5]=acc;
}
int main(){ double* x; unsigned* f; unsigned long long* o; long long* oc;
 cudaMalloc(&x, 8<<20); cudaMemset(x,0,8<<20); cudaMalloc(&f, 4096); cudaMemset(f,0,4096); cudaMallocManaged(&o, 64); cudaMallocManaged(&oc,64);
 for(int r=0;r<3;r++){ k<<<1,1>>>(x,f,o,oc); cudaDeviceSynchronize();
 printf("per op ns: ldcg %.1f  st+st.release %.1f  ld.acquire %.1f  st+threadfence %.1f | cycles: %.0f %.0f %.0f %.0f\n", o[0]/32., o[1]/32., o[2]/32., o[3]/32., oc[0]/32., oc[1]/32., oc[2]/32., oc[3]/32.);}
}
