// tma.cuh — Tensor Memory Accelerator helpers: 2D tiles of a lattice vector
// (fp64, rows of LD doubles) copied into shared memory by one thread with
// cp.async.bulk.tensor; out-of-range coordinates (negative or past the
// lattice) are zero-filled by the hardware, which gives the halo of boundary
// tiles for free.  The inner start coordinate must be 16-byte aligned (an
// even column for fp64): an odd one traps with an illegal instruction.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "internal.cuh"

namespace cf {

namespace host {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CF_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    require(p != nullptr && q == cudaDriverEntryPointSuccess, ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = (EncodeFn)p;
  }
  return fn;
}

// tensor map of an NL x LD fp64 lattice vector with box (bw columns, bh rows)
inline CUtensorMap lattice_tmap(const double* base, int nl, int ld, int bw, int bh) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)nl};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
  cuuint32_t box[2] = {(cuuint32_t)bw, (cuuint32_t)bh};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)base, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  require(r == CUDA_SUCCESS, ERR_CUDA, "cuTensorMapEncodeTiled failed");
  return m;
}

// tensor map of an NL x NL x LD fp64 3D lattice vector with box (bw, bh, bd)
inline CUtensorMap lattice_tmap3(const double* base, int nl, int ld, int bw, int bh, int bd) {
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)ld, (cuuint64_t)nl, (cuuint64_t)nl};
  cuuint64_t strides[2] = {(cuuint64_t)ld * sizeof(double), (cuuint64_t)ld * nl * sizeof(double)};
  cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, (cuuint32_t)bd};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)base, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  require(r == CUDA_SUCCESS, ERR_CUDA, "cuTensorMapEncodeTiled (3D) failed");
  return m;
}
}  // namespace host

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
// 2D tile (x0, y0) of the tensor map into shared memory, completing on bar
__device__ __forceinline__ void tma_load_2d(void* smem, const CUtensorMap* map, int x0, int y0, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          (unsigned)__cvta_generic_to_shared(smem)),
      "l"(map), "r"(x0), "r"(y0), "r"((unsigned)__cvta_generic_to_shared(bar))
      : "memory");
}

// L2 prefetch of [p, p + bytes) (bulk async, no shared memory); the range is
// widened to 16-byte alignment
__device__ __forceinline__ void prefetch_l2(const void* p, size_t bytes) {
  const size_t a = (size_t)p & ~(size_t)15, e = ((size_t)p + bytes + 15) & ~(size_t)15;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a), "r"((unsigned)(e - a)) : "memory");
}

// 3D box (x0, y0, z0) of the tensor map into shared memory, completing on bar
__device__ __forceinline__ void tma_load_3d(void* smem, const CUtensorMap* map, int x0, int y0, int z0, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          (unsigned)__cvta_generic_to_shared(smem)),
      "l"(map), "r"(x0), "r"(y0), "r"(z0), "r"((unsigned)__cvta_generic_to_shared(bar))
      : "memory");
}

}  // namespace cf
