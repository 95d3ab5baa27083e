"""B200-native CutFEM vertex-patch multigrid (arxiv 2508.11608 hot path).

The product is libcutfem_mg.so (C ABI in include/cutfem_mg.h) built from
csrc/ for sm_100a; `cutfem` is its thin ctypes binding.
"""
