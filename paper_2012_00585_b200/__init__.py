"""B200-native FE stiffness assembly (arXiv 2012.00585 hot path): CSR / CRAC scatter-add.

The compute lives in libfea_gpu.so (hand-written sm_100a CUDA behind the C ABI in
include/fea_gpu.h). This package is the Python host side used by bench.py and the tests;
the C++ host side mirroring the reference API is csrc/fea_gpu.hpp.
"""
from .assembly import (STRATEGIES, AssemblyError, FeaError, Plan, exclusive_sum, fill_seeded_k,  # noqa: F401
                       sort_pairs, spmv_crac, spmv_csr)

__all__ = ["Plan", "AssemblyError", "FeaError", "fill_seeded_k", "spmv_csr", "spmv_crac", "STRATEGIES",
           "exclusive_sum", "sort_pairs"]
