"""B200-native FlexQuant decode engine (arxiv 2506.12024 capabilities, hot path only).

Layout:
  csrc/        CUDA kernels + the C-ABI implementation (libfq_cuda.so, include/fq_cuda.h)
  host/        C++ host library mirroring the reference C++ API (libflexquant_b200.so)
  capi.py      ctypes binding of the C-ABI (tests, bench)
"""
__all__ = ["capi"]
