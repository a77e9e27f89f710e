"""B200-native data-parallel core of PUMP (arXiv 1607.06886).

Host-side Python mirror of the reference's ``pump`` API over the C ABI of
``libpump_gpu.so`` (include/pump_gpu.h).  The CUDA library is loaded lazily by
``paper_1607_06886_b200.api.lib()``; it fails loudly if the library is
missing — there is no CPU fallback.
"""
__all__ = ["api"]
