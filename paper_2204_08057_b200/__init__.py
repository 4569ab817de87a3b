"""B200-native (sm_100a, fp64) Kronecker CG / Sylvester solver of arxiv 2204.08057.

The product is the C-ABI library ``lib/libkroncg.so`` (include/kroncg.h) built from ``csrc/``;
``kroncg`` is its thin ctypes binding.  Import of ``kroncg`` fails loudly when the library is
missing -- there is no CPU fallback.
"""

__all__ = ["kroncg", "sharding"]
