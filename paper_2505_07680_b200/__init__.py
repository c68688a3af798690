"""paper_2505_07680_b200 -- B200-native multi-level speculative-decoding verification.

The product is ``libmsd.so`` (CUDA for sm_100a behind the C ABI in ``include/msd.h``);
this package is its thin ctypes binding (``api``) plus the seeded input generator
(``synth``).  Importing ``api`` loads ``libmsd.so`` and fails loudly if it is absent:
there is no CPU fallback.
"""
from . import synth  # noqa: F401  (no native dependency)
