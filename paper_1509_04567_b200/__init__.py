"""paper_1509_04567_b200 — B200-native (sm_100a, fp64) Paraexp-EBK hot path.

The product is the C-ABI library ``libpexp.so`` (include/pexp.h, sources in csrc/);
``pexp.py`` is its thin ctypes binding.  Importing ``paper_1509_04567_b200.pexp`` fails
loudly when the library is missing: there is no CPU fallback.
"""
__all__ = ["pexp", "build"]
