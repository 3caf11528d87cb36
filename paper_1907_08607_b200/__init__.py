"""paper_1907_08607_b200 -- B200-native exact butterfly counting (ParButterfly's
hot path, arXiv 1907.08607) behind a C ABI (include/bf.h, libbf.so).

The product is libbf.so (csrc/*.cu, sm_100a).  ``bf`` is the thin ctypes
binding; import it explicitly (``from paper_1907_08607_b200 import bf``) so that
building does not require the library to exist yet.
"""
__all__ = ["bf"]
