"""B200-native ECHO-3DHPC time-step library (arXiv 1810.04597 hot path).

The product is ``libecho_b200.so`` (C-ABI in include/echo.h, sm_100a kernels in
csrc/); ``paper_1810_04597_b200.echo`` is its ctypes binding.  Build with
``python -m paper_1810_04597_b200.build``.
"""

__all__ = ["echo"]
