"""B200-native sharded LAMB step of MegaScale (arXiv 2402.15627): C-ABI library liblamb.so
(include/lamb.h) with hand-written sm_100a kernels, and its Python binding `lamb`.

    from paper_2402_15627_b200 import lamb      # raises if liblamb.so is not built
"""
__all__ = ["lamb", "build"]
