"""B200-native (sm_100a) SGNS node-embedding training engine -- the hot path of
arXiv 2005.13789 ("A Distributed Multi-GPU System for Large-Scale Node
Embedding at Tencent") behind the C ABI in include/ne.h.

    from paper_2005_13789_b200 import ne     # ctypes binding, same names as ne.h
    from paper_2005_13789_b200.engine import Engine   # convenience wrapper

The CUDA library is libne_b200.so (built by paper_2005_13789_b200/build.py).
"""
from .build import OUT as LIBRARY_PATH  # noqa: F401
