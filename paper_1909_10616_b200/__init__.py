"""B200-native hot path of arXiv 1909.10616 (G-BFS / N-A2C GEMM-tiling tuners).

The product is the C-ABI library ``libtiletune.so`` (include/tiletune.h) built from ``csrc/``
for sm_100a; ``tiletune`` is its thin ctypes binding and ``dist`` the multi-GPU plumbing
(torch.distributed).  Importing ``tiletune`` raises if the library is missing -- there is no
CPU fallback.
"""
