"""B200-native Sync-Switch (arXiv 2104.08364) synchronization path.

The product is the C-ABI library ``libsyncswitch.so`` (include/syncswitch.h; CUDA sm_100a kernels + NCCL) and the
thin ctypes binding in :mod:`paper_2104_08364_b200.syncswitch`. Build with ``python -m paper_2104_08364_b200.build``.
"""
__all__ = ["syncswitch", "build"]
