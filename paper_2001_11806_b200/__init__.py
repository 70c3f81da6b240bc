"""B200-native fused lattice Boltzmann stream-collide library (arXiv 2001.11806 hot path).

The compute path is the CUDA C-ABI library ``liblbm_b200.so`` (include/lbm.h); ``lbm`` is its
thin ctypes binding. Import ``paper_2001_11806_b200.lbm`` after building with
``python -m paper_2001_11806_b200.build``.
"""
__all__ = ["lbm", "build"]
