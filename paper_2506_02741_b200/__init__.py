"""paper_2506_02741_b200 — B200-native hot path of VTGaussian-SLAM (arxiv 2506.02741):
differentiable splatting of view-tied isotropic 3D Gaussians as sm_100a CUDA kernels behind a
C ABI (include/vtgs.h), with this thin ctypes binding (`paper_2506_02741_b200.vtgs`).

Importing the binding loads libvtgs.so; build it with `python -m paper_2506_02741_b200.build`.
"""
__all__ = ["vtgs", "build"]
