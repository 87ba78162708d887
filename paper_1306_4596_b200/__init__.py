"""B200-native (sm_100a) Schwarz waveform relaxation for the Kolmogorov equation (arXiv 1306.4596).

The product is the C-ABI library ``libkfp.so`` (``include/kfp.h``); ``kfp`` is its
ctypes binding and ``dist`` the one-process-per-GPU driver (torch.distributed / NCCL
for the cross-GPU trace exchange).
"""
from .kfp import KfpError, Problem, load, LIB_PATH  # noqa: F401

__all__ = ["Problem", "KfpError", "load", "LIB_PATH"]
