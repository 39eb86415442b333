"""B200-native batched projected-gradient-ascent MaxCut (arXiv 2509.18612 hot path).

``libliftcut_b200.so`` (sm_100a CUDA + C++ runtime, C ABI in ``include/liftcut_b200.h``)
does the work; ``liftcut`` mirrors the reference's ``liftcut::`` API on top of it;
``dist`` carries the one-process-per-GPU NCCL plumbing.
"""
from . import liftcut  # noqa: F401
from ._abi import LCB_FP32, LCB_FP64, LIB_PATH, lib  # noqa: F401

__all__ = ["liftcut", "lib", "LIB_PATH", "LCB_FP32", "LCB_FP64"]
