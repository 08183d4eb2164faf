"""B200-native fused multi-LoRA linear layer (tLoRA hot path, arXiv 2602.07263).

The arithmetic lives in libtlora.so (sm_100a tcgen05/TMA kernels behind the C-ABI in
include/tlora.h). This package is the Python mirror of the reference operator API.
"""
from .capi import TloraError, lib  # noqa: F401

__all__ = ["TloraError", "lib"]
