"""perrk_b200: B200-native (sm_100a, FP64) P-ERRK + entropy-conservative
DGSEM hot path, a drop-in for the reference's Semidiscretization / perk_step
/ run path (arxiv/paper_2507_04991, proj/core).

Compute runs only in libperrk_b200.so (CUDA); see include/perrk_b200.h.
"""
from .capi import PerrkError, lib  # noqa: F401
from .perrk import *  # noqa: F401,F403
from . import perrk, workloads  # noqa: F401
