"""B200-native PolyMage-GPU hot path: fused stencil pipelines as warp-overlapped (OTPW) + hybrid-tiled
sm_100a kernels behind the C ABI of include/pmg.h (PAPER.md arXiv 1909.07190, §4-§6).

The package holds only what the path needs: csrc/ (C++ host library + hand-written device header),
libpmg.so (built in-tree) and the ctypes binding.  It never imports oracle/.
"""
from ._binding import EXPORTED, PmgError, lib  # noqa: F401
from .pipeline import (IO, Pipeline, Plan, empty_pitched, gpu_spec, query_gpu_spec, sched_opts,  # noqa: F401
                       selftest_shuffle, weights)

__all__ = ["Pipeline", "Plan", "PmgError", "gpu_spec", "query_gpu_spec", "weights", "sched_opts", "empty_pitched",
           "selftest_shuffle"]
