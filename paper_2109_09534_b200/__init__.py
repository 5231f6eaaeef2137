"""ntc-b200: B200-native hot path of arXiv 2109.09534 (nonnegative tensor
completion by AO + accelerated stochastic projected gradient, S_NMC).

The compute path is libntcb.so (hand-written CUDA for sm_100a behind the
C-ABI of include/ntc_b200.h); this package is the host-side mirror of the
reference's proj/core API (see ntc.py) plus multi-GPU sharding (dist.py).
"""
from .ntc import (AoConfig, AoResult, Context, FactorSet, MetricsRecord, NmcConfig, PinnedArray, RngStream,
                  SnmcStats, SparseTensor, ao_ntc, epoch_fraction, initial_factors, objective, pinned_like,
                  relative_error, s_nmc, sample_row, sweep_stream, term_cond)
from ._lib import CudaError, DomainError, InvalidArgument, NtcRuntimeError, OutOfRange

__all__ = ["AoConfig", "AoResult", "Context", "FactorSet", "MetricsRecord", "NmcConfig", "PinnedArray",
           "pinned_like",
           "RngStream", "SnmcStats", "SparseTensor", "ao_ntc", "epoch_fraction",
           "initial_factors", "objective", "relative_error", "s_nmc", "sample_row",
           "sweep_stream", "term_cond", "CudaError", "DomainError", "InvalidArgument",
           "NtcRuntimeError", "OutOfRange"]
