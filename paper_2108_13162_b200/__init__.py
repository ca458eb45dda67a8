"""paper_2108_13162_b200 — B200-native (sm_100a) FP64 sparse Krylov solvers.

The hot path of arxiv 2108.13162 ("Auto-tuned Krylov methods on cluster of GPUs"; the
reference implementation is the krysp C++ library) rebuilt as hand-written CUDA behind a
C-ABI (include/krysp_gpu.h, libkrysp_gpu.so).  This package is the Python mirror of the
reference API used by the tests and bench; include/krysp_gpu.hpp is the C++ mirror.
"""
from ._lib import (Breakdown, BufferLengthMismatch, ClockUnavailable, CudaError, DimensionMismatch,  # noqa: F401
                   DisconnectedAssignment, EllBlowup, EmptySubdomain, Error, IndexOutOfRange, NcclError,
                   NonFinite, ParseError, ProtocolDeadlock, UnsupportedField, load)
from .api import *  # noqa: F401,F403
from .api import __doc__ as _api_doc  # noqa: F401
