"""B200-native FAST-HALS / PL-NMF engine (arxiv/paper_1904_07935).

The product is the CUDA shared library ``libplnmf_gpu.so`` behind the C-ABI in
``include/plnmf_gpu.h``; :mod:`.plnmf` mirrors the reference's C++ interface on
top of it.  Nothing here imports or calls the oracle.
"""
from .plnmf import (Algorithm, ConvergenceTrace, CsrMatrix, DeviceError, DomainError, Engine,  # noqa: F401
                    ErrorReport, FactorPair, InputMatrix, InvalidArgument, Math, NonFiniteObjective,
                    PhaseTimes, SolverConfig, TilingPlan, TraceRecord, device_count, init_factors,
                    iterate, plan_tiles, synth_csr)

__all__ = ["Algorithm", "ConvergenceTrace", "CsrMatrix", "DeviceError", "DomainError", "Engine", "ErrorReport",
           "FactorPair", "InputMatrix", "InvalidArgument", "Math", "NonFiniteObjective", "PhaseTimes",
           "SolverConfig", "TilingPlan", "TraceRecord", "device_count", "init_factors", "iterate", "plan_tiles",
           "synth_csr"]
