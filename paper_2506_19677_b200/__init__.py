"""paper_2506_19677_b200 — B200-native engine for the SABER simulation/fit hot path.

The product is the C ABI library ``libsaber_b200.so`` (include/saber_cuda.h):
sm_100a kernels plus C++ host orchestration.  This package is its Python face,
mirroring the reference's API names (see api.py).
"""
from .api import *  # noqa: F401,F403
from .api import (BatchResult, CalibrationError, DomainError, FitError, InvalidArgument,  # noqa: F401
                  FitBatchResult, LoadSpeedSample, CalibrationReport, fit, fit_batch, calibrate,
                  BurstyArrivals, McResult, mc_sweep, mc_trace, profile, profile_batch,
                  ROW_DTYPE, SweepPlan, run_batch, sweep_row_keys)
from ._native import LIB_PATH, SaberError, lib  # noqa: F401

__version__ = "0.1.0"
