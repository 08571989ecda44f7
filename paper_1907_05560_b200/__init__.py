"""oscflat-b200: B200-native (sm_100a, FP64) drop-in for the reference's
per-step neutrino beam evolution (XFLAT / oscflat ``solver::Engine``).

The product is the native library ``_oscb200.so`` (C-ABI in
``include/oscflat_b200.h``); this package is a thin host mirror of the
reference's ``solver`` API used by the tests and the bench.
"""
from .config import BASELINE_CONFIGS, RunConfig, baseline_config, parse_config  # noqa: F401
from .engine import (ConfigError, Engine, Environment, HookInfo, IoError,  # noqa: F401
                     NumericError, ParallelError, RecordMeta, RunSummary, StepControl,
                     comm_unique_id, fermi_integral, should_dump)

__all__ = ["BASELINE_CONFIGS", "RunConfig", "baseline_config", "parse_config", "Engine",
           "Environment", "StepControl", "RunSummary", "HookInfo", "RecordMeta", "should_dump", "ConfigError",
           "NumericError", "IoError", "ParallelError", "comm_unique_id", "fermi_integral"]
