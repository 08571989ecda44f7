"""ctypes binding of the C-ABI (include/oscflat_b200.h) — plumbing only.

Loads the in-tree ``_oscb200.so``.  There is no fallback: if the library is
missing or cannot load, importing the product path raises.
"""
from __future__ import annotations

import ctypes as C
import os

from .build import LIB
from .config import ConfigError as _ConfigErrorBase

_dp = C.POINTER(C.c_double)


class OscDesc(C.Structure):
    _fields_ = [("model", C.c_int), ("abins", C.c_int), ("pbins", C.c_int), ("ebins", C.c_int),
                ("Rnu", C.c_double),
                ("cos2_theta0", _dp), ("sin_theta0", _dp), ("cos_phi", _dp), ("sin_phi", _dp),
                ("vac_h11", _dp), ("vac_h12", _dp), ("fw", _dp),
                ("couplings", C.c_double * 4), ("perturb", C.c_double),
                ("matter_profile", C.c_int), ("Ye", C.c_double), ("nb0", C.c_double),
                ("hNS", C.c_double), ("Mns", C.c_double), ("gs", C.c_double), ("S", C.c_double),
                ("nflav", C.c_int), ("vac3", _dp), ("fw6", _dp), ("couplings6", C.c_double * 6)]


class OscComm(C.Structure):
    _fields_ = [("rank", C.c_int), ("nranks", C.c_int), ("device", C.c_int),
                ("nccl_unique_id", C.c_void_p), ("flags", C.c_int)]


COMM_FORCE_COLLECTIVES = 1
GROUP_ORDERED = 1
GROUP_PEER = 2


class OscStepControl(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("dr", "dr_max", "dr_min", "eps0", "kappa", "r", "R0",
                                           "Rn")] + [("iter", C.c_uint64), ("Ts", C.c_uint64),
                                                     ("Tn", C.c_double)]


class OscRunSummary(C.Structure):
    _fields_ = [("final_r", C.c_double), ("iterations", C.c_uint64), ("accepted", C.c_uint64),
                ("rejected", C.c_uint64), ("wall_s", C.c_double),
                ("phase_hamiltonian_s", C.c_double), ("phase_evolve_s", C.c_double),
                ("phase_io_s", C.c_double), ("max_worker_wait_s", C.c_double),
                ("final_max_norm_dev", C.c_double), ("termination", C.c_int)]


class OscHookInfo(C.Structure):
    _fields_ = [("iter", C.c_uint64), ("r", C.c_double), ("dr", C.c_double),
                ("t_wall", C.c_double)]


HOOK_FN = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(OscHookInfo), _dp, C.c_size_t)


class OscDumpGates(C.Structure):
    _fields_ = [("r_step", C.c_double), ("t_step", C.c_double), ("itr_step", C.c_uint64)]


class OscRecordMeta(C.Structure):
    _fields_ = [("iter", C.c_uint64), ("r", C.c_double), ("dr", C.c_double), ("t_wall", C.c_double)]


DUMP_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int, C.POINTER(OscRecordMeta), _dp, C.c_size_t)


class OscParams(C.Structure):
    _fields_ = [("model", C.c_int), ("abins", C.c_int), ("pbins", C.c_int), ("ebins", C.c_int),
                ("Rnu", C.c_double), ("E0", C.c_double), ("E1", C.c_double),
                ("dm2", C.c_double), ("theta", C.c_double), ("hvv_scale", C.c_double),
                ("perturb", C.c_double), ("L", C.c_double * 4), ("T", C.c_double * 4),
                ("Emean", C.c_double * 4), ("eta", C.c_double * 4),
                ("matter_profile", C.c_int), ("Ye", C.c_double), ("nb0", C.c_double),
                ("hNS", C.c_double), ("Mns", C.c_double), ("gs", C.c_double), ("S", C.c_double),
                ("nflav", C.c_int), ("dm2_31", C.c_double), ("theta13", C.c_double),
                ("theta23", C.c_double), ("delta_cp", C.c_double), ("L_tau", C.c_double * 2),
                ("T_tau", C.c_double * 2), ("Emean_tau", C.c_double * 2),
                ("eta_tau", C.c_double * 2)]


# Every symbol the header declares (checked by tests/test_abi.py).
SYMBOLS = [
    "osc_last_error", "osc_version", "osc_comm_unique_id", "osc_create", "osc_destroy",
    "osc_local_range", "osc_init_states", "osc_set_state", "osc_get_state",
    "osc_set_state_device", "osc_get_state_device", "osc_trial_step_error", "osc_run", "osc_run_dumps", "osc_extract_mode2",
    "osc_max_norm_dev", "osc_begin", "osc_enqueue_steps", "osc_query", "osc_synchronize",
    "osc_stream", "osc_launches_per_step", "osc_debug_sums", "osc_set_schedule", "osc_set_launch_mode", "osc_get_launch_mode", "osc_comm_export", "osc_comm_connect", "osc_launch_count",
    "osc_fp64_peak", "osc_profile_stages", "osc_debug_evolve_bin", "osc_debug_exp3", "osc_debug_trace", "osc_env_build", "osc_env_desc", "osc_env_destroy", "osc_fermi_integral",
    "osc_create_group", "osc_group_info", "osc_device_count",
]

_lib = None


def lib() -> C.CDLL:
    """Load the native library (raises if it is absent — no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("OSC_LIB", LIB)  # variant sweeps (tools/) may point elsewhere
    if not os.path.exists(path):
        raise RuntimeError(f"native library {path} is missing; run __graft_entry__.build()")
    L = C.CDLL(path, mode=C.RTLD_GLOBAL)
    vp = C.c_void_p
    L.osc_last_error.restype = C.c_char_p
    L.osc_comm_unique_id.argtypes = [vp]
    L.osc_create.argtypes = [C.POINTER(OscDesc), C.POINTER(OscComm), C.POINTER(vp)]
    L.osc_destroy.argtypes = [vp]
    L.osc_create_group.argtypes = [C.POINTER(OscDesc), C.c_int, C.POINTER(C.c_int), C.c_int, C.POINTER(vp)]
    L.osc_group_info.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    L.osc_device_count.argtypes = [C.POINTER(C.c_int)]
    L.osc_local_range.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                  C.POINTER(C.c_size_t)]
    L.osc_init_states.argtypes = [vp]
    for f in ("osc_set_state", "osc_get_state", "osc_set_state_device", "osc_get_state_device"):
        getattr(L, f).argtypes = [vp, vp, C.c_size_t]
    L.osc_trial_step_error.argtypes = [vp, C.c_double, C.c_double, _dp]
    L.osc_run.argtypes = [vp, C.POINTER(OscStepControl), HOOK_FN, vp, C.POINTER(OscRunSummary)]
    L.osc_run_dumps.argtypes = [vp, C.POINTER(OscStepControl), C.POINTER(OscDumpGates), C.c_int, DUMP_FN, vp,
                                C.POINTER(OscRunSummary)]
    L.osc_extract_mode2.argtypes = [vp, _dp, C.c_size_t]
    L.osc_max_norm_dev.argtypes = [vp, _dp]
    L.osc_begin.argtypes = [vp, C.POINTER(OscStepControl)]
    L.osc_enqueue_steps.argtypes = [vp, C.c_int]
    L.osc_query.argtypes = [vp, _dp, _dp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                            C.POINTER(C.c_uint64), _dp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    L.osc_synchronize.argtypes = [vp]
    L.osc_stream.argtypes = [vp]
    L.osc_stream.restype = vp
    L.osc_launches_per_step.argtypes = [vp]
    L.osc_debug_sums.argtypes = [vp, _dp]
    L.osc_set_schedule.argtypes = [vp, C.c_int]
    L.osc_set_launch_mode.argtypes = [vp, C.c_int]
    L.osc_comm_export.argtypes = [vp, vp]
    L.osc_comm_connect.argtypes = [vp, vp]
    L.osc_get_launch_mode.argtypes = [vp]
    L.osc_launch_count.argtypes = [vp]
    L.osc_launch_count.restype = C.c_ulonglong
    L.osc_fp64_peak.argtypes = [C.c_int, _dp, _dp]
    L.osc_profile_stages.argtypes = [vp, C.c_int, C.POINTER(C.c_float)]
    L.osc_debug_trace.argtypes = [C.POINTER(C.c_ulonglong), C.c_size_t]
    L.osc_debug_evolve_bin.argtypes = [C.c_int, C.c_size_t, _dp, _dp, _dp, _dp, C.c_int]
    L.osc_debug_exp3.argtypes = [C.c_int, C.c_size_t, _dp, _dp, _dp, C.c_int]
    L.osc_env_build.argtypes = [C.POINTER(OscParams), C.POINTER(vp)]
    L.osc_env_desc.argtypes = [vp, C.POINTER(OscDesc), _dp]
    L.osc_env_destroy.argtypes = [vp]
    L.osc_fermi_integral.argtypes = [C.c_int, C.c_double]
    L.osc_fermi_integral.restype = C.c_double
    _lib = L
    return L


class OscError(RuntimeError):
    """Base for errors raised from a non-zero OscStatus."""

    status = 0


class ConfigError(OscError, _ConfigErrorBase):
    status = 1


class NumericError(OscError):
    status = 2


class IoError(OscError):
    status = 3


class ParallelError(OscError):
    status = 4


class CudaError(OscError):
    status = 5


_BY_STATUS = {1: ConfigError, 2: NumericError, 3: IoError, 4: ParallelError, 5: CudaError}


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().osc_last_error().decode(errors="replace")
        raise _BY_STATUS.get(rc, OscError)(msg)
