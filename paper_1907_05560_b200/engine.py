"""Python mirror of the reference's ``solver`` API over the C-ABI.

Reference: ``include/oscflat/solver.hpp:20-153``.  Names and argument meaning
follow the reference so the parity tests read like ``test_solver.cpp``:

* ``Environment.from_config(cfg)``  ->  solver::Environment::from_config
* ``Engine(env, gpus)``             ->  solver::Engine(env, lanes)
* ``engine.init_states()``, ``engine.state()``, ``engine.trial_step_error(r, dr)``,
  ``engine.run(ctl, hook)``          ->  the same-named Engine members
* ``StepControl.from_config(cfg)``  ->  solver::StepControl::from_config
* errors: ConfigError / NumericError / IoError / ParallelError (types.hpp:43-51)

All compute happens in the native library; there is no CPU path here.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import native
from .config import RunConfig
from .native import (DUMP_FN, HOOK_FN, OscComm, OscDesc, OscDumpGates, OscParams, OscRunSummary,
                     OscStepControl, check, lib)


@dataclass
class StepControl:
    """solver::StepControl (solver.hpp:20-34)."""

    dr: float = 1e-3
    dr_max: float = 1.0
    dr_min: float = 1e-12
    eps0: float = 1e-8
    kappa: float = 0.8
    r: float = 0.0
    R0: float = 0.0
    Rn: float = 0.0
    iter: int = 0
    Ts: int = 0
    Tn: float = 0.0

    @classmethod
    def from_config(cls, cfg: RunConfig) -> "StepControl":
        v = cfg.values
        return cls(dr=v["dr"], dr_max=v["max_dr"], dr_min=v["min_dr"], eps0=v["eps0"],
                   kappa=v["kappa"], r=v["R0"], R0=v["R0"], Rn=v["Rn"], iter=0, Ts=v["Ts"],
                   Tn=v["Tn"])

    def to_c(self) -> OscStepControl:
        return OscStepControl(dr=self.dr, dr_max=self.dr_max, dr_min=self.dr_min, eps0=self.eps0,
                              kappa=self.kappa, r=self.r, R0=self.R0, Rn=self.Rn, iter=self.iter,
                              Ts=self.Ts, Tn=self.Tn)


@dataclass
class RunSummary:
    """solver::RunSummary (solver.hpp:85-99)."""

    final_r: float
    iterations: int
    accepted: int
    rejected: int
    wall_s: float
    phase_hamiltonian_s: float
    phase_evolve_s: float
    phase_io_s: float
    max_worker_wait_s: float
    final_max_norm_dev: float
    termination: str


@dataclass
class HookInfo:
    iter: int
    r: float
    dr: float
    t_wall: float


def should_dump(gates, r: float, t_wall: float, it: int, last) -> bool:
    """io::should_dump (snapshot.cpp:237-243): gates = (r_step, t_step,
    itr_step), last = (r, t, iter) of the previous dump of that mode."""
    r_step, t_step, itr_step = gates
    if r_step > 0.0 and r - last[0] >= r_step:
        return True
    if t_step > 0.0 and t_wall - last[1] >= t_step:
        return True
    return itr_step > 0 and it - last[2] >= itr_step


@dataclass
class RecordMeta:
    """io::RecordMeta (snapshot.hpp:40-45) of a dump."""
    iter: int
    r: float
    dr: float
    t_wall: float


class Environment:
    """solver::Environment (solver.hpp:71-85): grid, vacuum table, spectra,
    couplings and matter parameters, built by the native host code."""

    def __init__(self, cfg: RunConfig):
        # like the reference, from_config does not run io::require_runnable
        # (the CLI does); the native builder validates what it consumes
        v = cfg.values
        p = OscParams()
        p.model = cfg.model_id
        p.abins, p.pbins, p.ebins = v["Abins"], v["Pbins"], v["Ebins"]
        p.Rnu, p.E0, p.E1, p.dm2, p.theta = v["Rv"], v["E0"], v["E1"], v["dm2"], v["theta"]
        p.hvv_scale, p.perturb = v["hvvScale"], v["perturb"]
        for arr, name in ((p.L, "L"), (p.T, "T"), (p.Emean, "E"), (p.eta, "eta")):
            for i, x in enumerate(cfg.species(name)):
                arr[i] = x
        p.matter_profile = cfg.matter_id
        p.Ye, p.nb0, p.hNS, p.Mns, p.gs, p.S = (v["Ye"], v["nb0"], v["hNS"], v["Mns"], v["gs"],
                                                 v["S"])
        p.nflav = v["Flvs"]
        if p.nflav == 3:
            prov = cfg.provided
            p.dm2 = v["dm2_21"] if "dm2_21" in prov else v["dm2"]
            p.theta = v["theta12"] if "theta12" in prov else v["theta"]
            p.dm2_31, p.theta13, p.theta23, p.delta_cp = (v["dm2_31"], v["theta13"],
                                                           v["theta23"], v["deltaCP"])
            for arr, name in ((p.L_tau, "L"), (p.T_tau, "T"), (p.Emean_tau, "E"),
                              (p.eta_tau, "eta")):
                for i, x in enumerate(cfg.tau(name)):
                    arr[i] = x
        self.cfg = cfg
        self._h = C.c_void_p()
        check(lib().osc_env_build(C.byref(p), C.byref(self._h)))
        self.desc = OscDesc()
        emean = (C.c_double * 4)()
        check(lib().osc_env_desc(self._h, C.byref(self.desc), emean))
        self.emean = list(emean)
        d = self.desc
        self.model, self.abins, self.pbins, self.ebins = d.model, d.abins, d.pbins, d.ebins
        self.nflav = 3 if d.nflav == 3 else 2
        self.species_count = 6 if self.nflav == 3 else 4
        self.comps = 6 if self.nflav == 3 else 4

    @classmethod
    def from_config(cls, cfg: RunConfig) -> "Environment":
        return cls(cfg)

    def __del__(self):
        try:
            lib().osc_env_destroy(self._h)
        except Exception:
            pass

    def tables(self) -> dict:
        d = self.desc
        T, P, E = d.abins, d.pbins, d.ebins
        arr = lambda p, n: np.ctypeslib.as_array(p, shape=(n,)).copy()
        t = dict(cos2=arr(d.cos2_theta0, T), sin0=arr(d.sin_theta0, T),
                 cphi=arr(d.cos_phi, P), sphi=arr(d.sin_phi, P), vac11=arr(d.vac_h11, E),
                 vac12=arr(d.vac_h12, E), fw=arr(d.fw, 4 * E).reshape(4, E),
                 couplings=np.array(list(d.couplings)), emean=np.array(self.emean))
        if self.nflav == 3:
            t.update(vac3=arr(d.vac3, 9 * E).reshape(E, 9), fw6=arr(d.fw6, 6 * E).reshape(6, E),
                     couplings6=np.array(list(d.couplings6)))
        return t

    @property
    def trajectories(self) -> int:
        return self.abins * self.pbins

    @property
    def cells(self) -> int:
        return self.trajectories * self.ebins


_TERM = {1: "radius", 2: "iterations", 3: "walltime"}


class Engine:
    """solver::Engine (solver.hpp:128-153) on one GPU per process.

    ``rank``/``nranks`` shard the theta bins like the reference's lanes
    (make_partitions); ``nccl_id`` is the 128-byte id shared by all ranks."""

    def __init__(self, env: Environment, rank: int = 0, nranks: int = 1, device: int = 0,
                 nccl_id: bytes | None = None, force_collectives: bool = False):
        self.env = env  # borrowed, kept alive (solver.hpp:152)
        self._idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id else None
        comm = OscComm(rank=rank, nranks=nranks, device=device,
                       nccl_unique_id=C.cast(self._idbuf, C.c_void_p) if self._idbuf else None,
                       flags=native.COMM_FORCE_COLLECTIVES if force_collectives else 0)
        self._ctx = C.c_void_p()
        check(lib().osc_create(C.byref(env.desc), C.byref(comm), C.byref(self._ctx)))
        lo, hi, n = C.c_int(), C.c_int(), C.c_size_t()
        check(lib().osc_local_range(self._ctx, C.byref(lo), C.byref(hi), C.byref(n)))
        self.t_lo, self.t_hi, self.state_doubles = lo.value, hi.value, n.value
        self.rank, self.nranks = rank, nranks
        self.ordered = False

    @classmethod
    def group(cls, env: Environment, nranks: int, devices=None, peer: bool = False) -> "Engine":
        """Engine(env, lanes) over ``nranks`` GPUs in this process
        (osc_create_group): theta blocks by make_partitions, one context per
        rank, driven through one handle whose state() covers every
        trajectory.  ``devices`` lists the GPU of each rank (default q mod
        the device count).  The stage moments move stream-ordered between
        the ranks; ``peer=True`` asks for the device-initiated exchange over
        peer pointers (distinct GPUs with peer access only)."""
        self = cls.__new__(cls)
        self.env = env
        self._idbuf = None
        self._ctx = C.c_void_p()
        dev = (C.c_int * nranks)(*devices) if devices is not None else None
        check(lib().osc_create_group(C.byref(env.desc), nranks, dev, native.GROUP_PEER if peer else 0,
                                     C.byref(self._ctx)))
        lo, hi, n = C.c_int(), C.c_int(), C.c_size_t()
        check(lib().osc_local_range(self._ctx, C.byref(lo), C.byref(hi), C.byref(n)))
        self.t_lo, self.t_hi, self.state_doubles = lo.value, hi.value, n.value
        nr, od = C.c_int(), C.c_int()
        check(lib().osc_group_info(self._ctx, C.byref(nr), C.byref(od)))
        self.rank, self.nranks, self.ordered = 0, nr.value, bool(od.value)
        return self

    def close(self):
        if getattr(self, "_ctx", None):
            lib().osc_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- reference API ---------------------------------------------------
    def init_states(self) -> None:
        check(lib().osc_init_states(self._ctx))

    def state(self) -> np.ndarray:
        """Committed psi0 as the mode-1 payload [traj][species][comp][ebin]."""
        out = np.empty(self.state_doubles, dtype=np.float64)
        check(lib().osc_get_state(self._ctx, out.ctypes.data, out.size))
        return out

    def set_state(self, mode1) -> None:
        a = np.ascontiguousarray(mode1, dtype=np.float64).ravel()
        check(lib().osc_set_state(self._ctx, a.ctypes.data, a.size))

    def trial_step_error(self, r: float, dr: float) -> float:
        err = C.c_double()
        check(lib().osc_trial_step_error(self._ctx, r, dr, C.byref(err)))
        return err.value

    def run(self, ctl: StepControl, hook=None) -> RunSummary:
        s = OscRunSummary()
        if hook is not None:
            def _tramp(user, info, state, n):
                i = info.contents
                hook(HookInfo(i.iter, i.r, i.dr, i.t_wall),
                     np.ctypeslib.as_array(state, shape=(n,)).copy())
            cb = HOOK_FN(_tramp)
        else:
            cb = HOOK_FN()
        check(lib().osc_run(self._ctx, C.byref(ctl.to_c()), cb, None, C.byref(s)))
        return RunSummary(s.final_r, s.iterations, s.accepted, s.rejected, s.wall_s,
                          s.phase_hamiltonian_s, s.phase_evolve_s, s.phase_io_s,
                          s.max_worker_wait_s, s.final_max_norm_dev,
                          _TERM.get(s.termination, "radius"))

    def run_dumps(self, ctl: StepControl, gates, mode_mask: int, callback, copy: bool = True) -> RunSummary:
        """Engine.run with the CLI's snapshot gating on the device
        (tools/oscflat.cpp:46-118 DumpDriver): gates = [(r_step, t_step,
        itr_step) for mode 1, same for mode 2]; callback(mode, RecordMeta,
        payload) receives copies (copy=False: a view of the engine's pinned
        buffer, valid only during the call), in dump order.  Mode-1 payloads are the
        local state (extract_mode1 layout), mode-2 payloads
        trajectories x species energy averages (extract_mode2)."""
        g = (OscDumpGates * 2)(*[OscDumpGates(float(a), float(b), int(c)) for a, b, c in gates])

        def _tramp(user, mode, meta, payload, n):
            m = meta.contents
            v = np.ctypeslib.as_array(payload, shape=(n,))
            callback(int(mode), RecordMeta(m.iter, m.r, m.dr, m.t_wall), v.copy() if copy else v)

        cb = DUMP_FN(_tramp)
        s = OscRunSummary()
        check(lib().osc_run_dumps(self._ctx, C.byref(ctl.to_c()), g, int(mode_mask), cb, None, C.byref(s)))
        return RunSummary(s.final_r, s.iterations, s.accepted, s.rejected, s.wall_s,
                          s.phase_hamiltonian_s, s.phase_evolve_s, s.phase_io_s,
                          s.max_worker_wait_s, s.final_max_norm_dev,
                          _TERM.get(s.termination, "radius"))

    def mode2(self) -> np.ndarray:
        """solver::extract_mode2 of the current state, computed on the device:
        [trajectory][species] energy-averaged |psi_e|^2 (solver.cpp:160-174)."""
        nsp = 6 if self.env.nflav == 3 else 4
        out = np.zeros(self.state_doubles // (nsp * (6 if nsp == 6 else 4) * self.env.ebins) * nsp)
        check(lib().osc_extract_mode2(self._ctx, out.ctypes.data_as(C.POINTER(C.c_double)), out.size))
        return out

    # -- device-resident helpers (bench / tests) -------------------------
    def max_norm_dev(self) -> float:
        v = C.c_double()
        check(lib().osc_max_norm_dev(self._ctx, C.byref(v)))
        return v.value

    def set_state_device(self, ptr: int, n: int) -> None:
        check(lib().osc_set_state_device(self._ctx, C.c_void_p(ptr), n))

    def get_state_device(self, ptr: int, n: int) -> None:
        check(lib().osc_get_state_device(self._ctx, C.c_void_p(ptr), n))

    def set_state_host_ptr(self, ptr: int, n: int) -> None:
        check(lib().osc_set_state(self._ctx, C.c_void_p(ptr), n))

    def get_state_host_ptr(self, ptr: int, n: int) -> None:
        check(lib().osc_get_state(self._ctx, C.c_void_p(ptr), n))

    def begin(self, ctl: StepControl) -> None:
        check(lib().osc_begin(self._ctx, C.byref(ctl.to_c())))

    def enqueue_steps(self, n: int) -> None:
        check(lib().osc_enqueue_steps(self._ctx, n))

    def query(self) -> dict:
        r, dr, err = C.c_double(), C.c_double(), C.c_double()
        it, acc, rej = C.c_uint64(), C.c_uint64(), C.c_uint64()
        st, term = C.c_int(), C.c_int()
        check(lib().osc_query(self._ctx, C.byref(r), C.byref(dr), C.byref(it), C.byref(acc),
                              C.byref(rej), C.byref(err), C.byref(st), C.byref(term)))
        return dict(r=r.value, dr=dr.value, iter=it.value, accepted=acc.value,
                    rejected=rej.value, err=err.value, status=st.value, terminate=term.value)

    def synchronize(self) -> None:
        check(lib().osc_synchronize(self._ctx))

    def stream(self) -> int:
        return lib().osc_stream(self._ctx) or 0

    def launches_per_step(self) -> int:
        return lib().osc_launches_per_step(self._ctx)

    def debug_sums(self) -> np.ndarray:
        out = np.zeros(60)
        check(lib().osc_debug_sums(self._ctx, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out.reshape(5, 12)

    def profile_stages(self, nsteps: int) -> list:
        out = (C.c_float * 3)()
        check(lib().osc_profile_stages(self._ctx, nsteps, out))
        return [float(x) for x in out]

    def set_schedule(self, schedule: int) -> None:
        check(lib().osc_set_schedule(self._ctx, schedule))

    def comm_export(self) -> bytes:
        """128-byte token (CUDA IPC handles of this rank's exchange slots)."""
        buf = C.create_string_buffer(128)
        check(lib().osc_comm_export(self._ctx, buf))
        return buf.raw

    def comm_connect(self, tokens) -> None:
        """Switch the stage exchange from NCCL to device-initiated peer stores;
        tokens = every rank's comm_export() in rank order."""
        blob = b"".join(tokens)
        check(lib().osc_comm_connect(self._ctx, C.create_string_buffer(blob, len(blob))))

    LAUNCH_STAGES, LAUNCH_RESIDENT = 0, 2

    def set_launch_mode(self, mode: int) -> None:
        """0: stage kernels (PDL, CUDA graphs); 2: persistent kernel with the
        state resident in shared memory (the default where it fits).  Raises
        ConfigError if unavailable."""
        check(lib().osc_set_launch_mode(self._ctx, int(mode)))

    @property
    def launch_mode(self) -> int:
        return int(lib().osc_get_launch_mode(self._ctx))

    def launch_count(self) -> int:
        """Kernels this engine has launched so far (graph nodes included)."""
        return int(lib().osc_launch_count(self._ctx))


def device_count() -> int:
    n = C.c_int()
    check(lib().osc_device_count(C.byref(n)))
    return n.value


def fp64_peak(device: int = 0) -> float:
    """Thread-level DFMA instructions per second measured on `device`."""
    v, ms = C.c_double(), C.c_double()
    check(lib().osc_fp64_peak(device, C.byref(v), C.byref(ms)))
    return v.value


def debug_evolve_bin(h, dl, psi, path: int = 0, device: int = 0):
    """flavor::evolve_bin (beam.hpp:105-121) through the device propagator
    code (path 0: the stage kernels' branch-free chain + fallback branch; 1:
    the safe path).  h [n,3], dl [n], psi [n,4] -> [n,4]."""
    import numpy as np

    h = np.ascontiguousarray(h, dtype=np.float64).reshape(-1, 3)
    n = h.shape[0]
    dl = np.ascontiguousarray(dl, dtype=np.float64).reshape(n)
    psi = np.ascontiguousarray(psi, dtype=np.float64).reshape(n, 4)
    out = np.zeros((n, 4))
    dp = C.POINTER(C.c_double)
    check(lib().osc_debug_evolve_bin(device, n, h.ctypes.data_as(dp), dl.ctypes.data_as(dp),
                                     psi.ctypes.data_as(dp), out.ctypes.data_as(dp), path))
    return out


def debug_exp3(H9, tau, path: int = 0, device: int = 0):
    """exp(-i H tau) of packed 3x3 Hermitian matrices through the device code
    of the 3-flavour stages (csrc/su3_exp.cuh).  H9 [n,9], tau [n] -> complex
    [n,3,3]."""
    import numpy as np

    H9 = np.ascontiguousarray(H9, dtype=np.float64).reshape(-1, 9)
    n = H9.shape[0]
    tau = np.ascontiguousarray(tau, dtype=np.float64).reshape(n)
    out = np.zeros((n, 18))
    dp = C.POINTER(C.c_double)
    check(lib().osc_debug_exp3(device, n, H9.ctypes.data_as(dp), tau.ctypes.data_as(dp),
                               out.ctypes.data_as(dp), path))
    return (out[:, 0::2] + 1j * out[:, 1::2]).reshape(n, 3, 3)


def comm_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib().osc_comm_unique_id(buf))
    return buf.raw


def fermi_integral(k: int, eta: float) -> float:
    return lib().osc_fermi_integral(k, eta)


ConfigError = native._ConfigErrorBase  # base of native.ConfigError and config errors
NumericError = native.NumericError
IoError = native.IoError
ParallelError = native.ParallelError
