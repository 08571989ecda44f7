"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the CPU checkers.

* ``Ref``    — the unmodified reference core compiled by ``oracle/Makefile``
               (``oracle/_ref/libref_oscflat_<arch>.so``), driven through
               ``oracle/ref_harness.cpp``.
* ``Oracle`` — the plain-C restatement ``oracle/oscflat_oracle.c``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module (it is the checker, never the
product path).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
_dp = C.POINTER(C.c_double)


def build(quiet: bool = True) -> None:
    """Build the checkers (reference compiled where its sources lie, if present)."""
    out = subprocess.run(["make", "-C", HERE, "-j8", "all"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout[-4000:] + out.stderr[-4000:])
    if not quiet:
        print(out.stdout)


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def host_isa() -> str:
    try:
        flags = open("/proc/cpuinfo").read()
    except OSError:
        return "v3"
    need = ("avx512f", "avx512dq", "avx512bw", "avx512vl", "avx512cd")
    return "v4" if all(f in flags for f in need) else "v3"


# --------------------------------------------------------------------------- ref
_REF_DUMP_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int, C.c_uint64, C.c_double, C.c_double,
                           C.POINTER(C.c_double), C.c_size_t)


class Ref:
    """Reference engine (solver::Engine) over a config text."""

    def __init__(self, variant: str | None = None):
        variant = variant or host_isa()
        path = os.path.join(REF_DIR, f"libref_oscflat_{variant}.so")
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing; run `make -C oracle` where "
                                    "/root/reference is present")
        self.variant = variant
        self.lib = L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_env_dims.argtypes = [C.c_char_p, C.POINTER(C.c_int)]
        L.ref_env_tables.argtypes = [C.c_char_p] + [_dp] * 9
        L.ref_matter.argtypes = [C.c_char_p, C.c_double]
        L.ref_matter.restype = C.c_double
        L.ref_fermi_integral.argtypes = [C.c_int, C.c_double]
        L.ref_fermi_integral.restype = C.c_double
        L.ref_run.argtypes = [C.c_char_p, C.c_int, _dp, C.c_double, C.c_double, C.c_uint64,
                              C.c_uint64, _dp, _dp]
        L.ref_trial_step.argtypes = [C.c_char_p, _dp, C.c_double, C.c_double, _dp, _dp]
        L.ref_init_state.argtypes = [C.c_int, C.c_int, C.c_double, C.c_uint64, _dp]
        L.ref_evolve_bin.argtypes = [_dp, C.c_double, _dp, _dp]
        L.ref_density.argtypes = [_dp, _dp]
        L.ref_e_sum.argtypes = [C.c_int, _dp, _dp, _dp]
        L.ref_partial_hvv.argtypes = [C.c_char_p, C.c_double, _dp, _dp, _dp]
        L.ref_fill_cache.argtypes = [C.c_char_p, C.c_double, _dp]
        L.ref_run_dumps.argtypes = [C.c_char_p, C.c_int, _dp, _dp, C.c_int, _REF_DUMP_FN, C.c_void_p, _dp]
        L.ref_extract_mode2.argtypes = [C.c_char_p, _dp, _dp]

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(f"reference error {rc}: {self.lib.ref_last_error().decode()}")

    def dims(self, cfg_text: str):
        d = (C.c_int * 5)()
        self._check(self.lib.ref_env_dims(cfg_text.encode(), d))
        return dict(model=d[0], abins=d[1], pbins=d[2], ebins=d[3], padded=d[4])

    def tables(self, cfg_text: str) -> dict:
        d = self.dims(cfg_text)
        T, P, E = d["abins"], d["pbins"], d["ebins"]
        t = dict(cos2=np.zeros(T), sin0=np.zeros(T), cphi=np.zeros(P), sphi=np.zeros(P),
                 vac11=np.zeros(E), vac12=np.zeros(E), fw=np.zeros(4 * E),
                 couplings=np.zeros(4), emean=np.zeros(4))
        self._check(self.lib.ref_env_tables(cfg_text.encode(), *[_ptr(t[k]) for k in (
            "cos2", "sin0", "cphi", "sphi", "vac11", "vac12", "fw", "couplings", "emean")]))
        t["fw"] = t["fw"].reshape(4, E)
        return t

    def state_size(self, cfg_text: str) -> int:
        d = self.dims(cfg_text)
        return d["abins"] * d["pbins"] * 16 * d["ebins"]

    def run(self, cfg_text: str, lanes: int = 1, state=None, r=-1.0, dr=0.0, it=0, ts=0):
        n = self.state_size(cfg_text)
        out = np.zeros(n)
        summ = np.zeros(7)
        sin = None if state is None else np.ascontiguousarray(state, dtype=np.float64)
        self._check(self.lib.ref_run(cfg_text.encode(), lanes, None if sin is None else _ptr(sin),
                                     r, dr, it, ts, _ptr(out), _ptr(summ)))
        keys = ("final_r", "iterations", "accepted", "rejected", "wall_s", "final_max_norm_dev",
                "phase_evolve_s")
        return out, dict(zip(keys, summ.tolist()))

    def run_dumps(self, cfg_text: str, gates, mode_mask: int, lanes: int = 1, state=None):
        """Engine::run + the CLI's DumpDriver gating; returns ([(mode, iter, r,
        dr, payload)], final mode-1 state)."""
        g = np.ascontiguousarray(np.asarray(gates, dtype=np.float64).ravel())
        dumps = []

        def _cb(user, mode, it, r, dr, payload, n):
            dumps.append((int(mode), int(it), r, dr, np.ctypeslib.as_array(payload, shape=(n,)).copy()))

        cb = _REF_DUMP_FN(_cb)
        out = np.zeros(self.state_size(cfg_text))
        sin = None if state is None else np.ascontiguousarray(state, dtype=np.float64)
        self._check(self.lib.ref_run_dumps(cfg_text.encode(), lanes, None if sin is None else _ptr(sin),
                                           _ptr(g), mode_mask, cb, None, _ptr(out)))
        return dumps, out

    def extract_mode2(self, cfg_text: str, state):
        d = self.dims(cfg_text)
        out = np.zeros(d["abins"] * d["pbins"] * 4)
        sin = np.ascontiguousarray(state, dtype=np.float64)
        self._check(self.lib.ref_extract_mode2(cfg_text.encode(), _ptr(sin), _ptr(out)))
        return out

    def trial_step(self, cfg_text: str, r: float, dr: float, state=None):
        n = self.state_size(cfg_text)
        after = np.zeros(n)
        err = C.c_double()
        sin = None if state is None else np.ascontiguousarray(state, dtype=np.float64)
        self._check(self.lib.ref_trial_step(cfg_text.encode(), None if sin is None else _ptr(sin),
                                            r, dr, C.byref(err), _ptr(after)))
        return err.value, after

    def init_state(self, species, ebins, eps, seed):
        out = np.zeros(4 * ebins)
        self._check(self.lib.ref_init_state(species, ebins, eps, seed, _ptr(out)))
        return out.reshape(4, ebins)

    def evolve_bin(self, h, dl, psi):
        h = np.ascontiguousarray(h, dtype=np.float64)
        psi = np.ascontiguousarray(psi, dtype=np.float64)
        out = np.zeros(4)
        self.lib.ref_evolve_bin(_ptr(h), dl, _ptr(psi), _ptr(out))
        return out

    def density(self, psi):
        psi = np.ascontiguousarray(psi, dtype=np.float64)
        out = np.zeros(3)
        self.lib.ref_density(_ptr(psi), _ptr(out))
        return out

    def e_sum(self, beam, fw):
        beam = np.ascontiguousarray(beam, dtype=np.float64)
        fw = np.ascontiguousarray(fw, dtype=np.float64)
        out = np.zeros(3)
        self._check(self.lib.ref_e_sum(beam.shape[1], _ptr(beam), _ptr(fw), _ptr(out)))
        return out

    def partial_hvv(self, cfg_text, r, rows):
        d = self.dims(cfg_text)
        rows = np.ascontiguousarray(rows, dtype=np.float64)
        sums = np.zeros(12)
        hvv = np.zeros((d["abins"] * d["pbins"], 3))
        self._check(self.lib.ref_partial_hvv(cfg_text.encode(), r, _ptr(rows), _ptr(sums),
                                             _ptr(hvv)))
        return sums, hvv

    def fill_cache(self, cfg_text, r):
        d = self.dims(cfg_text)
        out = np.zeros(3 * d["abins"])
        self._check(self.lib.ref_fill_cache(cfg_text.encode(), r, _ptr(out)))
        return out.reshape(3, d["abins"])

    def matter(self, cfg_text, r):
        return self.lib.ref_matter(cfg_text.encode(), r)

    def fermi_integral(self, k, eta):
        return self.lib.ref_fermi_integral(k, eta)


# ------------------------------------------------------------------------ oracle
class _Params(C.Structure):
    _fields_ = [("model", C.c_int), ("abins", C.c_int), ("pbins", C.c_int), ("ebins", C.c_int),
                ("Rnu", C.c_double), ("E0", C.c_double), ("E1", C.c_double),
                ("dm2", C.c_double), ("theta", C.c_double), ("hvv_scale", C.c_double),
                ("perturb", C.c_double), ("L", C.c_double * 4), ("T", C.c_double * 4),
                ("Emean", C.c_double * 4), ("eta", C.c_double * 4),
                ("matter_profile", C.c_int), ("Ye", C.c_double), ("nb0", C.c_double),
                ("hNS", C.c_double), ("Mns", C.c_double), ("gs", C.c_double), ("S", C.c_double)]


class _Ctl(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("dr", "dr_max", "dr_min", "eps0", "kappa", "r", "R0",
                                           "Rn")] + [("iter", C.c_uint64), ("Ts", C.c_uint64)]


class _Summary(C.Structure):
    _fields_ = [("final_r", C.c_double), ("iterations", C.c_uint64), ("accepted", C.c_uint64),
                ("rejected", C.c_uint64), ("final_max_norm_dev", C.c_double),
                ("termination", C.c_int)]


_oracle_lib = None


def _olib():
    global _oracle_lib
    if _oracle_lib is None:
        path = os.path.join(REF_DIR, "liboscflat_oracle.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.orc_last_error.restype = C.c_char_p
        L.orc_env_create.argtypes = [C.POINTER(_Params), C.POINTER(C.c_void_p)]
        L.orc_env_destroy.argtypes = [C.c_void_p]
        L.orc_env_tables.argtypes = [C.c_void_p] + [_dp] * 9
        L.orc_fermi_integral.argtypes = [C.c_int, C.c_double]
        L.orc_fermi_integral.restype = C.c_double
        L.orc_matter_potential.argtypes = [C.c_void_p, C.c_double]
        L.orc_matter_potential.restype = C.c_double
        L.orc_evolve_bin.argtypes = [_dp, C.c_double, _dp, _dp]
        L.orc_density.argtypes = [_dp, _dp]
        L.orc_init_state.argtypes = [C.c_int, C.c_int, C.c_double, C.c_uint64, _dp]
        L.orc_engine_create.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.orc_engine_destroy.argtypes = [C.c_void_p]
        L.orc_init_states.argtypes = [C.c_void_p]
        L.orc_set_state.argtypes = [C.c_void_p, _dp]
        L.orc_get_state.argtypes = [C.c_void_p, _dp]
        L.orc_prepare.argtypes = [C.c_void_p, C.c_double, C.c_double]
        L.orc_stage.argtypes = [C.c_void_p, C.c_int, _dp]
        L.orc_stage_set.argtypes = [C.c_void_p, C.c_int, _dp]
        L.orc_commit.argtypes = [C.c_void_p]
        L.orc_trial_step.argtypes = [C.c_void_p, C.c_double, C.c_double, _dp]
        L.orc_run.argtypes = [C.c_void_p, C.POINTER(_Ctl), C.POINTER(_Summary)]
        L.orc_max_norm_dev.argtypes = [C.c_void_p]
        L.orc_max_norm_dev.restype = C.c_double
        L.orc_make_partitions.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_int)]
        L.orc_hvv_from_rows.argtypes = [C.c_void_p, C.c_double, _dp, _dp, _dp]
        _oracle_lib = L
    return _oracle_lib


def params_from_config(cfg) -> _Params:
    v = cfg.values
    p = _Params()
    p.model = cfg.model_id
    p.abins, p.pbins, p.ebins = v["Abins"], v["Pbins"], v["Ebins"]
    p.Rnu, p.E0, p.E1, p.dm2, p.theta = v["Rv"], v["E0"], v["E1"], v["dm2"], v["theta"]
    p.hvv_scale, p.perturb = v["hvvScale"], v["perturb"]
    for arr, name in ((p.L, "L"), (p.T, "T"), (p.Emean, "E"), (p.eta, "eta")):
        for i, x in enumerate(cfg.species(name)):
            arr[i] = x
    p.matter_profile = cfg.matter_id
    p.Ye, p.nb0, p.hNS, p.Mns, p.gs, p.S = v["Ye"], v["nb0"], v["hNS"], v["Mns"], v["gs"], v["S"]
    return p


class _Params3(C.Structure):
    _fields_ = [("model", C.c_int), ("abins", C.c_int), ("pbins", C.c_int), ("ebins", C.c_int),
                ("Rnu", C.c_double), ("E0", C.c_double), ("E1", C.c_double),
                ("dm21", C.c_double), ("dm31", C.c_double), ("th12", C.c_double),
                ("th13", C.c_double), ("th23", C.c_double), ("dcp", C.c_double),
                ("hvv_scale", C.c_double), ("perturb", C.c_double), ("L", C.c_double * 6),
                ("T", C.c_double * 6), ("Emean", C.c_double * 6), ("eta", C.c_double * 6),
                ("matter_profile", C.c_int), ("Ye", C.c_double), ("nb0", C.c_double),
                ("hNS", C.c_double), ("Mns", C.c_double), ("gs", C.c_double), ("S", C.c_double)]


def params3_from_config(cfg) -> _Params3:
    v, prov = cfg.values, cfg.provided
    p = _Params3()
    p.model = cfg.model_id
    p.abins, p.pbins, p.ebins = v["Abins"], v["Pbins"], v["Ebins"]
    p.Rnu, p.E0, p.E1 = v["Rv"], v["E0"], v["E1"]
    p.dm21 = v["dm2_21"] if "dm2_21" in prov else v["dm2"]
    p.th12 = v["theta12"] if "theta12" in prov else v["theta"]
    p.dm31, p.th13, p.th23, p.dcp = v["dm2_31"], v["theta13"], v["theta23"], v["deltaCP"]
    p.hvv_scale, p.perturb = v["hvvScale"], v["perturb"]
    for arr, name in ((p.L, "L"), (p.T, "T"), (p.Emean, "E"), (p.eta, "eta")):
        vals = cfg.species(name) + cfg.tau(name)
        for i, x in enumerate(vals):
            arr[i] = x
    p.matter_profile = cfg.matter_id
    p.Ye, p.nb0, p.hNS, p.Mns, p.gs, p.S = v["Ye"], v["nb0"], v["hNS"], v["Mns"], v["gs"], v["S"]
    return p


class Oracle3:
    """3-flavour C restatement (oracle/oscflat3_oracle.c; parity unpinned)."""

    def __init__(self, cfg, t_lo=None, t_hi=None):
        self.L = L = _olib()
        for f in ("orc3_env_create", "orc3_engine_create"):
            pass
        L.orc3_last_error.restype = C.c_char_p
        L.orc3_env_create.argtypes = [C.POINTER(_Params3), C.POINTER(C.c_void_p)]
        L.orc3_env_destroy.argtypes = [C.c_void_p]
        L.orc3_env_tables.argtypes = [C.c_void_p, _dp, _dp, _dp]
        L.orc3_engine_create.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.orc3_engine_destroy.argtypes = [C.c_void_p]
        L.orc3_init_states.argtypes = [C.c_void_p]
        L.orc3_set_state.argtypes = [C.c_void_p, _dp]
        L.orc3_get_state.argtypes = [C.c_void_p, _dp]
        L.orc3_trial_step.argtypes = [C.c_void_p, C.c_double, C.c_double, _dp]
        L.orc3_run.argtypes = [C.c_void_p, C.POINTER(_Ctl), C.POINTER(_Summary)]
        L.orc3_expm.argtypes = [_dp, C.c_double, _dp]
        self.cfg = cfg
        self.params = params3_from_config(cfg)
        env = C.c_void_p()
        if L.orc3_env_create(C.byref(self.params), C.byref(env)) != 0:
            raise RuntimeError(L.orc3_last_error().decode())
        self.env = env
        p = self.params
        self.T = 1 if p.model == 0 else p.abins
        self.P = 1
        self.E = p.ebins
        self.t_lo = 0 if t_lo is None else t_lo
        self.t_hi = self.T if t_hi is None else t_hi
        eng = C.c_void_p()
        if L.orc3_engine_create(env, self.t_lo, self.t_hi, C.byref(eng)) != 0:
            raise RuntimeError(L.orc3_last_error().decode())
        self.eng = eng
        self.n = (self.t_hi - self.t_lo) * self.P * 36 * self.E
        L.orc3_init_states(eng)

    def __del__(self):
        try:
            self.L.orc3_engine_destroy(self.eng)
            self.L.orc3_env_destroy(self.env)
        except Exception:
            pass

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(f"oracle3 error {rc}: {self.L.orc3_last_error().decode()}")

    def tables(self):
        E = self.E
        vac, fw, c = np.zeros(9 * E), np.zeros(6 * E), np.zeros(6)
        self.L.orc3_env_tables(self.env, _ptr(vac), _ptr(fw), _ptr(c))
        return dict(vac3=vac.reshape(E, 9), fw6=fw.reshape(6, E), couplings6=c)

    def get_state(self):
        out = np.zeros(self.n)
        self.L.orc3_get_state(self.eng, _ptr(out))
        return out

    def set_state(self, mode1):
        a = np.ascontiguousarray(mode1, dtype=np.float64).ravel()
        self.L.orc3_set_state(self.eng, _ptr(a))

    def trial_step(self, r, dr):
        err = C.c_double()
        self._check(self.L.orc3_trial_step(self.eng, r, dr, C.byref(err)))
        return err.value

    def run(self, r=None, dr=None, it=0, ts=None):
        v = self.cfg.values
        c = _Ctl(dr=v["dr"] if dr is None else dr, dr_max=v["max_dr"], dr_min=v["min_dr"],
                 eps0=v["eps0"], kappa=v["kappa"], r=v["R0"] if r is None else r, R0=v["R0"],
                 Rn=v["Rn"], iter=it, Ts=v["Ts"] if ts is None else ts)
        s = _Summary()
        self._check(self.L.orc3_run(self.eng, C.byref(c), C.byref(s)))
        return dict(final_r=s.final_r, iterations=s.iterations, accepted=s.accepted,
                    rejected=s.rejected, final_max_norm_dev=s.final_max_norm_dev)

    def expm(self, h9, tau):
        h9 = np.ascontiguousarray(h9, dtype=np.float64)
        out = np.zeros(18)
        self.L.orc3_expm(_ptr(h9), tau, _ptr(out))
        return out[0::2].reshape(3, 3) + 1j * out[1::2].reshape(3, 3)


def make_partitions(length: int, workers: int):
    out = (C.c_int * (2 * workers))()
    if _olib().orc_make_partitions(length, workers, out) != 0:
        raise ValueError(_olib().orc_last_error().decode())
    return [(out[2 * w], out[2 * w + 1]) for w in range(workers)]


class Oracle:
    """C restatement engine over the theta partition [t_lo, t_hi)."""

    def __init__(self, cfg, t_lo: int | None = None, t_hi: int | None = None):
        self.L = L = _olib()
        self.cfg = cfg
        self.params = params_from_config(cfg)
        env = C.c_void_p()
        if L.orc_env_create(C.byref(self.params), C.byref(env)) != 0:
            raise RuntimeError(L.orc_last_error().decode())
        self.env = env
        p = self.params
        if p.model == 0:
            self.T, self.P = 1, 1
        else:
            self.T, self.P = p.abins, (p.pbins if p.model >= 2 else 1)
        self.E = p.ebins
        self.t_lo = 0 if t_lo is None else t_lo
        self.t_hi = self.T if t_hi is None else t_hi
        eng = C.c_void_p()
        if L.orc_engine_create(env, self.t_lo, self.t_hi, C.byref(eng)) != 0:
            raise RuntimeError(L.orc_last_error().decode())
        self.eng = eng
        self.n = (self.t_hi - self.t_lo) * self.P * 16 * self.E
        L.orc_init_states(eng)

    def __del__(self):
        try:
            self.L.orc_engine_destroy(self.eng)
            self.L.orc_env_destroy(self.env)
        except Exception:
            pass

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(f"oracle error {rc}: {self.L.orc_last_error().decode()}")

    def tables(self) -> dict:
        T, P, E = self.T, self.P, self.E
        t = dict(cos2=np.zeros(T), sin0=np.zeros(T), cphi=np.zeros(P), sphi=np.zeros(P),
                 vac11=np.zeros(E), vac12=np.zeros(E), fw=np.zeros(4 * E),
                 couplings=np.zeros(4), emean=np.zeros(4))
        self.L.orc_env_tables(self.env, *[_ptr(t[k]) for k in (
            "cos2", "sin0", "cphi", "sphi", "vac11", "vac12", "fw", "couplings", "emean")])
        t["fw"] = t["fw"].reshape(4, E)
        return t

    def init_states(self):
        self.L.orc_init_states(self.eng)

    def set_state(self, mode1):
        a = np.ascontiguousarray(mode1, dtype=np.float64).ravel()
        assert a.size == self.n
        self.L.orc_set_state(self.eng, _ptr(a))

    def get_state(self):
        out = np.zeros(self.n)
        self.L.orc_get_state(self.eng, _ptr(out))
        return out

    def prepare(self, r, dr):
        self._check(self.L.orc_prepare(self.eng, r, dr))

    def stage(self, k):
        out = np.zeros(24)
        self._check(self.L.orc_stage(self.eng, k, _ptr(out)))
        return out[: (24 if k == 1 else 12 if k in (0, 2) else 1)]

    def stage_set(self, k, total):
        buf = np.zeros(24)
        buf[: len(total)] = total
        self._check(self.L.orc_stage_set(self.eng, k, _ptr(buf)))

    def commit(self):
        self.L.orc_commit(self.eng)

    def trial_step(self, r, dr):
        err = C.c_double()
        self._check(self.L.orc_trial_step(self.eng, r, dr, C.byref(err)))
        return err.value

    def run(self, r=None, dr=None, it=0, ts=None):
        v = self.cfg.values
        c = _Ctl(dr=v["dr"] if dr is None else dr, dr_max=v["max_dr"], dr_min=v["min_dr"],
                 eps0=v["eps0"], kappa=v["kappa"], r=v["R0"] if r is None else r, R0=v["R0"],
                 Rn=v["Rn"], iter=it, Ts=v["Ts"] if ts is None else ts)
        s = _Summary()
        self._check(self.L.orc_run(self.eng, C.byref(c), C.byref(s)))
        return dict(final_r=s.final_r, iterations=s.iterations, accepted=s.accepted,
                    rejected=s.rejected, final_max_norm_dev=s.final_max_norm_dev,
                    termination={1: "radius", 2: "iterations"}.get(s.termination, "?"))

    def evolve_bin(self, h, dl, psi):
        h = np.ascontiguousarray(h, dtype=np.float64)
        psi = np.ascontiguousarray(psi, dtype=np.float64)
        out = np.zeros(4)
        self.L.orc_evolve_bin(_ptr(h), dl, _ptr(psi), _ptr(out))
        return out

    def hvv_from_rows(self, r, rows):
        rows = np.ascontiguousarray(rows, dtype=np.float64)
        ntraj = (self.t_hi - self.t_lo) * self.P
        sums, hvv = np.zeros(12), np.zeros((ntraj, 3))
        self._check(self.L.orc_hvv_from_rows(self.eng, r, _ptr(rows), _ptr(sums), _ptr(hvv)))
        return sums, hvv


def oracle_fermi_integral(k, eta):
    return _olib().orc_fermi_integral(k, eta)


def oracle_init_state(species, ebins, eps, seed):
    out = np.zeros(4 * ebins)
    _olib().orc_init_state(species, ebins, eps, seed, _ptr(out))
    return out.reshape(4, ebins)


if __name__ == "__main__":  # pragma: no cover
    build(quiet=False)
    sys.exit(0)
