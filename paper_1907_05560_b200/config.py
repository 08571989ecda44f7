"""`Keyword= value` run configuration, restricted to the keys the hot path reads.

Mirrors ``oscflat::io::RunConfig`` (reference ``include/oscflat/config.hpp:17-99``,
``src/config.cpp:56-179``): one keyword per line, ``#`` starts a comment, unknown
keywords are collected as warnings.  Only the physics / step-control keys the
evolution step consumes are typed here; I/O, autotune and CLI keys are accepted
and ignored (they are out of scope).
"""
from __future__ import annotations

from dataclasses import dataclass, field

MODEL_IDS = {"sa": 0, "single-angle": 0, "bulb": 1, "ebulb": 2, "extended-bulb": 2,
             "plane": 3, "cylinder": 4}  # plane/cylinder: BASELINE configs[3]/[4] (not in the reference)
MATTER_IDS = {"powerlaw": 0, "exp": 1, "sum": 2}  # matter.hpp:9 (Off = 3)
MATTER_OFF = 3

_FLOAT = {
    "Tn", "eps0", "kappa", "dr", "max_dr", "min_dr", "dm2", "theta", "R0", "Rn", "E0", "E1",
    "hvvScale", "perturb", "Ye", "nb0", "Rv", "Mns", "gs", "S", "hNS",
    "Lve", "Lvae", "Lvt", "Lvat", "Tve", "Tvae", "Tvt", "Tvat", "Eve", "Evae", "Evt", "Evat",
    "eta_ve", "eta_vae", "eta_vt", "eta_vat",
    # 3-flavour extension (BASELINE configs[1]; the reference accepts Flvs = 2 only)
    "dm2_21", "dm2_31", "theta12", "theta13", "theta23", "deltaCP",
    "Lvtau", "Lvatau", "Tvtau", "Tvatau", "Evtau", "Evatau", "eta_vtau", "eta_vatau",
}
_INT = {"Ts", "Abins", "Pbins", "Ebins", "SPoints", "Flvs", "lanes", "hasMatter"}
_STR = {"model", "matterProfile"}
# Keys of the reference vocabulary that do not touch the evolution step.
_IGNORED = {
    "dumpMode", "filePrefix", "newFile_step", "sync_step", "r_step1", "r_step2", "t_step1",
    "t_step2", "itr_step1", "itr_step2", "designatedWriter", "start_beam", "end_beam",
    "multiNodeBench", "minNodes", "maxNodes", "ratio_min", "ratio_max", "ratio_step",
    "knee_threshold", "cpu_threads", "accel_threads", "cpu_per_beam_us", "accel_per_beam_us",
}

_DEFAULTS = dict(  # config.hpp:19-99
    Tn=0.0, Ts=0, eps0=1e-8, kappa=0.8, dr=1e-3, max_dr=1.0, min_dr=1e-12, dm2=0.0, theta=0.0,
    R0=0.0, Rn=0.0, E0=0.0, E1=0.0, Abins=1, Pbins=1, Ebins=1, SPoints=1, Flvs=2, model="bulb",
    hvvScale=1.0, perturb=0.0, lanes=1, hasMatter=0, matterProfile="sum", Ye=0.0, nb0=0.0,
    Rv=10.0, Mns=1.4, gs=1.0, S=100.0, hNS=1.0,
    Lve=-1.0, Lvae=-1.0, Lvt=-1.0, Lvat=-1.0, Tve=-1.0, Tvae=-1.0, Tvt=-1.0, Tvat=-1.0,
    Eve=-1.0, Evae=-1.0, Evt=-1.0, Evat=-1.0, eta_ve=0.0, eta_vae=0.0, eta_vt=0.0, eta_vat=0.0,
)


class ConfigError(ValueError):
    """Mirrors oscflat::ConfigError (types.hpp:43-45)."""


@dataclass
class RunConfig:
    values: dict = field(default_factory=lambda: dict(_DEFAULTS))
    provided: set = field(default_factory=set)
    warnings: list = field(default_factory=list)

    def __getattr__(self, k):
        v = self.__dict__.get("values")
        if v is not None and k in v:
            return v[k]
        raise AttributeError(k)

    def set(self, key: str, value: str) -> None:
        if key in _FLOAT:
            try:
                self.values[key] = float(value)
            except ValueError as e:
                raise ConfigError(f"bad value for '{key}': {value}") from e
        elif key in _INT:
            try:
                self.values[key] = int(float(value)) if "e" in value.lower() else int(value)
            except ValueError as e:
                raise ConfigError(f"bad value for '{key}': {value}") from e
        elif key in _STR:
            self.values[key] = value
        elif key in _IGNORED:
            self.values[key] = value  # (kept verbatim for render)
        else:
            raise KeyError(key)
        self.provided.add(key)

    def override(self, key_value: str) -> "RunConfig":
        """io::apply_override (config.cpp:181-191)."""
        if "=" not in key_value:
            raise ConfigError("override must be key=value, got: " + key_value)
        k, v = key_value.split("=", 1)
        try:
            self.set(k.strip(), v.strip())
        except KeyError:
            raise ConfigError(f"override: unknown keyword '{k.strip()}'") from None
        return self

    # -- derived ---------------------------------------------------------
    @property
    def model_id(self) -> int:
        m = self.values["model"]
        if m not in MODEL_IDS:
            raise ConfigError("model must be one of sa|bulb|ebulb|plane|cylinder, got: " + m)
        return MODEL_IDS[m]

    @property
    def matter_id(self) -> int:
        if self.values["hasMatter"] == 0:
            return MATTER_OFF
        p = self.values["matterProfile"]
        if p not in MATTER_IDS:
            raise ConfigError("matterProfile must be powerlaw|exp|sum, got: " + p)
        return MATTER_IDS[p]

    def tau(self, name: str) -> list:
        """3-flavour tau-sector spectrum keys; default to the x species."""
        keys = {"L": (("Lvtau", "Lvt"), ("Lvatau", "Lvat")),
                "T": (("Tvtau", "Tvt"), ("Tvatau", "Tvat")),
                "E": (("Evtau", "Evt"), ("Evatau", "Evat")),
                "eta": (("eta_vtau", "eta_vt"), ("eta_vatau", "eta_vat"))}[name]
        return [self.values[k] if k in self.provided else self.values[d] for k, d in keys]

    def species(self, name: str) -> list:
        keys = {"L": ("Lve", "Lvae", "Lvt", "Lvat"), "T": ("Tve", "Tvae", "Tvt", "Tvat"),
                "E": ("Eve", "Evae", "Evt", "Evat"),
                "eta": ("eta_ve", "eta_vae", "eta_vt", "eta_vat")}[name]
        return [self.values[k] for k in keys]

    def require_runnable(self) -> None:
        """io::require_runnable (config.cpp:287-306)."""
        need = ["dm2", "theta", "R0", "Rn", "dr", "max_dr", "E0", "E1", "Abins", "Ebins",
                "eps0", "kappa", "Rv", "Lve", "Lvae", "Lvt", "Lvat"]
        missing = [k for k in need if k not in self.provided]
        for t, e in zip(("Tve", "Tvae", "Tvt", "Tvat"), ("Eve", "Evae", "Evt", "Evat")):
            if t not in self.provided and e not in self.provided:
                missing.append(f"{t}|{e}")
        if self.values["hasMatter"]:
            prof = self.values["matterProfile"]
            need_m = ["Ye"]
            if prof in ("exp", "sum"):
                need_m += ["nb0", "hNS"]
            if prof in ("powerlaw", "sum"):
                need_m += ["Mns", "gs", "S"]
            missing += [k for k in need_m if k not in self.provided]
        if missing:
            raise ConfigError("config leaves required keys uninitialized: " + " ".join(missing))
        v = self.values
        if not v["R0"] < v["Rn"]:
            raise ConfigError("config: need R0 < Rn")
        if not v["E0"] < v["E1"]:
            raise ConfigError("config: need E0 < E1")
        if min(v["Abins"], v["Pbins"], v["Ebins"]) < 1:
            raise ConfigError("config: Abins, Pbins, Ebins must be >= 1")
        if v["Flvs"] not in (2, 3):
            raise ConfigError("config: Flvs must be 2 or 3")
        if v["Flvs"] == 3 and self.model_id > 1:
            raise ConfigError("config: Flvs= 3 supports the sa and bulb models")
        if not (0.0 < v["kappa"] <= 1.0):
            raise ConfigError("config: kappa must be in (0, 1]")
        if not v["eps0"] > 0.0:
            raise ConfigError("config: eps0 must be > 0")
        if v["R0"] < v["Rv"] and self.model_id != 3:
            raise ConfigError("config: R0 must be >= Rv")
        self.model_id
        self.matter_id

    def render(self) -> str:
        """Canonical text (only provided keys, so the reference parses it identically)."""
        out = []
        for k in sorted(self.provided):
            val = self.values.get(k)
            if isinstance(val, float):
                out.append(f"{k}= {val!r}")
            elif val is not None:
                out.append(f"{k}= {val}")
        return "\n".join(out) + "\n"


def parse_config(text: str) -> RunConfig:
    """io::parse_config (config.cpp:140-171)."""
    cfg = RunConfig()
    for lineno, line in enumerate(text.splitlines(), 1):
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise ConfigError(f"config line {lineno}: expected 'Keyword= value', got: {line}")
        k, v = line.split("=", 1)
        k, v = k.strip(), v.strip()
        try:
            cfg.set(k, v)
        except KeyError:
            cfg.warnings.append(f"unknown keyword '{k}' (line {lineno}) ignored")
    return cfg


# ---------------------------------------------------------------------------
# BASELINE.json configs expressed in the reference vocabulary.
# Fixed-step mode is eps0=1e30, dr=max_dr=(Rn-R0)/steps, Ts=steps
# (test_solver.cpp:123-136).
_COMMON = """\
E0= 1
E1= 80
Tve= 2.76
Tvae= 4.01
Tvt= 6.26
Tvat= 6.26
eta_ve= 0
eta_vae= 0
eta_vt= 0
eta_vat= 0
Lve= 1e51
Lvae= 1e51
Lvt= 1e51
Lvat= 1e51
Rv= 10
dm2= -2.35e-3
theta= 0.1
kappa= 0.8
eps0= 1e30
"""

BASELINE_CONFIGS = {
    # configs[0]: bulb, 256 angle bins x 100 energy bins, r = 10 -> 250 km, 2000 steps
    "configs0": _COMMON + "model= bulb\nAbins= 256\nPbins= 1\nEbins= 100\nhasMatter= 0\n"
    "perturb= 1e-10\nR0= 10\nRn= 250\ndr= 0.12\nmax_dr= 0.12\nTs= 2000\n",
    # configs[2]: large bulb, 4096 angle bins x 256 energy bins, 1000 steps
    "configs2": _COMMON + "model= bulb\nAbins= 4096\nPbins= 1\nEbins= 256\nhasMatter= 0\n"
    "perturb= 1e-10\nR0= 10\nRn= 250\ndr= 0.24\nmax_dr= 0.24\nTs= 1000\n",
    # configs[1]: 3-flavour bulb, 512 angle x 128 energy bins, power-law matter
    # normalised to Ye = 0.5, rho = 1e7 g/cm^3 at 100 km (gs scales the
    # reference's 4.2e30 (10 km/r)^3 law: n_b(100 km) = 1e7 / m_u), 4000 fixed
    # steps over 10-250 km (range not given by BASELINE)
    "configs1": _COMMON + "Flvs= 3\nmodel= bulb\nAbins= 512\nPbins= 1\nEbins= 128\n"
    "dm2_21= 7.5e-5\ndm2_31= -2.4e-3\ntheta12= 0.59\ntheta13= 0.15\ntheta23= 0.785\n"
    "deltaCP= 0\nhasMatter= 1\nmatterProfile= powerlaw\nYe= 0.5\nMns= 1.4\nS= 100\n"
    "gs= 1433.8282\nperturb= 1e-10\nR0= 10\nRn= 250\ndr= 0.06\nmax_dr= 0.06\nTs= 4000\n",
    # configs[3]: plane emission, 256 zenith x 64 azimuth x 64 energy bins, 1000
    # fixed steps over 0-200 km, 1e-8 symmetry-breaking noise
    "configs3": _COMMON + "model= plane\nAbins= 256\nPbins= 64\nEbins= 64\nhasMatter= 0\n"
    "perturb= 1e-8\nR0= 0\nRn= 200\ndr= 0.2\nmax_dr= 0.2\nTs= 1000\n",
    # configs[4]: line source (cylinder), 512 polar x 128 axial-tilt x 32 energy
    # bins, 1000 fixed steps in distance from the axis 10-250 km
    "configs4": _COMMON + "model= cylinder\nAbins= 512\nPbins= 128\nEbins= 32\nhasMatter= 0\n"
    "perturb= 1e-8\nR0= 10\nRn= 250\ndr= 0.24\nmax_dr= 0.24\nTs= 1000\n",
}


def baseline_config(name: str, **overrides) -> RunConfig:
    cfg = parse_config(BASELINE_CONFIGS[name])
    for k, v in overrides.items():
        cfg.override(f"{k}={v}")
    return cfg
