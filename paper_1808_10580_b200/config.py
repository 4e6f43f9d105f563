"""Run configuration files (config/IO parity).

The reference's JSON config schema and its diagnostics (`include/scalarmc/
config.hpp`, `src/config.cpp:1-652`): the same keys, defaults, validation
order and `ConfigError("<json path>", "<what>")` messages, so a config file
that scalarmc accepts builds the same problem here and one it rejects is
rejected with the same text.  Behaviour kept on purpose:

* objects are checked for unknown keys in sorted key order (nlohmann::json
  objects are std::map-ordered);
* booleans are not numbers; "1.0" is not an integer;
* an error inside the Fourier velocity block is re-wrapped with the block's
  path (`config.cpp:127-132`), including errors of the max_wavenumber value;
* ScalarField / Domain constructor errors keep their std::invalid_argument
  type where the reference lets them escape (bump sharpness) and are wrapped
  where it wraps them (domains, prior, spec validation).

Malformed JSON is a ConfigError at "<origin>:<line>:<col>" like the
reference, but the parser's own message text (Python's json vs nlohmann) and
its exact error position differ.
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from typing import Any, Optional

from . import api as S


class ConfigError(RuntimeError):
    """config.hpp:18-22: `where: what`."""

    def __init__(self, where: str, what: str):
        super().__init__(f"{where}: {what}")
        self.where, self.what = where, what


def _fail(where: str, what: str):
    raise ConfigError(where, what)


# ---------------------------------------------------------------------------
# sections (config.hpp:26-90)
# ---------------------------------------------------------------------------
@dataclass
class McmcSection:
    steps: int = 10000
    beta: float = 0.02
    burn_in: int = 0
    thin: int = 1


@dataclass
class LikelihoodSection:
    data: list = field(default_factory=list)
    noise_std: float = -1.0  # <= 0: 0.1 * RMS of the data
    forward_seed: int = 0


@dataclass
class OptimizeSection:
    centers: list = field(default_factory=list)
    sharpness: float = 4.0
    target: list = field(default_factory=list)
    initial: list = field(default_factory=list)
    options: S.NelderMeadOptions = field(default_factory=S.NelderMeadOptions)


@dataclass
class ReferenceSection:
    galerkin_cutoff: int = 16
    dt_ref: float = -1.0
    fd_grid: int = 257
    field_grid: int = 101


@dataclass
class BenchmarkSection:
    cutoffs: list = field(default_factory=lambda: [8, 16, 32])
    repetitions: int = 5
    n_particles: int = 500
    n_observations: int = 2
    t_final: float = 0.05
    dt: float = 5e-4
    kappa: float = 0.01
    prior_s0: float = 1.0
    prior_alpha: float = 2.5
    seed: int = 0
    run_reference: bool = True


@dataclass
class RunConfig:
    problem: str = "ad"
    velocity: S.VelocityField = field(default_factory=S.VelocityField)
    kappa: float = 0.0
    initial_condition: S.ScalarField = field(default_factory=S.ScalarField)
    forcing: S.ScalarField = field(default_factory=S.ScalarField)
    boundary_data: S.ScalarField = field(default_factory=S.ScalarField)
    domain: S.Domain = field(default_factory=lambda: S.Domain.box((0.0, 0.0), (1.0, 1.0)))
    ad_observations: list = field(default_factory=list)
    bvp_observations: list = field(default_factory=list)
    particles: int = 10000
    dt: float = 0.0
    scheme: S.StepScheme = S.StepScheme.euler_maruyama
    max_steps: int = 10_000_000
    seed: int = 0
    workers: int = 0
    prior: Optional[S.PriorSpec] = None
    likelihood: Optional[LikelihoodSection] = None
    mcmc: Optional[McmcSection] = None
    optimize: Optional[OptimizeSection] = None
    reference: Optional[ReferenceSection] = None
    benchmark: Optional[BenchmarkSection] = None


# ---------------------------------------------------------------------------
# JSON value helpers (config.cpp:17-80)
# ---------------------------------------------------------------------------
def _is_number(j: Any) -> bool:
    return isinstance(j, (int, float)) and not isinstance(j, bool)


def _is_integer(j: Any) -> bool:
    return isinstance(j, int) and not isinstance(j, bool)


def _expect_object(j, where):
    if not isinstance(j, dict):
        _fail(where, "expected an object")


def _reject_unknown_keys(obj: dict, where: str, allowed):
    for key in sorted(obj):  # std::map order
        if key not in allowed:
            _fail(where + "." + key, "unknown key")


def _as_number(j, where) -> float:
    if not _is_number(j):
        _fail(where, "expected a number")
    return float(j)


def _as_integer(j, where) -> int:
    if not _is_integer(j):
        _fail(where, "expected an integer")
    return int(j)


def _as_seed(j, where) -> int:
    if not _is_integer(j):
        _fail(where, "expected an integer seed")
    # get<std::int64_t>() < 0: unsigned values >= 2^63 wrap negative and are rejected too
    if j < 0 or j >= 2 ** 63:
        _fail(where, "seed must be >= 0")
    return int(j)


def _number_or(obj, key, where, fallback) -> float:
    return _as_number(obj[key], where + "." + key) if key in obj else fallback


def _integer_or(obj, key, where, fallback) -> int:
    return _as_integer(obj[key], where + "." + key) if key in obj else fallback


def _as_vec2(j, where) -> S.Vec2:
    if not isinstance(j, list) or len(j) != 2:
        _fail(where, "expected [x1, x2]")
    return S.Vec2(_as_number(j[0], where + "[0]"), _as_number(j[1], where + "[1]"))


def _as_number_list(j, where) -> list:
    if not isinstance(j, list):
        _fail(where, "expected an array of numbers")
    return [_as_number(v, f"{where}[{i}]") for i, v in enumerate(j)]


# ---------------------------------------------------------------------------
# blocks
# ---------------------------------------------------------------------------
def _parse_velocity(j, where) -> S.VelocityField:
    """config.cpp:82-133."""
    _expect_object(j, where)
    kind = j.get("kind")
    if not isinstance(kind, str):
        _fail(where + ".kind", 'expected "constant" or "fourier"')
    if kind == "constant":
        _reject_unknown_keys(j, where, {"kind", "value"})
        if "value" not in j:
            _fail(where + ".value", "missing")
        return S.VelocityField.constant(_as_vec2(j["value"], where + ".value"))
    if kind == "fourier":
        _reject_unknown_keys(j, where, {"kind", "max_wavenumber", "modes"})
        if "max_wavenumber" not in j:
            _fail(where + ".max_wavenumber", "missing")
        modes = j.get("modes")
        if not isinstance(modes, list):
            _fail(where + ".modes", "expected an array")
        vm = []
        for i, m in enumerate(modes):
            mw = f"{where}.modes[{i}]"
            if not isinstance(m, list) or len(m) != 4:
                _fail(mw, "expected [k1, k2, re, im]")
            k1 = _as_integer(m[0], mw + "[0]")
            k2 = _as_integer(m[1], mw + "[1]")
            vm.append(S.VelocityMode(k1, k2, complex(_as_number(m[2], mw + "[2]"), _as_number(m[3], mw + "[3]"))))
        try:
            maxk = _as_integer(j["max_wavenumber"], where + ".max_wavenumber")
            return S.VelocityField.fourier(S.FourierVelocityField(vm, maxk))
        except (ValueError, IndexError, RuntimeError) as e:  # every std::exception, re-wrapped
            _fail(where, str(e))
    _fail(where + ".kind", f'unknown velocity kind "{kind}"')


def _parse_scalar_field(j, where) -> S.ScalarField:
    """config.cpp:152-224."""
    _expect_object(j, where)
    kind = j.get("kind")
    if not isinstance(kind, str):
        _fail(where + ".kind", 'expected "constant", "cosine", "bumps" or "linear"')
    if kind == "constant":
        _reject_unknown_keys(j, where, {"kind", "value"})
        if "value" not in j:
            _fail(where + ".value", "missing")
        return S.ScalarField.constant(_as_number(j["value"], where + ".value"))
    if kind == "cosine":
        _reject_unknown_keys(j, where, {"kind", "terms"})
        terms = j.get("terms")
        if not isinstance(terms, list):
            _fail(where + ".terms", "expected an array")
        out = []
        for i, t in enumerate(terms):
            tw = f"{where}.terms[{i}]"
            _expect_object(t, tw)
            _reject_unknown_keys(t, tw, {"amplitude", "phase", "k", "freq"})
            amplitude = _number_or(t, "amplitude", tw, 1.0)
            phase = _number_or(t, "phase", tw, 0.0)
            if ("k" in t) == ("freq" in t):
                _fail(tw, 'give exactly one of "k" (integer torus mode) or "freq" (radians)')
            if "k" in t:
                ki = _as_vec2(t["k"], tw + ".k")
                freq = S.Vec2(2.0 * math.pi * ki[0], 2.0 * math.pi * ki[1])
            else:
                freq = _as_vec2(t["freq"], tw + ".freq")
            out.append(S.CosineTerm(amplitude, freq, phase))
        return S.ScalarField.cosine_series(out)
    if kind == "linear":
        _reject_unknown_keys(j, where, {"kind", "offset", "gradient"})
        if "gradient" not in j:
            _fail(where + ".gradient", "missing")
        gradient = _as_vec2(j["gradient"], where + ".gradient")
        return S.ScalarField.affine(_number_or(j, "offset", where, 0.0), gradient)
    if kind == "bumps":
        _reject_unknown_keys(j, where, {"kind", "amplitudes", "centers", "sharpness"})
        if "amplitudes" not in j:
            _fail(where + ".amplitudes", "missing")
        centers = j.get("centers")
        if not isinstance(centers, list):
            _fail(where + ".centers", "expected an array")
        amplitudes = _as_number_list(j["amplitudes"], where + ".amplitudes")
        if len(amplitudes) != len(centers):
            _fail(where, "amplitudes and centers must have equal length")
        bumps = [S.Bump(a, _as_vec2(c, f"{where}.centers[{i}]")) for i, (a, c) in enumerate(zip(amplitudes, centers))]
        # the ScalarField ctor's invalid_argument escapes unwrapped (config.cpp:216-217)
        return S.ScalarField.gaussian_bumps(bumps, _number_or(j, "sharpness", where, 4.0))
    _fail(where + ".kind", f'unknown scalar field kind "{kind}"')


def _parse_domain(j, where) -> S.Domain:
    """config.cpp:263-298."""
    _expect_object(j, where)
    kind = j.get("kind")
    if not isinstance(kind, str):
        _fail(where + ".kind", 'expected "torus", "box" or "disk"')
    try:
        if kind == "torus":
            _reject_unknown_keys(j, where, {"kind"})
            return S.Domain.unit_torus()
        if kind == "box":
            _reject_unknown_keys(j, where, {"kind", "lower", "upper"})
            if "lower" not in j or "upper" not in j:
                _fail(where, 'box needs "lower" and "upper"')
            upper = _as_vec2(j["upper"], where + ".upper")  # g++ evaluates call arguments right to left
            lower = _as_vec2(j["lower"], where + ".lower")
            return S.Domain.box(lower, upper)
        if kind == "disk":
            _reject_unknown_keys(j, where, {"kind", "center", "radius"})
            if "center" not in j or "radius" not in j:
                _fail(where, 'disk needs "center" and "radius"')
            radius = _as_number(j["radius"], where + ".radius")
            center = _as_vec2(j["center"], where + ".center")
            return S.Domain.disk(center, radius)
    except ConfigError:
        raise
    except (ValueError, IndexError, RuntimeError) as e:
        _fail(where, str(e))
    _fail(where + ".kind", f'unknown domain kind "{kind}"')


def _parse_scheme(j, where) -> S.StepScheme:
    if not isinstance(j, str):
        _fail(where, 'expected "euler-maruyama" or "milstein"')
    if j == "euler-maruyama":
        return S.StepScheme.euler_maruyama
    if j == "milstein":
        return S.StepScheme.milstein
    _fail(where, f'unknown scheme "{j}"')


_ROOT_KEYS = {"problem", "velocity", "diffusion", "initial_condition", "forcing", "boundary", "domain",
              "observations", "particles", "dt", "scheme", "max_steps", "seed", "workers", "prior", "likelihood",
              "mcmc", "optimize", "reference", "benchmark"}


def parse_config(text: str, origin: str = "<config>") -> RunConfig:
    """parse_config (config.cpp:310-495)."""
    try:
        root = json.loads(text)
    except json.JSONDecodeError as e:
        _fail(f"{origin}:{e.lineno}:{e.colno}", e.msg)
    _expect_object(root, origin)
    _reject_unknown_keys(root, origin, _ROOT_KEYS)
    cfg = RunConfig()
    problem = root.get("problem")
    if not isinstance(problem, str):
        _fail(origin + ".problem", 'expected "ad" or "bvp"')
    if problem not in ("ad", "bvp"):
        _fail(origin + ".problem", f'unknown problem kind "{problem}"')
    cfg.problem = problem

    if "velocity" in root:
        cfg.velocity = _parse_velocity(root["velocity"], origin + ".velocity")
    if "diffusion" in root:
        d, dw = root["diffusion"], origin + ".diffusion"
        _expect_object(d, dw)
        _reject_unknown_keys(d, dw, {"kappa"})
        cfg.kappa = _number_or(d, "kappa", dw, 0.0)
        if cfg.kappa < 0.0:
            _fail(dw + ".kappa", "must be >= 0")
    if "initial_condition" in root:
        cfg.initial_condition = _parse_scalar_field(root["initial_condition"], origin + ".initial_condition")
    if "forcing" in root:
        cfg.forcing = _parse_scalar_field(root["forcing"], origin + ".forcing")
    if "boundary" in root:
        cfg.boundary_data = _parse_scalar_field(root["boundary"], origin + ".boundary")
    if "domain" in root:
        cfg.domain = _parse_domain(root["domain"], origin + ".domain")

    if "observations" in root:
        obs = root["observations"]
        if not isinstance(obs, list):
            _fail(origin + ".observations", "expected an array")
        for i, o in enumerate(obs):
            ow = f"{origin}.observations[{i}]"
            _expect_object(o, ow)
            if cfg.problem == "ad":
                _reject_unknown_keys(o, ow, {"t", "x"})
                if "t" not in o or "x" not in o:
                    _fail(ow, 'observation needs "t" and "x"')
                t = _as_number(o["t"], ow + ".t")
                cfg.ad_observations.append(S.AdObservation(t, _as_vec2(o["x"], ow + ".x")))
            else:
                _reject_unknown_keys(o, ow, {"x"})
                if "x" not in o:
                    _fail(ow, 'observation needs "x"')
                cfg.bvp_observations.append(_as_vec2(o["x"], ow + ".x"))

    cfg.particles = _integer_or(root, "particles", origin, cfg.particles)
    cfg.dt = _number_or(root, "dt", origin, cfg.dt)
    if "scheme" in root:
        cfg.scheme = _parse_scheme(root["scheme"], origin + ".scheme")
    cfg.max_steps = _integer_or(root, "max_steps", origin, cfg.max_steps)
    if "seed" in root:
        cfg.seed = _as_seed(root["seed"], origin + ".seed")
    cfg.workers = _integer_or(root, "workers", origin, cfg.workers)

    if "prior" in root:
        p, pw = root["prior"], origin + ".prior"
        _expect_object(p, pw)
        _reject_unknown_keys(p, pw, {"cutoff", "s0", "alpha"})
        prior = S.PriorSpec(_integer_or(p, "cutoff", pw, 8), _number_or(p, "s0", pw, 1.0),
                            _number_or(p, "alpha", pw, 2.5))
        try:
            prior.validate()
        except ValueError as e:
            _fail(pw, str(e))
        cfg.prior = prior
    if "likelihood" in root:
        l, lw = root["likelihood"], origin + ".likelihood"
        _expect_object(l, lw)
        _reject_unknown_keys(l, lw, {"data", "noise_std", "forward_seed"})
        if "data" not in l:
            _fail(lw + ".data", "missing")
        like = LikelihoodSection(_as_number_list(l["data"], lw + ".data"), _number_or(l, "noise_std", lw, -1.0))
        if "forward_seed" in l:
            like.forward_seed = _as_seed(l["forward_seed"], lw + ".forward_seed")
        cfg.likelihood = like
    if "mcmc" in root:
        m, mw = root["mcmc"], origin + ".mcmc"
        _expect_object(m, mw)
        _reject_unknown_keys(m, mw, {"steps", "beta", "burn_in", "thin"})
        mc = McmcSection()
        mc.steps = _integer_or(m, "steps", mw, mc.steps)
        mc.beta = _number_or(m, "beta", mw, mc.beta)
        mc.burn_in = _integer_or(m, "burn_in", mw, mc.burn_in)
        mc.thin = _integer_or(m, "thin", mw, mc.thin)
        if not (mc.beta > 0.0 and mc.beta <= 1.0):
            _fail(mw + ".beta", "must be in (0, 1]")
        cfg.mcmc = mc
    if "optimize" in root:
        o, ow = root["optimize"], origin + ".optimize"
        _expect_object(o, ow)
        _reject_unknown_keys(o, ow, {"centers", "sharpness", "target", "initial", "x_tol", "f_tol", "max_iter",
                                     "initial_step"})
        opt = OptimizeSection()
        centers = o.get("centers")
        if not isinstance(centers, list):
            _fail(ow + ".centers", "expected an array")
        opt.centers = [_as_vec2(c, f"{ow}.centers[{i}]") for i, c in enumerate(centers)]
        opt.sharpness = _number_or(o, "sharpness", ow, 4.0)
        if "target" in o:
            opt.target = _as_number_list(o["target"], ow + ".target")
        if "initial" in o:
            opt.initial = _as_number_list(o["initial"], ow + ".initial")
        if not opt.initial:
            opt.initial = [0.0] * len(opt.centers)
        nm = opt.options
        nm.x_tol = _number_or(o, "x_tol", ow, nm.x_tol)
        nm.f_tol = _number_or(o, "f_tol", ow, nm.f_tol)
        nm.max_iter = _integer_or(o, "max_iter", ow, nm.max_iter)
        nm.initial_step = _number_or(o, "initial_step", ow, nm.initial_step)
        cfg.optimize = opt
    if "reference" in root:
        r, rw = root["reference"], origin + ".reference"
        _expect_object(r, rw)
        _reject_unknown_keys(r, rw, {"galerkin_cutoff", "dt_ref", "fd_grid", "field_grid"})
        cfg.reference = ReferenceSection(_integer_or(r, "galerkin_cutoff", rw, 16), _number_or(r, "dt_ref", rw, -1.0),
                                         _integer_or(r, "fd_grid", rw, 257), _integer_or(r, "field_grid", rw, 101))
    if "benchmark" in root:
        b, bw = root["benchmark"], origin + ".benchmark"
        _expect_object(b, bw)
        _reject_unknown_keys(b, bw, {"cutoffs", "repetitions", "particles", "observations", "t_final", "dt",
                                     "kappa", "s0", "alpha", "run_reference"})
        bench = BenchmarkSection()
        if "cutoffs" in b:
            if not isinstance(b["cutoffs"], list):
                _fail(bw + ".cutoffs", "expected an array")
            bench.cutoffs = [_as_integer(c, f"{bw}.cutoffs[{i}]") for i, c in enumerate(b["cutoffs"])]
        bench.repetitions = _integer_or(b, "repetitions", bw, bench.repetitions)
        bench.n_particles = _integer_or(b, "particles", bw, bench.n_particles)
        bench.n_observations = _integer_or(b, "observations", bw, bench.n_observations)
        bench.t_final = _number_or(b, "t_final", bw, bench.t_final)
        bench.dt = _number_or(b, "dt", bw, bench.dt)
        bench.kappa = _number_or(b, "kappa", bw, bench.kappa)
        bench.prior_s0 = _number_or(b, "s0", bw, bench.prior_s0)
        bench.prior_alpha = _number_or(b, "alpha", bw, bench.prior_alpha)
        if "run_reference" in b:
            if not isinstance(b["run_reference"], bool):
                _fail(bw + ".run_reference", "expected a boolean")
            bench.run_reference = b["run_reference"]
        cfg.benchmark = bench
    return cfg


def load_config(path: str) -> RunConfig:
    """load_config (config.cpp:497-503)."""
    try:
        with open(path, encoding="utf-8") as f:
            text = f.read()
    except OSError:
        _fail(path, "cannot open config file")
    return parse_config(text, path)


# ---------------------------------------------------------------------------
# problem builders (config.cpp:567-650)
# ---------------------------------------------------------------------------
def make_ad_spec(cfg: RunConfig) -> S.AdProblemSpec:
    if cfg.problem != "ad":
        raise ConfigError("problem", 'expected an "ad" configuration')
    spec = S.AdProblemSpec(velocity=cfg.velocity, diffusion=S.DiffusionModel.isotropic(cfg.kappa),
                           initial_condition=cfg.initial_condition, observations=list(cfg.ad_observations),
                           dt=cfg.dt, n_particles=cfg.particles, scheme=cfg.scheme)
    try:
        spec.validate()
    except (ValueError, IndexError, RuntimeError) as e:
        raise ConfigError("observations", str(e)) from None
    return spec


def make_bvp_spec(cfg: RunConfig) -> S.BvpProblemSpec:
    if cfg.problem != "bvp":
        raise ConfigError("problem", 'expected a "bvp" configuration')
    spec = S.BvpProblemSpec(velocity=cfg.velocity, diffusion=S.DiffusionModel.isotropic(cfg.kappa),
                            forcing=cfg.forcing, boundary_data=cfg.boundary_data, domain=cfg.domain,
                            observations=list(cfg.bvp_observations), dt=cfg.dt, n_particles=cfg.particles,
                            scheme=cfg.scheme, max_steps=cfg.max_steps)
    try:
        spec.validate()
    except (ValueError, IndexError, RuntimeError) as e:
        raise ConfigError("observations", str(e)) from None
    return spec


def make_likelihood(cfg: RunConfig) -> S.LikelihoodSpec:
    if cfg.prior is None:
        raise ConfigError("prior", "section required for sampling")
    if cfg.likelihood is None:
        raise ConfigError("likelihood", "section required for sampling")
    data = list(cfg.likelihood.data)
    forward = make_ad_spec(cfg)
    if cfg.likelihood.noise_std > 0.0:
        noise_std = cfg.likelihood.noise_std
    else:
        ss = 0.0
        for y in data:
            ss += y * y
        rms = math.sqrt(ss / len(data)) if data else 0.0
        noise_std = 0.1 * rms
        if not noise_std > 0.0:
            raise ConfigError("likelihood.noise_std", "default rule needs nonzero data")
    like = S.LikelihoodSpec(data=data, noise_std=noise_std, forward=forward,
                            forward_seed=cfg.likelihood.forward_seed)
    try:
        like.validate()
    except (ValueError, IndexError, RuntimeError) as e:
        raise ConfigError("likelihood", str(e)) from None
    return like


def make_forcing_control(cfg: RunConfig) -> S.ForcingControl:
    if cfg.optimize is None:
        raise ConfigError("optimize", "section required for optimization")
    control = S.ForcingControl(initial_amplitudes=list(cfg.optimize.initial), centers=list(cfg.optimize.centers),
                               sharpness=cfg.optimize.sharpness, target=list(cfg.optimize.target),
                               observation_points=list(cfg.bvp_observations))
    try:
        control.validate()
    except ValueError as e:
        raise ConfigError("optimize", str(e)) from None
    return control
