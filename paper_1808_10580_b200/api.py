"""Python host mirror of the reference forward-map interface.

Same names, argument meaning and error behaviour as the reference C++ API of
scalarmc (/root/reference/proj/include/scalarmc/*.hpp), bound over the C ABI
(include/scalarmc_b200.h) with ctypes:

    reference (C++)                                this module
    -----------------------------------------      -------------------------------
    observe_ad(spec, seed, workers)                observe_ad(spec, seed, workers)
      (forward_ad.hpp:39-40)
    observe_ad_single(spec, j, seed, workers)      observe_ad_single(...)
      (forward_ad.hpp:43-44)
    observe_bvp(spec, seed, workers)               observe_bvp(...)
      (forward_bvp.hpp:35-36)
    LikelihoodSpec::misfit (inference.hpp:58)      LikelihoodSpec.misfit
    forcing_cost (optimize.hpp:59-60)              forcing_cost
    std::invalid_argument / out_of_range /         ValueError / IndexError /
    runtime_error                                  RuntimeError

plus the batched entry point `observe_ad_batched` (many parameter samples per
launch).  `workers` is accepted and ignored: the device is the context's GPU.
Every forward map runs on the GPU; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field, replace
from enum import IntEnum
from typing import Iterable, NamedTuple, Sequence

import numpy as np

from . import _abi as A


# ---------------------------------------------------------------------------
# value types (geometry.hpp, fields.hpp, executor.hpp)
# ---------------------------------------------------------------------------
class Vec2(NamedTuple):
    x1: float = 0.0
    x2: float = 0.0


Point2 = Vec2


class StepScheme(IntEnum):
    euler_maruyama = A.EULER_MARUYAMA
    milstein = A.MILSTEIN


class Precision(IntEnum):
    fp64 = A.FP64
    fp32 = A.FP32
    fp64_strict = A.FP64_STRICT


@dataclass(frozen=True)
class ParticleEstimate:
    """executor.hpp:13-19."""
    mean: float = 0.0
    std_error: float = 0.0
    n_particles: int = 0
    n_failed: int = 0
    aux_mean: float = 0.0

    @staticmethod
    def _from(e: A.smc_estimate) -> "ParticleEstimate":
        return ParticleEstimate(e.mean, e.std_error, e.n_particles, e.n_failed, e.aux_mean)


class Domain:
    """Domain (geometry.hpp:36-74): unit torus, box or disk."""

    def __init__(self, kind: int, lower=(0.0, 0.0), upper=(1.0, 1.0), center=(0.0, 0.0), radius=0.0):
        self.kind = kind
        self.lower = Vec2(*map(float, lower))
        self.upper = Vec2(*map(float, upper))
        self.center = Vec2(*map(float, center))
        self.radius = float(radius)

    @staticmethod
    def unit_torus() -> "Domain":
        return Domain(A.DOMAIN_TORUS)

    @staticmethod
    def box(lower, upper) -> "Domain":
        if not (lower[0] < upper[0] and lower[1] < upper[1]):
            raise ValueError("Domain::box: lower corner must be strictly below upper")
        return Domain(A.DOMAIN_BOX, lower=lower, upper=upper)

    @staticmethod
    def disk(center, radius: float) -> "Domain":
        if not radius > 0.0:
            raise ValueError("Domain::disk: radius must be positive")
        return Domain(A.DOMAIN_DISK, center=center, radius=radius)

    def is_periodic(self) -> bool:
        return self.kind == A.DOMAIN_TORUS

    def is_bounded(self) -> bool:
        return not self.is_periodic()

    def contains(self, x) -> bool:
        if self.kind == A.DOMAIN_BOX:
            return self.lower[0] < x[0] < self.upper[0] and self.lower[1] < x[1] < self.upper[1]
        if self.kind == A.DOMAIN_DISK:
            q1, q2 = x[0] - self.center[0], x[1] - self.center[1]
            return q1 * q1 + q2 * q2 < self.radius * self.radius
        return True

    def _pod(self) -> A.smc_domain:
        d = A.smc_domain()
        d.kind = self.kind
        d.lower[:] = self.lower
        d.upper[:] = self.upper
        d.center[:] = self.center
        d.radius = self.radius
        return d


@dataclass(frozen=True)
class VelocityMode:
    """fields.hpp:13-17: one stored +/-k representative."""
    k1: int
    k2: int
    coeff: complex


class FourierVelocityField:
    """Divergence-free Fourier velocity (fields.hpp:24-64).  The constructor's
    checks (fields.cpp:35-69) run in the native library."""

    def __init__(self, modes: Iterable[VelocityMode] = (), max_wavenumber: int | None = None):
        modes = [m if isinstance(m, VelocityMode) else VelocityMode(int(m[0]), int(m[1]), complex(m[2]))
                 for m in modes]
        self._empty = max_wavenumber is None and not modes
        self.max_wavenumber = int(max_wavenumber) if max_wavenumber is not None else 0
        self.k = np.ascontiguousarray([[m.k1, m.k2] for m in modes], dtype=np.int32).reshape(-1, 2)
        self.coeff = np.ascontiguousarray([[m.coeff.real, m.coeff.imag] for m in modes],
                                          dtype=np.float64).reshape(-1, 2)
        if not self._empty:
            _check(A.load_library().smc_velocity_validate(C.byref(self._pod())))

    @staticmethod
    def from_arrays(k: np.ndarray, coeff: np.ndarray, max_wavenumber: int) -> "FourierVelocityField":
        f = FourierVelocityField.__new__(FourierVelocityField)
        f._empty = False
        f.max_wavenumber = int(max_wavenumber)
        f.k = np.ascontiguousarray(k, dtype=np.int32).reshape(-1, 2)
        f.coeff = np.ascontiguousarray(coeff, dtype=np.float64).reshape(-1, 2)
        _check(A.load_library().smc_velocity_validate(C.byref(f._pod())))
        return f

    @property
    def n_modes(self) -> int:
        return int(self.k.shape[0])

    def amplitude_bound(self) -> float:
        return float(sum(2.0 * math.hypot(a, b) for a, b in self.coeff))

    def _pod(self) -> A.smc_velocity:
        v = A.smc_velocity()
        if self._empty:  # default-constructed zero field == constant (0, 0)
            v.is_constant = 1
            return v
        v.is_constant = 0
        v.max_wavenumber = self.max_wavenumber
        v.n_modes = self.n_modes
        v.k = A.iptr(self.k)
        v.coeff = A.dptr(self.coeff)
        return v


class VelocityField:
    """VelocityField (fields.hpp:67-86): constant vector or Fourier field."""

    def __init__(self):
        self.is_constant = True
        self.constant_value = Vec2(0.0, 0.0)
        self.fourier_field: FourierVelocityField | None = None

    @staticmethod
    def constant(v) -> "VelocityField":
        f = VelocityField()
        f.constant_value = Vec2(float(v[0]), float(v[1]))
        return f

    @staticmethod
    def fourier(field: FourierVelocityField) -> "VelocityField":
        f = VelocityField()
        f.is_constant = False
        f.fourier_field = field
        return f

    def amplitude_bound(self) -> float:
        if self.is_constant:
            return math.hypot(*self.constant_value)
        return self.fourier_field.amplitude_bound()

    def _pod(self) -> A.smc_velocity:
        if self.is_constant:
            v = A.smc_velocity()
            v.is_constant = 1
            v.constant[:] = self.constant_value
            return v
        return self.fourier_field._pod()


class DiffusionModel:
    """DiffusionModel (fields.hpp:91-116).  Only the isotropic model has a
    device representation; a diagonal std::function model is rejected at
    observe time with ValueError (the reference would run it on the CPU)."""

    def __init__(self, kappa: float = 0.0, diagonal: bool = False):
        self._kappa = kappa
        self._diagonal = diagonal

    @staticmethod
    def isotropic(kappa: float) -> "DiffusionModel":
        if not kappa >= 0.0:
            raise ValueError("DiffusionModel: kappa must be >= 0")
        return DiffusionModel(float(kappa))

    @staticmethod
    def diagonal(*fns) -> "DiffusionModel":
        return DiffusionModel(0.0, diagonal=True)

    def is_isotropic(self) -> bool:
        return not self._diagonal

    def kappa(self) -> float:
        if self._diagonal:
            raise RuntimeError("DiffusionModel: kappa is defined only for isotropic models")
        return self._kappa


@dataclass(frozen=True)
class CosineTerm:
    amplitude: float = 0.0
    freq: Vec2 = Vec2()
    phase: float = 0.0


@dataclass(frozen=True)
class Bump:
    amplitude: float = 0.0
    center: Vec2 = Vec2()


class ScalarField:
    """ScalarField (fields.hpp:121-164): constant, cosine series, Gaussian
    bumps or affine.  __call__ evaluates on the host (test convenience; the
    forward maps evaluate on the device)."""

    def __init__(self, kind=A.SCALAR_CONSTANT, constant=0.0, terms=(), bumps=(), sharpness=4.0,
                 gradient=(0.0, 0.0)):
        self.kind = kind
        self.constant_value = float(constant)
        self.terms = tuple(terms)
        self.bumps = tuple(bumps)
        self.sharpness = float(sharpness)
        self.gradient = Vec2(*map(float, gradient))
        self._arrays()

    def _arrays(self):
        t = self.terms
        self._amp = np.ascontiguousarray([x.amplitude for x in (t or self.bumps)], dtype=np.float64)
        self._freq = np.ascontiguousarray([[x.freq[0], x.freq[1]] for x in t], dtype=np.float64).reshape(-1, 2)
        self._phase = np.ascontiguousarray([x.phase for x in t], dtype=np.float64)
        self._center = np.ascontiguousarray([[b.center[0], b.center[1]] for b in self.bumps],
                                            dtype=np.float64).reshape(-1, 2)

    @staticmethod
    def constant(value: float) -> "ScalarField":
        return ScalarField(A.SCALAR_CONSTANT, constant=value)

    @staticmethod
    def affine(offset: float, gradient) -> "ScalarField":
        return ScalarField(A.SCALAR_LINEAR, constant=offset, gradient=gradient)

    @staticmethod
    def cosine_series(terms: Sequence) -> "ScalarField":
        ts = [t if isinstance(t, CosineTerm) else CosineTerm(float(t[0]), Vec2(*t[1]), float(t[2]) if len(t) > 2 else 0.0)
              for t in terms]
        return ScalarField(A.SCALAR_COSINE, terms=ts)

    @staticmethod
    def cosine_mode(k1: int, k2: int, amplitude: float, phase: float = 0.0) -> "ScalarField":
        tp = 2.0 * math.pi
        return ScalarField.cosine_series([CosineTerm(amplitude, Vec2(tp * k1, tp * k2), phase)])

    @staticmethod
    def gaussian_bumps(bumps: Sequence, sharpness: float = 4.0) -> "ScalarField":
        if not sharpness > 0.0:
            raise ValueError("ScalarField: sharpness must be positive")
        bs = [b if isinstance(b, Bump) else Bump(float(b[0]), Vec2(*b[1])) for b in bumps]
        return ScalarField(A.SCALAR_BUMPS, bumps=bs, sharpness=sharpness)

    def with_bump_amplitudes(self, amplitudes: Sequence[float]) -> "ScalarField":
        if self.kind != A.SCALAR_BUMPS:
            raise RuntimeError("ScalarField: amplitude replacement applies to bump sums only")
        if len(amplitudes) != len(self.bumps):
            raise ValueError("ScalarField: amplitude count mismatch")
        return ScalarField(A.SCALAR_BUMPS, bumps=[Bump(float(a), b.center) for a, b in zip(amplitudes, self.bumps)],
                           sharpness=self.sharpness)

    def __call__(self, x) -> float:
        x1, x2 = float(x[0]), float(x[1])
        if self.kind == A.SCALAR_COSINE:
            s = 0.0
            for t in self.terms:
                s += t.amplitude * math.cos(t.freq[0] * x1 + t.freq[1] * x2 + t.phase)
            return s
        if self.kind == A.SCALAR_BUMPS:
            s = 0.0
            for b in self.bumps:
                d1, d2 = x1 - b.center[0], x2 - b.center[1]
                s += b.amplitude * math.exp(-self.sharpness * (d1 * d1 + d2 * d2))
            return s
        if self.kind == A.SCALAR_LINEAR:
            return self.constant_value + (self.gradient[0] * x1 + self.gradient[1] * x2)
        return self.constant_value

    def _pod(self) -> A.smc_scalar_field:
        f = A.smc_scalar_field()
        f.kind = self.kind
        f.constant = self.constant_value
        f.gradient[:] = self.gradient
        f.sharpness = self.sharpness
        if self.kind == A.SCALAR_COSINE:
            f.n_terms = len(self.terms)
            f.amplitude, f.freq, f.phase = A.dptr(self._amp), A.dptr(self._freq), A.dptr(self._phase)
        elif self.kind == A.SCALAR_BUMPS:
            f.n_terms = len(self.bumps)
            f.amplitude, f.center = A.dptr(self._amp), A.dptr(self._center)
        return f


# ---------------------------------------------------------------------------
# problem specs (forward_ad.hpp:15-34, forward_bvp.hpp:16-30)
# ---------------------------------------------------------------------------
class AdObservation(NamedTuple):
    t: float
    x: Vec2


def _diffusion_kappa(d: DiffusionModel) -> float:
    if not d.is_isotropic():
        raise ValueError("scalarmc_b200: only isotropic diffusion has a device representation")
    return d.kappa()


@dataclass
class AdProblemSpec:
    velocity: VelocityField = field(default_factory=VelocityField)
    diffusion: DiffusionModel = field(default_factory=lambda: DiffusionModel.isotropic(0.0))
    initial_condition: ScalarField = field(default_factory=ScalarField)
    observations: list = field(default_factory=list)
    dt: float = 0.0
    n_particles: int = 10000
    scheme: StepScheme = StepScheme.euler_maruyama
    precision: Precision = Precision.fp64

    def _pod(self) -> tuple[A.smc_ad_problem, list]:
        keep = []
        p = A.smc_ad_problem()
        p.velocity = self.velocity._pod()
        p.kappa = _diffusion_kappa(self.diffusion)
        p.initial_condition = self.initial_condition._pod()
        obs = [o if isinstance(o, AdObservation) else AdObservation(float(o[0]), Vec2(*o[1]))
               for o in self.observations]
        t = np.ascontiguousarray([o.t for o in obs], dtype=np.float64)
        x = np.ascontiguousarray([[o.x[0], o.x[1]] for o in obs], dtype=np.float64).reshape(-1, 2)
        keep += [t, x, self.velocity, self.initial_condition]
        p.n_obs = len(obs)
        p.obs_t, p.obs_x = A.dptr(t), A.dptr(x)
        p.dt = float(self.dt)
        p.n_particles = int(self.n_particles)
        p.scheme = int(self.scheme)
        p.precision = int(self.precision)
        return p, keep

    def resolved_dt(self) -> float:
        p, keep = self._pod()
        out = C.c_double()
        _check(A.load_library().smc_ad_resolved_dt(C.byref(p), C.byref(out)))
        return out.value

    def validate(self) -> None:
        p, keep = self._pod()
        _check(A.load_library().smc_ad_validate(C.byref(p)))


@dataclass
class BvpProblemSpec:
    velocity: VelocityField = field(default_factory=VelocityField)
    diffusion: DiffusionModel = field(default_factory=lambda: DiffusionModel.isotropic(0.0))
    forcing: ScalarField = field(default_factory=ScalarField)
    boundary_data: ScalarField = field(default_factory=ScalarField)
    domain: Domain = field(default_factory=lambda: Domain.box((0.0, 0.0), (1.0, 1.0)))
    observations: list = field(default_factory=list)
    dt: float = 0.0
    n_particles: int = 10000
    scheme: StepScheme = StepScheme.euler_maruyama
    max_steps: int = 10_000_000
    precision: Precision = Precision.fp64

    def _pod(self) -> tuple[A.smc_bvp_problem, list]:
        p = A.smc_bvp_problem()
        p.velocity = self.velocity._pod()
        p.kappa = _diffusion_kappa(self.diffusion)
        p.forcing = self.forcing._pod()
        p.boundary_data = self.boundary_data._pod()
        p.domain = self.domain._pod()
        x = np.ascontiguousarray([[o[0], o[1]] for o in self.observations], dtype=np.float64).reshape(-1, 2)
        p.n_obs = len(self.observations)
        p.obs_x = A.dptr(x)
        p.dt = float(self.dt)
        p.n_particles = int(self.n_particles)
        p.scheme = int(self.scheme)
        p.precision = int(self.precision)
        p.max_steps = int(self.max_steps)
        return p, [x, self.velocity, self.forcing, self.boundary_data]

    def resolved_dt(self) -> float:
        p, keep = self._pod()
        out = C.c_double()
        _check(A.load_library().smc_bvp_resolved_dt(C.byref(p), C.byref(out)))
        return out.value

    def validate(self) -> None:
        p, keep = self._pod()
        _check(A.load_library().smc_bvp_validate(C.byref(p)))


# ---------------------------------------------------------------------------
# device context
# ---------------------------------------------------------------------------
def _check(status: int) -> None:
    if status == A.SMC_OK:
        return
    msg = A.load_library().smc_last_error().decode()
    if status == A.SMC_EINVAL:
        raise ValueError(msg)
    if status == A.SMC_ERANGE:
        raise IndexError(msg)
    raise RuntimeError(msg)


class Context:
    """One CUDA device context (stream + persistent buffers), smc_ctx."""

    def __init__(self, device: int | None = None):
        if device is None:
            device = int(os.environ.get("LOCAL_RANK", "0"))
        self.device = device
        self.lib = A.load_library()
        h = C.c_void_p()
        _check(self.lib.smc_create(device, C.byref(h)))
        self.handle = h

    def close(self):
        if self.handle:
            self.lib.smc_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return int(self.lib.smc_stream(self.handle) or 0)

    def stats(self) -> A.smc_stats:
        s = A.smc_stats()
        _check(self.lib.smc_last_stats(self.handle, C.byref(s)))
        return s

    def fp64_peak_tflops(self, ms: float = 200.0) -> float:
        out = C.c_double()
        _check(self.lib.smc_fp64_peak(self.handle, ms, C.byref(out)))
        return out.value


_contexts: dict[int, Context] = {}


def default_context(device: int | None = None) -> Context:
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", "0"))
    ctx = _contexts.get(device)
    if ctx is None:
        ctx = _contexts[device] = Context(device)
    return ctx


# ---------------------------------------------------------------------------
# forward maps
# ---------------------------------------------------------------------------
def observe_ad(spec: AdProblemSpec, seed: int, workers: int = 1, ctx: Context | None = None) -> list[ParticleEstimate]:
    """observe_ad (forward_ad.hpp:39-40, forward_ad.cpp:53-60) on the GPU."""
    ctx = ctx or default_context()
    p, keep = spec._pod()
    out = (A.smc_estimate * max(p.n_obs, 1))()
    _check(ctx.lib.smc_ad_observe(ctx.handle, C.byref(p), C.c_uint64(seed), out))
    return [ParticleEstimate._from(out[j]) for j in range(p.n_obs)]


def observe_ad_single(spec: AdProblemSpec, obs_index: int, seed: int, workers: int = 1,
                      ctx: Context | None = None) -> ParticleEstimate:
    """observe_ad_single (forward_ad.hpp:43-44, forward_ad.cpp:62-69)."""
    ctx = ctx or default_context()
    p, keep = spec._pod()
    out = A.smc_estimate()
    if obs_index < 0:
        raise IndexError("observe_ad_single: observation index out of range")
    _check(ctx.lib.smc_ad_observe_single(ctx.handle, C.byref(p), C.c_uint64(obs_index), C.c_uint64(seed),
                                         C.byref(out)))
    return ParticleEstimate._from(out)


def observe_bvp(spec: BvpProblemSpec, seed: int, workers: int = 1, ctx: Context | None = None) -> list[ParticleEstimate]:
    """observe_bvp (forward_bvp.hpp:35-36, forward_bvp.cpp:34-49) on the GPU."""
    ctx = ctx or default_context()
    p, keep = spec._pod()
    out = (A.smc_estimate * max(p.n_obs, 1))()
    _check(ctx.lib.smc_bvp_observe(ctx.handle, C.byref(p), C.c_uint64(seed), out))
    return [ParticleEstimate._from(out[j]) for j in range(p.n_obs)]


def observe_bvp_range(spec: BvpProblemSpec, seed: int, obs_begin: int, obs_count: int,
                      ctx: Context | None = None) -> list[ParticleEstimate]:
    """observe_bvp for observations [obs_begin, obs_begin + obs_count) with
    their original stream slots (observation sharding across GPUs)."""
    ctx = ctx or default_context()
    p, keep = spec._pod()
    out = (A.smc_estimate * max(obs_count, 1))()
    _check(ctx.lib.smc_bvp_observe_range(ctx.handle, C.byref(p), C.c_uint64(seed), obs_begin, obs_count, out))
    return [ParticleEstimate._from(out[j]) for j in range(obs_count)]


def observe_ad_batched(spec: AdProblemSpec, prior: "PriorSpec", u: np.ndarray, seed: int,
                       seeds: np.ndarray | None = None, ctx: Context | None = None) -> np.ndarray:
    """Batched AD forward map: row b of u (prior order) -> estimates [B][n_obs]
    as a structured array (mean, std_error, n_particles, n_failed, aux_mean)."""
    ctx = ctx or default_context()
    u = np.ascontiguousarray(u, dtype=np.float64)
    if u.ndim != 2 or u.shape[1] != prior.dimension():
        raise ValueError("velocity_from_coefficients: coefficient size mismatch")
    p, keep = spec._pod()
    B = u.shape[0]
    out = np.zeros((B, p.n_obs), dtype=ESTIMATE_DTYPE)
    sp = None
    if seeds is not None:
        seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
        sp = seeds.ctypes.data_as(C.POINTER(C.c_uint64))
    _check(ctx.lib.smc_ad_observe_batched(ctx.handle, C.byref(p), C.byref(prior._pod()), B, A.dptr(u), sp,
                                          C.c_uint64(seed), out.ctypes.data_as(C.POINTER(A.smc_estimate))))
    return out


ESTIMATE_DTYPE = np.dtype([("mean", "<f8"), ("std_error", "<f8"), ("n_particles", "<i8"),
                           ("n_failed", "<i8"), ("aux_mean", "<f8")])


def ad_particle_values(spec: AdProblemSpec, obs_index: int, seed: int, n: int,
                       ctx: Context | None = None) -> np.ndarray:
    """Per-particle theta_0(X_T) of particles [0, n) of one observation."""
    ctx = ctx or default_context()
    p, keep = spec._pod()
    out = np.empty(n, dtype=np.float64)
    _check(ctx.lib.smc_ad_particle_values(ctx.handle, C.byref(p), obs_index, C.c_uint64(seed), n, A.dptr(out)))
    return out


def bvp_particle_values(spec: BvpProblemSpec, obs_index: int, seed: int, n: int, ctx: Context | None = None):
    ctx = ctx or default_context()
    p, keep = spec._pod()
    vals = np.empty(n, dtype=np.float64)
    aux = np.empty(n, dtype=np.float64)
    failed = np.empty(n, dtype=np.uint8)
    _check(ctx.lib.smc_bvp_particle_values(ctx.handle, C.byref(p), obs_index, C.c_uint64(seed), n, A.dptr(vals),
                                           A.dptr(aux), failed.ctypes.data_as(C.POINTER(C.c_uint8))))
    return vals, aux, failed


def normal_pairs_device(seed: int, obs: int, particle: int, n_blocks: int, ctx: Context | None = None) -> np.ndarray:
    ctx = ctx or default_context()
    out = np.empty((n_blocks, 2), dtype=np.float64)
    _check(ctx.lib.smc_normal_pairs_device(ctx.handle, C.c_uint64(seed), C.c_uint64(obs), C.c_uint64(particle),
                                           n_blocks, A.dptr(out)))
    return out


def philox_device(ctr: np.ndarray, key: np.ndarray, ctx: Context | None = None) -> np.ndarray:
    ctx = ctx or default_context()
    ctr = np.ascontiguousarray(ctr, dtype=np.uint32).reshape(-1, 4)
    key = np.ascontiguousarray(key, dtype=np.uint32).reshape(-1, 2)
    out = np.empty_like(ctr)
    P = C.POINTER(C.c_uint32)
    _check(ctx.lib.smc_philox_device(ctx.handle, ctr.shape[0], ctr.ctypes.data_as(P), key.ctypes.data_as(P),
                                     out.ctypes.data_as(P)))
    return out


# ---------------------------------------------------------------------------
# u -> G callers (inference.hpp, optimize.hpp)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class PriorSpec:
    """PriorSpec (inference.hpp:22-38)."""
    cutoff: int = 8
    s0: float = 1.0
    alpha: float = 2.5

    def validate(self) -> None:
        if self.cutoff < 1:
            raise ValueError("PriorSpec: cutoff must be >= 1")
        if not self.s0 >= 0.0:
            raise ValueError("PriorSpec: s0 must be >= 0")
        if not math.isfinite(self.alpha):
            raise ValueError("PriorSpec: alpha must be finite")

    def modes(self) -> list[tuple[int, int]]:
        """Canonical modes ordered by |k|^2 then (k1, k2) (inference.cpp:24-40)."""
        K = self.cutoff
        out = [(k1, k2) for k1 in range(-K, K + 1) for k2 in range(-K, K + 1)
               if (k1 > 0 or (k1 == 0 and k2 > 0)) and float(k1) * k1 + float(k2) * k2 <= float(K) * K]
        out.sort(key=lambda m: (float(m[0]) * m[0] + float(m[1]) * m[1], m[0], m[1]))
        return out

    def component_stds(self) -> np.ndarray:
        s = [self.s0 * math.pow(math.sqrt(float(a) * a + float(b) * b), -self.alpha) for a, b in self.modes()]
        return np.repeat(np.asarray(s, dtype=np.float64), 2)

    def dimension(self) -> int:
        return 2 * len(self.modes())

    def _pod(self) -> A.smc_prior:
        p = A.smc_prior()
        p.cutoff, p.s0, p.alpha = self.cutoff, self.s0, self.alpha
        return p


def prior_draw(prior: PriorSpec, seed: int, obs_index: int, particle_index: int, ctx: Context | None = None) -> np.ndarray:
    """prior_draw (inference.cpp:55-61) for a fresh NormalStream{seed, obs,
    particle}: u_i = s_i * normal(), normals drawn pairwise (rng.cpp:74-83) on
    the device."""
    prior.validate()
    stds = prior.component_stds()
    z = normal_pairs_device(seed, obs_index, particle_index, len(stds) // 2 + 1, ctx).reshape(-1)
    return stds * z[: len(stds)]


def velocity_from_coefficients(prior: PriorSpec, u: Sequence[float]) -> FourierVelocityField:
    """inference.cpp:63-73."""
    modes = prior.modes()
    u = np.asarray(u, dtype=np.float64)
    if u.shape != (2 * len(modes),):
        raise ValueError("velocity_from_coefficients: coefficient size mismatch")
    return FourierVelocityField.from_arrays(np.asarray(modes, dtype=np.int32), u.reshape(-1, 2), prior.cutoff)


@dataclass
class LikelihoodSpec:
    """LikelihoodSpec (inference.hpp:52-59)."""
    data: list
    noise_std: float = 0.1
    forward: AdProblemSpec = field(default_factory=AdProblemSpec)
    forward_seed: int = 0
    workers: int = 1

    def validate(self) -> None:
        if len(self.data) != len(self.forward.observations):
            raise ValueError("LikelihoodSpec: data length must match observation count")
        if not self.noise_std > 0.0:
            raise ValueError("LikelihoodSpec: noise_std must be positive")

    def misfit(self, prior: PriorSpec, u: Sequence[float]) -> float:
        """Phi(u) = |y - G(u)|^2 / (2 sigma_n^2) (inference.cpp:93-104)."""
        if math.isinf(self.noise_std):
            return 0.0
        spec = replace(self.forward, velocity=VelocityField.fourier(velocity_from_coefficients(prior, u)))
        est = observe_ad(spec, self.forward_seed, self.workers)
        ss = 0.0
        for y, e in zip(self.data, est):
            r = y - e.mean
            ss += r * r
        return ss / (2.0 * self.noise_std * self.noise_std)

    def misfit_batched(self, prior: PriorSpec, U: np.ndarray) -> np.ndarray:
        """Phi for every row of U in one batched launch (common random numbers,
        the same forward_seed for every row, as misfit)."""
        est = observe_ad_batched(self.forward, prior, U, self.forward_seed)
        r = np.asarray(self.data, dtype=np.float64)[None, :] - est["mean"]
        return (r * r).sum(axis=1) / (2.0 * self.noise_std * self.noise_std)


@dataclass
class ChainConfig:
    """ChainConfig (inference.hpp:87-93)."""
    n_steps: int = 10000
    beta: float = 0.02
    burn_in: int = 0
    thin: int = 1
    seed: int = 0


def run_chains(config: ChainConfig, prior: PriorSpec, likelihood: LikelihoodSpec, seeds: Sequence[int],
               u0: np.ndarray | None = None, keep_samples: bool = True, keep_trace: bool = True,
               ctx: Context | None = None) -> dict:
    """len(seeds) independent pCN chains on the device (run_chain,
    inference.cpp:170-194): chain c is run_chain(config with seed=seeds[c]),
    and every step evaluates all chains' proposals in one batched forward
    map.  Returns arrays: final_u [B][dim], final_phi [B], map_u [B][dim],
    map_objective [B], accepted [B], acceptance_rate [B], phi_trace
    [B][n_steps], samples [B][n_samples][dim]."""
    ctx = ctx or default_context()
    likelihood.validate()
    p, keep = likelihood.forward._pod()
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    B, dim = len(seeds), prior.dimension()
    cfg = A.smc_chain_config(config.n_steps, config.beta, config.burn_in, config.thin)
    ns = int(ctx.lib.smc_pcn_num_samples(C.byref(cfg)))
    res = {"final_u": np.zeros((B, dim)), "final_phi": np.zeros(B), "map_u": np.zeros((B, dim)),
           "map_objective": np.zeros(B), "accepted": np.zeros(B, dtype=np.int64)}
    res["phi_trace"] = np.zeros((B, max(config.n_steps, 1))) if keep_trace else None
    res["samples"] = np.zeros((B, max(ns, 1), dim)) if keep_samples and ns > 0 else None
    out = A.smc_chain_outputs(A.dptr(res["final_u"]), A.dptr(res["final_phi"]), A.dptr(res["map_u"]),
                              A.dptr(res["map_objective"]), res["accepted"].ctypes.data_as(C.POINTER(C.c_int64)),
                              A.dptr(res["phi_trace"]), A.dptr(res["samples"]))
    d = np.ascontiguousarray(likelihood.data, dtype=np.float64)
    u0p = A.dptr(np.ascontiguousarray(u0, dtype=np.float64).reshape(B, dim)) if u0 is not None else A.dptr(None)
    _check(ctx.lib.smc_pcn_chains(ctx.handle, C.byref(p), C.byref(prior._pod()), A.dptr(d),
                                  C.c_double(likelihood.noise_std), C.c_uint64(likelihood.forward_seed), B,
                                  seeds.ctypes.data_as(C.POINTER(C.c_uint64)), u0p, C.byref(cfg), C.byref(out)))
    if keep_trace:
        res["phi_trace"] = res["phi_trace"][:, : config.n_steps]
    if res["samples"] is not None:
        res["samples"] = res["samples"][:, :ns]
    res["acceptance_rate"] = res["accepted"] / max(config.n_steps, 1) if config.n_steps > 0 else np.zeros(B)
    return res


@dataclass
class ForcingControl:
    """ForcingControl (optimize.hpp:45-54)."""
    initial_amplitudes: list
    centers: list
    sharpness: float = 4.0
    target: list = field(default_factory=list)
    observation_points: list = field(default_factory=list)

    def validate(self) -> None:
        if not self.centers:
            raise ValueError("ForcingControl: no forcing centers")
        if len(self.initial_amplitudes) != len(self.centers):
            raise ValueError("ForcingControl: amplitude/center count mismatch")
        if len(self.target) != len(self.observation_points):
            raise ValueError("ForcingControl: target and observation lengths must match")
        if not self.sharpness > 0.0:
            raise ValueError("ForcingControl: sharpness must be positive")


def _control_spec(control: ForcingControl, base: BvpProblemSpec, amplitudes: Sequence[float]) -> BvpProblemSpec:
    """control_spec (optimize.cpp:147-157)."""
    return replace(base, forcing=ScalarField.gaussian_bumps(
        [Bump(float(a), Vec2(*c)) for a, c in zip(amplitudes, control.centers)], control.sharpness),
        observations=list(control.observation_points))


@dataclass(frozen=True)
class ForcingBasis:
    """One Dirichlet pass under common random numbers, linear in the bump
    amplitudes F: mean_j(F) = bc[j] - basis[j] . F (smc_bvp_forcing_basis)."""
    bc: np.ndarray        # [n_obs] E[theta_bc(X_tau)]
    basis: np.ndarray     # [n_obs][n_bumps] E[int phi_k(X_t) dt]
    exit_time: np.ndarray # [n_obs]
    n_failed: np.ndarray  # [n_obs]

    def means(self, amplitudes: Sequence[float]) -> np.ndarray:
        return self.bc - self.basis @ np.asarray(amplitudes, dtype=np.float64)


def forcing_basis(control: ForcingControl, base: BvpProblemSpec, seed: int, ctx: Context | None = None) -> ForcingBasis:
    ctx = ctx or default_context()
    control.validate()
    spec = _control_spec(control, base, [1.0] * len(control.centers))
    p, keep = spec._pod()
    nb, no = len(control.centers), len(control.observation_points)
    bc, tau = np.zeros(no), np.zeros(no)
    basis = np.zeros((no, nb))
    nf = np.zeros(no, dtype=np.int64)
    _check(ctx.lib.smc_bvp_forcing_basis(ctx.handle, C.byref(p), C.c_uint64(seed), A.dptr(bc), A.dptr(basis),
                                         A.dptr(tau), nf.ctypes.data_as(C.POINTER(C.c_int64))))
    return ForcingBasis(bc, basis, tau, nf)


@dataclass
class NelderMeadOptions:
    """NelderMeadOptions (optimize.hpp:13-21)."""
    x_tol: float = 1e-6
    f_tol: float = 1e-9
    max_iter: int = 2000
    initial_step: float = 1.0


def nelder_mead(objective, x0: Sequence[float], options: NelderMeadOptions = NelderMeadOptions()) -> dict:
    """nelder_mead (optimize.cpp:37-134): coefficients (1, 2, 0.5, 0.5),
    non-finite values as +inf, stops on simplex diameter < x_tol, value spread
    < f_tol, or max_iter (the reference's algorithm, restated on the host)."""
    dim = len(x0)
    if dim == 0:
        raise ValueError("nelder_mead: empty start point")
    if not all(math.isfinite(v) for v in x0):
        raise ValueError("nelder_mead: non-finite start point")

    def guarded(x):
        v = objective(x)
        return v if math.isfinite(v) else math.inf

    verts = [list(map(float, x0)) for _ in range(dim + 1)]
    for i in range(dim):
        verts[i + 1][i] += options.initial_step
    vals = [guarded(v) for v in verts]

    def sort_simplex():
        nonlocal verts, vals
        order = sorted(range(dim + 1), key=lambda i: vals[i])  # stable, like std::stable_sort
        verts = [verts[i] for i in order]
        vals = [vals[i] for i in order]

    def diameter():
        d = 0.0
        for i in range(1, dim + 1):
            s = 0.0
            for c in range(dim):
                diff = verts[i][c] - verts[0][c]
                s += diff * diff
            d = max(d, math.sqrt(s))
        return d

    sort_simplex()
    trace = [(0, vals[0], list(verts[0]))]
    it, reason = 0, "max_iter"
    while it < options.max_iter:
        if diameter() < options.x_tol:
            reason = "x_tol"
            break
        if math.isfinite(vals[dim]) and vals[dim] - vals[0] < options.f_tol:
            reason = "f_tol"
            break
        centroid = [0.0] * dim
        for i in range(dim):
            for c in range(dim):
                centroid[c] += verts[i][c] / float(dim)

        def along(t):
            return [centroid[c] + t * (centroid[c] - verts[dim][c]) for c in range(dim)]

        refl = along(1.0)
        f_refl = guarded(refl)
        if f_refl < vals[0]:
            exp_ = along(2.0)
            f_exp = guarded(exp_)
            if f_exp < f_refl:
                verts[dim], vals[dim] = exp_, f_exp
            else:
                verts[dim], vals[dim] = refl, f_refl
        elif f_refl < vals[dim - 1]:
            verts[dim], vals[dim] = refl, f_refl
        else:
            outside = f_refl < vals[dim]
            con = along(0.5 if outside else -0.5)
            f_con = guarded(con)
            if f_con < min(vals[dim], f_refl):
                verts[dim], vals[dim] = con, f_con
            else:
                for i in range(1, dim + 1):
                    verts[i] = [verts[0][c] + 0.5 * (verts[i][c] - verts[0][c]) for c in range(dim)]
                    vals[i] = guarded(verts[i])
        sort_simplex()
        it += 1
        trace.append((it, vals[0], list(verts[0])))
    return {"argmin": verts[0], "min_value": vals[0], "iterations": it, "stop_reason": reason, "trace": trace}


def optimize_forcing(control: ForcingControl, base: BvpProblemSpec, options: NelderMeadOptions, seed: int,
                     ctx: Context | None = None) -> dict:
    """optimize_forcing (optimize.cpp:175-185) with every Nelder-Mead vertex
    evaluated from ONE device pass (forcing_basis): under the fixed seed the
    objective |Y - G(F)|_2 is exactly the reference's forcing_cost up to
    summation order (G is linear in F)."""
    control.validate()
    fb = forcing_basis(control, base, seed, ctx)
    Y = np.asarray(control.target, dtype=np.float64)

    def cost(F):
        r = Y - fb.means(F)
        return math.sqrt(float(np.sum(r * r)))
    res = nelder_mead(cost, control.initial_amplitudes, options)
    res["basis"] = fb
    return res


def forcing_cost(amplitudes: Sequence[float], control: ForcingControl, base: BvpProblemSpec, seed: int,
                 workers: int = 1) -> float:
    """|Y - G(F)|_2 with G = observe_bvp under a fixed seed (optimize.cpp:161-173)."""
    control.validate()
    if len(amplitudes) != len(control.centers):
        raise ValueError("forcing_cost: amplitude count mismatch")
    est = observe_bvp(_control_spec(control, base, amplitudes), seed, workers)
    ss = 0.0
    for y, e in zip(control.target, est):
        r = y - e.mean
        ss += r * r
    return math.sqrt(ss)


# ---------------------------------------------------------------------------
# spectral Galerkin reference solver
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class GalerkinBasis:
    """GalerkinBasis (galerkin.hpp:14-18): `box` keeps max(|l1|,|l2|) <= cutoff,
    `disk` keeps |l|_2 <= cutoff."""
    kind: str = "box"
    cutoff: int = 8

    def _pod(self) -> A.smc_galerkin_basis:
        if self.kind not in ("box", "disk"):
            raise ValueError("GalerkinBasis: kind must be 'box' or 'disk'")
        return A.smc_galerkin_basis(0 if self.kind == "box" else 1, int(self.cutoff))

    def modes(self) -> list[tuple[int, int]]:
        lib = A.load_library()
        b = self._pod()
        n = int(lib.smc_galerkin_n_basis(C.byref(b)))
        if n < 0:
            _check(lib.smc_galerkin_modes(C.byref(b), None))
        out = np.zeros((n, 2), dtype=np.int32)
        _check(lib.smc_galerkin_modes(C.byref(b), out.ctypes.data_as(C.POINTER(C.c_int32))))
        return [(int(a), int(c)) for a, c in out]


@dataclass
class GalerkinResult:
    """GalerkinResult (galerkin.hpp:20-27)."""
    observation_values: np.ndarray
    coefficients_at_observations: np.ndarray | None
    final_coefficients: np.ndarray
    basis_modes: list
    dt_used: float
    steps: int


def _basis(basis) -> GalerkinBasis:
    return basis if isinstance(basis, GalerkinBasis) else GalerkinBasis("box", int(basis))


def galerkin_spectral_radius(spec: AdProblemSpec, basis, ctx: Context | None = None) -> float:
    """galerkin_spectral_radius (galerkin.cpp:151-157)."""
    ctx = ctx or default_context()
    p, keep = spec._pod()
    b = _basis(basis)._pod()
    out = C.c_double()
    _check(ctx.lib.smc_galerkin_spectral_radius(ctx.handle, C.byref(p), C.byref(b), C.byref(out)))
    return out.value


def galerkin_solve_ad(spec: AdProblemSpec, basis, dt_ref: float, keep_observation_coefficients: bool = False,
                      ctx: Context | None = None) -> GalerkinResult:
    """galerkin_solve_ad (galerkin.hpp:36-40, galerkin.cpp:159-231) on the
    device; `basis` is a GalerkinBasis or a box cutoff (the int overload)."""
    ctx = ctx or default_context()
    b = _basis(basis)
    modes = b.modes()
    nb = len(modes)
    p, keep = spec._pod()
    vals = np.zeros(len(spec.observations))
    final = np.zeros((nb, 2))
    cat = np.zeros((len(spec.observations), nb, 2)) if keep_observation_coefficients else None
    r = A.smc_galerkin_result(A.dptr(vals), A.dptr(cat), A.dptr(final), 0.0, 0)
    _check(ctx.lib.smc_galerkin_solve_ad(ctx.handle, C.byref(p), C.byref(b._pod()), C.c_double(dt_ref), C.byref(r)))
    to_c = (lambda a: a[..., 0] + 1j * a[..., 1])
    return GalerkinResult(vals, to_c(cat) if cat is not None else None, to_c(final), modes, r.dt_used, int(r.steps))


def galerkin_field_grid(result: GalerkinResult, n: int, basis=None, ctx: Context | None = None) -> np.ndarray:
    """galerkin_field_grid (galerkin.cpp:233-250): n x n grid, row-major,
    x2 fastest (result.basis_modes must be the basis' mode order)."""
    ctx = ctx or default_context()
    if basis is None:
        L = max(max(abs(a), abs(c)) for a, c in result.basis_modes)
        box = len(result.basis_modes) == (2 * L + 1) ** 2
        basis = GalerkinBasis("box" if box else "disk", L)
    b = _basis(basis)._pod()
    c = np.ascontiguousarray(np.stack([result.final_coefficients.real, result.final_coefficients.imag], axis=-1))
    out = np.zeros(int(n) * int(n)) if n >= 2 else np.zeros(1)
    _check(ctx.lib.smc_galerkin_field_grid(ctx.handle, C.byref(b), A.dptr(c), int(n), A.dptr(out)))
    return out
