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
    """A device context (stream + persistent buffers), smc_ctx.

    Context(device): one GPU.  Context(devices=[0, 1, ...]): one process
    driving several GPUs (smc_create_multi); the forward maps then shard over
    them and return the same bits as one GPU.  Context.for_rank(...): one GPU
    of a one-process-per-GPU group (smc_create_rank; see
    distributed.rank_context for the torch.distributed plumbing)."""

    def __init__(self, device: int | None = None, *, devices: Sequence[int] | None = None):
        self.lib = A.load_library()
        h = C.c_void_p()
        if devices is not None:
            devs = (C.c_int * len(devices))(*[int(d) for d in devices])
            _check(self.lib.smc_create_multi(len(devices), devs, C.byref(h)))
            device = int(devices[0])
        else:
            if device is None:
                device = int(os.environ.get("LOCAL_RANK", "0"))
            _check(self.lib.smc_create(device, C.byref(h)))
        self.device = device
        self.handle = h

    @classmethod
    def for_rank(cls, device: int, rank: int, world: int, unique_id: bytes) -> "Context":
        """Collective over the `world` ranks (ncclCommInitRank): every rank
        calls it with the unique id rank 0 got from nccl_unique_id()."""
        self = cls.__new__(cls)
        self.lib = A.load_library()
        h = C.c_void_p()
        uid = (C.c_uint8 * A.SMC_UNIQUE_ID_BYTES).from_buffer_copy(bytes(unique_id))
        _check(self.lib.smc_create_rank(int(device), int(rank), int(world), uid, C.byref(h)))
        self.device = int(device)
        self.handle = h
        return self

    def group(self) -> dict:
        """World size, this context's rank, local devices and exchange kind."""
        g = A.smc_group_desc()
        _check(self.lib.smc_group_query(self.handle, C.byref(g)))
        return {"world": g.world, "rank": g.rank, "n_local": g.n_local, "nccl": bool(g.nccl),
                "devices": [d for d in g.devices if d >= 0]}

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

    def fp32_peak_tflops(self, ms: float = 200.0) -> float:
        out = C.c_double()
        _check(self.lib.smc_fp32_peak(self.handle, ms, C.byref(out)))
        return out.value


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId (rank 0 of a smc_create_rank group)."""
    buf = (C.c_uint8 * A.SMC_UNIQUE_ID_BYTES)()
    _check(A.load_library().smc_nccl_unique_id(buf))
    return bytes(buf)


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


# The callers above the forward maps live in their own modules (mirroring the
# reference's inference / optimize / galerkin headers); re-exported here.
from .inference import (ChainConfig, LikelihoodSpec, PriorSpec, prior_draw, run_chains,  # noqa: E402,F401
                        velocity_from_coefficients)
from .optimize import (ForcingBasis, ForcingControl, NelderMeadOptions, _control_spec, forcing_basis,  # noqa: E402,F401
                       forcing_cost, nelder_mead, optimize_forcing)
from .galerkin import (GalerkinBasis, GalerkinResult, galerkin_field_grid, galerkin_solve_ad,  # noqa: E402,F401
                       galerkin_spectral_radius)
