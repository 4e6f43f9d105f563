"""Parameter priors, the likelihood and the device-resident multi-chain pCN
driver (include/scalarmc/inference.hpp, src/inference.cpp; SURVEY.md §8(f)
rank 1)."""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field, replace
from typing import Sequence

import numpy as np

from . import _abi as A
from .api import (AdProblemSpec, Context, FourierVelocityField, VelocityField, VelocityMode, _check,
                  default_context, normal_pairs_device, observe_ad, observe_ad_batched)

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


def run_chains(config: ChainConfig, prior: PriorSpec, likelihood: LikelihoodSpec | None, seeds: Sequence[int],
               u0: np.ndarray | None = None, keep_samples: bool = True, keep_trace: bool = True,
               ctx: Context | None = None) -> dict:
    """len(seeds) independent pCN chains on the device (run_chain,
    inference.cpp:170-194): chain c is run_chain(config with seed=seeds[c]),
    and every step evaluates all chains' proposals in one batched forward
    map.  Returns arrays: final_u [B][dim], final_phi [B], map_u [B][dim],
    map_objective [B], accepted [B], acceptance_rate [B], phi_trace
    [B][n_steps], samples [B][n_samples][dim]."""
    ctx = ctx or default_context()
    if likelihood is not None:
        likelihood.validate()
        p, keep = likelihood.forward._pod()
    else:  # run_chain(..., likelihood = nullptr): Phi == 0
        p, keep = None, None
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
    d = np.ascontiguousarray(likelihood.data if likelihood is not None else [0.0], dtype=np.float64)
    u0p = A.dptr(np.ascontiguousarray(u0, dtype=np.float64).reshape(B, dim)) if u0 is not None else A.dptr(None)
    noise = likelihood.noise_std if likelihood is not None else 1.0
    fseed = likelihood.forward_seed if likelihood is not None else 0
    _check(ctx.lib.smc_pcn_chains(ctx.handle, C.byref(p) if p is not None else None, C.byref(prior._pod()),
                                  A.dptr(d), C.c_double(noise), C.c_uint64(fseed), B,
                                  seeds.ctypes.data_as(C.POINTER(C.c_uint64)), u0p, C.byref(cfg), C.byref(out)))
    if keep_trace:
        res["phi_trace"] = res["phi_trace"][:, : config.n_steps]
    if res["samples"] is not None:
        res["samples"] = res["samples"][:, :ns]
    res["acceptance_rate"] = res["accepted"] / max(config.n_steps, 1) if config.n_steps > 0 else np.zeros(B)
    return res
