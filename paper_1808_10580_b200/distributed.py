"""Multi-GPU forward map: one process per GPU, torch.distributed over NCCL.

Particle sharding for a single evaluation: the N_p particles
of every observation are cut into aligned chunks of SMC_CHUNK (1024); rank r
owns the contiguous chunk range chunk_range(C, r, W).  Each rank runs the
fused particle kernel on its range and reduces every chunk with the exact
pairwise tree (executor.cpp:11-26).  The only exchange is an all-gather of the
tiny per-chunk partial sums (N_o x C doubles) — once for the sums, once for
the squared deviations of the two-pass variance (executor.cpp:104-112).
Every rank then finishes the same tree over all chunks, so the estimates are
bit-identical for any world size, including 1.

Sample sharding for batched evaluation needs no collective: rank r evaluates
its contiguous block of parameter samples.

The exchange logic is written against a small `ShardOps` interface so the
same code runs on the GPU (DeviceOps: the C ABI + NCCL) and, in the CPU tests,
with a numpy restatement of the chunk tree over gloo.
"""
from __future__ import annotations

import ctypes as C
from typing import Protocol

import numpy as np

from . import _abi as A
from .api import AdProblemSpec, Context, ParticleEstimate, _check, default_context

CHUNK = A.SMC_CHUNK


def num_chunks(n_particles: int) -> int:
    return (n_particles + CHUNK - 1) // CHUNK


def chunk_range(n_chunks: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced chunk range of `rank` (chunk-aligned shards keep
    every partial an aligned subtree of the reference's pairwise tree)."""
    return (n_chunks * rank) // world, (n_chunks * (rank + 1)) // world


def estimates_from_sums(sums: np.ndarray, sumsq: np.ndarray, n: int) -> list[ParticleEstimate]:
    """reduce_observation's tail (executor.cpp:103-116) for all-valid particles."""
    nd = float(n)
    out = []
    for s, q in zip(sums, sumsq):
        mean = s / nd
        se = float(np.sqrt((q / (nd - 1.0)) / nd)) if n > 1 else 0.0
        out.append(ParticleEstimate(float(mean), se, n, 0, 0.0))
    return out


class ShardOps(Protocol):
    def partials(self, begin: int, end: int): ...           # [n_obs][end-begin] chunk sums (this rank)
    def sq_partials(self, means, begin: int, end: int): ...  # [n_obs][end-begin] chunk sums of (v-mean)^2
    def finish(self, partials) -> np.ndarray: ...           # [n_obs][C] -> [n_obs] tree sums
    def all_gather(self, local, counts: list[int]): ...     # rank-ordered concat along axis 1


def sharded_estimates(ops: ShardOps, n_particles: int, rank: int, world: int) -> list[ParticleEstimate]:
    n_chunks = num_chunks(n_particles)
    counts = [chunk_range(n_chunks, r, world)[1] - chunk_range(n_chunks, r, world)[0] for r in range(world)]
    b, e = chunk_range(n_chunks, rank, world)
    full = ops.all_gather(ops.partials(b, e), counts)
    sums = ops.finish(full)
    means = ops.divide(sums, n_particles)
    fullsq = ops.all_gather(ops.sq_partials(means, b, e), counts)
    sumsq = ops.finish(fullsq)
    return estimates_from_sums(ops.to_host(sums), ops.to_host(sumsq), n_particles)


class DeviceOps:
    """ShardOps on the GPU: the C ABI for compute, torch.distributed (NCCL)
    for the all-gather, device tensors throughout."""

    def __init__(self, spec: AdProblemSpec, seed: int, ctx: Context | None = None, group=None):
        import torch
        self.torch = torch
        self.ctx = ctx or default_context()
        self.spec, self.seed, self.group = spec, seed, group
        self.pod, self.keep = spec._pod()
        self.n_obs = len(spec.observations)
        self.dev = torch.device("cuda", self.ctx.device)

    def partials(self, begin: int, end: int):
        out = self.torch.empty((self.n_obs, max(end - begin, 1)), dtype=self.torch.float64, device=self.dev)
        _check(self.ctx.lib.smc_ad_shard_partials(self.ctx.handle, C.byref(self.pod), C.c_uint64(self.seed),
                                                  begin, end, C.c_void_p(out.data_ptr())))
        return out[:, : end - begin]

    def sq_partials(self, means, begin: int, end: int):
        out = self.torch.empty((self.n_obs, max(end - begin, 1)), dtype=self.torch.float64, device=self.dev)
        _check(self.ctx.lib.smc_ad_shard_sq_partials(self.ctx.handle, C.c_void_p(means.data_ptr()), self.n_obs,
                                                     begin, end, C.c_void_p(out.data_ptr())))
        return out[:, : end - begin]

    def finish(self, partials):
        partials = partials.contiguous()
        sums = self.torch.empty(self.n_obs, dtype=self.torch.float64, device=self.dev)
        _check(self.ctx.lib.smc_tree_finish(self.ctx.handle, C.c_void_p(partials.data_ptr()), self.n_obs,
                                            partials.shape[1], C.c_void_p(sums.data_ptr())))
        return sums

    def divide(self, sums, n: int):
        # IEEE division, as executor.cpp:103.  Tensor / tensor: dividing by a
        # Python scalar lets ATen multiply by the rounded reciprocal instead,
        # which is off by an ulp for some sums.
        return sums / self.torch.full_like(sums, float(n))

    def all_gather(self, local, counts: list[int]):
        """Rank-ordered concatenation of every rank's [n_obs][count_r] chunk
        sums (NCCL all_gather_into_tensor on device buffers; over a gloo group
        the tensors travel through the host, which the CPU/1-GPU tests use)."""
        torch = self.torch
        import torch.distributed as dist
        world = len(counts)
        if world == 1:
            return local
        width = max(counts)
        on_host = dist.get_backend(self.group) == "gloo"
        dev = torch.device("cpu") if on_host else self.dev
        buf = torch.zeros((self.n_obs, width), dtype=torch.float64, device=dev)
        buf[:, : local.shape[1]] = local.to(dev)
        if on_host:
            parts = [torch.empty_like(buf) for _ in range(world)]
            dist.all_gather(parts, buf, group=self.group)
            gathered = torch.stack(parts)
        else:
            gathered = torch.empty((world, self.n_obs, width), dtype=torch.float64, device=dev)
            dist.all_gather_into_tensor(gathered, buf, group=self.group)
        return torch.cat([gathered[r, :, : counts[r]] for r in range(world)], dim=1).to(self.dev)

    def to_host(self, t) -> np.ndarray:
        return t.double().cpu().numpy()


def observe_ad_sharded(spec: AdProblemSpec, seed: int, rank: int, world: int, ctx: Context | None = None,
                       group=None) -> list[ParticleEstimate]:
    """observe_ad over `world` ranks (call on every rank of the group)."""
    return sharded_estimates(DeviceOps(spec, seed, ctx, group), spec.n_particles, rank, world)


class _EmulatedOps(DeviceOps):
    """All ranks' shards run one after another on one GPU (tests only: no
    kernel waits on another, so this is safe on a single device)."""

    def __init__(self, spec, seed, world, ctx=None):
        super().__init__(spec, seed, ctx)
        self.world = world


def observe_ad_emulated(spec: AdProblemSpec, seed: int, world: int, ctx: Context | None = None):
    """Bit-identity check of the sharded path on one GPU: every rank's partials
    are computed in turn and concatenated in rank order, exactly what the
    all-gather delivers."""
    import torch
    ops = _EmulatedOps(spec, seed, world, ctx)
    n_chunks = num_chunks(spec.n_particles)
    ranges = [chunk_range(n_chunks, r, world) for r in range(world)]
    full = torch.cat([ops.partials(b, e).clone() for b, e in ranges], dim=1)
    sums = ops.finish(full)
    means = ops.divide(sums, spec.n_particles)
    sq = []
    for b, e in ranges:
        ops.partials(b, e)  # recompute this rank's particle values
        sq.append(ops.sq_partials(means, b, e).clone())
    sumsq = ops.finish(torch.cat(sq, dim=1))
    return estimates_from_sums(ops.to_host(sums), ops.to_host(sumsq), spec.n_particles)


def sample_range(n_samples: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block of parameter samples for rank (batched evaluation)."""
    return (n_samples * rank) // world, (n_samples * (rank + 1)) // world
