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

Walker sharding for a single Dirichlet evaluation (observe_bvp_sharded): rank
r runs its walker range of every observation; the per-walker results are
all-gathered in walker order and reduced once (the reference compacts valid
walkers before its tree, so partial sums would not be split-invariant).

The exchange logic is written against a small `ShardOps` interface so the
same code runs on the GPU (DeviceOps: the C ABI + NCCL) and, in the CPU tests,
with a numpy restatement of the chunk tree over gloo.
"""
from __future__ import annotations

import ctypes as C
from typing import Protocol

import numpy as np

from . import _abi as A
from .api import AdProblemSpec, BvpProblemSpec, Context, ParticleEstimate, _check, default_context

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
        buf = torch.zeros((self.n_obs, width), dtype=local.dtype, device=dev)
        buf[:, : local.shape[1]] = local.to(dev)
        if on_host:
            parts = [torch.empty_like(buf) for _ in range(world)]
            dist.all_gather(parts, buf, group=self.group)
            gathered = torch.stack(parts)
        else:
            gathered = torch.empty((world, self.n_obs, width), dtype=local.dtype, device=dev)
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


# ---------------------------------------------------------------------------
# Dirichlet (BVP) walker sharding (single evaluation)
# ---------------------------------------------------------------------------
def walker_range(n_walkers: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous walker range of every observation for rank."""
    return (n_walkers * rank) // world, (n_walkers * (rank + 1)) // world


class BvpDeviceOps(DeviceOps):
    """Walker sharding of observe_bvp: each rank runs its walker range of every
    observation (smc_bvp_shard_values), the ranks all-gather the per-walker
    results in walker order, and every rank reduces the whole set
    (smc_bvp_reduce_values).  The reference compacts the valid walkers before
    its tree (executor.cpp:93-101), so a walker's tree position depends on
    failures anywhere before it: the exchange carries walker results (C3: 25 x
    1e6 x 17 B over NVLink) rather than partial sums, and the estimates equal
    observe_bvp bit for bit for any split."""

    def __init__(self, spec: BvpProblemSpec, seed: int, ctx: Context | None = None, group=None):
        super().__init__(spec, seed, ctx, group)

    def shard(self, begin: int, end: int):
        torch = self.torch
        span = max(end - begin, 0)
        vals = torch.empty((self.n_obs, span), dtype=torch.float64, device=self.dev)
        aux = torch.empty_like(vals)
        failed = torch.empty((self.n_obs, span), dtype=torch.uint8, device=self.dev)
        _check(self.ctx.lib.smc_bvp_shard_values(self.ctx.handle, C.byref(self.pod), C.c_uint64(self.seed), begin,
                                                 end, C.c_void_p(vals.data_ptr()), C.c_void_p(aux.data_ptr()),
                                                 C.c_void_p(failed.data_ptr())))
        return vals, aux, failed

    def reduce(self, vals, aux, failed) -> list[ParticleEstimate]:
        vals, aux, failed = vals.contiguous(), aux.contiguous(), failed.contiguous()
        out = (A.smc_estimate * self.n_obs)()
        _check(self.ctx.lib.smc_bvp_reduce_values(self.ctx.handle, C.c_void_p(vals.data_ptr()),
                                                  C.c_void_p(aux.data_ptr()), C.c_void_p(failed.data_ptr()),
                                                  vals.shape[1], self.n_obs, out))
        return [ParticleEstimate._from(out[j]) for j in range(self.n_obs)]


def observe_bvp_sharded(spec: BvpProblemSpec, seed: int, rank: int, world: int, ctx: Context | None = None,
                        group=None) -> list[ParticleEstimate]:
    """observe_bvp over `world` ranks by walker ranges (call on every rank)."""
    ops = BvpDeviceOps(spec, seed, ctx, group)
    n = spec.n_particles
    counts = [walker_range(n, r, world)[1] - walker_range(n, r, world)[0] for r in range(world)]
    b, e = walker_range(n, rank, world)
    vals, aux, failed = ops.shard(b, e)
    return ops.reduce(ops.all_gather(vals, counts), ops.all_gather(aux, counts), ops.all_gather(failed, counts))


def observe_bvp_emulated(spec: BvpProblemSpec, seed: int, world: int, ctx: Context | None = None):
    """The walker-sharded path with every rank's range run in turn on one GPU
    and concatenated in rank order (what the all-gather delivers)."""
    import torch
    ops = BvpDeviceOps(spec, seed, ctx)
    parts = [tuple(t.clone() for t in ops.shard(*walker_range(spec.n_particles, r, world))) for r in range(world)]
    return ops.reduce(*(torch.cat([p[i] for p in parts], dim=1) for i in range(3)))


def sample_range(n_samples: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block of parameter samples for rank (batched evaluation)."""
    return (n_samples * rank) // world, (n_samples * (rank + 1)) // world
