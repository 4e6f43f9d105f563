"""Multi-GPU forward maps: host plumbing for the C ABI's
multi-device contexts, and the restatement of their shard plans and exchanges
that the CPU tests run over gloo.

The sharding runs inside the library (csrc/capi_group.cu).  A context over
several GPUs — one process driving all of them, `Context(devices=[0, ..., 7])`,
or one process per GPU, `rank_context()` under torchrun — makes observe_ad,
observe_ad_single, observe_bvp, observe_ad_batched and run_chains shard their
work and combine the ranks with a small deterministic exchange (NCCL over
NVLink), on the context's stream, in ONE C-ABI call per evaluation.  Every
rank gets the full result, bit-identical to one GPU for any split:

  observe_ad   units = (observation, 1024-particle chunk) pairs, contiguous
               ranges balanced by particle-steps (unit_bounds).  Each rank
               sends its units' exact chunk partials of the reference's
               pairwise tree (executor.cpp:11-26); all ranks finish the tree,
               divide, and repeat for the squared deviations (:103-112).
               Exchange: 2 x n_obs x chunks doubles.
  observe_bvp  walker ranges per rank (walker_range).  The reference compacts
               the valid walkers before its tree (executor.cpp:93-101), so the
               ranks first exchange their valid counts; rank r then owns the
               interval [off, off + cnt) of each observation's compacted order
               and sends the tree sums of its aligned dyadic blocks
               (dyadic_decompose), which every rank merges into the exact
               root (merge_blocks).  Exchange: ~1.5 KB per observation per rank.
  batched/pCN  contiguous blocks of parameter samples / chains (sample_range),
               results gathered.

Over a gloo process group (the plumbing tests: several ranks on one GPU, which
NCCL refuses) rank_context() builds the host-staged variant whose exchange is
an all-gather over torch.distributed; the arithmetic is the same.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _abi as A
from .api import Context, _check, nccl_unique_id

CHUNK = A.SMC_CHUNK


def num_chunks(n_particles: int) -> int:
    return (n_particles + CHUNK - 1) // CHUNK


# ---------------------------------------------------------------------------
# shard plans (the library's, restated; tests compare them)
# ---------------------------------------------------------------------------
def weighted_split(costs, world: int) -> list[int]:
    """capi_group.cu weighted_split: contiguous ranges of items balanced by
    cost; bounds[r] = first item of rank r, bounds[world] = len(costs)."""
    n = len(costs)
    prefix = [0.0]
    for c in costs:
        prefix.append(prefix[-1] + float(c))
    total = prefix[-1]
    b = [0] + [n] * world
    i = 0
    for r in range(1, world):
        target = total * r / world
        while i < n and prefix[i + 1] <= target:
            i += 1
        cut = i
        if i < n and (target - prefix[i]) > (prefix[i + 1] - target):
            cut = i + 1
        b[r] = max(b[r - 1], min(cut, n))
    return b


def unit_bounds(obs_steps, n_particles: int, world: int) -> list[int]:
    """observe_ad's (observation, chunk) unit ranges: unit u = obs * C + chunk,
    cost = n_steps(obs) x particles in the chunk."""
    cpo = num_chunks(n_particles)
    costs = [obs_steps[u // cpo] * min(CHUNK, n_particles - (u % cpo) * CHUNK) for u in range(len(obs_steps) * cpo)]
    return weighted_split(costs, world)


def walker_range(n_walkers: int, rank: int, world: int) -> tuple[int, int]:
    """observe_bvp: rank's contiguous walker range of every observation."""
    return (n_walkers * rank) // world, (n_walkers * (rank + 1)) // world


def sample_range(n_samples: int, rank: int, world: int) -> tuple[int, int]:
    """Batched evaluation / pCN: rank's contiguous block of samples (chains)."""
    return (n_samples * rank) // world, (n_samples * (rank + 1)) // world


# ---------------------------------------------------------------------------
# the Dirichlet exchange: aligned dyadic blocks (reduce_kernels.cu restated)
# ---------------------------------------------------------------------------
def dyadic_decompose(a: int, b: int) -> list[tuple[int, int]]:
    """Greedy (maximal) decomposition of [a, b) into aligned blocks
    [i 2^L, (i+1) 2^L) -> [(L, first leaf)]."""
    out = []
    p = a
    while p < b:
        L = 62 if p == 0 else (p & -p).bit_length() - 1
        while (1 << L) > b - p:
            L -= 1
        out.append((L, p))
        p += 1 << L
    return out


def tree_root(v: np.ndarray) -> float:
    """The reference's pairwise_sum (executor.cpp:11-26) as the aligned tree
    over v padded with -0.0."""
    v = np.asarray(v, dtype=np.float64)
    if len(v) == 0:
        return 0.0
    m = 1 << max(0, (len(v) - 1).bit_length())
    x = np.full(m, -0.0)
    x[: len(v)] = v
    while len(x) > 1:
        x = x[0::2] + x[1::2]
    return float(x[0])


def block_sums(local: np.ndarray, off: int) -> list[float]:
    """A rank's record: the tree sum of each block of its interval
    [off, off + len(local)) in the global compacted order."""
    return [tree_root(local[s - off: s - off + (1 << L)]) for L, s in dyadic_decompose(off, off + len(local))]


def merge_blocks(counts, records) -> float:
    """dyadic_finish_kernel: merge every rank's blocks (rank order) into the
    root of the tree over all of them."""
    stack: list[list] = []  # [level, index, value]

    def merge():
        while len(stack) >= 2 and stack[-1][0] == stack[-2][0] and stack[-2][1] % 2 == 0 \
                and stack[-1][1] == stack[-2][1] + 1:
            right = stack.pop()
            left = stack[-1]
            left[2] = float(np.float64(left[2]) + np.float64(right[2]))
            left[0] += 1
            left[1] >>= 1

    off = 0
    for cnt, rec in zip(counts, records):
        for (L, s), v in zip(dyadic_decompose(off, off + cnt), rec):
            stack.append([L, s >> L, v])
            merge()
        off += cnt
    while len(stack) > 1:  # trailing left children through the -0.0 padding
        stack[-1][0] += 1
        stack[-1][1] >>= 1
        merge()
    return stack[0][2] if stack else 0.0


# ---------------------------------------------------------------------------
# torch.distributed plumbing
# ---------------------------------------------------------------------------
class _HostedExchange:
    """smc_exchange_fn over torch.distributed (gloo): all-gather of every
    rank's byte slice of the library's staging buffer."""

    def __init__(self, rank: int, group):
        self.rank, self.group = rank, group
        self.fn = A.EXCHANGE_FN(self)

    def __call__(self, user, buf, displ, nbytes, world):
        try:
            import torch
            import torch.distributed as dist
            d = [int(displ[i]) for i in range(world)]
            b = [int(nbytes[i]) for i in range(world)]
            total = max(x + y for x, y in zip(d, b))
            arr = np.ctypeslib.as_array(buf, shape=(total,))
            width = max(max(b), 1)
            mine = torch.zeros(width, dtype=torch.uint8)
            r = self.rank
            mine[: b[r]] = torch.from_numpy(arr[d[r]: d[r] + b[r]].copy())
            parts = [torch.empty(width, dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(parts, mine, group=self.group)
            for q in range(world):
                if q != r:
                    arr[d[q]: d[q] + b[q]] = parts[q][: b[q]].numpy()
            return 0
        except Exception:  # noqa: BLE001 — reported by the library as a runtime error
            return 1


def rank_context(device: int | None = None, group=None) -> Context:
    """This process's GPU as one rank of a sharded context over the
    torch.distributed group (every rank must call it; collective).  NCCL
    process group: rank 0's NCCL unique id is broadcast and the library owns
    its own communicator (smc_create_rank).  gloo: host-staged exchange through
    torch.distributed (smc_create_rank_hosted)."""
    import torch.distributed as dist
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", "0"))
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if world == 1:
        return Context(device)
    if dist.get_backend(group) == "nccl":
        box = [nccl_unique_id() if rank == 0 else None]
        src = 0 if group is None else dist.get_global_rank(group, 0)
        dist.broadcast_object_list(box, src=src, group=group)
        return Context.for_rank(device, rank, world, box[0])
    ctx = Context.__new__(Context)
    ctx.lib = A.load_library()
    ex = _HostedExchange(rank, group)
    h = C.c_void_p()
    _check(ctx.lib.smc_create_rank_hosted(int(device), rank, world, ex.fn, None, C.byref(h)))
    ctx.device, ctx.handle, ctx._exchange = int(device), h, ex  # the callback lives as long as the context
    return ctx
