"""The multi-GPU shard plans and exchanges on CPU: world_size 2 and 3 over gloo.

The library shards inside the C ABI (csrc/capi_group.cu); these tests run the
numpy restatement of the same plans (paper_1808_10580_b200.distributed) over
real torch.distributed process groups, with per-particle values from the
plain-C oracle, and require the oracle's single-process estimates bit for bit:

  observe_ad   (observation, chunk) units balanced by particle-steps, chunk
               partials all-gathered (variable sizes), tree finished, two-pass
               variance;
  observe_bvp  valid counts exchanged, then each rank's aligned dyadic blocks
               of its interval of the compacted order, merged in rank order.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1808_10580_b200 import distributed as D


def chunk_tree(v: np.ndarray) -> float:
    """One unit's partial: the aligned 1024-leaf tree padded with -0.0."""
    x = np.full(D.CHUNK, -0.0)
    x[: len(v)] = v
    while len(x) > 1:
        x = x[0::2] + x[1::2]
    return float(x[0])


def all_gather_v(local: np.ndarray, counts: list[int]) -> np.ndarray:
    """Rank-ordered concatenation of variable-length float64 vectors."""
    width = max(max(counts), 1)
    buf = torch.zeros(width, dtype=torch.float64)
    buf[: len(local)] = torch.from_numpy(np.ascontiguousarray(local, dtype=np.float64))
    parts = [torch.empty_like(buf) for _ in counts]
    dist.all_gather(parts, buf)
    return np.concatenate([p[:c].numpy() for p, c in zip(parts, counts)])


def sharded_ad(values: np.ndarray, obs_steps, rank: int, world: int):
    """observe_ad's group plan (capi_group.cu group_ad_observe) on numpy."""
    n_obs, n = values.shape
    cpo = D.num_chunks(n)
    bounds = D.unit_bounds(obs_steps, n, world)
    counts = [bounds[r + 1] - bounds[r] for r in range(world)]
    mine = range(bounds[rank], bounds[rank + 1])

    def unit_values(u):
        j, c = divmod(u, cpo)
        return values[j, c * D.CHUNK: min((c + 1) * D.CHUNK, n)]

    full = all_gather_v(np.array([chunk_tree(unit_values(u)) for u in mine]), counts).reshape(n_obs, cpo)
    sums = np.array([D.tree_root(row) for row in full])
    means = sums / np.full(n_obs, float(n))
    sq = []
    for u in mine:
        d = unit_values(u) - means[u // cpo]
        sq.append(chunk_tree(d * d))
    fullsq = all_gather_v(np.array(sq), counts).reshape(n_obs, cpo)
    sumsq = np.array([D.tree_root(row) for row in fullsq])
    se = np.sqrt((sumsq / (n - 1.0)) / n)
    return list(zip(means.tolist(), se.tolist()))


def sharded_bvp(values, failed, rank: int, world: int):
    """observe_bvp's group plan (group_bvp_observe): counts, dyadic blocks,
    merge; then the squared deviations the same way."""
    n_obs, n = values.shape
    b, e = D.walker_range(n, rank, world)
    out = []
    for j in range(n_obs):
        local = values[j, b:e][failed[j, b:e] == 0]
        cnt = torch.tensor([len(local)], dtype=torch.int64)
        parts = [torch.empty_like(cnt) for _ in range(world)]
        dist.all_gather(parts, cnt)
        counts = [int(p.item()) for p in parts]
        off = sum(counts[:rank])
        rec = D.block_sums(local, off)
        recs = all_gather_v(np.array(rec + [0.0] * (64 - len(rec))), [64] * world).reshape(world, 64)
        total = sum(counts)
        mean = D.merge_blocks(counts, recs) / float(total)
        d = local - mean
        rec2 = D.block_sums(d * d, off)
        recs2 = all_gather_v(np.array(rec2 + [0.0] * (64 - len(rec2))), [64] * world).reshape(world, 64)
        sumsq = D.merge_blocks(counts, recs2)
        out.append((mean, float(np.sqrt((sumsq / (total - 1.0)) / total)), n - total))
    return out


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(kind, rank, world, port, payload, expected, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if kind == "ad":
            got = sharded_ad(*payload, rank, world)
        else:
            got = sharded_bvp(*payload, rank, world)
        result_q.put((rank, got == expected, got))
    finally:
        dist.destroy_process_group()


def _run(kind, world, payload, expected):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    prt = _free_port()
    procs = [ctx.Process(target=_worker, args=(kind, r, world, prt, payload, expected, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in results), results


@pytest.mark.parametrize("world,n_particles", [(2, 5000), (3, 2048), (2, 700), (3, 3001)])
def test_sharded_ad_plan_bit_identical(port, world, n_particles):
    """C1's three observations (200/300/400 steps) make the unit costs
    unequal, so the split is not at observation boundaries."""
    import specs
    spec = specs.c1_two_mode(n_particles=n_particles)
    values = np.stack([port.ad_particle_values(spec, j, 7, n_particles) for j in range(3)])
    ref = port.observe_ad(spec, 7)
    expected = [(float(e["mean"]), float(e["std_error"])) for e in ref]
    assert D.tree_root(values[0]) == port.pairwise_sum(values[0])
    _run("ad", world, (values, [200, 300, 400]), expected)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_bvp_plan_bit_identical(port, world):
    """Walkers that fail (max_steps 150) are compacted out before the tree, so
    each rank's interval starts at a count only the exchange reveals."""
    import specs
    spec = specs.paper_bvp(n_particles=2500, amplitudes=(1.0, -0.5, 2.0))
    spec.max_steps = 150
    vals, failed = [], []
    for j in range(len(spec.observations)):
        v, _, f, _ = port.bvp_particle_values(spec, j, 606, spec.n_particles)
        vals.append(v)
        failed.append(f)
    vals, failed = np.stack(vals), np.stack(failed)
    assert failed.any() and not failed.all(axis=1).any()
    ref = port.observe_bvp(spec, 606)
    expected = [(float(e["mean"]), float(e["std_error"]), int(e["n_failed"])) for e in ref]
    _run("bvp", world, (vals, failed), expected)


def test_dyadic_merge_equals_pairwise_tree(port):
    """Any split of a compacted sequence into rank intervals, each sent as the
    tree sums of its aligned dyadic blocks, merges into exactly the
    reference's pairwise_sum (including empty ranks and 1-element ranks)."""
    rng = np.random.default_rng(3)
    for trial in range(200):
        n = int(rng.integers(0, 5000))
        v = rng.normal(size=n) * 10.0 ** rng.integers(-3, 4, size=n)
        world = int(rng.integers(1, 9))
        cuts = np.sort(rng.integers(0, n + 1, size=world - 1))
        edges = [0, *cuts.tolist(), n]
        counts = [edges[r + 1] - edges[r] for r in range(world)]
        recs = [D.block_sums(v[edges[r]: edges[r + 1]], edges[r]) for r in range(world)]
        want = port.pairwise_sum(v) if n else 0.0
        assert D.merge_blocks(counts, recs) == want, (trial, n, counts)
        assert all(len(r) <= 64 for r in recs)


def test_dyadic_decompose_is_maximal_tiling():
    for a, b in [(0, 0), (0, 1), (3, 8), (5, 1029), (1023, 1025), (0, 1 << 20), (12345, 999_999)]:
        blocks = D.dyadic_decompose(a, b)
        p = a
        for L, s in blocks:
            assert s == p and s % (1 << L) == 0
            p += 1 << L
        assert p == b
        # maximal: no two adjacent blocks are siblings
        for (L1, s1), (L2, s2) in zip(blocks, blocks[1:]):
            assert not (L1 == L2 and (s1 >> L1) % 2 == 0)


def test_unit_bounds_partition_and_balance():
    for steps in ([1000] * 9, [200, 300, 400], [63 * k for k in range(1, 9)] * 8):
        for n in (700, 5000, 32768, 100_000):
            cpo = D.num_chunks(n)
            for world in (1, 2, 3, 4, 8):
                b = D.unit_bounds(steps, n, world)
                assert b[0] == 0 and b[-1] == len(steps) * cpo and all(x <= y for x, y in zip(b, b[1:]))
                cost = [steps[u // cpo] * min(D.CHUNK, n - (u % cpo) * D.CHUNK) for u in range(len(steps) * cpo)]
                loads = [sum(cost[b[r]: b[r + 1]]) for r in range(world)]
                assert max(loads) <= sum(cost) / world + max(cost) + 1e-6


def test_walker_and_sample_ranges_partition():
    for n in (2, 7, 1000, 1_000_000):
        for world in (1, 2, 3, 8):
            for fn in (D.walker_range, D.sample_range):
                rs = [fn(n, r, world) for r in range(world)]
                assert rs[0][0] == 0 and rs[-1][1] == n
                assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
                assert max(e - b for b, e in rs) - min(e - b for b, e in rs) <= 1
