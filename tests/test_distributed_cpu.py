"""The multi-GPU exchange logic on CPU: world_size 2 (and 3) over gloo.

paper_1808_10580_b200.distributed.sharded_estimates is run with a numpy
ShardOps — per-particle values from the plain-C oracle, chunk partials by a
numpy restatement of the aligned pairwise tree — so the shard plan, the
all-gather assembly and the two-pass finish are exercised exactly as on the
GPUs.  The result must be bit-identical to the oracle's single-process
observe_ad (which is bit-identical to the reference)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1808_10580_b200 import distributed as D


def tree_chunks(v: np.ndarray, chunk: int = D.CHUNK) -> np.ndarray:
    """Aligned pairwise tree per chunk, leaves padded with -0.0."""
    m = max(1, -(-len(v) // chunk))
    x = np.full(m * chunk, -0.0)
    x[: len(v)] = v
    x = x.reshape(m, chunk)
    while x.shape[1] > 1:
        x = x[:, 0::2] + x[:, 1::2]
    return x[:, 0]


def tree_sum(v: np.ndarray) -> float:
    while len(v) > 1:
        v = tree_chunks(v)
    return float(v[0]) if len(v) else 0.0


class NumpyOps:
    def __init__(self, values: np.ndarray):
        self.values = values  # [n_obs][n]

    def partials(self, b, e):
        n = self.values.shape[1]
        return np.stack([tree_chunks(row[b * D.CHUNK: min(e * D.CHUNK, n)])[: e - b] if e > b else np.zeros(0)
                         for row in self.values])

    def sq_partials(self, means, b, e):
        n = self.values.shape[1]
        out = []
        for row, m in zip(self.values, means):
            d = row[b * D.CHUNK: min(e * D.CHUNK, n)] - m
            out.append(tree_chunks(d * d)[: e - b] if e > b else np.zeros(0))
        return np.stack(out)

    def finish(self, partials):
        return np.array([tree_sum(row) for row in partials])

    def divide(self, sums, n):
        return sums / float(n)

    def all_gather(self, local, counts):
        width = max(counts)
        buf = torch.zeros((local.shape[0], width), dtype=torch.float64)
        buf[:, : local.shape[1]] = torch.from_numpy(np.ascontiguousarray(local))
        parts = [torch.empty_like(buf) for _ in counts]
        dist.all_gather(parts, buf)
        return np.concatenate([p[:, :c].numpy() for p, c in zip(parts, counts)], axis=1)

    def to_host(self, x):
        return np.asarray(x)


def _worker(rank, world, port, values, expected, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        est = D.sharded_estimates(NumpyOps(values), values.shape[1], rank, world)
        ok = all(e.mean == x[0] and e.std_error == x[1] for e, x in zip(est, expected))
        result_q.put((rank, ok, [(e.mean, e.std_error) for e in est]))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,n_particles", [(2, 5000), (3, 2048), (2, 700)])
def test_sharded_exchange_bit_identical(port, world, n_particles):
    import specs
    spec = specs.c1_two_mode(n_particles=n_particles)
    values = np.stack([port.ad_particle_values(spec, j, 7, n_particles) for j in range(3)])
    ref = port.observe_ad(spec, 7)
    expected = [(float(e["mean"]), float(e["std_error"])) for e in ref]
    # the numpy tree itself equals the oracle's pairwise_sum
    assert tree_sum(values[0]) == port.pairwise_sum(values[0])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    prt = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, prt, values, expected, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in results), results


def test_chunk_ranges_partition():
    for n_chunks in (1, 7, 98, 977):
        for world in (1, 2, 3, 4, 8):
            rs = [D.chunk_range(n_chunks, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n_chunks
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            assert max(e - b for b, e in rs) - min(e - b for b, e in rs) <= 1


def _gather_worker(rank, world, port, n, result_q):
    """DeviceOps.all_gather over gloo with ragged walker ranges, float64 and
    uint8 (the Dirichlet walker-sharding exchange): the rank-ordered result
    must be the unsharded [n_obs][n] array."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ops = D.DeviceOps.__new__(D.DeviceOps)  # the exchange only: no device context
        ops.torch, ops.n_obs, ops.dev, ops.group = torch, 4, torch.device("cpu"), None
        full_v = torch.arange(4 * n, dtype=torch.float64).reshape(4, n) * 0.5
        full_f = (torch.arange(4 * n).reshape(4, n) % 7 == 0).to(torch.uint8)
        counts = [D.walker_range(n, r, world)[1] - D.walker_range(n, r, world)[0] for r in range(world)]
        b, e = D.walker_range(n, rank, world)
        gv = ops.all_gather(full_v[:, b:e].clone(), counts)
        gf = ops.all_gather(full_f[:, b:e].clone(), counts)
        result_q.put((rank, bool(torch.equal(gv, full_v)) and bool(torch.equal(gf, full_f)) and gf.dtype == torch.uint8))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 1001), (3, 10)])
def test_walker_sharding_gather(world, n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    prt = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, prt, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in results), results


def test_walker_ranges_partition():
    for n in (2, 7, 1000, 1_000_000):
        for world in (1, 2, 3, 8):
            rs = [D.walker_range(n, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
