"""One process per GPU through the C ABI (smc_create_rank_hosted): two and
three ranks on the one B200, started by torch.multiprocessing with a gloo
process group, each calling the forward maps with the same arguments; every
rank must return the single-device result bit for bit.  This is the torchrun
plumbing of distributed.rank_context with the exchange staged through
torch.distributed (NCCL refuses several ranks on one GPU); the shard plans and
the finishing arithmetic are the ones the NCCL ranks run."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

PCN_DATA = [-0.9065, -0.7528, -0.6665, -0.8091, -0.6508, -0.5135, -0.5185, -0.4553, -0.4066]


def workloads(S, specs, ctx):
    u = S.prior_draw(specs.C2_PRIOR, 808, 0xBE9C4, 0, ctx)
    ad = specs.c2_spec(u, n_particles=4100)
    ad.observations = [S.AdObservation(t, o.x) for t, o in zip((0.05, 0.2, 0.11), ad.observations[:3])]
    bvp = specs.paper_bvp(n_particles=3000)
    bvp.max_steps = 150
    U = np.stack([u * (1.0 + 0.01 * b) for b in range(5)])
    base = specs.c4_base(n_particles=300)
    fwd = specs.c4_base(n_particles=160)
    fwd.dt = 0.006
    like = S.LikelihoodSpec(data=PCN_DATA, noise_std=0.05, forward=fwd, forward_seed=1234)
    out = {"ad": [(x.mean, x.std_error, x.n_particles, x.n_failed, x.aux_mean) for x in S.observe_ad(ad, 808, ctx=ctx)],
           "bvp": [(x.mean, x.std_error, x.n_particles, x.n_failed, x.aux_mean) for x in
                   S.observe_bvp(bvp, 606, ctx=ctx)],
           "batched": S.observe_ad_batched(base, specs.C2_PRIOR, U, 808, ctx=ctx).tobytes()}
    res = S.run_chains(S.ChainConfig(n_steps=8, beta=0.3, burn_in=1, thin=2), S.PriorSpec(2, 0.6, 2.5), like,
                       [40, 41, 42, 43, 44], ctx=ctx)
    out["pcn"] = {k: v.tobytes() for k, v in res.items() if v is not None}
    return out


def _worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "tests")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    import paper_1808_10580_b200 as S
    from paper_1808_10580_b200 import distributed as D
    import specs
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ctx = D.rank_context(0)
        g = ctx.group()
        q.put((rank, g, workloads(S, specs, ctx)))
        ctx.close()
    except Exception as e:  # noqa: BLE001
        q.put((rank, None, repr(e)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_rank_contexts_bit_identical(world):
    import paper_1808_10580_b200 as S
    import specs
    want = workloads(S, specs, S.default_context(0))
    mctx = mp.get_context("spawn")
    q = mctx.Queue()
    port = _free_port()
    procs = [mctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, g, got in results:
        assert g is not None, got
        assert g["world"] == world and g["rank"] == rank and not g["nccl"]
        for k in ("ad", "bvp", "batched"):
            assert got[k] == want[k], (rank, k)
        assert got["pcn"] == want["pcn"], rank
