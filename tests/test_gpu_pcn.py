"""Device-resident multi-chain pCN against the
reference's run_chain (src/inference.cpp:170-194).

Three chains run together (one batched forward map per step); chain c must
reproduce the reference's run_chain with seed = seeds[c]: the same accepted
count, Phi trace within the forward map's parity gate, and the same states.
"""
import numpy as np
import pytest

import paper_1808_10580_b200 as S
import specs
from conftest import unhex

pytestmark = pytest.mark.gpu

DATA = [-0.9065, -0.7528, -0.6665, -0.8091, -0.6508, -0.5135, -0.5185, -0.4553, -0.4066]


def likelihood():
    fwd = specs.c4_base(n_particles=160)
    fwd.dt = 0.006
    return S.LikelihoodSpec(data=DATA, noise_std=0.05, forward=fwd, forward_seed=1234)


def test_chains_match_reference_run_chain(ctx, golden):
    g = golden["pcn"]
    prior = S.PriorSpec(2, 0.6, 2.5)
    cfg = S.ChainConfig(n_steps=g["n_steps"], beta=g["beta"], burn_in=g["burn_in"], thin=g["thin"])
    seeds = [c["seed"] for c in g["chains"]]
    res = S.run_chains(cfg, prior, likelihood(), seeds, ctx=ctx)
    for b, ref in enumerate(g["chains"]):
        assert res["accepted"][b] == ref["accepted"]
        trace = unhex(ref["phi_trace"])
        assert np.allclose(res["phi_trace"][b], trace, rtol=1e-8, atol=1e-10)
        assert np.allclose(res["final_u"][b], unhex(ref["final_u"]), rtol=0, atol=1e-12)
        assert np.allclose(res["map_u"][b], unhex(ref["map_u"]), rtol=0, atol=1e-12)
        assert abs(res["map_objective"][b] - float.fromhex(ref["map_objective"])) <= 1e-8 * abs(
            float.fromhex(ref["map_objective"]))
        samples = unhex(ref["samples"])
        assert res["samples"][b].shape == samples.shape
        assert np.allclose(res["samples"][b], samples, rtol=0, atol=1e-12)


def test_chain_with_given_start_and_single_chain(ctx, golden):
    prior = S.PriorSpec(2, 0.6, 2.5)
    u0 = S.prior_draw(prior, 5, 0, 0, ctx)
    cfg = S.ChainConfig(n_steps=10, beta=0.3, burn_in=0, thin=1)
    one = S.run_chains(cfg, prior, likelihood(), [11], u0=u0[None, :], ctx=ctx)
    two = S.run_chains(cfg, prior, likelihood(), [11, 12], u0=np.stack([u0, u0]), ctx=ctx)
    # chains are independent of their batch neighbours
    assert np.array_equal(one["phi_trace"][0], two["phi_trace"][0])
    assert np.array_equal(one["final_u"][0], two["final_u"][0])
    assert one["samples"].shape == (1, 10, prior.dimension())


def test_chain_validation(ctx):
    prior = S.PriorSpec(2, 0.6, 2.5)
    with pytest.raises(ValueError, match="beta must be in"):
        S.run_chains(S.ChainConfig(n_steps=3, beta=1.5), prior, likelihood(), [1], ctx=ctx)
    with pytest.raises(ValueError, match="thin must be"):
        S.run_chains(S.ChainConfig(n_steps=3, beta=0.1, thin=0), prior, likelihood(), [1], ctx=ctx)


@pytest.mark.parametrize("n_steps,burn_in,thin", [(37, 5, 3), (16, 0, 1), (33, -2, 4)])
def test_graph_replay_matches_step_loop(ctx, monkeypatch, n_steps, burn_in, thin):
    """The CUDA-graph path (device step counter, 16-step groups + remainder)
    must be bit-identical to the per-step host loop."""
    prior = S.PriorSpec(2, 0.6, 2.5)
    cfg = S.ChainConfig(n_steps=n_steps, beta=0.3, burn_in=burn_in, thin=thin)
    seeds = [3, 4, 5]
    monkeypatch.setenv("SMC_PCN_GRAPH", "0")
    loop = S.run_chains(cfg, prior, likelihood(), seeds, ctx=ctx)
    monkeypatch.setenv("SMC_PCN_GRAPH", "1")
    graph = S.run_chains(cfg, prior, likelihood(), seeds, ctx=ctx)
    for key in ("phi_trace", "final_u", "map_u", "map_objective", "accepted", "samples"):
        assert np.array_equal(np.asarray(loop[key]), np.asarray(graph[key])), key


def test_k25_chains_match_reference(ctx, reference):
    """Chains on the C4 prior (K = 25, dimension 1960): the device pCN driver
    then runs the tiled disk kernel every step; two short chains against the
    reference's run_chain (workers = all host cores)."""
    prior = S.PriorSpec(25, 1.0, 2.5)
    cfg = S.ChainConfig(n_steps=6, beta=0.05, burn_in=1, thin=2)
    res = S.run_chains(cfg, prior, likelihood(), [21, 22], ctx=ctx)
    for b, seed in enumerate((21, 22)):
        ref = reference.run_chain(likelihood(), prior, 6, 0.05, 1, 2, seed)
        assert res["accepted"][b] == ref["accepted"]
        assert np.allclose(res["phi_trace"][b], ref["phi_trace"], rtol=1e-8, atol=1e-10)
        assert np.allclose(res["final_u"][b], ref["final_u"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("burn_in,thin", [(-2, 4), (-5, 3), (3, 5)])
def test_sample_schedule_matches_reference(ctx, reference, burn_in, thin):
    """The recorded iterations (i > burn_in, (i - burn_in - 1) % thin == 0,
    inference.cpp:183-185), negative burn-in included: same sample count and
    states as the reference's run_chain."""
    prior = S.PriorSpec(2, 0.6, 2.5)
    n = 17
    res = S.run_chains(S.ChainConfig(n_steps=n, beta=0.3, burn_in=burn_in, thin=thin), prior, likelihood(), [9],
                       ctx=ctx)
    ref = reference.run_chain(likelihood(), prior, n, 0.3, burn_in, thin, 9)
    want = [i for i in range(1, n + 1) if i > burn_in and (i - burn_in - 1) % thin == 0]
    assert res["samples"].shape[1] == len(want) == ref["samples"].shape[0]
    assert np.allclose(res["samples"][0], ref["samples"], rtol=0, atol=1e-12)
