"""Multi-device contexts on the GPU: the sharded forward maps
inside the C ABI, bit-identical to one device.

One B200 is available here, so the groups repeat device 0: the library then
replaces NCCL by event-ordered peer copies (the "emulated" exchange) but runs
the same shard plans, kernels and finishing arithmetic as over NCCL.  The NCCL
calls themselves are exercised by one-rank groups forced with
SMC_GROUP_FORCE=1 (ncclCommInitAll / ncclCommInitRank of one device and the
in-place broadcasts of the exchange)."""
import os

import numpy as np
import pytest

import paper_1808_10580_b200 as S
import specs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return S.default_context(0)


_groups = {}


def group(world):
    g = _groups.get(world)
    if g is None:
        g = _groups[world] = S.Context(devices=[0] * world)
    return g


def fields(e):
    return (e.mean, e.std_error, e.n_particles, e.n_failed, e.aux_mean)


def same(a, b):
    return [fields(x) for x in a] == [fields(y) for y in b]


def ragged_c2(ctx, n=5000):
    u = S.prior_draw(specs.C2_PRIOR, 808, 0xBE9C4, 0, ctx)
    spec = specs.c2_spec(u, n_particles=n)
    # three observation times: unequal unit costs, so splits fall inside observations
    spec.observations = [S.AdObservation(t, o.x) for t, o in zip((0.05, 0.2, 0.11, 0.3), spec.observations[:4])]
    return spec


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_group_query(world):
    g = group(world).group()
    assert g["world"] == world and g["n_local"] == world and g["rank"] == 0 and not g["nccl"]
    assert g["devices"] == [0] * world


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("n", [5000, 1024, 2])
def test_ad_group_bit_identical(ctx, world, n):
    spec = ragged_c2(ctx, n)
    want = S.observe_ad(spec, 808, ctx=ctx)
    got = S.observe_ad(spec, 808, ctx=group(world))
    assert same(got, want)
    st = group(world).stats()
    assert st.particle_kernel_ms > 0 and st.kernel_launches > 0


@pytest.mark.parametrize("world", [2, 8])
def test_ad_single_group(ctx, world):
    spec = ragged_c2(ctx)
    for j in (0, 3):
        want = S.observe_ad_single(spec, j, 808, ctx=ctx)
        got = S.observe_ad_single(spec, j, 808, ctx=group(world))
        assert fields(got) == fields(want)


@pytest.mark.parametrize("precision", [S.Precision.fp32, S.Precision.fp64_strict])
def test_ad_group_other_precisions(ctx, precision):
    spec = ragged_c2(ctx, 3000)
    spec.precision = precision
    assert same(S.observe_ad(spec, 808, ctx=group(3)), S.observe_ad(spec, 808, ctx=ctx))


def test_ad_group_generic_lattice(ctx):
    """K = 25 prior field (tiled lattice kernel, not the compile-time disk)."""
    u = S.prior_draw(specs.C4_PRIOR, 808, 0xBE9C4, 1, ctx)
    spec = specs.c4_base(n_particles=2100)
    spec.velocity = S.VelocityField.fourier(S.velocity_from_coefficients(specs.C4_PRIOR, u))
    assert same(S.observe_ad(spec, 808, ctx=group(3)), S.observe_ad(spec, 808, ctx=ctx))


def test_ad_group_constant_velocity_c1(ctx, golden):
    spec = specs.c1_two_mode(n_particles=10000)
    assert same(S.observe_ad(spec, 7, ctx=group(8)), S.observe_ad(spec, 7, ctx=ctx))


@pytest.mark.parametrize("max_steps", [10_000_000, 150])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_bvp_group_bit_identical(ctx, world, max_steps):
    """Walker ranges per rank; the valid counts and then the aligned dyadic
    block sums are exchanged.  max_steps 150 makes walkers fail, so each
    rank's interval of the compacted order depends on the other ranks."""
    spec = specs.paper_bvp(n_particles=5000)
    spec.max_steps = max_steps
    want = S.observe_bvp(spec, 606, ctx=ctx)
    got = S.observe_bvp(spec, 606, ctx=group(world))
    if max_steps == 150:
        assert sum(e.n_failed for e in want) > 0
    assert same(got, want)
    assert group(world).stats().particle_steps == ctx.stats().particle_steps


def test_bvp_group_more_ranks_than_walkers(ctx):
    spec = specs.paper_bvp(n_particles=5)
    assert same(S.observe_bvp(spec, 606, ctx=group(8)), S.observe_bvp(spec, 606, ctx=ctx))


def test_bvp_group_range(ctx):
    spec = specs.paper_bvp(n_particles=3000)
    want = S.observe_bvp_range(spec, 606, 1, 2, ctx=ctx)
    assert same(S.observe_bvp_range(spec, 606, 1, 2, ctx=group(3)), want)


def test_bvp_group_all_failed_raises(ctx):
    spec = specs.paper_bvp(n_particles=64)
    spec.max_steps = 1
    with pytest.raises(RuntimeError, match="every particle"):
        S.observe_bvp(spec, 606, ctx=ctx)
    with pytest.raises(RuntimeError, match="every particle"):
        S.observe_bvp(spec, 606, ctx=group(2))


def test_group_validation_errors_match(ctx):
    spec = ragged_c2(ctx)
    spec.n_particles = 1
    with pytest.raises(ValueError) as a:
        S.observe_ad(spec, 808, ctx=ctx)
    with pytest.raises(ValueError) as b:
        S.observe_ad(spec, 808, ctx=group(2))
    assert str(a.value) == str(b.value)


def test_forced_one_rank_nccl_groups(ctx, monkeypatch):
    """The NCCL code path on one GPU: ncclCommInitAll / ncclCommInitRank of a
    single device and the in-place broadcasts of every exchange."""
    monkeypatch.setenv("SMC_GROUP_FORCE", "1")
    multi = S.Context(devices=[0])
    rank = S.Context.for_rank(0, 0, 1, S.nccl_unique_id())
    try:
        for g in (multi, rank):
            assert g.group()["nccl"] and g.group()["world"] == 1
            spec = ragged_c2(ctx)
            assert same(S.observe_ad(spec, 808, ctx=g), S.observe_ad(spec, 808, ctx=ctx))
            bvp = specs.paper_bvp(n_particles=3000)
            bvp.max_steps = 150
            assert same(S.observe_bvp(bvp, 606, ctx=g), S.observe_bvp(bvp, 606, ctx=ctx))
    finally:
        multi.close()
        rank.close()


def test_repeated_group_calls_reuse_buffers(ctx):
    """Back-to-back evaluations of different shapes on one group context."""
    g = group(3)
    for n in (4000, 1500, 9000):
        spec = ragged_c2(ctx, n)
        assert same(S.observe_ad(spec, 808, ctx=g), S.observe_ad(spec, 808, ctx=ctx))
        bvp = specs.paper_bvp(n_particles=n)
        assert same(S.observe_bvp(bvp, 606, ctx=g), S.observe_bvp(bvp, 606, ctx=ctx))


# ---------------------------------------------------- batched and pCN ------
@pytest.mark.parametrize("world", [2, 3, 8])
def test_batched_group_sample_sharding(ctx, world):
    prior = specs.C2_PRIOR
    u0 = S.prior_draw(prior, 808, 0xBE9C4, 0, ctx)
    U = np.stack([u0 * (1.0 + 0.01 * b) for b in range(7)])
    base = specs.c4_base(n_particles=500)
    want = S.observe_ad_batched(base, prior, U, 808, ctx=ctx)
    got = S.observe_ad_batched(base, prior, U, 808, ctx=group(world))
    assert got.tobytes() == want.tobytes()
    seeds = np.arange(7, dtype=np.uint64) + 100
    want = S.observe_ad_batched(base, prior, U, 808, seeds=seeds, ctx=ctx)
    got = S.observe_ad_batched(base, prior, U, 808, seeds=seeds, ctx=group(world))
    assert got.tobytes() == want.tobytes()


def test_batched_group_non_finite_raises(ctx):
    prior = specs.C2_PRIOR
    U = np.zeros((4, prior.dimension()))
    U[3, 5] = np.nan
    base = specs.c4_base(n_particles=64)
    with pytest.raises(ValueError, match="non-finite"):
        S.observe_ad_batched(base, prior, U, 808, ctx=group(2))


PCN_DATA = [-0.9065, -0.7528, -0.6665, -0.8091, -0.6508, -0.5135, -0.5185, -0.4553, -0.4066]


@pytest.mark.parametrize("world,chains", [(2, 5), (3, 2), (8, 9)])
def test_pcn_group_chain_sharding(ctx, world, chains):
    fwd = specs.c4_base(n_particles=160)
    fwd.dt = 0.006
    like = S.LikelihoodSpec(data=PCN_DATA, noise_std=0.05, forward=fwd, forward_seed=1234)
    prior = S.PriorSpec(2, 0.6, 2.5)
    cfg = S.ChainConfig(n_steps=12, beta=0.3, burn_in=2, thin=3)
    seeds = list(range(40, 40 + chains))
    want = S.run_chains(cfg, prior, like, seeds, ctx=ctx)
    got = S.run_chains(cfg, prior, like, seeds, ctx=group(world))
    for k in ("final_u", "final_phi", "map_u", "map_objective", "accepted", "phi_trace", "samples"):
        assert np.array_equal(got[k], want[k]), k


@pytest.mark.parametrize("world", [2, 8])
def test_serialised_group_bit_identical(ctx, monkeypatch, world):
    """SMC_GROUP_SERIAL=1 (tools/shard_model.py: every member on one stream,
    so each shard runs alone and its kernel time is one rank's) must not
    change results: with all members' work queued behind each other, any
    host write into a buffer an earlier queued copy still reads shows up here
    (it caught the Dirichlet map's step-count readback into the image's
    staging buffer)."""
    monkeypatch.setenv("SMC_GROUP_SERIAL", "1")
    g = S.Context(devices=[0] * world)
    ad = ragged_c2(ctx)
    assert same(S.observe_ad(ad, 808, ctx=g), S.observe_ad(ad, 808, ctx=ctx))
    bvp = specs.paper_bvp(n_particles=20000, amplitudes=(1.0, -0.5, 2.0))
    assert same(S.observe_bvp(bvp, 606, ctx=g), S.observe_bvp(bvp, 606, ctx=ctx))
