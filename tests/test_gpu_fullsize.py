"""Parity at the BASELINE configurations' full sizes.

The oracle cannot run a whole full-size evaluation in test time, so a
full-size run is pinned through size-independent properties:

* particle prefix — every particle is keyed by (seed, obs, particle) alone,
  so the first particles of a full-size run must be the oracle's particles
  (the oracle runs only those);
* the estimate is the reference's reduction of the per-particle values the
  kernel produced: mean = pairwise_sum / n, var = pairwise_sum((v - mean)^2)
  / (n - 1), se = sqrt(var / n) — bit-exact with the oracle's pairwise_sum
  (executor.cpp:11-26, :87-116);
* sharding / observation-range / batch splits reproduce the whole run
  bit-for-bit.
"""
import math
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_1808_10580_b200 as S
from paper_1808_10580_b200 import distributed as D
import specs

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def reference_reduction(port, values):
    """reduce_observation (executor.cpp:87-116) over already-valid values."""
    n = values.size
    mean = port.pairwise_sum(values) / n
    var = port.pairwise_sum((values - mean) ** 2) / (n - 1) if n > 1 else 0.0
    return mean, math.sqrt(var / n)


@pytest.fixture(scope="module")
def c2(ctx):
    u = S.prior_draw(specs.C2_PRIOR, 808, 0xBE9C4, 0, ctx)  # bench.py / benchmark.cpp:69-71 recipe
    spec = specs.c2_spec(u, n_particles=100_000)
    return spec, S.observe_ad(spec, 808, ctx=ctx)


def test_c2_full_estimates_are_the_reference_reduction(ctx, port, c2):
    spec, est = c2
    for j in (0, 4, 8):
        vals = S.ad_particle_values(spec, j, 808, spec.n_particles, ctx)
        mean, se = reference_reduction(port, vals)
        assert est[j].mean == mean and est[j].std_error == se


def test_c2_full_particle_prefix_matches_oracle(ctx, port, c2):
    spec, _ = c2
    for j in (0, 8):
        got = S.ad_particle_values(spec, j, 808, 192, ctx)
        want = port.ad_particle_values(spec, j, 808, 192)
        assert np.max(np.abs(got - want)) < 1e-11


def test_c2_full_sharded_bit_identical(ctx, c2):
    spec, est = c2
    for world in (2, 8):
        assert S.observe_ad(spec, 808, ctx=S.Context(devices=[0] * world)) == est


def test_c3_full_observation_split_and_prefix(ctx, port):
    spec = specs.c3_spec(n_particles=1_000_000)
    est = S.observe_bvp(spec, 606, ctx=ctx)
    head = S.observe_bvp_range(spec, 606, 0, 12, ctx=ctx)
    tail = S.observe_bvp_range(spec, 606, 12, len(spec.observations) - 12, ctx=ctx)
    assert list(head) + list(tail) == list(est)
    assert all(e.n_failed == 0 for e in est)
    # walker prefix of observation 0 against the oracle
    vals, aux, failed = S.bvp_particle_values(spec, 0, 606, 256, ctx)
    pv, pa, pf, _ = port.bvp_particle_values(spec, 0, 606, 256)
    assert np.array_equal(failed, pf)
    assert np.max(np.abs(vals - pv)) < 1e-9
    assert np.max(np.abs(aux - pa)) < 1e-12


def test_c3_full_estimate_is_the_reference_reduction(ctx, port):
    spec = specs.c3_spec(n_particles=1_000_000)
    spec.observations = spec.observations[:2]
    est = S.observe_bvp(spec, 606, ctx=ctx)
    for j in range(2):
        vals, aux, failed = S.bvp_particle_values(spec, j, 606, spec.n_particles, ctx)
        ok = failed == 0  # executor.cpp:93-101: failed walkers excluded
        mean, se = reference_reduction(port, vals[ok])
        assert est[j].mean == mean and est[j].std_error == se
        assert est[j].n_failed == int(np.sum(~ok))


def test_c4_full_batch_equals_single_calls(ctx):
    prior = specs.C4_PRIOR
    u0 = S.prior_draw(prior, 808, 0xBE9C4, 1, ctx)
    B = 4096
    xi = np.stack([S.prior_draw(prior, 4242, 0xFFFFFFFF, b, ctx) for b in (0, 1, 2047, 4095)])
    U = np.repeat((math.sqrt(1 - 0.02 ** 2) * u0)[None, :], B, axis=0)
    for row, b in zip(xi, (0, 1, 2047, 4095)):
        U[b] += 0.02 * row
    base = specs.c4_base(n_particles=1024)
    out = S.observe_ad_batched(base, prior, U, 808, ctx=ctx)
    for b in (0, 1, 2047, 4095):
        spec = specs.c4_base(n_particles=1024)
        spec.velocity = S.VelocityField.fourier(S.velocity_from_coefficients(prior, U[b]))
        single = S.observe_ad(spec, 808, ctx=ctx)  # K=25: both run the tiled lattice kernel
        for j, f in enumerate(single):
            assert out[b, j]["mean"] == f.mean and out[b, j]["std_error"] == f.std_error


def test_c5_full_prefix_matches_oracle(ctx, port):
    sys.path.insert(0, str(ROOT))
    import bench
    u = S.prior_draw(S.PriorSpec(80, 1.0, 2.5), 808, 0xBE9C4, 2, ctx)
    spec = bench.c5_spec(S, u)
    est = S.observe_ad(spec, 808, ctx=ctx)
    assert len(est) == 64 and all(np.isfinite(e.mean) for e in est)
    for j in (0, 63):
        got = S.ad_particle_values(spec, j, 808, 32, ctx)
        want = port.ad_particle_values(spec, j, 808, 32)
        assert np.max(np.abs(got - want)) < 1e-11
    vals = S.ad_particle_values(spec, 63, 808, spec.n_particles, ctx)
    mean, se = reference_reduction(port, vals)
    assert est[63].mean == mean and est[63].std_error == se
