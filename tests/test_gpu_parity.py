"""Parity of the CUDA forward map with the reference (GPU, -m gpu).

Every forward map goes through the C ABI (the ctypes mirror in
paper_1808_10580_b200.api).  Expected values are the golden fixtures made by
running the real reference (tests/golden/make_golden.py) or, where a fixture
would be too large, the plain-C oracle on the same inputs.

Tolerances (north_star / SURVEY.md §8(d) parity gate):
  FP64 means:   |gpu - ref| <= 1e-10 * max(|ref|, theta_scale)
  FP64 SE:      relative 1e-8
  FP32 means:   |gpu32 - ref| <= 3 SE_ref (+ the FP64 tolerance)
Integer / index work (Philox words, counts, n_failed) is bit-exact.
"""
import math

import numpy as np
import pytest

import paper_1808_10580_b200 as S
import specs
from conftest import est_from, unhex

pytestmark = pytest.mark.gpu

MEAN_RTOL = 1e-10
SE_RTOL = 1e-8


def theta_scale(field: S.ScalarField) -> float:
    if field.kind == 1:
        return sum(abs(t.amplitude) for t in field.terms)
    return 1.0


def assert_estimates(got, ref_list, scale=1.0, exact_counts=True):
    assert len(got) == len(ref_list)
    for j, (e, r) in enumerate(zip(got, ref_list)):
        r = est_from(r) if isinstance(r, dict) else r
        tol = MEAN_RTOL * max(abs(r["mean"]), scale)
        assert abs(e.mean - r["mean"]) <= tol, (j, e.mean, r["mean"], abs(e.mean - r["mean"]))
        assert abs(e.std_error - r["std_error"]) <= SE_RTOL * abs(r["std_error"]) + 1e-300, (j, e.std_error, r["std_error"])
        assert abs(e.aux_mean - r["aux_mean"]) <= MEAN_RTOL * max(abs(r["aux_mean"]), 1.0)
        if exact_counts:
            assert e.n_particles == r["n_particles"] and e.n_failed == r["n_failed"]


# ---------------------------------------------------------------- RNG ------
def test_device_philox_is_bit_exact(ctx, golden):
    g = golden["philox"]
    out = S.philox_device(np.array(g["ctr"]), np.array(g["key"]), ctx)
    assert out.tolist() == g["out"]


def test_device_normals_match_reference(ctx, golden):
    worst = 0.0
    identical = total = 0
    for rec in golden["normal_pairs"]:
        seed, obs, particle = rec["key"]
        got = S.normal_pairs_device(seed, obs, particle, 64, ctx)
        want = unhex(rec["pairs"])
        worst = max(worst, float(np.max(np.abs(got - want))))
        identical += int(np.sum(got.view(np.uint64) == want.view(np.uint64)))
        total += got.size
    assert worst < 1e-14
    # sincospi(2 u1) vs glibc sin/cos(2 pi u1): equal except in the last ulp
    assert identical / total > 0.3


# ---------------------------------------------------------------- AD -------
@pytest.mark.parametrize("precision", [S.Precision.fp64, S.Precision.fp64_strict])
def test_c1_matches_reference(ctx, golden, precision):
    g = golden["c1"]
    spec = specs.c1_two_mode(precision=precision)
    est = S.observe_ad(spec, 7, ctx=ctx)
    assert_estimates(est, g["estimates"], theta_scale(spec.initial_condition))
    assert abs(est[0].mean - (-0.795097030819361)) < 1e-10  # SURVEY.md §8c golden


@pytest.mark.parametrize("precision", [S.Precision.fp64, S.Precision.fp64_strict])
def test_c1_particles_match_reference(ctx, golden, precision):
    spec = specs.c1_two_mode(precision=precision)
    same = total = 0
    for j in range(3):
        got = S.ad_particle_values(spec, j, 7, 256, ctx)
        want = unhex(golden["c1"]["particles"][j])
        assert np.max(np.abs(got - want)) < 1e-12
        same += int(np.sum(got.view(np.uint64) == want.view(np.uint64)))
        total += got.size
    if precision == S.Precision.fp64_strict:
        # reference operation order: only libm rounding differs
        assert same / total > 0.2, same / total


def test_c2_matches_reference(ctx, golden):
    g = golden["c2"]
    u = unhex(g["u"])
    spec = specs.c2_spec(u, n_particles=g["n_particles"])
    assert_estimates(S.observe_ad(spec, 808, ctx=ctx), g["estimates"], 1.0)
    for idx, j in enumerate((0, 4, 8)):
        got = S.ad_particle_values(spec, j, 808, 128, ctx)
        assert np.max(np.abs(got - unhex(g["particles"][idx]))) < 1e-11


def test_c2_lattice_kernel_matches_reference(ctx, golden, monkeypatch):
    monkeypatch.setenv("SMC_DISABLE_DISK", "1")
    g = golden["c2"]
    spec = specs.c2_spec(unhex(g["u"]), n_particles=g["n_particles"])
    assert_estimates(S.observe_ad(spec, 808, ctx=ctx), g["estimates"], 1.0)


@pytest.mark.parametrize("ppt", ["1", "2"])
def test_c2_disk_particles_per_thread(ctx, golden, monkeypatch, ppt):
    monkeypatch.setenv("SMC_DISK_P", ppt)
    g = golden["c2"]
    spec = specs.c2_spec(unhex(g["u"]), n_particles=g["n_particles"])
    assert_estimates(S.observe_ad(spec, 808, ctx=ctx), g["estimates"], 1.0)


def test_c2_strict_matches_reference(ctx, golden):
    g = golden["c2"]
    spec = specs.c2_spec(unhex(g["u"]), n_particles=g["n_particles"], precision=S.Precision.fp64_strict)
    assert_estimates(S.observe_ad(spec, 808, ctx=ctx), g["estimates"], 1.0)


def test_heat_matches_reference_and_analytic(ctx, golden):
    spec = specs.heat_spec(0.01, 0.5, (0.0, 0.0), 20000, 1e-3)
    est = S.observe_ad(spec, 20240501, ctx=ctx)
    assert_estimates(est, golden["heat"]["estimates"], 1.0)
    target = math.exp(-4.0 * math.pi ** 2 * 0.01 * 0.5)  # acceptance.cpp:42
    assert abs(est[0].mean - target) <= 3.0 * est[0].std_error + 0.01


def test_batched_matches_reference_per_sample(ctx, golden):
    g = golden["c4"]
    U = unhex(g["U"])
    base = specs.c4_base(n_particles=g["n_particles"])
    out = S.observe_ad_batched(base, specs.C4_PRIOR, U, 808, ctx=ctx)
    for b in range(U.shape[0]):
        got = [S.ParticleEstimate(*[out[b, j][k] for k in out.dtype.names]) for j in range(out.shape[1])]
        assert_estimates(got, g["estimates"][b], 1.0)


def test_batched_equals_single_calls(ctx):
    rng = np.random.default_rng(1)
    prior = S.PriorSpec(4, 1.0, 2.0)
    U = rng.normal(size=(5, prior.dimension())) * 0.3
    base = specs.c4_base(n_particles=300)
    out = S.observe_ad_batched(base, prior, U, 99, ctx=ctx)
    for b in range(5):
        spec = specs.c4_base(n_particles=300)
        spec.velocity = S.VelocityField.fourier(S.velocity_from_coefficients(prior, U[b]))
        single = S.observe_ad(spec, 99, ctx=ctx)
        for j, e in enumerate(single):
            # batched runs the generic lattice kernel, single calls the disk kernel
            assert abs(out[b, j]["mean"] - e.mean) <= 1e-13
            assert abs(out[b, j]["std_error"] - e.std_error) <= 1e-12 * e.std_error


@pytest.mark.parametrize("K,n_particles", [(8, 160), (8, 100), (3, 40), (14, 96), (25, 160), (25, 70)])
def test_batched_grid_orders_identical(ctx, monkeypatch, K, n_particles):
    """Batched launches pick a grid order (sample-major; observation-major
    longest-first; observation-major over flattened (sample, particle)
    ranges) by launch size.  Every particle's path is addressed by (seed, obs,
    particle, step), so all orders give bit-identical estimates — including
    particle counts that are not a multiple of 32 (warps straddle samples), the
    generic tiled kernel (K = 14) and the tiled disk kernel (K = 25)."""
    prior = S.PriorSpec(K, 1.0, 2.5)
    U = np.random.default_rng(K).normal(size=(7, prior.dimension())) * 0.3
    base = specs.c4_base(n_particles=n_particles)
    want = S.observe_ad_batched(base, prior, U, 31, ctx=ctx)
    for env in ({"SMC_BATCH_ORDER": "sample"}, {"SMC_BATCH_ORDER": "obs", "SMC_NO_FLAT": "1"},
                {"SMC_BATCH_ORDER": "obs"}):
        with monkeypatch.context() as m:
            for k, v in env.items():
                m.setenv(k, v)
            got = S.observe_ad_batched(base, prior, U, 31, ctx=ctx)
        for f in ("mean", "std_error", "n_particles"):
            assert np.array_equal(got[f], want[f]), (env, f)


def test_batched_per_sample_seeds(ctx):
    prior = S.PriorSpec(3, 1.0, 2.0)
    U = np.tile(np.random.default_rng(2).normal(size=prior.dimension()) * 0.2, (3, 1))
    base = specs.c4_base(n_particles=256)
    crn = S.observe_ad_batched(base, prior, U, 5, ctx=ctx)
    assert np.array_equal(crn["mean"][0], crn["mean"][1])
    seeded = S.observe_ad_batched(base, prior, U, 5, seeds=np.array([5, 6, 7], dtype=np.uint64), ctx=ctx)
    assert np.array_equal(seeded["mean"][0], crn["mean"][0])
    assert not np.array_equal(seeded["mean"][1], crn["mean"][1])


def test_misfit_matches_reference(ctx, golden):
    g = golden["misfit"]
    prior = S.PriorSpec(2, 0.6, 2.5)
    fwd = specs.c4_base(n_particles=160)
    fwd.dt = 0.006
    like = S.LikelihoodSpec(data=g["data"], noise_std=g["noise_std"], forward=fwd, forward_seed=g["forward_seed"])
    phi = like.misfit(prior, unhex(g["u"]))
    ref = float.fromhex(g["phi"])
    assert abs(phi - ref) <= 1e-9 * max(abs(ref), 1.0)
    assert abs(like.misfit_batched(prior, unhex(g["u"])[None, :])[0] - ref) <= 1e-9 * max(abs(ref), 1.0)


# ------------------------------------------- reference unit tests, on GPU ----
def test_zero_diffusion_is_exact(ctx):
    # test_forward.cpp:34-47
    spec = S.AdProblemSpec(diffusion=S.DiffusionModel.isotropic(0.0),
                           initial_condition=S.ScalarField.cosine_mode(1, 0, 1.0), n_particles=4096,
                           observations=[S.AdObservation(0.5, S.Vec2(0.0, 0.25)),
                                         S.AdObservation(1.0, S.Vec2(0.125, 0.5))])
    for prec in (S.Precision.fp64, S.Precision.fp64_strict):
        spec.precision = prec
        est = S.observe_ad(spec, 1, ctx=ctx)
        for j, o in enumerate(spec.observations):
            assert est[j].mean == spec.initial_condition(o.x)
            assert est[j].std_error == 0.0


def test_single_slot_equivalence_and_determinism(ctx):
    # test_forward.cpp:59-82
    spec = specs.heat_spec(0.02, 0.25, (0.0, 0.0), 2000, 2e-3)
    spec.observations += [S.AdObservation(0.5, S.Vec2(0.25, 0.75)), S.AdObservation(0.6, S.Vec2(0.5, 0.5))]
    full = S.observe_ad(spec, 5, ctx=ctx)
    for j in range(3):
        single = S.observe_ad_single(spec, j, 5, ctx=ctx)
        assert single == full[j]
    with pytest.raises(IndexError):
        S.observe_ad_single(spec, 3, 5, ctx=ctx)
    truncated = specs.heat_spec(0.02, 0.25, (0.0, 0.0), 2000, 2e-3)
    truncated.observations += [S.AdObservation(0.5, S.Vec2(0.25, 0.75))]
    part = S.observe_ad(truncated, 5, ctx=ctx)
    assert part[0] == full[0] and part[1] == full[1]
    assert S.observe_ad(spec, 5, ctx=ctx) == full


def test_linearity_in_theta0(ctx):
    # test_forward.cpp:84-94
    base = specs.heat_spec(0.03, 0.2, (0.3, 0.6), 3000, 1e-3)
    base.initial_condition = S.ScalarField.cosine_mode(1, 1, 1.0, 0.4)
    scaled = specs.heat_spec(0.03, 0.2, (0.3, 0.6), 3000, 1e-3)
    scaled.initial_condition = S.ScalarField.cosine_series([(-2.5, (2 * math.pi, 2 * math.pi), 0.4),
                                                            (1.25, (0.0, 0.0), 0.0)])
    g = S.observe_ad(base, 21, ctx=ctx)[0]
    h = S.observe_ad(scaled, 21, ctx=ctx)[0]
    assert abs(h.mean - (-2.5 * g.mean + 1.25)) <= 1e-12 * abs(-2.5 * g.mean + 1.25)


def test_maximum_principle_property(ctx):
    # acceptance.cpp:362-406, 200 random configurations, N_p = 32
    rng = np.random.default_rng(4096)
    violations = 0
    for trial in range(200):
        f = specs.random_fourier(rng, int(rng.integers(1, 4)), 3)
        c, a = 4 * rng.random() - 2, 2 * rng.random() - 1
        tk1, tk2 = (int(v) for v in rng.integers(-3, 4, size=2))
        if tk1 == 0 and tk2 == 0:
            tk1 = 1
        t = 0.05 + 0.25 * rng.random()
        spec = S.AdProblemSpec(velocity=S.VelocityField.fourier(f),
                               diffusion=S.DiffusionModel.isotropic(0.1 * rng.random()),
                               initial_condition=S.ScalarField.cosine_series(
                                   [(a, (2 * math.pi * tk1, 2 * math.pi * tk2), 0.0), (c, (0.0, 0.0), 0.0)]),
                               observations=[S.AdObservation(t, S.Vec2(rng.random(), rng.random()))],
                               dt=t / 20.0, n_particles=32)
        m = S.observe_ad(spec, 5000 + trial, ctx=ctx)[0].mean
        violations += not (c - abs(a) <= m <= c + abs(a))
    assert violations == 0


def test_validation_errors_on_device_path(ctx):
    spec = S.AdProblemSpec()
    with pytest.raises(ValueError, match="no observations"):
        S.observe_ad(spec, 0, ctx=ctx)
    spec.observations = [S.AdObservation(0.0, S.Vec2(0.5, 0.5))]
    with pytest.raises(ValueError, match="times must be positive"):
        S.observe_ad(spec, 0, ctx=ctx)
    spec.observations = [S.AdObservation(0.5, S.Vec2(1.5, 0.5))]
    with pytest.raises(ValueError, match=r"\[0,1\)\^2"):
        S.observe_ad(spec, 0, ctx=ctx)


# ------------------------------------------------ sharded (multi-GPU) path ----
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_sharded_partials_are_bit_identical(ctx, world):
    u = S.prior_draw(specs.C2_PRIOR, 808, 0xBE9C4, 0, ctx)
    spec = specs.c2_spec(u, n_particles=5000)
    spec.observations = spec.observations[:3]
    spec.observations = [S.AdObservation(0.2, o.x) for o in spec.observations]
    whole = S.observe_ad(spec, 808, ctx=ctx)
    est = S.observe_ad(spec, 808, ctx=S.Context(devices=[0] * world))
    for a, b in zip(whole, est):
        assert a.mean == b.mean and a.std_error == b.std_error


def test_more_observations_than_one_grid_dimension(ctx):
    """70 000 observations (> 65 535, one grid dimension) run in chunks; each
    estimate depends only on its own observation slot, so it equals the
    single-observation call for that slot in either chunk."""
    rng = np.random.default_rng(5)
    xs = rng.random((70000, 2))
    spec = S.AdProblemSpec(diffusion=S.DiffusionModel.isotropic(0.02),
                           initial_condition=S.ScalarField.cosine_mode(1, 1, 1.0),
                           observations=[S.AdObservation(0.01, S.Vec2(*x)) for x in xs], n_particles=4, dt=0.005)
    est = S.observe_ad(spec, 9, ctx=ctx)
    assert len(est) == 70000
    for j in (0, 65534, 65535, 69999):
        one = S.observe_ad_single(spec, j, 9, ctx=ctx)
        assert one.mean == est[j].mean and one.std_error == est[j].std_error, j


@pytest.mark.parametrize("max_steps", [10_000_000, 150])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_bvp_walker_sharding_bit_identical(ctx, world, max_steps):
    """SURVEY.md 8(e) for the Dirichlet map: walker ranges per rank, valid
    counts and aligned dyadic block sums exchanged — equal to observe_bvp bit
    for bit for any split, including runs where walkers fail (max_steps 150:
    the compaction before the reference's tree then depends on failures in
    other ranks' ranges)."""
    spec = specs.paper_bvp(n_particles=5000)
    spec.max_steps = max_steps
    want = S.observe_bvp(spec, 606, ctx=ctx)
    got = S.observe_bvp(spec, 606, ctx=S.Context(devices=[0] * world))
    if max_steps == 150:
        assert sum(e.n_failed for e in want) > 0
    for a, b in zip(got, want):
        assert (a.mean, a.std_error, a.n_particles, a.n_failed, a.aux_mean) == \
            (b.mean, b.std_error, b.n_particles, b.n_failed, b.aux_mean)


# ---------------------------------------------------------------- FP32 -----
def test_fp32_within_three_standard_errors(ctx, golden):
    spec = specs.c1_two_mode(n_particles=10000, precision=S.Precision.fp32)
    est = S.observe_ad(spec, 7, ctx=ctx)
    for e, r in zip(est, golden["c1"]["estimates"]):
        r = est_from(r)
        assert abs(e.mean - r["mean"]) <= 3.0 * r["std_error"]
    u = unhex(golden["c2"]["u"])
    spec2 = specs.c2_spec(u, n_particles=512, precision=S.Precision.fp32)
    for e, r in zip(S.observe_ad(spec2, 808, ctx=ctx), golden["c2"]["estimates"]):
        r = est_from(r)
        assert abs(e.mean - r["mean"]) <= 3.0 * r["std_error"]


def test_fp32_param_path_matches_shared_memory_path(ctx, golden, monkeypatch):
    """FP32 single-sample launches take the coefficient block as a kernel
    parameter (converted to float on the host); the shared-memory kernel
    (SMC_DISK_P=2) converts on the device.  Same floats, same arithmetic per
    particle: identical particle values."""
    u = unhex(golden["c2"]["u"])
    spec = specs.c2_spec(u, n_particles=4096, precision=S.Precision.fp32)
    a = [S.ad_particle_values(spec, j, 808, 4096, ctx) for j in (0, 8)]
    monkeypatch.setenv("SMC_DISK_P", "2")
    b = [S.ad_particle_values(spec, j, 808, 4096, ctx) for j in (0, 8)]
    for x, y in zip(a, b):
        assert np.array_equal(x, y), float(np.max(np.abs(x - y)))


@pytest.mark.parametrize("K", [1, 5, 12, 25])
def test_fp32_param_path_matches_batched_path(ctx, K):
    """The packed FP32 kernel-parameter form (FFMA2) against the batched
    shared-memory kernel on the same single sample, across the disk sizes:
    identical estimates."""
    prior = S.PriorSpec(K, 1.0, 2.5)
    u = np.random.default_rng(100 + K).normal(size=prior.dimension()) * 0.4
    base = specs.c4_base(n_particles=1000, precision=S.Precision.fp32)
    batched = S.observe_ad_batched(base, prior, u[None, :], 77, ctx=ctx)
    spec = specs.c4_base(n_particles=1000, precision=S.Precision.fp32)
    spec.velocity = S.VelocityField.fourier(S.velocity_from_coefficients(prior, u))
    single = S.observe_ad(spec, 77, ctx=ctx)
    for j, e in enumerate(single):
        assert batched[0, j]["mean"] == e.mean and batched[0, j]["std_error"] == e.std_error, j


@pytest.mark.parametrize("disable_disk,K", [(False, 14), (False, 25), (True, 6)])
def test_fp32_tiled_kernel_within_three_standard_errors(ctx, monkeypatch, disable_disk, K):
    """The FP32 tiled lattice kernel (packed FFMA2 pair updates; FP32 dense
    fields above K = 12 take it too — the tiled disk kernel is FP64 only)
    against the FP64 parity path on the same streams."""
    if disable_disk:
        monkeypatch.setenv("SMC_DISABLE_DISK", "1")
    prior = S.PriorSpec(K, 1.0, 2.5)
    U = np.random.default_rng(3).normal(size=(2, prior.dimension())) * 0.5
    b64 = S.observe_ad_batched(specs.c4_base(n_particles=4000), prior, U, 12, ctx=ctx)
    b32 = S.observe_ad_batched(specs.c4_base(n_particles=4000, precision=S.Precision.fp32), prior, U, 12, ctx=ctx)
    assert np.all(np.abs(b32["mean"] - b64["mean"]) <= 3.0 * b64["std_error"])
    spec = specs.c4_base(n_particles=4000, precision=S.Precision.fp32)
    spec.velocity = S.VelocityField.fourier(S.velocity_from_coefficients(prior, U[0]))
    single = S.observe_ad(spec, 12, ctx=ctx)
    assert all(abs(e.mean - m) <= 3.0 * se for e, m, se in zip(single, b64["mean"][0], b64["std_error"][0]))


# ---------------------------------------------------------------- BVP ------
def test_bvp_box_matches_reference(ctx, golden):
    g = golden["bvp_box"]
    spec = specs.paper_bvp()
    est = S.observe_bvp(spec, 606, ctx=ctx)
    assert_estimates(est, g["estimates"], 1.0)
    vals, aux, failed = S.bvp_particle_values(spec, 0, 606, 256, ctx)
    p = g["particles"]
    assert failed.tolist() == p["failed"]
    assert np.max(np.abs(vals - unhex(p["values"]))) < 1e-11
    assert np.max(np.abs(aux - unhex(p["aux"]))) < 1e-12


def test_bvp_strict_matches_reference(ctx, golden):
    spec = specs.paper_bvp(precision=S.Precision.fp64_strict)
    assert_estimates(S.observe_bvp(spec, 606, ctx=ctx), golden["bvp_box"]["estimates"], 1.0)


def test_c3_shape_matches_reference(ctx, golden):
    assert_estimates(S.observe_bvp(specs.c3_spec(n_particles=512), 606, ctx=ctx), golden["c3"]["estimates"], 1.0)


def test_bvp_disk_fourier_matches_reference(ctx, golden):
    disk = specs.paper_bvp(n_particles=1000, amplitudes=(1.0, -0.5, 2.0), observations=[(0.5, 0.5), (0.3, 0.6)],
                           velocity=S.VelocityField.fourier(specs.random_fourier(np.random.default_rng(5), 6, 3)))
    disk.domain = S.Domain.disk((0.5, 0.5), 0.5)
    disk.dt = 5e-4
    assert_estimates(S.observe_bvp(disk, 5, ctx=ctx), golden["bvp_disk"]["estimates"], 1.0)


def test_bvp_max_steps_failures_excluded(ctx, golden):
    fail = specs.paper_bvp(n_particles=300, observations=[(0.94, 0.94), (0.8, 0.5)])
    fail.max_steps = 300
    assert_estimates(S.observe_bvp(fail, 77, ctx=ctx), golden["bvp_maxsteps"]["estimates"], 1.0)
    fail.observations = [(0.5, 0.5)]
    fail.max_steps = 5
    with pytest.raises(RuntimeError, match="every particle of an observation failed"):
        S.observe_bvp(fail, 77, ctx=ctx)


def test_bvp_constant_boundary_exact(ctx):
    # test_forward.cpp:112-126
    spec = S.BvpProblemSpec(diffusion=S.DiffusionModel.isotropic(0.2), boundary_data=S.ScalarField.constant(3.5),
                            observations=[(0.5, 0.5), (0.25, 0.7)], n_particles=1024, dt=1e-3)
    for e in S.observe_bvp(spec, 9, ctx=ctx):
        assert e.mean == 3.5 and e.std_error == 0.0 and e.aux_mean > 0.0 and e.n_failed == 0


def test_bvp_manufactured_solution(ctx):
    # test_forward.cpp:128-141 / acceptance.cpp:88-104
    spec = S.BvpProblemSpec(velocity=S.VelocityField.constant((1.0, 1.0)), diffusion=S.DiffusionModel.isotropic(0.25),
                            forcing=S.ScalarField.constant(-2.0), boundary_data=S.ScalarField.affine(0.0, (1.0, 1.0)),
                            observations=[(0.5, 0.5)], n_particles=100000, dt=2e-4)
    e = S.observe_bvp(spec, 31415, ctx=ctx)[0]
    assert abs(e.mean - 1.0) <= 3.0 * e.std_error + 0.01


def test_bvp_linearity(ctx):
    # test_forward.cpp:143-164
    h = math.pi / 2
    spec = S.BvpProblemSpec(velocity=S.VelocityField.constant((0.5, -0.25)), diffusion=S.DiffusionModel.isotropic(0.15),
                            forcing=S.ScalarField.gaussian_bumps([(1.0, (0.4, 0.4))], 4.0),
                            boundary_data=S.ScalarField.cosine_series([(0.5, (h, 0.0), 0.0), (0.5, (0.0, h), 0.0)]),
                            observations=[(0.5, 0.5), (0.3, 0.8)], n_particles=2000, dt=5e-4)
    a = -3.0
    scaled = S.BvpProblemSpec(velocity=spec.velocity, diffusion=spec.diffusion,
                              forcing=spec.forcing.with_bump_amplitudes([a]),
                              boundary_data=S.ScalarField.cosine_series([(a * 0.5, (h, 0.0), 0.0),
                                                                         (a * 0.5, (0.0, h), 0.0)]),
                              observations=spec.observations, n_particles=2000, dt=5e-4)
    for b, m in zip(S.observe_bvp(spec, 17, ctx=ctx), S.observe_bvp(scaled, 17, ctx=ctx)):
        assert abs(m.mean - a * b.mean) <= 1e-12 * abs(a * b.mean)


def test_forcing_cost_matches_reference(ctx, golden):
    for rec in golden["forcing_cost"]:
        control = S.ForcingControl(initial_amplitudes=rec["F"], centers=[(0.68, 0.4), (0.4, 0.68), (0.82, 0.82)],
                                   sharpness=4.0, target=rec["target"],
                                   observation_points=[(0.88, 0.6), (0.6, 0.88), (0.94, 0.94)])
        cost = S.forcing_cost(rec["F"], control, specs.paper_bvp(n_particles=400), rec["seed"])
        ref = float.fromhex(rec["cost"])
        assert abs(cost - ref) <= 1e-9 * max(ref, 1.0)


def test_bvp_fp32_within_three_standard_errors(ctx, golden):
    spec = specs.paper_bvp(precision=S.Precision.fp32)
    for e, r in zip(S.observe_bvp(spec, 606, ctx=ctx), golden["bvp_box"]["estimates"]):
        r = est_from(r)
        assert abs(e.mean - r["mean"]) <= 3.0 * r["std_error"]


def test_batched_non_finite_coefficient_rejected(ctx):
    """velocity_from_coefficients -> FourierVelocityField ctor (fields.cpp:46-47)
    throws std::invalid_argument before any work; the device packer checks
    every coefficient it reads."""
    prior = S.PriorSpec(3, 1.0, 2.0)
    U = np.zeros((4, prior.dimension()))
    U[2, 5] = np.inf
    with pytest.raises(ValueError, match="non-finite coefficient"):
        S.observe_ad_batched(specs.c4_base(n_particles=64), prior, U, 1, ctx=ctx)
    U[2, 5] = 0.0
    S.observe_ad_batched(specs.c4_base(n_particles=64), prior, U, 1, ctx=ctx)  # context still usable


@pytest.mark.parametrize("disk_velocity", [True, False])
def test_bvp_dense_fourier_velocity_matches_oracle(ctx, port, monkeypatch, disk_velocity):
    """C3b: the paper BVP with C2's K=8 prior-draw velocity.
    A dense field takes the walkers with the compile-time disk series
    (bvp_disk.cu); SMC_DISABLE_DISK forces the tiled lattice walkers."""
    if not disk_velocity:
        monkeypatch.setenv("SMC_DISABLE_DISK", "1")
    spec = specs.c3_spec(n_particles=400)
    spec.observations = spec.observations[:3]
    u = S.prior_draw(specs.C2_PRIOR, 808, 0xBE9C4, 0, ctx)
    spec.velocity = S.VelocityField.fourier(S.velocity_from_coefficients(specs.C2_PRIOR, u))
    got = S.observe_bvp(spec, 606, ctx=ctx)
    want = port.observe_bvp(spec, 606)
    assert_estimates(got, list(want), 1.0)


@pytest.mark.parametrize("n", [2, 3, 1023, 1024, 1025, 4097])
def test_ragged_particle_counts(ctx, port, n):
    """Chunk boundaries of K3 (1024-leaf chunks, -0.0 padding): the estimate
    is the reference's pairwise reduction of the kernel's own per-particle
    values, bit for bit, and the particles are the oracle's."""
    spec = specs.c1_two_mode(n_particles=n)
    est = S.observe_ad(spec, 7, ctx=ctx)
    for j in range(len(spec.observations)):
        vals = S.ad_particle_values(spec, j, 7, n, ctx)
        mean = port.pairwise_sum(vals) / n
        var = port.pairwise_sum((vals - mean) ** 2) / (n - 1)
        assert est[j].mean == mean and est[j].std_error == math.sqrt(var / n)
        assert est[j].n_particles == n and est[j].n_failed == 0
        assert np.max(np.abs(vals - port.ad_particle_values(spec, j, 7, n))) < 1e-12


@pytest.mark.parametrize("n", [2, 5, 1025])
def test_bvp_ragged_with_failures(ctx, port, n):
    """max_steps failures excluded before the tree (executor.cpp:93-101) at
    ragged walker counts."""
    spec = specs.paper_bvp(n_particles=n, observations=[(0.94, 0.94), (0.5, 0.5)])
    spec.max_steps = 60
    try:
        want = port.observe_bvp(spec, 606)
    except RuntimeError:
        with pytest.raises(RuntimeError):
            S.observe_bvp(spec, 606, ctx=ctx)
        return
    got = S.observe_bvp(spec, 606, ctx=ctx)
    assert_estimates(got, list(want), 1.0)


def test_milstein_equals_euler_maruyama_for_isotropic_diffusion(ctx):
    """milstein_step returns em_step for isotropic diffusion (sde.cpp:18-22):
    the scheme flag must not change a single bit."""
    spec = specs.c1_two_mode(n_particles=2000)
    em = S.observe_ad(spec, 7, ctx=ctx)
    spec.scheme = S.StepScheme.milstein
    assert S.observe_ad(spec, 7, ctx=ctx) == em
    bvp = specs.paper_bvp(n_particles=500)
    em_b = S.observe_bvp(bvp, 606, ctx=ctx)
    bvp.scheme = S.StepScheme.milstein
    assert S.observe_bvp(bvp, 606, ctx=ctx) == em_b


def test_concurrent_contexts_do_not_interfere():
    """Two contexts (own streams and buffers) driven from two host threads at
    once reproduce their serial results bit for bit — the kernel-parameter
    coefficient path and every buffer are per launch / per context."""
    import threading
    u = [S.prior_draw(specs.C2_PRIOR, 808, 0xBE9C4, j, None) for j in range(2)]
    spec = [specs.c2_spec(u[j], n_particles=20000) for j in range(2)]
    for sp in spec:
        sp.observations = sp.observations[:3]
    ctxs = [S.Context(0), S.Context(0)]
    serial = [S.observe_ad(spec[j], 808, ctx=ctxs[j]) for j in range(2)]
    bvp = specs.paper_bvp(n_particles=2000)
    serial_b = S.observe_bvp(bvp, 606, ctx=ctxs[1])
    out = [None, None, None]

    def run(j):
        for _ in range(3):
            out[j] = S.observe_ad(spec[j], 808, ctx=ctxs[j])
            if j == 1:
                out[2] = S.observe_bvp(bvp, 606, ctx=ctxs[1])
    threads = [threading.Thread(target=run, args=(j,)) for j in range(2)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert out[0] == serial[0] and out[1] == serial[1] and out[2] == serial_b
    for c in ctxs:
        c.close()


def test_k25_dense_field_paths(ctx, port, monkeypatch):
    """The tiled disk kernels (K = 25, the C4 prior): the single-sample
    shared-memory form, the batched form and the unit-mode parameter form
    (a 3-rank group on one GPU) give identical estimates; the runtime-tiled
    lattice kernel agrees to rounding; particles are the oracle's."""
    prior = specs.C4_PRIOR
    u = S.prior_draw(prior, 808, 0xBE9C4, 1, ctx)
    spec = specs.c4_base(n_particles=1500)
    spec.velocity = S.VelocityField.fourier(S.velocity_from_coefficients(prior, u))
    disk = S.observe_ad(spec, 808, ctx=ctx)
    batched = S.observe_ad_batched(specs.c4_base(n_particles=1500), prior, u[None, :], 808, ctx=ctx)
    grouped = S.observe_ad(spec, 808, ctx=S.Context(devices=[0, 0, 0]))
    for j, e in enumerate(disk):
        assert (batched[0, j]["mean"], batched[0, j]["std_error"]) == (e.mean, e.std_error)
        assert (grouped[j].mean, grouped[j].std_error) == (e.mean, e.std_error)
    for j in (0, 4, 8):
        vals = S.ad_particle_values(spec, j, 808, 64, ctx)
        assert np.max(np.abs(vals - port.ad_particle_values(spec, j, 808, 64))) < 1e-11
    spec32 = specs.c4_base(n_particles=1500, precision=S.Precision.fp32)
    spec32.velocity = spec.velocity
    single32 = S.observe_ad(spec32, 808, ctx=ctx)
    grouped32 = S.observe_ad(spec32, 808, ctx=S.Context(devices=[0, 0]))
    assert [(e.mean, e.std_error) for e in single32] == [(e.mean, e.std_error) for e in grouped32]
    assert all(abs(a.mean - b.mean) <= 3.0 * b.std_error for a, b in zip(single32, disk))
    monkeypatch.setenv("SMC_DISABLE_DISK", "1")
    lattice = S.observe_ad(spec, 808, ctx=ctx)
    for a, b in zip(lattice, disk):
        assert abs(a.mean - b.mean) <= 1e-12 and abs(a.std_error - b.std_error) <= 1e-10 * b.std_error


@pytest.mark.parametrize("sharpness", [4.0, 150.0, 2000.0])
def test_bvp_bump_exponent_range_paths(ctx, port, sharpness):
    """The walkers' table exponential (fm::exp_bump) is valid for exponents in
    [-708, 0]; prepare_bvp proves -a|x - c|^2 >= -700 over the domain's
    bounding box (a = 4 and 150: proved, table path) or falls back to the
    generic evaluator (a = 2000: max a d^2 ~ 1600).  Both match the oracle."""
    centers = [(0.68, 0.4), (0.4, 0.68), (0.82, 0.82)]
    spec = specs.c3_spec(n_particles=600)
    spec.observations = [(0.7, 0.42), (0.5, 0.5), (0.83, 0.8)]
    spec.forcing = S.ScalarField.gaussian_bumps(
        [S.Bump(a, S.Vec2(*c)) for a, c in zip((1.0, -0.5, 2.0), centers)], sharpness)
    got = S.observe_bvp(spec, 606, ctx=ctx)
    want = port.observe_bvp(spec, 606)
    assert_estimates(got, list(want), 1.0)


def test_forward_maps_on_a_busy_stream(ctx):
    """The problem image's H2D copy reads pinned staging memory; when the
    context's stream is busy (here: a 0.1 s sleep kernel queued ahead, as the
    bench's L2 flush or a caller's own work can be) that copy is still
    pending while the host enqueues the rest of the call, so nothing else may
    write the staging buffer before the call's final sync (the Dirichlet
    map's walker-step readback once did).  Results equal the idle-stream ones."""
    import torch
    busy = S.Context(0)
    s = torch.cuda.Stream(device=0)
    S.load_library().smc_set_stream(busy.handle, s.cuda_stream)
    bvp = specs.paper_bvp(n_particles=3000, amplitudes=(1.0, -0.5, 2.0))
    ad = specs.c1_two_mode(n_particles=4096)
    for run in (lambda c: S.observe_bvp(bvp, 606, ctx=c), lambda c: S.observe_ad(ad, 7, ctx=c)):
        want = run(ctx)
        with torch.cuda.stream(s):
            torch.cuda._sleep(200_000_000)
        got = run(busy)
        for a, b in zip(got, want):
            assert (a.mean, a.std_error, a.aux_mean, a.n_particles, a.n_failed) == \
                (b.mean, b.std_error, b.aux_mean, b.n_particles, b.n_failed)
