"""Pin the oracle (CPU): the plain-C restatement must reproduce the real
reference bit for bit — against the committed golden fixtures (generated from
the reference compiled from its own sources) and, when oracle/_ref is built,
directly against the reference on fresh random inputs."""
import math

import numpy as np
import pytest

import paper_1808_10580_b200 as S
import specs
from conftest import est_from, unhex


def bits(a):
    return np.asarray(a, dtype=np.float64).view(np.uint64)


def same(a, b):
    return np.array_equal(bits(a), bits(b))


def test_philox_known_answers(port, golden):
    g = golden["philox"]
    out = port.philox(g["ctr"], g["key"])
    assert out.tolist() == g["out"]
    # Random123 philox4x32-10 KAT
    assert [f"{w:08x}" for w in out[0]] == ["6627e8d5", "e169c58d", "bc57ac4c", "9b00dbd8"]
    assert [f"{w:08x}" for w in out[1]] == ["408f276d", "41c83b0e", "a20bc7c6", "6d5451fd"]
    assert [f"{w:08x}" for w in out[2]] == ["d16cfe09", "94fdcceb", "5001e420", "24126ea1"]


def test_normal_pairs_bitwise(port, golden):
    for rec in golden["normal_pairs"]:
        seed, obs, particle = rec["key"]
        assert same(port.normal_pairs(seed, obs, particle, 64), unhex(rec["pairs"]))
    first = port.normal_pairs(0, 0, 0, 1)[0]
    assert first[0] == -0.39766753844418196 and first[1] == -0.31039547880173834


def test_stream_caches_bitwise(port, golden):
    g = golden["stream_draws"]
    assert same(port.stream_draws(*g["key"], g["ops"]), unhex(g["out"]))


def test_pairwise_sum_bitwise(port, golden):
    for rec in golden["pairwise_sum"]:
        v = unhex(rec["values"]) if rec["values"] else np.zeros(0)
        assert same(port.pairwise_sum(v), float.fromhex(rec["sum"]))


def test_pairwise_sum_power_of_two_exact(port):
    # test_rng_executor.cpp:82-84
    assert port.pairwise_sum(np.full(4096, 0.8207058237)) == 4096.0 * 0.8207058237
    assert port.pairwise_sum(np.zeros(0)) == 0.0


def test_velocity_bitwise(port, golden):
    for rec in golden["velocity"]:
        f = S.FourierVelocityField.from_arrays(np.array(rec["k"]), unhex(rec["coeff"]), rec["K"])
        got = port.velocity_eval(S.VelocityField.fourier(f), unhex(rec["x"]))
        assert same(got, unhex(rec["v"]))


def test_velocity_single_pair_hand_value(port):
    # test_fields.cpp:51-72: k=(1,0), v_k = i/2 -> v2 at x1=0.25 is -1.
    f = S.VelocityField.fourier(S.FourierVelocityField([S.VelocityMode(1, 0, 0.5j)], 1))
    v = port.velocity_eval(f, [[0.25, 0.0]])
    assert v[0, 0] == 0.0
    assert abs(v[0, 1] + 1.0) < 1e-15


def _check_estimates(got, ref_list):
    assert len(got) == len(ref_list)
    for e, r in zip(got, ref_list):
        r = est_from(r)
        for k in ("mean", "std_error", "aux_mean"):
            assert same(e[k], r[k]), (k, e[k], r[k])
        assert int(e["n_particles"]) == r["n_particles"] and int(e["n_failed"]) == r["n_failed"]


def test_c1_forward_map_bitwise(port, golden):
    g = golden["c1"]
    spec = specs.c1_two_mode()
    _check_estimates(port.observe_ad(spec, 7), g["estimates"])
    assert float.fromhex(g["estimates"][0]["mean"]) == -0.795097030819361
    for j in range(3):
        assert same(port.ad_particle_values(spec, j, 7, 256), unhex(g["particles"][j]))


def test_c2_particles_bitwise(port, golden):
    g = golden["c2"]
    u = unhex(g["u"])
    spec = specs.c2_spec(u, n_particles=g["n_particles"])
    for idx, j in enumerate((0, 4, 8)):
        assert same(port.ad_particle_values(spec, j, 808, 32), unhex(g["particles"][idx])[:32])


def test_prior_modes_and_draw(port, golden):
    assert port.prior_modes(8).tolist() == golden["prior"]["modes8"]
    assert port.prior_modes(8).tolist() == [list(m) for m in specs.C2_PRIOR.modes()]
    assert same(port.prior_draw(specs.C2_PRIOR, 808, 0xBE9C4, 0), unhex(golden["prior"]["draw8"]))


def test_bvp_box_bitwise(port, golden):
    g = golden["bvp_box"]
    spec = specs.paper_bvp()
    vals, aux, failed, steps = port.bvp_particle_values(spec, 0, 606, 256)
    p = g["particles"]
    assert same(vals, unhex(p["values"])) and same(aux, unhex(p["aux"]))
    assert failed.tolist() == p["failed"] and steps.tolist() == p["steps"]


@pytest.mark.slow
def test_bvp_box_estimates_bitwise(port, golden):
    _check_estimates(port.observe_bvp(specs.paper_bvp(), 606), golden["bvp_box"]["estimates"])


def test_bvp_failures_bitwise(port, golden):
    fail = specs.paper_bvp(n_particles=300, observations=[(0.94, 0.94), (0.8, 0.5)])
    fail.max_steps = 300
    _check_estimates(port.observe_bvp(fail, 77), golden["bvp_maxsteps"]["estimates"])


def test_bvp_disk_fourier_bitwise(port, golden):
    disk = specs.paper_bvp(n_particles=1000, amplitudes=(1.0, -0.5, 2.0), observations=[(0.5, 0.5), (0.3, 0.6)],
                           velocity=S.VelocityField.fourier(specs.random_fourier(np.random.default_rng(5), 6, 3)))
    disk.domain = S.Domain.disk((0.5, 0.5), 0.5)
    disk.dt = 5e-4
    _check_estimates(port.observe_bvp(disk, 5), golden["bvp_disk"]["estimates"])


# ---- direct comparison with the compiled reference (when built) ----------
def test_port_matches_reference_random_fields(port, reference):
    rng = np.random.default_rng(99)
    for trial in range(6):
        f = specs.random_fourier(rng, int(rng.integers(1, 20)), int(rng.integers(1, 7)))
        x = rng.random((64, 2))
        assert same(port.velocity_eval(S.VelocityField.fourier(f), x),
                    reference.velocity_eval(S.VelocityField.fourier(f), x))
        spec = specs.c1_two_mode(n_particles=64)
        spec.velocity = S.VelocityField.fourier(f)
        spec.diffusion = S.DiffusionModel.isotropic(float(rng.random() * 0.1))
        for j in range(3):
            assert same(port.ad_particle_values(spec, j, trial, 64), reference.ad_particle_values(spec, j, trial, 64))


def test_port_matches_reference_scalar_fields(port, reference):
    rng = np.random.default_rng(3)
    x = rng.random((50, 2)) * 2 - 0.5
    fields = [S.ScalarField.constant(3.5), S.ScalarField.affine(0.3, (1.0, -2.0)),
              S.ScalarField.gaussian_bumps([(1.0, (0.4, 0.4)), (-2.0, (0.1, 0.9))], 3.0),
              S.ScalarField.cosine_series([(0.5, (math.pi / 2, 0.0), 0.1), (0.25, (1.0, 2.0), -0.3)])]
    for f in fields:
        assert same(port.scalar_eval(f, x), reference.scalar_eval(f, x))
