"""The C-ABI boundary on the CPU (no device calls): the in-tree library loads,
exports every entry point include/scalarmc_b200.h declares, agrees with the
ctypes struct layouts, and its host-side validation raises the reference's
exception types with the reference's messages."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

import paper_1808_10580_b200 as S
from paper_1808_10580_b200 import _abi as A
import specs

HEADER = Path(__file__).resolve().parents[1] / "include" / "scalarmc_b200.h"


def header_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"^[a-z_][\w \*]*?\b(smc_\w+)\s*\(", text, flags=re.M)))


def test_library_loads_and_exports_every_header_symbol():
    lib = A.load_library()
    names = header_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), f"{n} declared in include/scalarmc_b200.h but not exported"
        assert n in A._PROTOS, f"{n} missing from the ctypes prototype table"
    assert lib.smc_abi_version() == 1


def test_struct_layouts_match():
    lib = A.load_library()
    out = (C.c_int64 * 16)()
    n = lib.smc_struct_sizes(out, 16)
    mine = [C.sizeof(t) for t in (A.smc_estimate, A.smc_scalar_field, A.smc_velocity, A.smc_ad_problem,
                                  A.smc_domain, A.smc_bvp_problem, A.smc_prior, A.smc_stats)]
    assert list(out[:n]) == mine


def test_no_device_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError):
        S.Context(0)


def _ref_error(reference, fn, *args):
    try:
        fn(*args)
    except Exception as e:  # noqa: BLE001
        return type(e), str(e)
    return None, None


@pytest.mark.parametrize("case", range(8))
def test_validation_matches_reference(case, reference):
    spec = specs.c1_two_mode(n_particles=100)
    if case == 0:
        spec.observations = []
    elif case == 1:
        spec.observations = [S.AdObservation(0.0, S.Vec2(0.5, 0.5))]
    elif case == 2:
        spec.observations = [S.AdObservation(0.5, S.Vec2(1.5, 0.5))]
    elif case == 3:
        spec.observations = [S.AdObservation(0.5, S.Vec2(float("nan"), 0.5))]
    elif case == 4:
        spec.n_particles = 1
    elif case == 5:
        spec.observations = [S.AdObservation(0.5, S.Vec2(0.5, 1.0))]
    elif case == 6:
        spec.observations = [S.AdObservation(-1.0, S.Vec2(0.5, 0.5))]
    elif case == 7:
        spec.observations = [S.AdObservation(0.1, S.Vec2(0.0, 0.999))]
    ref_type, ref_msg = _ref_error(reference, reference.observe_ad, spec, 1, 1)
    try:
        spec.validate()
        mine = (None, None)
    except Exception as e:  # noqa: BLE001
        mine = (type(e), str(e))
    expected = {None: None, ValueError: ValueError, IndexError: IndexError, RuntimeError: RuntimeError}[ref_type]
    assert mine[0] is expected and mine[1] == ref_msg


@pytest.mark.parametrize("case", range(6))
def test_bvp_validation_matches_reference(case, reference):
    spec = specs.paper_bvp(n_particles=100)
    if case == 0:
        spec.domain = S.Domain.unit_torus()
    elif case == 1:
        spec.observations = [(1.5, 0.5)]
    elif case == 2:
        spec.observations = [(1.0, 0.5)]  # on the boundary: not strictly interior
    elif case == 3:
        spec.max_steps = 0
    elif case == 4:
        spec.observations = []
    elif case == 5:
        spec.n_particles = 1
    ref_type, ref_msg = _ref_error(reference, reference.observe_bvp, spec, 1, 1)
    with pytest.raises(ref_type) as ei:
        spec.validate()
    assert str(ei.value) == ref_msg


def test_field_constructor_errors_match_reference(reference):
    cases = [([S.VelocityMode(0, 0, 1.0)], 1), ([S.VelocityMode(2, 0, 1.0)], 1),
             ([S.VelocityMode(1, 0, complex(float("inf"), 0))], 1),
             ([S.VelocityMode(1, 1, 1.0), S.VelocityMode(-1, -1, 1.0)], 2), ([S.VelocityMode(1, 0, 1.0)], 0)]
    for modes, K in cases:
        with pytest.raises(ValueError) as mine:
            S.FourierVelocityField(modes, K)
        f = S.FourierVelocityField.__new__(S.FourierVelocityField)
        f._empty = False
        f.max_wavenumber = K
        f.k = np.array([[m.k1, m.k2] for m in modes], dtype=np.int32)
        f.coeff = np.array([[m.coeff.real, m.coeff.imag] for m in modes], dtype=np.float64)
        with pytest.raises(ValueError) as ref:
            reference.velocity_eval(S.VelocityField.fourier(f), [[0.1, 0.2]])
        assert str(mine.value) == str(ref.value)


def test_resolved_dt_matches_reference(reference, golden):
    c1 = specs.c1_two_mode()
    assert c1.resolved_dt() == reference.resolved_dt_ad(c1) == float.fromhex(golden["c1"]["resolved_dt"])
    for v in (S.VelocityField.constant((1.0, 1.0)), S.VelocityField.constant((0.0, 0.0)),
              S.VelocityField.fourier(specs.random_fourier(np.random.default_rng(1), 5, 3))):
        for kappa in (0.0, 0.282, 1e-4):
            for dom in (S.Domain.box((0, 0), (1, 1)), S.Domain.disk((0.5, 0.5), 0.5), S.Domain.box((0, 0), (40, 40))):
                spec = specs.paper_bvp(n_particles=10, observations=[(0.5, 0.5)], dt=0.0, velocity=v)
                spec.diffusion = S.DiffusionModel.isotropic(kappa)
                spec.domain = dom
                assert spec.resolved_dt() == reference.resolved_dt_bvp(spec)


def test_prior_modes_python_mirror(golden):
    assert [list(m) for m in S.PriorSpec(8).modes()] == golden["prior"]["modes8"]
    assert S.PriorSpec(8).dimension() == 196
    assert S.PriorSpec(25).dimension() == 1960
