"""Config-file parity: paper_1808_10580_b200.config
against the reference's own parse_config / make_*_spec / make_likelihood /
make_forcing_control (src/config.cpp, compiled in place; oracle/ref_cli.cpp).

Each case mutates a valid base configuration; the reference's verdict
(accepted, or the exception type and its what() text) must be reproduced
exactly.  Runs on CPU: the parser and the host-side validators need no GPU.
"""
import copy
import json
import math

import pytest

from paper_1808_10580_b200 import config as K
from paper_1808_10580_b200.records import RecordWriter, format_double

AD = {
    "problem": "ad",
    "velocity": {"kind": "fourier", "max_wavenumber": 2, "modes": [[1, 0, 0.25, -0.1], [1, -1, 0.05, 0.2]]},
    "diffusion": {"kappa": 0.03},
    "initial_condition": {"kind": "cosine", "terms": [{"k": [1, 0], "amplitude": 0.9},
                                                      {"freq": [0.0, 6.283185307179586], "phase": 0.4}]},
    "observations": [{"t": 0.05, "x": [0.3, 0.6]}, {"t": 0.08, "x": [0.9, 0.1]}],
    "particles": 2048, "dt": 0.002, "seed": 11, "workers": 0,
    "prior": {"cutoff": 2, "s0": 0.7, "alpha": 2.0},
    "likelihood": {"data": [0.5, -0.25], "noise_std": 0.08, "forward_seed": 5},
    "mcmc": {"steps": 40, "beta": 0.3, "burn_in": 4, "thin": 3},
}
BVP = {
    "problem": "bvp",
    "velocity": {"kind": "constant", "value": [0.5, -0.25]},
    "diffusion": {"kappa": 0.2},
    "forcing": {"kind": "bumps", "amplitudes": [0.5, 1.0], "centers": [[0.3, 0.3], [0.7, 0.6]], "sharpness": 3.0},
    "boundary": {"kind": "linear", "offset": 0.1, "gradient": [1.0, -0.5]},
    "domain": {"kind": "box", "lower": [0.0, 0.0], "upper": [1.0, 1.0]},
    "observations": [{"x": [0.4, 0.5]}, {"x": [0.8, 0.2]}],
    "particles": 1000, "dt": 0.0005, "max_steps": 100000, "seed": 3,
    "optimize": {"centers": [[0.3, 0.3], [0.7, 0.6]], "sharpness": 3.0, "target": [0.1, 0.2],
                 "x_tol": 0.01, "f_tol": 1e-3, "max_iter": 30, "initial_step": 0.5},
}

DEL = object()


def mutate(base, path, value):
    cfg = copy.deepcopy(base)
    node = cfg
    for k in path[:-1]:
        node = node[k]
    if value is DEL:
        del node[path[-1]]
    else:
        node[path[-1]] = value
    return cfg


CASES = [
    # root
    ("ad", ("zz_unknown",), 1), ("ad", ("aa_unknown",), 1), ("ad", ("problem",), "pde"), ("ad", ("problem",), 3),
    ("ad", ("problem",), DEL), ("ad", ("particles",), 1.5), ("ad", ("particles",), True), ("ad", ("dt",), "x"),
    ("ad", ("seed",), -4), ("ad", ("seed",), 2.0), ("ad", ("seed",), 18446744073709551615), ("ad", ("workers",), "8"),
    ("ad", ("scheme",), "rk4"), ("ad", ("scheme",), 1), ("ad", ("scheme",), "milstein"), ("ad", ("max_steps",), 1e3),
    ("ad", ("particles",), 1), ("ad", ("dt",), -1.0),
    # velocity
    ("ad", ("velocity", "kind"), "spectral"), ("ad", ("velocity", "kind"), DEL), ("ad", ("velocity", "extra"), 0),
    ("ad", ("velocity", "max_wavenumber"), DEL), ("ad", ("velocity", "max_wavenumber"), 1.5),
    ("ad", ("velocity", "max_wavenumber"), 0), ("ad", ("velocity", "max_wavenumber"), 1),
    ("ad", ("velocity", "modes"), {}), ("ad", ("velocity", "modes"), [[1, 0, 0.1]]),
    ("ad", ("velocity", "modes"), [[1.0, 0, 0.1, 0.2]]), ("ad", ("velocity", "modes"), [[0, 0, 0.1, 0.2]]),
    ("ad", ("velocity", "modes"), [[1, 0, 0.1, 0.2], [-1, 0, 0.3, 0.0]]),
    ("ad", ("velocity", "modes"), [[-1, 1, 0.1, 0.2]]), ("ad", ("velocity", "modes"), [[1, 0, "a", 0.2]]),
    ("ad", ("velocity",), {"kind": "constant"}), ("ad", ("velocity",), {"kind": "constant", "value": [1, 2, 3]}),
    ("ad", ("velocity",), {"kind": "constant", "value": [1, "b"]}), ("ad", ("velocity",), [1, 2]),
    # diffusion
    ("ad", ("diffusion",), {"kappa": -0.1}), ("ad", ("diffusion",), {"sigma": 1}), ("ad", ("diffusion",), 0.1),
    ("ad", ("diffusion",), {}),
    # scalar fields
    ("ad", ("initial_condition", "kind"), "gauss"), ("ad", ("initial_condition", "kind"), 7),
    ("ad", ("initial_condition", "terms"), {}), ("ad", ("initial_condition", "terms"), [{"amplitude": 1}]),
    ("ad", ("initial_condition", "terms"), [{"k": [1, 0], "freq": [1, 0]}]),
    ("ad", ("initial_condition", "terms"), [{"k": [1, 0], "wave": 2}]),
    ("ad", ("initial_condition", "terms"), [{"k": [1, 0], "amplitude": "x"}]),
    ("ad", ("initial_condition", "terms"), [3]), ("ad", ("initial_condition",), {"kind": "constant"}),
    ("ad", ("initial_condition",), {"kind": "constant", "value": 2.5}),
    ("ad", ("initial_condition",), {"kind": "linear", "offset": 1}),
    ("ad", ("initial_condition",), {"kind": "linear", "gradient": [1, 2]}),
    ("ad", ("initial_condition",), {"kind": "linear", "gradient": [1, 2], "offset": "z"}),
    ("ad", ("initial_condition",), {"kind": "linear", "gradient": [1], "offset": "z"}),
    ("bvp", ("forcing", "sharpness"), -1.0), ("bvp", ("forcing", "amplitudes"), DEL),
    ("bvp", ("forcing", "amplitudes"), [1.0]), ("bvp", ("forcing", "centers"), 5),
    ("bvp", ("forcing", "centers"), [[0.1, 0.2], [0.3]]), ("bvp", ("forcing", "amplitudes"), "a"),
    # observations
    ("ad", ("observations",), {}), ("ad", ("observations",), [{"t": 0.1}]), ("ad", ("observations",), [[0.1]]),
    ("ad", ("observations",), [{"t": 0.1, "x": [0.5, 0.5], "w": 1}]), ("ad", ("observations",), [{"t": "a", "x": "b"}]),
    ("ad", ("observations",), [{"t": 0.0, "x": [0.5, 0.5]}]), ("ad", ("observations",), [{"t": 0.1, "x": [1.5, 0.5]}]),
    ("ad", ("observations",), []), ("bvp", ("observations",), [{"x": [0.5, 0.5], "t": 1}]),
    ("bvp", ("observations",), [{"y": [0.5, 0.5]}]), ("bvp", ("observations",), [{"x": [0.0, 0.5]}]),
    ("bvp", ("observations",), [{"x": [2.0, 0.5]}]),
    # domain
    ("bvp", ("domain",), {"kind": "torus"}), ("bvp", ("domain",), {"kind": "torus", "r": 1}),
    ("bvp", ("domain",), {"kind": "box", "lower": [0, 0]}), ("bvp", ("domain",), {"kind": "box", "lower": [1, 1],
                                                                                    "upper": [0, 0]}),
    ("bvp", ("domain",), {"kind": "box", "lower": [0], "upper": "u"}),
    ("bvp", ("domain",), {"kind": "disk", "center": [0.5, 0.5], "radius": 0.0}),
    ("bvp", ("domain",), {"kind": "disk", "center": [0.5], "radius": "r"}),
    ("bvp", ("domain",), {"kind": "disk", "center": [0.5, 0.5], "radius": 0.5}),
    ("bvp", ("domain",), {"kind": "annulus"}), ("bvp", ("domain",), {"kind": 1}),
    ("bvp", ("max_steps",), 0), ("bvp", ("dt",), -0.1), ("bvp", ("particles",), 1),
    # sections
    ("ad", ("prior",), {"cutoff": 0}), ("ad", ("prior",), {"s0": -1.0}), ("ad", ("prior",), {"cut": 2}),
    ("ad", ("prior",), {"cutoff": 2.0}), ("ad", ("prior",), DEL), ("ad", ("likelihood",), DEL),
    ("ad", ("likelihood", "data"), DEL), ("ad", ("likelihood", "data"), [1.0]),
    ("ad", ("likelihood", "data"), [0.0, 0.0]), ("ad", ("likelihood", "noise_std"), DEL),
    ("ad", ("likelihood", "noise_std"), -3.0), ("ad", ("likelihood", "forward_seed"), -1),
    ("ad", ("likelihood", "extra"), 1), ("ad", ("mcmc", "beta"), 0.0), ("ad", ("mcmc", "beta"), 1.5),
    ("ad", ("mcmc", "thin"), 0.5), ("ad", ("mcmc", "steps"), "n"), ("ad", ("mcmc", "x"), 1),
    ("bvp", ("optimize",), DEL), ("bvp", ("optimize", "centers"), DEL), ("bvp", ("optimize", "centers"), []),
    ("bvp", ("optimize", "target"), [0.1]), ("bvp", ("optimize", "initial"), [1.0]),
    ("bvp", ("optimize", "initial"), []), ("bvp", ("optimize", "sharpness"), 0.0),
    ("bvp", ("optimize", "max_iter"), 2.5), ("bvp", ("optimize", "x_tol"), "t"), ("bvp", ("optimize", "zz"), 1),
    ("ad", ("reference",), {"galerkin_cutoff": 8, "dt_ref": 1e-4}), ("ad", ("reference",), {"fd": 1}),
    ("ad", ("reference",), {"field_grid": 1.5}),
    ("ad", ("benchmark",), {"cutoffs": [4, 8], "run_reference": False, "t_final": 0.1}),
    ("ad", ("benchmark",), {"cutoffs": 8}), ("ad", ("benchmark",), {"cutoffs": [4.5]}),
    ("ad", ("benchmark",), {"run_reference": 1}), ("ad", ("benchmark",), {"speed": 1}),
    ("ad", ("benchmark",), []),
]

OUR_KIND = {K.ConfigError: "ConfigError", ValueError: "invalid_argument", IndexError: "out_of_range",
            RuntimeError: "exception"}


def ours(text, origin, stage):
    try:
        cfg = K.parse_config(text, origin)
        if stage == 1:
            K.make_ad_spec(cfg)
        elif stage == 2:
            K.make_bvp_spec(cfg)
        elif stage == 3:
            K.make_likelihood(cfg)
        elif stage == 4:
            K.make_forcing_control(cfg)
    except Exception as e:  # noqa: BLE001
        for cls, name in OUR_KIND.items():
            if isinstance(e, cls):
                return name, str(e)
        raise
    return None, ""


@pytest.fixture(scope="module")
def refcli():
    from oracle.oracle import ReferenceCli, reference_available
    if not reference_available():
        pytest.skip("oracle/_ref not built")
    try:
        return ReferenceCli()
    except RuntimeError as e:
        pytest.skip(str(e))


@pytest.mark.parametrize("case", range(len(CASES)))
def test_config_diagnostics_match_reference(refcli, case):
    which, path, value = CASES[case]
    base = AD if which == "ad" else BVP
    text = json.dumps(mutate(base, path, value))
    stages = (0, 1, 3) if which == "ad" else (0, 2, 4)
    for stage in stages:
        want = refcli.config_check(text, "cfg.json", stage)
        got = ours(text, "cfg.json", stage)
        assert got == want, (stage, text)


def test_shipped_style_configs_accepted(refcli):
    for base, stages in ((AD, (1, 3)), (BVP, (2, 4))):
        for stage in stages:
            assert refcli.config_check(json.dumps(base), "c", stage) == (None, "")
            assert ours(json.dumps(base), "c", stage) == (None, "")


def test_parse_error_location(refcli):
    bad = '{\n  "problem": "ad",\n  "particles": 12,,\n}'
    kind, msg = refcli.config_check(bad, "f.json", 0)
    assert kind == "ConfigError" and msg.startswith("f.json:")
    with pytest.raises(K.ConfigError) as e:
        K.parse_config(bad, "f.json")
    assert str(e.value).startswith("f.json:3:")  # line/column of the fault; parser text differs
    assert ours("[1, 2]", "o", 0) == refcli.config_check("[1, 2]", "o", 0)


def test_load_config_missing_file(refcli, tmp_path):
    p = str(tmp_path / "missing.json")
    with pytest.raises(K.ConfigError, match="cannot open config file"):
        K.load_config(p)


def test_format_double_matches_reference(refcli):
    import numpy as np
    rng = np.random.default_rng(3)
    vals = list(rng.normal(size=300) * 10.0 ** rng.integers(-30, 30, size=300)) + [
        0.0, -0.0, 1.0, 0.1, 1 / 3, 2 ** 60, 1e-320, 5e-324, 1.7976931348623157e308, math.inf, -math.inf,
        123456789012345678.0, 0.5, 100.0, 1e21, 1e-5]
    for v in vals:
        assert format_double(v) == refcli.format_double(v), v
    assert format_double(math.nan) == "nan"


def test_record_writer_formats():
    import io
    buf = io.StringIO()
    w = RecordWriter(buf, "csv", ["a", "b"])
    w.write_row([1.0, 0.1])
    buf2 = io.StringIO()
    RecordWriter(buf2, "jsonl", ["a", "b"]).write_row([2.0, -0.5])
    assert buf.getvalue() == "a,b\n1,0.1\n"
    assert buf2.getvalue() == '{"a":2,"b":-0.5}\n'
    with pytest.raises(ValueError, match="column count mismatch"):
        w.write_row([1.0])


def _cli(*args):
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    return subprocess.run([sys.executable, "-m", "paper_1808_10580_b200.cli", *map(str, args)], cwd=root,
                          capture_output=True, text=True, timeout=300)


def test_cli_config_error_exit_code(refcli, tmp_path):
    """cli.cpp:296-302: ConfigError -> "config error: ..." and exit 2, before
    any device work (so this runs on CPU)."""
    bad = mutate(AD, ("velocity", "max_wavenumber"), 1.5)
    p = tmp_path / "bad.json"
    p.write_text(json.dumps(bad))
    r = _cli("forward-ad", "--config", p, "--out", tmp_path / "o.csv")
    _, want = refcli.config_check(json.dumps(bad), str(p), 1)
    assert r.returncode == 2 and r.stderr.strip() == f"config error: {want}"
    r = _cli("forward-bvp", "--config", p, "--out", tmp_path / "o.csv")  # an "ad" file given to forward-bvp
    assert r.returncode == 2 and "config error:" in r.stderr
    r = _cli("forward-ad", "--config", tmp_path / "missing.json", "--out", tmp_path / "o.csv")
    assert r.returncode == 2 and r.stderr.strip() == f"config error: {tmp_path / 'missing.json'}: cannot open config file"
    good = tmp_path / "bvp.json"
    good.write_text(json.dumps(mutate(BVP, ("forcing", "sharpness"), -2.0)))
    r = _cli("forward-bvp", "--config", good, "--out", tmp_path / "o.csv")
    assert r.returncode == 1 and r.stderr.strip() == "error: ScalarField: sharpness must be positive"


def test_cli_usage_errors(tmp_path):
    assert _cli().returncode == 2
    assert _cli("forward-ad", "--config", "x.json").returncode == 2  # --out required
    assert _cli("forward-ad", "--config", "x", "--out", "y", "--format", "xml").returncode == 2
    r = _cli("benchmark", "--config", "x", "--out", "y")
    assert r.returncode == 1 and "not part of the B200 forward-map path" in r.stderr
    p = tmp_path / "bvp.json"
    p.write_text(json.dumps(BVP))
    r = _cli("reference", "--config", p, "--out", tmp_path / "g.csv", "--method", "fd")
    assert r.returncode == 1 and "finite-difference" in r.stderr
