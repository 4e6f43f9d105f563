"""The command-line front end (paper_1808_10580_b200.cli) against the REAL
reference CLI's outputs for the same configuration files
(tests/golden/cli/, written by tests/golden/make_cli_golden.py from
oracle/ref_cli.cpp over the compiled reference).

Headers, row counts, observation coordinates, counts and the stdout layout
must match exactly; estimates within the FP64 forward-map gate (the GPU sums
in a different order), chain states / Nelder-Mead points within the
tolerances of tests/test_gpu_pcn.py and tests/test_gpu_forcing.py.
"""
import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLD = ROOT / "tests" / "golden" / "cli"

pytestmark = pytest.mark.gpu


def cli(*args, cwd=None):
    return subprocess.run([sys.executable, "-m", "paper_1808_10580_b200.cli", *map(str, args)], cwd=cwd or ROOT,
                          capture_output=True, text=True, timeout=600)


def read_csv(path):
    lines = Path(path).read_text().splitlines()
    return lines[0].split(","), [l.split(",") for l in lines[1:]]


def read_jsonl(path):
    rows = [json.loads(l) for l in Path(path).read_text().splitlines()]
    return list(rows[0].keys()), [[str(r[k]) for k in r] for r in rows], rows


def close(a, b, rel=1e-10, floor=1.0):
    a, b = float(a), float(b)
    return abs(a - b) <= rel * max(abs(b), floor)


def check_forward(got_rows, want_rows, cols):
    assert len(got_rows) == len(want_rows)
    for g, w in zip(got_rows, want_rows):
        for c, gv, wv in zip(cols, g, w):
            if c in ("mean",):
                assert close(gv, wv, 1e-10), (c, gv, wv)
            elif c in ("std_error", "mean_exit_time"):
                assert close(gv, wv, 1e-8, 0.0), (c, gv, wv)
            else:  # coordinates, times, counts: the same text
                assert gv == wv, (c, gv, wv)


def test_forward_ad_csv(tmp_path):
    r = cli("forward-ad", "--config", GOLD / "ad.json", "--out", tmp_path / "o" / "ad.csv")
    assert r.returncode == 0, r.stderr
    gh, gr = read_csv(tmp_path / "o" / "ad.csv")
    wh, wr = read_csv(GOLD / "ad.csv")
    assert gh == wh
    check_forward(gr, wr, wh)


def test_forward_ad_jsonl_seed_override(tmp_path):
    r = cli("forward-ad", "--config", GOLD / "ad.json", "--out", tmp_path / "ad.jsonl", "--format", "jsonl",
            "--seed", 5)
    assert r.returncode == 0, r.stderr
    gk, _, grows = read_jsonl(tmp_path / "ad.jsonl")
    wk, _, wrows = read_jsonl(GOLD / "ad_seed5.jsonl")
    assert gk == wk and len(grows) == len(wrows)
    for g, w in zip(grows, wrows):
        assert g["t"] == w["t"] and g["x1"] == w["x1"] and g["n_particles"] == w["n_particles"]
        assert close(g["mean"], w["mean"]) and close(g["std_error"], w["std_error"], 1e-8, 0.0)


def test_forward_bvp_csv(tmp_path):
    r = cli("forward-bvp", "--config", GOLD / "bvp.json", "--out", tmp_path / "bvp.csv")
    assert r.returncode == 0, r.stderr
    gh, gr = read_csv(tmp_path / "bvp.csv")
    wh, wr = read_csv(GOLD / "bvp.csv")
    assert gh == wh
    check_forward(gr, wr, wh)


def test_sample(tmp_path):
    out = tmp_path / "chain"
    r = cli("sample", "--config", GOLD / "sample.json", "--out", out)
    assert r.returncode == 0, r.stderr
    want = (GOLD / "sample.stdout").read_text().splitlines()
    got = r.stdout.splitlines()
    assert got[0] == want[0] and got[2] == want[2]  # acceptance_rate, samples: exact
    assert close(got[1].split()[1], want[1].split()[1], 1e-8)
    gh, gr = read_csv(out / "archive.csv")
    wh, wr = read_csv(GOLD / "sample_out" / "archive.csv")
    assert gh == wh and len(gr) == len(wr)
    for g, w in zip(gr, wr):
        assert g[0] == w[0]
        assert close(g[1], w[1], 1e-8)
        assert np.allclose(np.array(g[2:], float), np.array(w[2:], float), rtol=0, atol=1e-12)
    gh, gr = read_csv(out / "map.csv")
    wh, wr = read_csv(GOLD / "sample_out" / "map.csv")
    assert gh == wh and np.allclose(np.array(gr[0], float), np.array(wr[0], float), rtol=0, atol=1e-12)
    gh, gr = read_csv(out / "summary.csv")
    wh, wr = read_csv(GOLD / "sample_out" / "summary.csv")
    assert gh == wh
    for c, g, w in zip(wh, gr[0], wr[0]):
        if c in ("map_objective", "final_phi"):
            assert close(g, w, 1e-8), c
        else:
            assert g == w, c


def test_optimize(tmp_path):
    r = cli("optimize", "--config", GOLD / "optimize.json", "--out", tmp_path / "opt.csv")
    assert r.returncode == 0, r.stderr
    want = (GOLD / "optimize.stdout").read_text().splitlines()
    got = r.stdout.splitlines()
    assert got[1] == want[1]  # iterations N (reason)
    assert close(got[0].split()[1], want[0].split()[1], 1e-8, 1e-6)
    assert np.allclose(np.array(got[2].split()[1:], float), np.array(want[2].split()[1:], float), rtol=1e-8,
                       atol=1e-10)
    gh, gr = read_csv(tmp_path / "opt.csv")
    wh, wr = read_csv(GOLD / "optimize.csv")
    assert gh == wh and len(gr) == len(wr)
    for g, w in zip(gr, wr):
        assert g[0] == w[0]
        assert close(g[1], w[1], 1e-8, 1e-6)
        assert np.allclose(np.array(g[2:], float), np.array(w[2:], float), rtol=1e-8, atol=1e-10)


def test_reference_galerkin(tmp_path):
    """`reference --method galerkin` (cli.cpp:98-122): grid file + observation
    rows on stdout, against the numpy restatement of galerkin.cpp."""
    from oracle import galerkin_oracle as G
    from paper_1808_10580_b200.config import load_config, make_ad_spec
    from paper_1808_10580_b200.records import format_double
    cfg_path = tmp_path / "gal.json"
    cfg = json.loads((GOLD / "ad.json").read_text())
    cfg["reference"] = {"galerkin_cutoff": 5, "dt_ref": 2.5e-4, "field_grid": 9}
    cfg_path.write_text(json.dumps(cfg))
    r = cli("reference", "--config", cfg_path, "--out", tmp_path / "grid.csv", "--method", "galerkin")
    assert r.returncode == 0, r.stderr
    spec = make_ad_spec(load_config(str(cfg_path)))
    vals, theta, steps, modes = G.solve(spec, "box", 5, 2.5e-4)
    gh, gr = read_csv(tmp_path / "grid.csv")
    assert gh == ["x1", "x2", "value"] and len(gr) == 81
    want = G.field_grid(theta, modes, 9)
    for q, row in enumerate(gr):
        assert row[0] == format_double((q // 9) / 9) and row[1] == format_double((q % 9) / 9)
        assert abs(float(row[2]) - want[q]) < 1e-10
    lines = r.stdout.splitlines()
    assert lines[0] == "obs,x1,x2,value" and len(lines) == 1 + len(vals)
    for j, line in enumerate(lines[1:]):
        f = line.split(",")
        assert f[0] == str(j) and abs(float(f[3]) - vals[j]) < 1e-10 * max(1.0, abs(vals[j]))
