"""Generate tests/golden/cli/ from the REAL reference's CLI command bodies.

Writes four run configurations (this repo's own, exercising every command on
the B200 path: forward-ad, forward-bvp, sample, optimize) and the files and
stdout the reference produces for them (oracle/ref_cli.cpp over the compiled
reference: load_config, make_*_spec, observe_*, run_chain,
optimize_forcing, RecordWriter).  tests/test_gpu_cli.py runs
`python -m paper_1808_10580_b200.cli` on the same configs and compares.

    make -C oracle && python tests/golden/make_cli_golden.py
"""
from __future__ import annotations

import json
import shutil
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.oracle import ReferenceCli  # noqa: E402

OUT = Path(__file__).resolve().parent / "cli"

CONFIGS = {
    "ad": {
        "problem": "ad",
        "velocity": {"kind": "fourier", "max_wavenumber": 3,
                     "modes": [[1, 0, 0.2, -0.1], [0, 1, -0.15, 0.05], [1, -2, 0.05, 0.08], [2, 2, -0.04, 0.02]]},
        "diffusion": {"kappa": 0.02},
        "initial_condition": {"kind": "cosine", "terms": [{"k": [1, 0], "amplitude": 1.0},
                                                          {"k": [1, 1], "amplitude": 0.5, "phase": 0.3},
                                                          {"freq": [0.0, 12.566370614359172], "amplitude": 0.2}]},
        "observations": [{"t": 0.05, "x": [0.2, 0.4]}, {"t": 0.1, "x": [0.6, 0.3]}, {"t": 0.125, "x": [0.0, 0.9]}],
        "particles": 6000, "dt": 0.0025, "seed": 4242, "workers": 0,
    },
    "bvp": {
        "problem": "bvp",
        "velocity": {"kind": "constant", "value": [0.6, -0.3]},
        "diffusion": {"kappa": 0.15},
        "forcing": {"kind": "bumps", "amplitudes": [1.0, -0.5], "centers": [[0.35, 0.4], [0.7, 0.65]],
                    "sharpness": 5.0},
        "boundary": {"kind": "cosine", "terms": [{"freq": [1.5707963267948966, 0.0], "amplitude": 0.5},
                                                 {"freq": [0.0, 3.141592653589793], "amplitude": 0.25}]},
        "domain": {"kind": "box", "lower": [0.0, 0.0], "upper": [1.0, 1.0]},
        "observations": [{"x": [0.5, 0.5]}, {"x": [0.85, 0.2]}],
        "particles": 3000, "dt": 0.0004, "seed": 77, "workers": 0,
    },
    "sample": {
        "problem": "ad",
        "velocity": {"kind": "fourier", "max_wavenumber": 2, "modes": []},
        "diffusion": {"kappa": 0.05},
        "initial_condition": {"kind": "cosine", "terms": [{"k": [1, 0], "amplitude": 1.0},
                                                          {"k": [0, 1], "amplitude": 0.7}]},
        "observations": [{"t": 0.06, "x": [0.25, 0.25]}, {"t": 0.06, "x": [0.75, 0.5]},
                         {"t": 0.12, "x": [0.5, 0.75]}, {"t": 0.12, "x": [0.25, 0.5]}],
        "particles": 128, "dt": 0.006, "seed": 9, "workers": 0,
        "prior": {"cutoff": 2, "s0": 0.6, "alpha": 2.5},
        "likelihood": {"data": [-0.8, -0.6, -0.5, -0.45], "noise_std": 0.05, "forward_seed": 321},
        "mcmc": {"steps": 60, "beta": 0.25, "burn_in": 10, "thin": 5},
    },
    "optimize": {
        "problem": "bvp",
        "velocity": {"kind": "constant", "value": [1.0, 1.0]},
        "diffusion": {"kappa": 0.282},
        "forcing": {"kind": "bumps", "amplitudes": [0.0, 0.0], "centers": [[0.6, 0.45], [0.45, 0.6]],
                    "sharpness": 4.0},
        "boundary": {"kind": "constant", "value": 0.25},
        "domain": {"kind": "box", "lower": [0.0, 0.0], "upper": [1.0, 1.0]},
        "observations": [{"x": [0.85, 0.6]}, {"x": [0.6, 0.85]}],
        "particles": 400, "dt": 0.0005, "seed": 606, "workers": 0,
        "optimize": {"centers": [[0.6, 0.45], [0.45, 0.6]], "sharpness": 4.0, "target": [0.1, 0.05],
                     "x_tol": 0.005, "f_tol": 0.0001, "max_iter": 80, "initial_step": 1.0},
    },
}


def main() -> None:
    R = ReferenceCli()
    if OUT.exists():
        shutil.rmtree(OUT)
    OUT.mkdir(parents=True)
    for name, cfg in CONFIGS.items():
        (OUT / f"{name}.json").write_text(json.dumps(cfg, indent=2) + "\n")
    cfg = lambda n: str(OUT / f"{n}.json")  # noqa: E731
    R.forward(cfg("ad"), str(OUT / "ad.csv"), "csv")
    R.forward(cfg("ad"), str(OUT / "ad_seed5.jsonl"), "jsonl", seed=5)
    R.forward(cfg("bvp"), str(OUT / "bvp.csv"), "csv", bvp=True)
    (OUT / "sample.stdout").write_text(R.sample(cfg("sample"), str(OUT / "sample_out"), "csv"))
    (OUT / "optimize.stdout").write_text(R.optimize(cfg("optimize"), str(OUT / "optimize.csv"), "csv"))
    print("wrote", sorted(p.name for p in OUT.rglob("*") if p.is_file()))


if __name__ == "__main__":
    main()
