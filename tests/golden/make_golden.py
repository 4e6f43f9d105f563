"""Generate tests/golden/golden.json from the REAL reference.

Runs the reference scalarmc library compiled from /root/reference/proj/src
(oracle/Makefile -> oracle/_ref/libscalarmc_ref.so) on the configurations in
tests/specs.py and records its outputs bit-exactly (doubles as float.hex).
The fixtures pin the oracle restatement (CPU tests) and the CUDA path (GPU
tests) without /root/reference being present at test time.

    make -C oracle && python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import math
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import paper_1808_10580_b200 as S  # noqa: E402
import specs  # noqa: E402
from oracle.oracle import Reference  # noqa: E402

OUT = Path(__file__).resolve().parent / "golden.json"


def hx(a) -> list | str:
    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 0:
        return float(a).hex()
    return [hx(x) for x in a]


def est(e) -> dict:
    return {k: (float(e[k]).hex() if e.dtype[k].kind == "f" else int(e[k])) for k in e.dtype.names}


def main() -> None:
    R = Reference()
    rng = np.random.default_rng(20241018)
    g: dict = {"generator": "tests/golden/make_golden.py", "reference": "/root/reference/proj (compiled in place)"}

    # Philox4x32-10 known answers (Random123 KAT) + random inputs.
    ctr = [[0, 0, 0, 0], [0xFFFFFFFF] * 4, [0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344]]
    key = [[0, 0], [0xFFFFFFFF] * 2, [0xA4093822, 0x299F31D0]]
    ctr += rng.integers(0, 2**32, size=(13, 4), dtype=np.uint64).tolist()
    key += rng.integers(0, 2**32, size=(13, 2), dtype=np.uint64).tolist()
    g["philox"] = {"ctr": ctr, "key": key, "out": R.philox(ctr, key).tolist()}

    # Normal pairs and mixed cached draws for assorted keys.
    keys = [(0, 0, 0), (7, 0, 0), (7, 2, 9999), (2**64 - 1, 2**32 - 1, 2**32 - 1), (808, 0xBE9C4, 0), (123, 4, 56)]
    g["normal_pairs"] = [{"key": list(k), "pairs": hx(R.normal_pairs(*k, 64))} for k in keys]
    ops = rng.integers(0, 3, size=200).tolist()
    g["stream_draws"] = {"key": [31337, 0xFFFFFFFF, 0], "ops": ops, "out": hx(R.stream_draws(31337, 0xFFFFFFFF, 0, ops))}

    # pairwise_sum on edge sizes.
    sums = []
    for n in (0, 1, 2, 3, 5, 7, 64, 1000, 1023, 1024, 1025, 4097):
        v = rng.normal(size=n)
        sums.append({"values": hx(v), "sum": float(R.pairwise_sum(v)).hex()})
    g["pairwise_sum"] = sums

    # Velocity field evaluations (random fields, test_fields.cpp:24-41 style).
    vel = []
    for n_modes, kmax in ((1, 1), (8, 4), (12, 5), (40, 8)):
        f = specs.random_fourier(rng, n_modes, kmax)
        x = rng.random((32, 2))
        vel.append({"k": f.k.tolist(), "coeff": hx(f.coeff), "K": kmax, "x": hx(x),
                    "v": hx(R.velocity_eval(S.VelocityField.fourier(f), x))})
    g["velocity"] = vel

    # C1: the shipped forward_ad_two_mode.json (seed 7, N_p 1e4) — SURVEY §8c.
    c1 = specs.c1_two_mode()
    g["c1"] = {"seed": 7, "n_particles": 10000, "estimates": [est(e) for e in R.observe_ad(c1, 7, 0)],
               "particles": [hx(R.ad_particle_values(c1, j, 7, 256)) for j in range(3)],
               "resolved_dt": R.resolved_dt_ad(c1).hex()}

    # Heat equation (acceptance.cpp:34-48 at N_p 2e4) and zero diffusion (test_forward.cpp:34-47).
    heat = specs.heat_spec(0.01, 0.5, (0.0, 0.0), 20000, 1e-3)
    g["heat"] = {"seed": 20240501, "estimates": [est(e) for e in R.observe_ad(heat, 20240501, 0)]}

    # C2 at reduced N_p: the survey's benchmark recipe for u (benchmark.cpp:69-71).
    u2 = R.prior_draw(specs.C2_PRIOR, 808, 0xBE9C4, 0)
    c2 = specs.c2_spec(u2, n_particles=512)
    g["c2"] = {"u": hx(u2), "seed": 808, "n_particles": 512,
               "estimates": [est(e) for e in R.observe_ad(c2, 808, 0)],
               "particles": [hx(R.ad_particle_values(c2, j, 808, 128)) for j in (0, 4, 8)]}

    # C4-like batch: K=25 prior, pCN proposals u_b = sqrt(1-b^2) u0 + b xi_b.
    u0 = R.prior_draw(specs.C4_PRIOR, 808, 0xBE9C4, 1)
    beta = 0.02
    U = np.stack([math.sqrt(1 - beta * beta) * u0 + beta * R.prior_draw(specs.C4_PRIOR, 4242, 0xFFFFFFFF, b)
                  for b in range(4)])
    c4 = specs.c4_base(n_particles=64)
    g["c4"] = {"U": hx(U), "seed": 808, "n_particles": 64,
               "estimates": [[est(e) for e in R.observe_ad_u(c4, specs.C4_PRIOR, U[b], 808, 0)] for b in range(4)]}

    # misfit through the unchanged reference LikelihoodSpec (sample_k2.json shape).
    pk2 = S.PriorSpec(2, 0.6, 2.5)
    uk2 = R.prior_draw(pk2, 31337, 0xFFFFFFFF, 0)
    like = specs.c4_base(n_particles=160)
    like.dt = 0.006
    data = [-0.9065, -0.7528, -0.6665, -0.8091, -0.6508, -0.5135, -0.5185, -0.4553, -0.4066]
    g["misfit"] = {"u": hx(uk2), "data": data, "noise_std": 0.05, "forward_seed": 1234,
                   "phi": float(R.misfit(like, pk2, uk2, data, 0.05, 1234, 0)).hex()}

    # run_chain (pCN, inference.cpp:170-194) on the sample_k2.json shape for
    # three chain seeds, prior-drawn starts (the reference's own chain stream).
    likespec = S.LikelihoodSpec(data=data, noise_std=0.05, forward=like, forward_seed=1234)
    chains = []
    for cseed in (31337, 7, 99):
        r = R.run_chain(likespec, pk2, 40, 0.22, 5, 3, cseed)
        chains.append({"seed": cseed, "phi_trace": hx(r["phi_trace"]), "samples": hx(r["samples"]),
                       "final_u": hx(r["final_u"]), "map_u": hx(r["map_u"]), "final_phi": float(r["final_phi"]).hex(),
                       "map_objective": float(r["map_objective"]).hex(), "accepted": r["accepted"]})
    g["pcn"] = {"n_steps": 40, "beta": 0.22, "burn_in": 5, "thin": 3, "chains": chains}

    # Paper BVP (forward_bvp_box.json, seed 606, N_p 16000) — SURVEY §8c.
    bvp = specs.paper_bvp()
    vals, aux, failed, steps = R.bvp_particle_values(bvp, 0, 606, 256)
    g["bvp_box"] = {"seed": 606, "n_particles": 16000, "estimates": [est(e) for e in R.observe_bvp(bvp, 606, 0)],
                    "particles": {"values": hx(vals), "aux": hx(aux), "failed": failed.tolist(),
                                  "steps": steps.tolist()},
                    "resolved_dt": R.resolved_dt_bvp(bvp).hex()}

    # C3 shape at reduced N_p (F = (1, -0.5, 2), 25 observations).
    c3 = specs.c3_spec(n_particles=512)
    g["c3"] = {"seed": 606, "n_particles": 512, "estimates": [est(e) for e in R.observe_bvp(c3, 606, 0)]}

    # Disk domain with a Fourier velocity (C3b-like) and max_steps failures.
    disk = specs.paper_bvp(n_particles=1000, amplitudes=(1.0, -0.5, 2.0), observations=[(0.5, 0.5), (0.3, 0.6)],
                           velocity=S.VelocityField.fourier(specs.random_fourier(np.random.default_rng(5), 6, 3)))
    disk.domain = S.Domain.disk((0.5, 0.5), 0.5)
    disk.dt = 5e-4
    g["bvp_disk"] = {"seed": 5, "estimates": [est(e) for e in R.observe_bvp(disk, 5, 0)]}
    fail = specs.paper_bvp(n_particles=300, observations=[(0.94, 0.94), (0.8, 0.5)])
    fail.max_steps = 300
    g["bvp_maxsteps"] = {"seed": 77, "estimates": [est(e) for e in R.observe_bvp(fail, 77, 0)]}

    # forcing_cost through the unchanged reference optimize.cpp.
    fc = specs.paper_bvp(n_particles=400)
    g["forcing_cost"] = [{"F": F, "target": [0.0, 0.0, 0.0], "seed": 606,
                          "cost": float(R.forcing_cost(fc, F, [(0.68, 0.4), (0.4, 0.68), (0.82, 0.82)], 4.0,
                                                       [0.0, 0.0, 0.0], 606, 0)).hex()}
                         for F in ([0.0, 0.0, 0.0], [1.0, -0.5, 2.0])]

    # optimize_forcing (Nelder-Mead over observe_bvp, optimize.cpp:175-185) on
    # forward_bvp_box.json's "optimize" section at 300 walkers/obs.
    ob = specs.paper_bvp(n_particles=300)
    ctrs = [(0.68, 0.4), (0.4, 0.68), (0.82, 0.82)]
    for tgt in ([0.0, 0.0, 0.0], [0.2, 0.1, -0.05]):
        r = R.optimize_forcing(ob, [0.0, 0.0, 0.0], ctrs, 4.0, tgt, 0.005, 1e-4, 250, 1.0, 606)
        g.setdefault("optimize", []).append({"target": tgt, "argmin": hx(r["argmin"]),
                                             "min_value": float(r["min_value"]).hex(),
                                             "iterations": r["iterations"], "stop_reason": r["stop_reason"]})

    # Prior mode order (inference.cpp:24-40) and a prior draw.
    g["prior"] = {"modes8": R.prior_modes(8).tolist(), "draw8": hx(u2)}

    OUT.write_text(json.dumps(g, indent=0))
    print(f"wrote {OUT} ({OUT.stat().st_size / 1024:.0f} KiB)")


if __name__ == "__main__":
    main()
