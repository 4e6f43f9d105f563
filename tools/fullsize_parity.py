#!/usr/bin/env python
"""Full-size parity against the real reference (oracle/_ref, the reference
compiled from its own sources) on the GPU box's host cores.

    python tools/fullsize_parity.py [--out gpurun_out/r02_fullsize_parity.json] [--configs c2,c3,c4,c5]

  c2  all 9 observations at 1e5 particles: GPU observe_ad vs the reference's
      observe_ad (velocity from u, observe_ad_u) with workers = all cores
  c3  all 25 observations at 1e6 walkers: GPU observe_bvp vs the reference's
      observe_bvp; plus, for a 1e5-walker slice of several observations, the
      per-walker exit times compared walker by walker to count exit-step flips
      (a walker whose last step lands on the other side of the boundary in one
      implementation: SURVEY.md §8(c) "FP semantics", sde.cpp:63-74)
  c4  the first proposals of the 4096-proposal batch (rows of one batched
      launch) vs the reference's observe_ad_u per proposal
  c5  the shortest-time observations of the K=80 evaluation

Writes one JSON report (max |delta mean| / max(|ref|, 1), max relative SE
difference, flip counts, timings).  tests/test_gpu_fullsize_reference.py
asserts on it.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]


def compare(got, want) -> dict:
    dm = [abs(g.mean - float(w["mean"])) / max(abs(float(w["mean"])), 1.0) for g, w in zip(got, want)]
    ds = [abs(g.std_error - float(w["std_error"])) / float(w["std_error"]) for g, w in zip(got, want)]
    nf = [int(g.n_failed) == int(w["n_failed"]) for g, w in zip(got, want)]
    da = [abs(g.aux_mean - float(w["aux_mean"])) / max(abs(float(w["aux_mean"])), 1e-300) for g, w in zip(got, want)]
    return {"n_obs": len(dm), "max_rel_mean": max(dm), "max_rel_se": max(ds), "n_failed_equal": all(nf),
            "max_rel_aux": max(da), "means_gpu": [g.mean for g in got], "means_ref": [float(w["mean"]) for w in want]}


def run(configs="c2,c3,c4,c5", slice_walkers=100_000, slice_obs="0,6,12,18,24") -> dict:
    """Run the GPU path and the compiled reference on the full-size configs; return the report."""
    import paper_1808_10580_b200 as S
    import specs
    from oracle.oracle import Reference
    import bench
    R = Reference()
    cores = os.cpu_count() or 1
    ctx = S.Context(0)
    report: dict = {"cores": cores}
    cfgs = configs.split(",")
    if "c2" in cfgs:
        u = S.prior_draw(specs.C2_PRIOR, 808, 0xBE9C4, 0, ctx)
        spec = specs.c2_spec(u, n_particles=100_000)
        got = S.observe_ad(spec, 808, ctx=ctx)
        base = specs.c2_spec(u, n_particles=100_000)
        t0 = time.perf_counter()
        want = R.observe_ad(base, 808, cores)
        report["c2"] = dict(compare(got, want), ref_seconds=time.perf_counter() - t0)
    if "c3" in cfgs:
        spec = specs.c3_spec(n_particles=1_000_000)
        got = S.observe_bvp(spec, 606, ctx=ctx)
        t0 = time.perf_counter()
        want = R.observe_bvp(spec, 606, cores)
        rep = dict(compare(got, want), ref_seconds=time.perf_counter() - t0)
        dt = spec.resolved_dt()
        flips = {}
        total = 0
        worst_value = 0.0
        for j in [int(x) for x in slice_obs.split(",")]:
            gv, ga, gf = S.bvp_particle_values(spec, j, 606, slice_walkers, ctx)
            rv, ra, rf, rsteps = R.bvp_particle_values(spec, j, 606, slice_walkers)
            # an exit-step flip moves tau by about one dt; same-step walkers differ by rounding only
            flip = np.abs(ga - ra) > 0.5 * dt
            fail_diff = int(np.sum(gf != rf))
            same = ~flip & (gf == rf) & (gf == 0)
            worst_value = max(worst_value, float(np.max(np.abs(gv[same] - rv[same]))) if same.any() else 0.0)
            flips[j] = {"walkers": slice_walkers, "exit_step_flips": int(flip.sum()), "failed_flag_diffs": fail_diff,
                        "max_abs_value_diff_flipped": float(np.max(np.abs(gv[flip] - rv[flip]))) if flip.any() else 0.0}
            total += int(flip.sum())
        rep["flip_slices"] = flips
        rep["flips_per_walker"] = total / (slice_walkers * len(flips))
        rep["flips_per_evaluation_estimate"] = rep["flips_per_walker"] * 25 * 1_000_000
        rep["max_abs_value_diff_same_exit_step"] = worst_value
        report["c3"] = rep
    if "c4" in cfgs:
        prior = specs.C4_PRIOR
        u0 = S.prior_draw(prior, 808, 0xBE9C4, 1, ctx)
        B = 4096
        U = np.stack([math.sqrt(1 - 0.02 ** 2) * u0 + 0.02 * S.prior_draw(prior, 4242, 0xFFFFFFFF, b, ctx)
                      for b in range(B)])
        base = specs.c4_base(n_particles=1024)
        est = S.observe_ad_batched(base, prior, U, 808, ctx=ctx)
        rows = []
        t0 = time.perf_counter()
        for b in range(4):
            want = R.observe_ad_u(base, prior, U[b], 808, cores)
            got = [S.ParticleEstimate(*[e[k] for k in ("mean", "std_error", "n_particles", "n_failed", "aux_mean")])
                   for e in est[b]]
            rows.append(compare(got, want))
        report["c4"] = {"proposals_checked": 4, "max_rel_mean": max(r["max_rel_mean"] for r in rows),
                        "max_rel_se": max(r["max_rel_se"] for r in rows), "ref_seconds": time.perf_counter() - t0}
    if "c5" in cfgs:
        u = S.prior_draw(S.PriorSpec(80, 1.0, 2.5), 808, 0xBE9C4, 2, ctx)
        spec = bench.c5_spec(S, u)
        js = [0, 8]  # t = 1/16 at (0,0) and (1/8,1/8)
        got_all = S.observe_ad(spec, 808, ctx=ctx)
        got = [got_all[j] for j in js]
        t0 = time.perf_counter()
        want = [R.observe_ad_single(spec, j, 808, cores) for j in js]
        report["c5"] = dict(compare(got, want), observations=js, ref_seconds=time.perf_counter() - t0)
    return report


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "r02_fullsize_parity.json"))
    ap.add_argument("--configs", default="c2,c3,c4,c5")
    ap.add_argument("--slice", type=int, default=100_000, help="walkers per observation in the C3 flip count")
    ap.add_argument("--slice-obs", default="0,6,12,18,24")
    args = ap.parse_args()
    report = run(args.configs, args.slice, args.slice_obs)
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(report, indent=1) + "\n")
    print(json.dumps({k: ({kk: vv for kk, vv in v.items() if not kk.startswith("means")} if isinstance(v, dict) else v)
                      for k, v in report.items()}, indent=1))


if __name__ == "__main__":
    main()
