"""Per-rank time of a W-GPU sharded evaluation, modelled on ONE B200.

    python tools/shard_model.py [--config c2] [--worlds 1,2,4,8] [--reps 3]

An emulated group of W members on device 0 (SMC_GROUP_EXCHANGE=emulated,
duplicate device list) with SMC_GROUP_SERIAL=1 runs the members' shards one
after another on one stream, so each member's particle-kernel time (CUDA
events around its launches; ctx.stats() reports the max over members) is the
time one rank of a real W-GPU group spends in K1 — the quantity the driver's
strong-scaling run is bound by.  Prints one JSON line per W: the max per-rank
K1 ms, W x that against the one-GPU K1 ms (modelled K1 efficiency), and the
whole serial evaluation's ms.  Exchanges run as peer copies on one GPU here,
so the NCCL latency of a real group (~10-30 us per exchange) is not in it.
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
os.environ.setdefault("SMC_GROUP_EXCHANGE", "emulated")
os.environ["SMC_GROUP_SERIAL"] = "1"

import paper_1808_10580_b200 as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2", choices=["c2", "c3", "c5"])
ap.add_argument("--worlds", default="1,2,4,8")
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()

import bench  # noqa: E402  (the bench's workloads, same specs and seeds)

base = S.default_context(0)
kind, spec, _ = bench.build_workload(args.config, base)
if kind == "ad":
    run = lambda ctx: S.observe_ad(spec, 808, ctx=ctx)  # noqa: E731
else:
    run = lambda ctx: S.observe_bvp(spec, 606, ctx=ctx)  # noqa: E731

one = None
ref = None
for w in [int(x) for x in args.worlds.split(",")]:
    ctx = base if w == 1 else S.Context(devices=[0] * w)
    run(ctx)  # warm-up
    k1, wall = [], []
    for _ in range(args.reps):
        t0 = time.perf_counter()
        est = run(ctx)
        wall.append(1e3 * (time.perf_counter() - t0))
        k1.append(ctx.stats().particle_kernel_ms)
    means = [e.mean for e in est]
    if ref is None:
        ref = means
    per_rank = min(k1)
    if one is None:
        one = per_rank
    print(json.dumps({"config": args.config, "world": w, "per_rank_k1_ms": round(per_rank, 3),
                      "modelled_k1_efficiency": round(one / (w * per_rank), 4),
                      "serial_eval_ms": round(min(wall), 3), "bit_identical_to_w1": means == ref}))
