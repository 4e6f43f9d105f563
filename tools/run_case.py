"""Run one workload of bench.py a few times (for ncu / compute-sanitizer).

    python tools/run_case.py --config c2 --reps 2 [--particles N] [--lattice]
"""
import argparse
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--particles", type=int, default=0)
ap.add_argument("--lattice", action="store_true", help="disable the compile-time disk kernel")
ap.add_argument("--precision", default="fp64", choices=["fp64", "fp32", "fp64_strict"])
args = ap.parse_args()
if args.lattice:
    os.environ["SMC_DISABLE_DISK"] = "1"

import bench  # noqa: E402
import paper_1808_10580_b200 as S  # noqa: E402

ctx = S.default_context(0)
spec, steps, F, desc = bench.build_workload(args.config, ctx)
if args.particles:
    spec.n_particles = args.particles
spec.precision = S.Precision[args.precision]
for _ in range(args.reps):
    est = S.observe_ad(spec, 808, ctx=ctx)
st = ctx.stats()
print(f"{args.config}: kernel {st.particle_kernel_ms:.3f} ms reduce {st.reduce_ms:.3f} ms "
      f"steps {st.particle_steps} -> {st.particle_steps / st.particle_kernel_ms * 1e3:.4g} particle-steps/s; "
      f"mean[0]={est[0].mean:.15g}")
