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
ap.add_argument("--cutoff", type=int, default=0, help="C2 shape with a K=cutoff prior-draw velocity (0: as config)")
ap.add_argument("--constant-velocity", action="store_true", help="C2 shape with v = (0.3, -0.2)")
args = ap.parse_args()
if args.lattice:
    os.environ["SMC_DISABLE_DISK"] = "1"

import bench  # noqa: E402
import paper_1808_10580_b200 as S  # noqa: E402

ctx = S.default_context(0)
if args.config == "c4":
    # B pCN proposals u_b = sqrt(1-beta^2) u0 + beta xi_b, K=25 prior, CRN seed 808
    import math
    import numpy as np
    import specs
    B = args.particles or 4096
    prior = specs.C4_PRIOR
    u0 = S.prior_draw(prior, 808, 0xBE9C4, 1, ctx)
    stds = prior.component_stds()
    xi = np.random.default_rng(0).normal(size=(B, prior.dimension())) * stds
    U = math.sqrt(1 - 0.02 ** 2) * u0[None, :] + 0.02 * xi
    base = specs.c4_base(n_particles=1024, precision=S.Precision[args.precision])
    for _ in range(args.reps):
        out = S.observe_ad_batched(base, prior, U, 808, ctx=ctx)
    st = ctx.stats()
    print(f"c4 B={B}: kernel {st.particle_kernel_ms:.3f} ms reduce {st.reduce_ms:.3f} ms steps {st.particle_steps} -> "
          f"{st.particle_steps / st.particle_kernel_ms * 1e3:.4g} particle-steps/s; "
          f"{14 * 980 + 12 * 24 + 20} flop/step -> {(14 * 980 + 12 * 24 + 20) * st.particle_steps / st.particle_kernel_ms / 1e9:.2f} TFLOP/s")
    sys.exit(0)
if args.config in ("pcn", "pcn8"):
    # sample_k2.json shape (K=2) or the paper's Ex. 2 size (K=8, N_u=197): B chains
    import time
    import numpy as np
    import specs
    B = args.particles or 100
    prior = S.PriorSpec(2, 0.6, 2.5) if args.config == "pcn" else S.PriorSpec(8, 0.6, 2.5)
    fwd = specs.c4_base(n_particles=160)
    fwd.dt = 0.006
    like = S.LikelihoodSpec(data=[-0.9065, -0.7528, -0.6665, -0.8091, -0.6508, -0.5135, -0.5185, -0.4553, -0.4066],
                            noise_std=0.05, forward=fwd, forward_seed=1234)
    n_steps = int(os.environ.get('PCN_STEPS', '2000'))
    cfg = S.ChainConfig(n_steps=n_steps, beta=0.22, burn_in=min(200, n_steps // 2), thin=10)
    S.run_chains(S.ChainConfig(n_steps=5, beta=0.22), prior, like, list(range(B)), ctx=ctx)  # warm-up
    times, dev = [], []
    for _ in range(max(args.reps, 1)):
        t0 = time.perf_counter()
        res = S.run_chains(cfg, prior, like, list(range(B)), ctx=ctx)
        times.append(time.perf_counter() - t0)
        dev.append(ctx.stats().particle_kernel_ms)
    el = min(times)
    print(f"[wall {', '.join(f'{t / n_steps * 1e6:.0f}' for t in times)} us/step; "
          f"device {', '.join(f'{d / n_steps * 1e3:.0f}' for d in dev)} us/step]")
    print(f"{args.config} B={B} dim={prior.dimension()}: {n_steps} steps in {el:.3f} s (best of {len(times)}) -> "
          f"{B * n_steps / el:.4g} chain-steps/s ({el / n_steps * 1e6:.1f} us/step), "
          f"acceptance {res['acceptance_rate'].mean():.3f}")
    sys.exit(0)
if args.config == "galerkin":
    # the paper's Fig. 8 reference solve: C2's velocity, box cutoff L (default
    # 16: 1089 modes, A = 19 MB), dt_ref from the stability estimate, t = 1
    import math
    import time
    import numpy as np
    import specs
    L = args.cutoff or 16
    u = S.prior_draw(specs.C2_PRIOR, 808, 0xBE9C4, 0, ctx)
    spec = specs.c2_spec(u, n_particles=1000)
    radius = S.galerkin_spectral_radius(spec, L, ctx)
    dt = 1.0 / radius
    for rep in range(max(args.reps, 1)):
        t0 = time.perf_counter()
        res = S.galerkin_solve_ad(spec, L, dt, ctx=ctx)
        el = time.perf_counter() - t0
    nb = len(res.basis_modes)
    print(f"galerkin L={L} nb={nb} dt={dt:.3g} steps={res.steps}: {el * 1e3:.1f} ms -> {el / res.steps * 1e6:.2f} us/step, "
          f"{16.0 * nb * nb * res.steps / el / 1e12:.2f} TB/s of A streamed; obs[0]={res.observation_values[0]:.12g}")
    sys.exit(0)
if args.config in ("c3", "c3b"):
    # paper BVP, F=(1,-0.5,2), 25 obs, 1e6 walkers/obs, seed 606
    import specs
    spec = specs.c3_spec(n_particles=args.particles or 1_000_000, precision=S.Precision[args.precision])
    if args.config == "c3b":
        u = S.prior_draw(specs.C2_PRIOR, 808, 0xBE9C4, 0, ctx)
        spec.velocity = S.VelocityField.fourier(S.velocity_from_coefficients(specs.C2_PRIOR, u))
    for _ in range(args.reps):
        est = S.observe_bvp(spec, 606, ctx=ctx)
    st = ctx.stats()
    print(f"{args.config}: kernel {st.particle_kernel_ms:.3f} ms reduce {st.reduce_ms:.3f} ms walker-steps "
          f"{st.particle_steps} -> {st.particle_steps / st.particle_kernel_ms * 1e3:.4g} walker-steps/s; "
          f"mean[0]={est[0].mean:.15g} exit[0]={est[0].aux_mean:.6g} failed={sum(e.n_failed for e in est)}")
    sys.exit(0)
kind, spec, steps = bench.build_workload(args.config, ctx)
if args.cutoff:
    import specs
    prior = S.PriorSpec(args.cutoff, 1.0, 2.5)
    spec.velocity = S.VelocityField.fourier(S.velocity_from_coefficients(prior, S.prior_draw(prior, 808, 0xBE9C4, 0, ctx)))
if args.constant_velocity:
    spec.velocity = S.VelocityField.constant((0.3, -0.2))
if args.particles:
    spec.n_particles = args.particles
spec.precision = S.Precision[args.precision]
for _ in range(args.reps):
    est = S.observe_ad(spec, 808, ctx=ctx)
st = ctx.stats()
print(f"{args.config} K={args.cutoff} const={args.constant_velocity} P={os.environ.get('SMC_DISK_P', '-')}: kernel {st.particle_kernel_ms:.3f} ms reduce {st.reduce_ms:.3f} ms "
      f"steps {st.particle_steps} -> {st.particle_steps / st.particle_kernel_ms * 1e3:.4g} particle-steps/s; "
      f"mean[0]={est[0].mean:.15g}")
