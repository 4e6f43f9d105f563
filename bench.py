#!/usr/bin/env python
"""Benchmark of the B200 particle forward map (BASELINE.json metric:
particle-steps/s and forward-map evals/s, whole box).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

A "step" is one forward-map evaluation G(u) of the workload.  At N=1 the
workload is BASELINE configs[1] = SURVEY.md §8(d) C2: 2D advection-diffusion,
K=8 Fourier velocity (M=98 modes, N_u=197) drawn from the prior with the
reference's benchmark recipe (benchmark.cpp:69-71), 9 observations, 1e5
particles per observation, 1000 Euler-Maruyama steps (9e8 particle-steps per
evaluation), FP64.  Under torchrun (N>1) each evaluation is sharded over the
ranks by particle chunks with an NCCL all-gather of the chunk partial sums
(strong scaling: the evaluation is fixed).

Printed on rank 0, one JSON line:
  value       particle-steps/s from device time (CUDA events on the stream the
              kernels run on, inputs resident, max over ranks)
  e2e         the same metric through the public API (S.observe_ad / the
              sharded observe_ad) with host spec in, host estimates out
  roofline    dominant kernel K1 (ad_particles<double>): algorithmic FP64 flops
              (F_AD = 14 M + 12 (K-1) + 20 per particle-step)
              over its CUDA-event duration, against the FP64 DFMA peak measured
              in this run
  cpu_baseline  the reference (oracle/_ref, compiled from the reference's own
              sources) on this host's cores, bounded sample, rank 0 at N=1

--impl reference runs the reference's own CPU implementation (oracle/_ref) of
the same workload on all host cores instead.  --precision fp32 measures the
optional FP32 variant of the kernels (roofline against an FFMA peak measured
in the same run); the default and the headline are FP64.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

METRIC = "particle-steps/sec and forward-map evals/sec (whole box) at 1/2/4/8 B200"
PROFILES = ROOT / "profiles"


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------
def flops_ad(K: int, M: int) -> int:
    """F_AD = 14 M + 12 (K - 1) + 20 per particle-step."""
    return 14 * M + 12 * (K - 1) + 20


def flops_bvp(n_bumps: int, K: int = 0, M: int = 0) -> int:
    """F_BVP = 10 + 4 + 4 + 8 N_bump + 2 (+ F_velocity)."""
    return 10 + 4 + 4 + 8 * n_bumps + 2 + (14 * M + 12 * (K - 1) if M else 0)


def c5_spec(S, u):
    """K=80 (M=10040), kappa 3e-5, theta_0 = 100-term
    cosine series (|k| <= 8, random amplitudes), 64 observations
    (j/8, j/8) x t in {1/16 .. 8/16}, dt 5e-4, 32768 particles/obs."""
    prior = S.PriorSpec(80, 1.0, 2.5)
    rng = np.random.default_rng(5)
    terms = []
    for k1 in range(-8, 9):
        for k2 in range(-8, 9):
            if len(terms) < 100 and 0 < k1 * k1 + k2 * k2 <= 64:
                terms.append((float(rng.normal()) / (k1 * k1 + k2 * k2), (2 * math.pi * k1, 2 * math.pi * k2),
                              float(rng.random() * 2 * math.pi)))
    obs = [S.AdObservation(t / 16.0, S.Vec2(j / 8.0, j / 8.0)) for j in range(8) for t in range(1, 9)]
    return S.AdProblemSpec(velocity=S.VelocityField.fourier(S.velocity_from_coefficients(prior, u)),
                           diffusion=S.DiffusionModel.isotropic(3e-5),
                           initial_condition=S.ScalarField.cosine_series(terms), observations=obs, dt=5e-4,
                           n_particles=32768)


def build_workload(name: str, ctx, u_source=None):
    """-> (kind, payload, particle-steps per evaluation (None: counted on
    device), flops per particle-step, description).  u_source(prior, seed,
    obs, particle) draws prior coefficients (device normals on our arm, the
    reference's prior_draw on the reference arm)."""
    import paper_1808_10580_b200 as S
    import specs
    draw = u_source or (lambda prior, seed, obs, particle: S.prior_draw(prior, seed, obs, particle, ctx))
    if name == "c2":
        u = draw(specs.C2_PRIOR, 808, 0xBE9C4, 0)  # benchmark.cpp:69-71 recipe
        spec = specs.c2_spec(u, n_particles=100_000)
        K, M = 8, len(specs.C2_PRIOR.modes())
        desc = {"workload": "C2: AD forward map, K=8 Fourier velocity (M=98, N_u=197), 9 obs, 1e5 particles/obs, "
                            "1000 EM steps, FP64", "K": K, "modes": M, "n_obs": 9, "particles_per_obs": 100_000,
                "em_steps": 1000, "seed": 808}
        kind, payload, F = "ad", spec, flops_ad(K, M)
    elif name == "c1":
        spec = specs.c1_two_mode(n_particles=10_000)
        desc = {"workload": "C1: shipped forward_ad_two_mode.json (K=1, M=2, 3 obs, 1e4 particles)", "K": 1,
                "modes": 2, "n_obs": 3, "particles_per_obs": 10_000, "seed": 7}
        kind, payload, F = "ad", spec, flops_ad(1, 2)
    elif name == "c5":
        u = draw(S.PriorSpec(80, 1.0, 2.5), 808, 0xBE9C4, 2)
        spec = c5_spec(S, u)
        desc = {"workload": "C5: AD forward map, K=80 (M=10040, N_u=20081), 64 obs, 32768 particles/obs, FP64",
                "K": 80, "modes": 10040, "n_obs": 64, "particles_per_obs": 32768, "seed": 808}
        kind, payload, F = "ad", spec, flops_ad(80, 10040)
    elif name == "c3":
        spec = specs.c3_spec(n_particles=1_000_000)
        desc = {"workload": "C3: Dirichlet BVP, box, v=(1,1), kappa 0.282, 3 bumps F=(1,-0.5,2), 25 obs, "
                            "1e6 walkers/obs, dt 1.5e-4, FP64", "n_obs": 25, "walkers_per_obs": 1_000_000,
                "seed": 606}
        kind, payload, F = "bvp", spec, flops_bvp(3)
    elif name == "c4":
        prior = specs.C4_PRIOR
        u0 = draw(prior, 808, 0xBE9C4, 1)
        B = 4096
        # pCN proposals u_b = sqrt(1-beta^2) u0 + beta xi_b, xi_b ~ prior (inference.cpp:141-144)
        U = np.stack([math.sqrt(1 - 0.02 ** 2) * u0 + 0.02 * draw(prior, 4242, 0xFFFFFFFF, b) for b in range(B)])
        base = specs.c4_base(n_particles=1024)
        desc = {"workload": "C4: batched MCMC, 4096 pCN proposals per launch, K=25 (M=980) velocity, 9 obs, "
                            "1024 particles/obs, CRN seed 808, FP64", "K": 25, "modes": 980, "samples": B,
                "n_obs": 9, "particles_per_obs": 1024, "seed": 808}
        kind, payload, F = "batched", (base, prior, U), flops_ad(25, 980)
    else:
        raise SystemExit(f"unknown config {name}")
    if kind == "ad":
        dt = payload.resolved_dt()
        steps = sum(int(math.ceil(o.t / dt)) for o in payload.observations) * payload.n_particles
    elif kind == "batched":
        base, prior, U = payload
        steps = sum(int(math.ceil(o.t / base.resolved_dt())) for o in base.observations) * base.n_particles * len(U)
    else:
        steps = None  # exit times are random: counted on device
    return kind, payload, steps, F, desc


# ---------------------------------------------------------------------------
# clocks sampling (B200_PROFILING.md "clocks DURING the timed region")
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower() in ("active", "1"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU baseline: the reference compiled from its own sources (oracle/_ref)
# ---------------------------------------------------------------------------
def reference_runner(config: str, R, cores: int, budget_s: float):
    """A bounded sample of `config` on the reference (oracle/_ref, the
    reference compiled from its own sources) with workers = cores:
    -> (particle-steps per run, run(), description).  Inputs follow the same
    recipes as our arm, drawn with the reference's own prior_draw.  The
    reference's executor parallelises one observation over 1024-particle
    chunks (executor.cpp:45-85), so samples keep >= 1024 x cores particles per
    observation where the full config has them."""
    import copy
    kind, payload, steps, F, desc = build_workload(
        config, None, u_source=lambda prior, seed, obs, particle: R.prior_draw(prior, seed, obs, particle))
    rate = 3.0e9 / F * cores  # ~3 Gflop/s/core on the reference's mode loop
    if kind == "ad" and config != "c5":
        spec = payload
        per_particle = steps / spec.n_particles
        n = int(max(1024 * cores, budget_s * rate / per_particle))
        n = min(spec.n_particles, n)
        sample = copy.copy(spec)
        sample.n_particles = n
        return per_particle * n, lambda: R.observe_ad(sample, 808, cores), \
            f"observe_ad, all {len(spec.observations)} obs, {n} particles/obs (of {spec.n_particles}), " \
            f"workers={cores}"
    if kind in ("ad", "batched"):
        # one observation (the shortest time) of the evaluation, 1024 x cores particles
        if kind == "ad":
            spec = copy.copy(payload)
            u = None
        else:
            base, prior, U = payload
            spec = copy.copy(base)
            u = U[0]
        j = int(np.argmin([o.t for o in spec.observations]))
        spec.observations = [spec.observations[j]]
        spec.n_particles = 1024 * cores
        per = int(math.ceil(spec.observations[0].t / spec.resolved_dt())) * spec.n_particles
        if u is None:
            run = lambda: R.observe_ad(spec, 808, cores)  # noqa: E731
        else:
            run = lambda: R.observe_ad_u(spec, prior, u, 808, cores)  # noqa: E731
        return per, run, f"observe_ad on observation {j} only (t={spec.observations[0].t:g}), " \
                         f"{spec.n_particles} particles, workers={cores}" + \
                         (", proposal 0 of the batch" if u is not None else "")
    # bvp: walker-steps of the sample from the reference's own simulate_to_exit
    spec = payload
    sample = copy.copy(spec)
    n = int(max(64, min(spec.n_particles, 1024 * cores)))
    sample.n_particles = n
    probe = 32
    mean_steps = float(np.mean([R.bvp_particle_values(spec, j, 606, probe)[3].mean()
                                for j in range(len(spec.observations))]))
    return mean_steps * n * len(spec.observations), lambda: R.observe_bvp(sample, 606, cores), \
        f"observe_bvp with {n} walkers/obs (of {spec.n_particles}), workers={cores}; walker-steps from " \
        f"{probe} walkers/obs via the reference's simulate_to_exit"


def cpu_reference_sample(config: str, ctx, per_eval: float, budget_s: float = 4.0):
    """cpu_baseline: 1 warm-up + median of 5 bounded runs
    (benchmark.cpp:39-52 methodology; median of >= 5) on all
    host cores."""
    from oracle.oracle import Reference
    R = Reference()
    cores = os.cpu_count() or 1
    steps, run, sample = reference_runner(config, R, cores, budget_s)
    run()
    times = []
    for _ in range(5):
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
    return steps / statistics.median(times), cores, sample + ", median of 5 after 1 warm-up"


# ---------------------------------------------------------------------------
# ours
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1808_10580_b200 as S
    from paper_1808_10580_b200 import distributed as D

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) if args.device < 0 else args.device
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:  # multi-rank plumbing test on fewer GPUs (host-staged all-gathers)
            dist.init_process_group("gloo")
    red_dev = "cuda" if args.dist_backend == "nccl" else "cpu"
    ctx = S.default_context(local)
    stream = torch.cuda.Stream(device=local)
    torch.cuda.set_stream(stream)
    S.load_library().smc_set_stream(ctx.handle, stream.cuda_stream)

    kind, payload, steps_per_eval, F, desc = build_workload(args.config, ctx)
    fp32 = args.precision == "fp32"
    if fp32:  # the optional FP32 variant (north_star: within 3 SE of the FP64 result)
        target = payload[0] if kind == "batched" else payload
        target.precision = S.Precision.fp32
        desc = dict(desc, workload=desc["workload"].replace("FP64", "FP32 variant"), precision="fp32")
    peak = ctx.fp32_peak_tflops(300.0) if fp32 else ctx.fp64_peak_tflops(300.0)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # > 126 MB L2

    def timed(fn):
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        before = ctx.stats().total_launches
        t0.record(stream)
        k_ms, steps = fn()
        t1.record(stream)
        t1.synchronize()
        return t0.elapsed_time(t1), k_ms, ctx.stats().total_launches - before, steps

    if kind == "ad":
        spec = payload
        n_chunks = D.num_chunks(spec.n_particles)
        b, e = D.chunk_range(n_chunks, rank, world)
        counts = [D.chunk_range(n_chunks, r, world)[1] - D.chunk_range(n_chunks, r, world)[0] for r in range(world)]
        my_steps = steps_per_eval * (e - b) / n_chunks  # chunk-proportional (last chunk may be partial)

        def device_step():
            """One evaluation, inputs resident: at N=1 the single-GPU forward map
            (K1 + K3, one launch each), at N>1 the device-level sharded path."""
            if world == 1:
                def run1():
                    S.observe_ad(spec, 808, ctx=ctx)
                    return ctx.stats().particle_kernel_ms, my_steps
                return timed(run1)
            ops = D.DeviceOps(spec, 808, ctx)

            def run():
                parts = ops.partials(b, e)
                k = ctx.stats().particle_kernel_ms
                sums = ops.finish(ops.all_gather(parts, counts))
                means = ops.divide(sums, spec.n_particles)
                ops.finish(ops.all_gather(ops.sq_partials(means, b, e), counts))
                return k, my_steps
            return timed(run)

        def e2e_step():
            if world == 1:
                return S.observe_ad(spec, 808, ctx=ctx)
            return D.observe_ad_sharded(spec, 808, rank, world, ctx)
        api = ("paper_1808_10580_b200.observe_ad -> smc_ad_observe (C ABI)" if world == 1 else
               "paper_1808_10580_b200.distributed.observe_ad_sharded (C ABI + NCCL all-gather)")
        parallel = f"particle-shard x{world}" if world > 1 else "single GPU"
        scaling = "strong"
        h2d, d2h = _image_bytes(spec), 40 * len(spec.observations)
        kernel_name = "ad_particles (K1)"
    elif kind == "bvp":
        spec = payload
        n_obs = len(spec.observations)
        if world == 1:
            def device_step():
                def run():
                    S.observe_bvp(spec, 606, ctx=ctx)
                    st = ctx.stats()
                    return st.particle_kernel_ms, st.particle_steps
                return timed(run)

            def e2e_step():
                return S.observe_bvp(spec, 606, ctx=ctx)
            api = "paper_1808_10580_b200.observe_bvp -> smc_bvp_observe (C ABI)"
        else:  # walker sharding: every rank runs its walker range of all observations
            bops = D.BvpDeviceOps(spec, 606, ctx)
            wb, we = D.walker_range(spec.n_particles, rank, world)
            wcounts = [D.walker_range(spec.n_particles, r, world)[1] - D.walker_range(spec.n_particles, r, world)[0]
                       for r in range(world)]

            def device_step():
                def run():
                    vals, aux, failed = bops.shard(wb, we)
                    st = ctx.stats()
                    k, steps = st.particle_kernel_ms, st.particle_steps
                    bops.reduce(bops.all_gather(vals, wcounts), bops.all_gather(aux, wcounts),
                                bops.all_gather(failed, wcounts))
                    return k, steps
                return timed(run)

            def e2e_step():
                return D.observe_bvp_sharded(spec, 606, rank, world, ctx)
            api = ("paper_1808_10580_b200.distributed.observe_bvp_sharded (C ABI smc_bvp_shard_values + "
                   "all-gather of walker results + smc_bvp_reduce_values)")
        parallel = f"walker-shard x{world}" if world > 1 else "single GPU"
        scaling = "strong"
        h2d, d2h = 16 * n_obs + 512, 40 * n_obs
        kernel_name = "bvp_walkers (K2)"
    else:  # batched
        base, prior, U = payload
        sb, se = D.sample_range(len(U), rank, world)
        my_U = U[sb:se]
        my_steps = steps_per_eval * (se - sb) / len(U)

        def device_step():
            def run():
                S.observe_ad_batched(base, prior, my_U, 808, ctx=ctx)
                return ctx.stats().particle_kernel_ms, my_steps
            return timed(run)

        def e2e_step():
            return S.observe_ad_batched(base, prior, my_U, 808, ctx=ctx)
        api = "paper_1808_10580_b200.observe_ad_batched -> smc_ad_observe_batched (C ABI)"
        parallel = f"sample-shard x{world}" if world > 1 else "single GPU"
        scaling = "strong"
        h2d, d2h = my_U.nbytes + 2048, 40 * len(base.observations) * len(my_U)
        kernel_name = "ad_particles<double> generic tiled lattice (K1)"

    for _ in range(args.warmup):
        device_step()
        e2e_step()

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    dev_ms = k_ms = 0.0
    launches = 0
    my_total_steps = 0.0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for _ in range(args.steps):
        flush.zero_()  # L2 flush between timed iterations (outside the step's events)
        torch.cuda.synchronize()
        d, k, n, st = device_step()
        dev_ms += d
        k_ms += k
        launches += n
        my_total_steps += st
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # end-to-end through the public API (host inputs in, host estimates out)
    e2e_s = 0.0
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        e2e_step()
        e2e_s += time.perf_counter() - t0
    torch.cuda.synchronize()
    clocks = sampler.stop()

    tmax = torch.tensor([dev_ms, e2e_s], dtype=torch.float64, device=red_dev)
    tsum = torch.tensor([my_total_steps], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
    dev_ms, e2e_s = tmax.tolist()
    total_steps = tsum.item()
    per_eval = total_steps / args.steps
    value = total_steps / (dev_ms / 1e3)
    e2e_value = total_steps / e2e_s
    # roofline: this rank's algorithmic flops over its particle-kernel event time
    achieved = F * my_total_steps / (k_ms / 1e3) / 1e12

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "particle-steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f32" if fp32 else "f64",
            "data": "synthetic (prior-draw velocity, reference recipe)",
            "config": dict(desc, parallelism=parallel, l2="flushed between steps (256 MiB write)"),
            "evals_per_sec": value / per_eval,
            "e2e": {"value": e2e_value, "unit": "particle-steps/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "evals_per_sec": e2e_value / per_eval, "api": api},
            "roofline": {"bound": "fp32" if fp32 else "fp64", "kernel": kernel_name, "achieved": achieved,
                         "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                         "peak_source": ("FP32 FFMA microbenchmark measured in this run (smc_fp32_peak, all SMs, "
                                         "8 chains/thread); MEASURED_PEAKS.json has no FP32 entry" if fp32 else
                                         "FP64 DFMA microbenchmark measured in this run (smc_fp64_peak, all SMs, "
                                         "8 chains/thread); MEASURED_PEAKS.json has no FP64 entry"),
                         "flops_per_unit": F, "unit_of_work": "particle-step",
                         "flops_note": "algorithmic flops = SURVEY.md 8(d) F_AD (the reference's 14 flops per "
                                       "mode); the kernels execute fewer (4 FMA per mode, Chebyshev "
                                       "harmonics), so frac can exceed 1 — the hardware figure is "
                                       "traffic.pipe_active_frac, ncu's active fraction of the dominant pipe "
                                       "for this kernel",
                         "traffic": _ncu_traffic(args.config + ("_fp32" if fp32 else ""))},
            "gpu_launches": launches,
            "clocks": clocks,
        }
        if world == 1 and not args.no_cpu_baseline:
            try:
                v, cores, sample = cpu_reference_sample(args.config, ctx, per_eval)
                line["cpu_baseline"] = {"value": v, "unit": "particle-steps/s", "cores": cores, "kind": "reference",
                                        "sample": sample}
            except Exception as e:  # noqa: BLE001
                line["cpu_baseline"] = {"value": None, "unavailable": f"{type(e).__name__}: {e}"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _image_bytes(spec) -> int:
    """Bytes of the host->device problem image one observe_ad call uploads."""
    n_obs = len(spec.observations)
    b = 80 * n_obs  # AdObsImg
    ic = spec.initial_condition
    b += 32 * max(len(ic.terms), len(ic.bumps))
    v = spec.velocity
    if not v.is_constant:
        m = v.fourier_field.n_modes
        b += 40 * m + 8 * 4 * m + 256  # strict mode list + lattice coefficients (~4 doubles/mode) + index
    return int(b)


def _ncu_traffic(config: str = "c2"):
    """DRAM bytes per particle-kernel launch and the dominant pipe's active
    fraction from the committed ncu --set full capture of this config
    (profiles/rNN_k*_<config>[_reduced].json), if any."""
    caps = sorted(PROFILES.glob(f"r*_k*_{config}.json")) or sorted(PROFILES.glob(f"r*_k*_{config}_reduced.json"))
    if caps:
        try:
            d = json.loads(caps[-1].read_text())
            fp32 = config.endswith("_fp32")
            pipe = d.get("fma_pipe_pct_active" if fp32 else "fp64_pipe_pct_active")
            return {"dram_bytes_per_launch": d.get("dram_bytes_per_launch"), "source": f"profiles/{caps[-1].name}",
                    "pipe": "fma (FP32)" if fp32 else "fp64",
                    "pipe_active_frac": None if pipe is None else round(pipe / 100.0, 4),
                    "reduced_launch": caps[-1].name.endswith("_reduced.json")}
        except Exception:  # noqa: BLE001
            return None
    return None


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------
def run_reference(args):
    """The reference's own CPU implementation (oracle/_ref) on all host cores,
    same config/metric/unit as our arm; each step a bounded sample."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    from oracle.oracle import Reference
    R = Reference()
    cores = os.cpu_count() or 1
    kind, payload, steps_full, F, desc = build_workload(
        args.config, None, u_source=lambda prior, seed, obs, particle: R.prior_draw(prior, seed, obs, particle))
    steps, run, sample = reference_runner(args.config, R, cores, budget_s=4.0)
    for _ in range(args.warmup):
        run()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        run()
    el = time.perf_counter() - t0
    value = steps * args.steps / el
    per_eval = steps_full if steps_full else steps
    line = {"metric": METRIC, "impl": "reference", "value": value, "unit": "particle-steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (prior-draw velocity, reference recipe)",
            "config": dict(desc, parallelism=f"std::thread x{cores} (reference executor)"),
            "evals_per_sec": value / per_eval,
            "cpu_baseline": {"value": value, "unit": "particle-steps/s", "cores": cores, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": value, "unit": "particle-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="fp64", choices=["fp64", "fp32"],
                    help="fp32 = the optional FP32 variant of the kernels (our arm only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: test the multi-rank path with fewer GPUs than ranks")
    ap.add_argument("--device", type=int, default=-1, help="override LOCAL_RANK -> device (plumbing tests)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
