#!/usr/bin/env python
"""Benchmark of the B200 particle forward map (BASELINE.json metric:
particle-steps/s and forward-map evals/s, whole box).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

A "step" is one forward-map evaluation G(u) of the workload.  At N=1 the
workload is BASELINE configs[1] = SURVEY.md §8(d) C2: 2D advection-diffusion,
K=8 Fourier velocity (M=98 modes, N_u=197) drawn from the prior with the
reference's benchmark recipe (benchmark.cpp:69-71), 9 observations, 1e5
particles per observation, 1000 Euler-Maruyama steps (9e8 particle-steps per
evaluation), FP64.

--gpus N > 1 without a launcher re-executes itself under
`python -m torch.distributed.run --nproc-per-node N` (one process per GPU);
under torchrun WORLD_SIZE must equal N.  Every rank then calls the SAME public
forward map on a multi-device context (distributed.rank_context: the C ABI's
smc_create_rank, NCCL communicator inside the library), which shards the
evaluation (strong scaling: particles of C1/C2/C5, walkers of C3, proposals of
C4) and combines the ranks with the library's small deterministic exchange.

Printed on rank 0, one JSON line:
  value       particle-steps/s of the whole evaluation over the max-over-ranks
              device time (CUDA events on the stream the forward map runs on)
  e2e         the same metric through the public API call with host spec in
              and host estimates out, wall clock, max over ranks
  roofline    dominant kernel (K1 / K2): algorithmic FP64 flops (SURVEY.md
              §8(d) F_AD / F_BVP per particle-step) over its CUDA-event
              duration against the FP64 DFMA peak measured in this run, plus
              the EXECUTED FP64 flops (ncu DFMA/DADD/DMUL counts) over the same
              time, and the ncu pipe / DRAM figures of the committed capture
  cpu_baseline  the reference (oracle/_ref, compiled from the reference's own
              sources) on this host's cores, bounded sample, rank 0 at N=1

--impl reference runs the reference's own CPU implementation (oracle/_ref) of
the same workload on all host cores: no product code is imported or loaded in
that process (oracle/pods.py builds its problems).  --precision fp32 measures
the optional FP32 variant of the kernels.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "particle-steps/sec and forward-map evals/sec (whole box) at 1/2/4/8 B200"
PROFILES = ROOT / "profiles"

# Workload descriptions; both arms print exactly these.
CONFIGS = {
    "c1": {"workload": "C1: shipped forward_ad_two_mode.json (K=1, M=2, 3 obs, 1e4 particles)", "K": 1,
           "modes": 2, "n_obs": 3, "particles_per_obs": 10_000, "seed": 7},
    "c2": {"workload": "C2: AD forward map, K=8 Fourier velocity (M=98, N_u=197), 9 obs, 1e5 particles/obs, "
                       "1000 EM steps, FP64", "K": 8, "modes": 98, "n_obs": 9, "particles_per_obs": 100_000,
           "em_steps": 1000, "seed": 808},
    "c3": {"workload": "C3: Dirichlet BVP, box, v=(1,1), kappa 0.282, 3 bumps F=(1,-0.5,2), 25 obs, "
                       "1e6 walkers/obs, dt 1.5e-4, FP64", "n_obs": 25, "walkers_per_obs": 1_000_000, "seed": 606},
    "c4": {"workload": "C4: batched MCMC, 4096 pCN proposals per launch, K=25 (M=980) velocity, 9 obs, "
                       "1024 particles/obs, CRN seed 808, FP64", "K": 25, "modes": 980, "samples": 4096,
           "n_obs": 9, "particles_per_obs": 1024, "seed": 808},
    "c5": {"workload": "C5: AD forward map, K=80 (M=10040, N_u=20081), 64 obs, 32768 particles/obs, FP64",
           "K": 80, "modes": 10040, "n_obs": 64, "particles_per_obs": 32768, "seed": 808},
}
C4_BATCH, C4_BETA = 4096, 0.02


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------
def flops_ad(K: int, M: int) -> int:
    """F_AD = 14 M + 12 (K - 1) + 20 per particle-step."""
    return 14 * M + 12 * (K - 1) + 20


def flops_bvp(n_bumps: int, K: int = 0, M: int = 0) -> int:
    """F_BVP = 10 + 4 + 4 + 8 N_bump + 2 (+ F_velocity)."""
    return 10 + 4 + 4 + 8 * n_bumps + 2 + (14 * M + 12 * (K - 1) if M else 0)


FLOPS = {"c1": flops_ad(1, 2), "c2": flops_ad(8, 98), "c3": flops_bvp(3), "c4": flops_ad(25, 980),
         "c5": flops_ad(80, 10040)}


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


def build_workload(name: str, ctx):
    """Our arm: -> (kind, payload, particle-steps per evaluation (None:
    counted on device)).  Prior draws on the device (S.prior_draw, the
    reference's prior_draw bit for bit)."""
    import paper_1808_10580_b200 as S
    sys.path.insert(0, str(ROOT / "tests"))
    import specs
    if name == "c2":
        u = S.prior_draw(specs.C2_PRIOR, 808, 0xBE9C4, 0, ctx)  # benchmark.cpp:69-71 recipe
        kind, payload = "ad", specs.c2_spec(u, n_particles=100_000)
    elif name == "c1":
        kind, payload = "ad", specs.c1_two_mode(n_particles=10_000)
    elif name == "c5":
        kind, payload = "ad", c5_spec(S, S.prior_draw(S.PriorSpec(80, 1.0, 2.5), 808, 0xBE9C4, 2, ctx))
    elif name == "c3":
        kind, payload = "bvp", specs.c3_spec(n_particles=1_000_000)
    elif name == "c4":
        prior = specs.C4_PRIOR
        u0 = S.prior_draw(prior, 808, 0xBE9C4, 1, ctx)
        # pCN proposals u_b = sqrt(1-beta^2) u0 + beta xi_b, xi_b ~ prior (inference.cpp:141-144)
        U = np.stack([math.sqrt(1 - C4_BETA ** 2) * u0 + C4_BETA * S.prior_draw(prior, 4242, 0xFFFFFFFF, b, ctx)
                      for b in range(C4_BATCH)])
        kind, payload = "batched", (specs.c4_base(n_particles=1024), prior, U)
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
    return kind, payload, steps


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
# CPU baseline / reference arm: the reference compiled from its own sources
# (oracle/_ref), problems from oracle/pods.py — no product code involved
# ---------------------------------------------------------------------------
def reference_runner(config: str, R, cores: int, budget_s: float):
    """A bounded sample of `config` on the reference with workers = cores:
    -> (particle-steps per run, run(), description).  Inputs follow the same
    recipes as our arm, drawn with the reference's own prior_draw.  The
    reference's executor parallelises one observation over 1024-particle
    chunks (executor.cpp:45-85), so samples keep >= 1024 x cores particles per
    observation where the full config has them."""
    from oracle import pods as P
    rate = 3.0e9 / FLOPS[config] * cores  # ~3 Gflop/s/core on the reference's mode loop
    if config in ("c1", "c2"):
        full = P.c1() if config == "c1" else P.c2_base()
        per_particle = sum(int(math.ceil(t / R.resolved_dt_ad(full))) for t, _ in full.observations)
        n = int(min(full.n_particles, max(1024 * cores, budget_s * rate / per_particle)))
        sample = P.c1(n) if config == "c1" else P.c2_base(n)
        if config == "c1":
            run = lambda: R.observe_ad(sample, 7, cores)  # noqa: E731
        else:
            u = R.prior_draw(P.C2_PRIOR, 808, 0xBE9C4, 0)
            run = lambda: R.observe_ad_u(sample, P.C2_PRIOR, u, 808, cores)  # noqa: E731
        return per_particle * n, run, f"observe_ad, all {len(full.observations)} obs, {n} particles/obs " \
                                      f"(of {full.n_particles}), workers={cores}"
    if config in ("c4", "c5"):
        # one observation (the shortest time) of the evaluation, 1024 x cores particles
        if config == "c5":
            spec, prior = P.c5_base(1024 * cores), P.C5_PRIOR
            u = R.prior_draw(prior, 808, 0xBE9C4, 2)
        else:
            spec, prior = P.c4_base(1024 * cores), P.C4_PRIOR
            u = math.sqrt(1 - C4_BETA ** 2) * R.prior_draw(prior, 808, 0xBE9C4, 1) + \
                C4_BETA * R.prior_draw(prior, 4242, 0xFFFFFFFF, 0)
        j = int(np.argmin([t for t, _ in spec.observations]))
        spec.observations = [spec.observations[j]]
        per = int(math.ceil(spec.observations[0][0] / R.resolved_dt_ad(spec))) * spec.n_particles
        return per, lambda: R.observe_ad_u(spec, prior, u, 808, cores), \
            f"observe_ad on observation {j} only (t={spec.observations[0][0]:g}), {spec.n_particles} particles, " \
            f"workers={cores}" + (", proposal 0 of the batch" if config == "c4" else "")
    # c3: walker-steps of the sample from the reference's own simulate_to_exit
    full = P.c3()
    n = int(max(64, min(full.n_particles, 1024 * cores)))
    sample = P.c3(n)
    probe = 32
    mean_steps = float(np.mean([R.bvp_particle_values(full, j, 606, probe)[3].mean()
                                for j in range(len(full.observations))]))
    return mean_steps * n * len(full.observations), lambda: R.observe_bvp(sample, 606, cores), \
        f"observe_bvp with {n} walkers/obs (of {full.n_particles}), workers={cores}; walker-steps from " \
        f"{probe} walkers/obs via the reference's simulate_to_exit"


def cpu_reference_sample(config: str, budget_s: float = 4.0):
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


def loaded_native_libraries() -> list[str]:
    try:
        return sorted({ln.split()[-1] for ln in open("/proc/self/maps") if ln.rstrip().endswith(".so")
                       or ".so." in ln.split()[-1]})
    except OSError:
        return []


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
        else:  # plumbing test with fewer GPUs than ranks: host-staged exchange
            dist.init_process_group("gloo")
        ctx = D.rank_context(local)  # the library's multi-device context (NCCL inside)
    else:
        ctx = S.Context(local)
    red_dev = "cuda" if (world == 1 or args.dist_backend == "nccl") else "cpu"
    stream = torch.cuda.Stream(device=local)
    torch.cuda.set_stream(stream)
    S.load_library().smc_set_stream(ctx.handle, stream.cuda_stream)

    kind, payload, steps_per_eval = build_workload(args.config, ctx)
    F = FLOPS[args.config]
    desc = dict(CONFIGS[args.config])
    fp32 = args.precision == "fp32"
    if fp32:  # the optional FP32 variant (north_star: within 3 SE of the FP64 result)
        target = payload[0] if kind == "batched" else payload
        target.precision = S.Precision.fp32
        desc = dict(desc, workload=desc["workload"].replace("FP64", "FP32 variant"), precision="fp32")
    # the roofline denominator, measured on this GPU now; its clocks are
    # sampled the same way as the timed region's (roofline.peak_clocks)
    peak_sampler = ClockSampler(local)
    peak_sampler.start()
    time.sleep(0.3)
    peak = ctx.fp32_peak_tflops(300.0) if fp32 else ctx.fp64_peak_tflops(300.0)
    peak_clocks = peak_sampler.stop()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # > 126 MB L2

    if kind == "ad":
        spec = payload

        def evaluate():
            return S.observe_ad(spec, 808, ctx=ctx)
        h2d, d2h = _image_bytes(spec), 40 * len(spec.observations)
        api = "paper_1808_10580_b200.observe_ad -> smc_ad_observe (C ABI)"
        kernel_name = "ad_particles (K1)"
        shard = "particle chunks"
    elif kind == "bvp":
        spec = payload

        def evaluate():
            return S.observe_bvp(spec, 606, ctx=ctx)
        n_obs = len(spec.observations)
        h2d, d2h = 16 * n_obs + 512, 40 * n_obs
        api = "paper_1808_10580_b200.observe_bvp -> smc_bvp_observe (C ABI)"
        kernel_name = "bvp_walkers (K2)"
        shard = "walker ranges"
    else:
        base, prior, U = payload

        def evaluate():
            return S.observe_ad_batched(base, prior, U, 808, ctx=ctx)
        sb, se = D.sample_range(len(U), rank, world)
        h2d, d2h = U[sb:se].nbytes + 2048, 40 * len(base.observations) * len(U)
        api = "paper_1808_10580_b200.observe_ad_batched -> smc_ad_observe_batched (C ABI)"
        # FP64 K = 25 prior (C4): the compile-time tiled disk kernel; the FP32
        # variant keeps the generic tiled lattice kernel
        kernel_name = ("ad_particles<float> generic tiled lattice (K1)" if fp32
                       else "ad_particles_disk<25> tiled disk (K1)")
        shard = "parameter samples"
    if world > 1:
        g = ctx.group()
        parallel = f"{shard} sharded over {world} ranks ({'NCCL' if g['nccl'] else 'host-staged gloo'} exchange " \
                   f"inside the C ABI)"
    else:
        parallel = "single GPU"

    def device_step():
        """One evaluation timed with CUDA events on the forward map's stream:
        (event ms, this rank's particle-kernel ms, launches, this rank's
        particle-steps)."""
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        before = ctx.stats().total_launches
        t0.record(stream)
        evaluate()
        t1.record(stream)
        t1.synchronize()
        st = ctx.stats()
        return t0.elapsed_time(t1), st.particle_kernel_ms, st.total_launches - before, st.particle_steps

    for _ in range(args.warmup):
        device_step()

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    dev_ms = k_ms = 0.0
    launches = 0
    my_steps = 0.0
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
        my_steps += st
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # end to end through the public API (host inputs in, host estimates out)
    e2e_s = 0.0
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        evaluate()
        e2e_s += time.perf_counter() - t0
    torch.cuda.synchronize()
    clocks = sampler.stop()

    tmax = torch.tensor([dev_ms, e2e_s], dtype=torch.float64, device=red_dev)
    tsum = torch.tensor([my_steps], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
    dev_ms, e2e_s = tmax.tolist()
    total_steps = tsum.item()
    if steps_per_eval is not None:
        assert abs(total_steps - steps_per_eval * args.steps) < 1e-6 * total_steps, (total_steps, steps_per_eval)
    per_eval = total_steps / args.steps
    value = total_steps / (dev_ms / 1e3)
    e2e_value = total_steps / e2e_s
    # roofline: this rank's flops over its particle-kernel event time
    achieved = F * my_steps / (k_ms / 1e3) / 1e12
    traffic = _ncu_traffic(args.config + ("_fp32" if fp32 else ""))
    executed = None
    if traffic and traffic.get("executed_flops_per_unit"):
        ex = traffic["executed_flops_per_unit"] * my_steps / (k_ms / 1e3) / 1e12
        executed = {"achieved": ex, "frac": ex / peak, "flops_per_unit": traffic["executed_flops_per_unit"],
                    "source": traffic["source"] + " (ncu DFMA x2 + DADD + DMUL thread-instructions per unit)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "particle-steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32" if fp32 else "f64",
            "data": "synthetic (prior-draw velocity, reference recipe)", "config": desc,
            "parallelism": parallel, "l2": "flushed between steps (256 MiB write)",
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
                         "flops_note": "algorithmic flops = SURVEY.md 8(d) (the reference's 14 flops per mode); the "
                                       "kernels execute fewer (4 FMA per mode, Chebyshev harmonics), so frac can "
                                       "exceed 1 — `executed` is the hardware figure: the FP64 flops the kernel "
                                       "actually issues per particle-step (ncu) at the same rate",
                         "peak_clocks": peak_clocks,
                         "executed": executed,
                         # dram bytes per launch of the dominant kernel (ncu --set full capture), or null
                         "traffic": None if not traffic else traffic.get("dram_bytes_per_launch"),
                         "traffic_detail": traffic},
            "gpu_launches": launches,
            "clocks": clocks,
        }
        if world == 1 and not args.no_cpu_baseline:
            try:
                v, cores, sample = cpu_reference_sample(args.config)
                line["cpu_baseline"] = {"value": v, "unit": "particle-steps/s", "cores": cores, "kind": "reference",
                                        "sample": sample}
            except Exception as e:  # noqa: BLE001
                line["cpu_baseline"] = {"value": None, "unavailable": f"{type(e).__name__}: {e}"}
        print(json.dumps(line), flush=True)
    ctx.close()
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
    """DRAM bytes per particle-kernel launch, the dominant pipe's active
    fraction and the executed FP64 flops per unit from the committed ncu
    --set full capture of this config (profiles/rNN_k*_<config>[_reduced].json)."""
    caps = sorted(PROFILES.glob(f"r*_k*_{config}.json")) or sorted(PROFILES.glob(f"r*_k*_{config}_reduced.json"))
    if not caps:
        return None
    try:
        d = json.loads(caps[-1].read_text())
        fp32 = config.endswith("_fp32")
        pipe = d.get("fma_pipe_pct_active" if fp32 else "fp64_pipe_pct_active")
        return {"dram_bytes_per_launch": d.get("dram_bytes_per_launch"), "source": f"profiles/{caps[-1].name}",
                "pipe": "fma (FP32)" if fp32 else "fp64",
                "pipe_active_frac": None if pipe is None else round(pipe / 100.0, 4),
                "executed_flops_per_unit": d.get("executed_fp32_flops_per_unit" if fp32 else "executed_fp64_flops_per_unit"),
                "reduced_launch": caps[-1].name.endswith("_reduced.json")}
    except Exception:  # noqa: BLE001
        return None


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------
def run_reference(args):
    """The reference's own CPU implementation (oracle/_ref) on all host cores,
    same config/metric/unit as our arm; each step a bounded sample.  Nothing
    of the product (paper_1808_10580_b200, libscalarmc_b200.so) is imported or
    loaded in this process."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    from oracle import pods as P
    from oracle.oracle import Reference
    R = Reference()
    cores = os.cpu_count() or 1
    steps, run, sample = reference_runner(args.config, R, cores, budget_s=4.0)
    for _ in range(args.warmup):
        run()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        run()
    el = time.perf_counter() - t0
    native = loaded_native_libraries()
    leaked = [m for m in sys.modules if m.startswith("paper_1808_10580_b200")] + \
        [p for p in native if "libscalarmc_b200" in p]
    if leaked:
        raise SystemExit(f"reference arm loaded product code: {leaked}")
    value = steps * args.steps / el
    if args.config == "c3":
        full = P.c3()
        per_eval = steps / P.c3(int(max(64, min(full.n_particles, 1024 * cores)))).n_particles * full.n_particles
    elif args.config == "c4":
        per_eval = sum(int(math.ceil(t / 1e-3)) for t, _ in P.c4_base().observations) * 1024 * C4_BATCH
    elif args.config == "c5":
        per_eval = sum(int(math.ceil(t / 5e-4)) for t, _ in P.c5_base().observations) * 32768
    else:
        full = P.c1() if args.config == "c1" else P.c2_base()
        per_eval = sum(int(math.ceil(t / R.resolved_dt_ad(full))) for t, _ in full.observations) * full.n_particles
    line = {"metric": METRIC, "impl": "reference", "value": value, "unit": "particle-steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (prior-draw velocity, reference recipe)", "config": dict(CONFIGS[args.config]),
            "parallelism": f"std::thread x{cores} (reference executor)",
            "evals_per_sec": value / per_eval,
            "cpu_baseline": {"value": value, "unit": "particle-steps/s", "cores": cores, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": value, "unit": "particle-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "native_libraries": [p for p in native if "/oracle/" in p]}
    print(json.dumps(line), flush=True)


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="fp64", choices=["fp64", "fp32"],
                    help="fp32 = the optional FP32 variant of the kernels (our arm only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: test the multi-rank path with fewer GPUs than ranks (host-staged exchange)")
    ap.add_argument("--device", type=int, default=-1, help="override LOCAL_RANK -> device (plumbing tests)")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-execute under torch.distributed.run
        env = dict(os.environ, MASTER_ADDR="127.0.0.1")
        if args.dist_backend == "nccl":
            env.setdefault("NCCL_DEBUG", "INFO")  # NCCL's init lines (transport, NVLS) stay visible on stderr
            env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(Path(__file__).resolve()),
               *sys.argv[1:]]
        raise SystemExit(subprocess.run(cmd, env=env).returncode)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
