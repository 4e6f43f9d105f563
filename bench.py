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
the same workload on all host cores instead.
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


def build_workload(name: str, ctx):
    import paper_1808_10580_b200 as S
    import specs
    if name == "c2":
        u = S.prior_draw(specs.C2_PRIOR, 808, 0xBE9C4, 0, ctx)  # benchmark.cpp:69-71 recipe
        spec = specs.c2_spec(u, n_particles=100_000)
        K, M = 8, len(specs.C2_PRIOR.modes())
        desc = {"workload": "C2: AD forward map, K=8 Fourier velocity (M=98, N_u=197), 9 obs, 1e5 particles/obs, "
                            "1000 EM steps, FP64", "K": K, "modes": M, "n_obs": 9, "particles_per_obs": 100_000,
                "em_steps": 1000, "seed": 808}
    elif name == "c1":
        spec = specs.c1_two_mode(n_particles=10_000)
        K, M = 1, 2
        desc = {"workload": "C1: shipped forward_ad_two_mode.json (K=1, M=2, 3 obs, 1e4 particles)", "K": K,
                "modes": M, "n_obs": 3, "particles_per_obs": 10_000, "seed": 7}
    elif name == "c5":
        prior = S.PriorSpec(80, 1.0, 2.5)
        u = S.prior_draw(prior, 808, 0xBE9C4, 2, ctx)
        rng = np.random.default_rng(5)
        terms = []
        for k1 in range(-8, 9):
            for k2 in range(-8, 9):
                if len(terms) < 100 and 0 < k1 * k1 + k2 * k2 <= 64:
                    terms.append((float(rng.normal()) / (k1 * k1 + k2 * k2), (2 * math.pi * k1, 2 * math.pi * k2),
                                  float(rng.random() * 2 * math.pi)))
        obs = [S.AdObservation(t / 16.0, S.Vec2(j / 8.0, j / 8.0)) for j in range(8) for t in range(1, 9)]
        spec = S.AdProblemSpec(velocity=S.VelocityField.fourier(S.velocity_from_coefficients(prior, u)),
                               diffusion=S.DiffusionModel.isotropic(3e-5),
                               initial_condition=S.ScalarField.cosine_series(terms), observations=obs, dt=5e-4,
                               n_particles=32768)
        K, M = 80, len(prior.modes())
        desc = {"workload": "C5: AD forward map, K=80 (M=10040), 64 obs, 32768 particles/obs, FP64", "K": K,
                "modes": M, "n_obs": 64, "particles_per_obs": 32768, "seed": 808}
    else:
        raise SystemExit(f"unknown config {name}")
    dt = spec.resolved_dt()
    steps = sum(int(math.ceil(o.t / dt)) for o in spec.observations) * spec.n_particles
    return spec, steps, flops_ad(K, M), desc


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
def cpu_reference_sample(spec, steps_per_eval: int, budget_s: float = 20.0):
    """Time the reference observe_ad (workers = all host cores) on a bounded
    sample of the workload: same spec, fewer particles per observation.
    1 warm-up + median of 3 (benchmark.cpp:39-52 methodology)."""
    import copy
    from oracle.oracle import Reference
    R = Reference()
    cores = os.cpu_count() or 1
    sample = copy.copy(spec)
    per_particle = steps_per_eval / spec.n_particles
    # size so one run is ~budget/5 s at ~1.5e6 particle-steps/s/core (K=8 rate)
    n = int(max(64, min(spec.n_particles, (budget_s / 5.0) * 1.5e6 * cores / per_particle)))
    sample.n_particles = n
    sample.precision = spec.precision
    R.observe_ad(sample, 808, cores)  # warm-up
    times = []
    for _ in range(3):
        t0 = time.perf_counter()
        R.observe_ad(sample, 808, cores)
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    return (per_particle * n) / t, cores, f"observe_ad with {n} particles/obs (of {spec.n_particles}), " \
                                          f"median of 3 after 1 warm-up, workers={cores}"


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
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = S.default_context(local)
    stream = torch.cuda.Stream(device=local)
    torch.cuda.set_stream(stream)
    S.load_library().smc_set_stream(ctx.handle, stream.cuda_stream)

    spec, steps_per_eval, F, desc = build_workload(args.config, ctx)
    peak = ctx.fp64_peak_tflops(300.0)

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # > 126 MB L2

    def device_step():
        """One evaluation through the device-level (sharded) path: inputs
        resident, returns (kernel_ms, launches)."""
        ops = D.DeviceOps(spec, 808, ctx)
        n_chunks = D.num_chunks(spec.n_particles)
        b, e = D.chunk_range(n_chunks, rank, world)
        counts = [D.chunk_range(n_chunks, r, world)[1] - D.chunk_range(n_chunks, r, world)[0] for r in range(world)]
        before = ctx.stats().total_launches
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        parts = ops.partials(b, e)
        k_ms = ctx.stats().particle_kernel_ms
        full = ops.all_gather(parts, counts)
        sums = ops.finish(full)
        means = ops.divide(sums, spec.n_particles)
        fullsq = ops.all_gather(ops.sq_partials(means, b, e), counts)
        ops.finish(fullsq)
        t1.record(stream)
        t1.synchronize()
        return t0.elapsed_time(t1), k_ms, ctx.stats().total_launches - before

    def e2e_step():
        if world == 1:
            return S.observe_ad(spec, 808, ctx=ctx)
        return D.observe_ad_sharded(spec, 808, rank, world, ctx)

    for _ in range(args.warmup):
        device_step()
        e2e_step()

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    dev_ms = k_ms = 0.0
    launches = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for _ in range(args.steps):
        flush.zero_()  # L2 flush between timed iterations (outside the step's events)
        torch.cuda.synchronize()
        d, k, n = device_step()
        dev_ms += d
        k_ms += k
        launches += n
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # end-to-end through the public API (host spec in, host estimates out)
    e2e_s = 0.0
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        est = e2e_step()
        e2e_s += time.perf_counter() - t0
    torch.cuda.synchronize()
    clocks = sampler.stop()

    t = torch.tensor([dev_ms, k_ms, e2e_s], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_ms, k_ms, e2e_s = t.tolist()

    total_steps = steps_per_eval * args.steps
    value = total_steps / (dev_ms / 1e3)
    e2e_value = total_steps / e2e_s
    local_steps_per_eval = steps_per_eval * (D.chunk_range(D.num_chunks(spec.n_particles), rank, world)[1] -
                                             D.chunk_range(D.num_chunks(spec.n_particles), rank, world)[0]) / max(
        1, D.num_chunks(spec.n_particles))
    achieved = F * local_steps_per_eval * args.steps / (k_ms / 1e3) / 1e12  # per-launch algorithmic flops / duration
    h2d = _image_bytes(spec)
    d2h = 40 * len(spec.observations)

    if rank == 0:
        traffic = _ncu_traffic()
        line = {
            "metric": METRIC, "value": value, "unit": "particle-steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (prior-draw velocity, reference recipe)",
            "config": dict(desc, parallelism=f"particle-shard x{world}" if world > 1 else "single GPU",
                           l2="flushed between steps (256 MiB write)"),
            "evals_per_sec": value / steps_per_eval,
            "e2e": {"value": e2e_value, "unit": "particle-steps/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "evals_per_sec": e2e_value / steps_per_eval,
                    "api": "paper_1808_10580_b200.observe_ad -> smc_ad_observe (C ABI)" if world == 1 else
                           "paper_1808_10580_b200.distributed.observe_ad_sharded"},
            "roofline": {"bound": "fp64", "kernel": "ad_particles<double> (K1)", "achieved": achieved,
                         "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                         "peak_source": "FP64 DFMA microbenchmark measured in this run (smc_fp64_peak, all SMs, "
                                        "8 chains/thread); MEASURED_PEAKS.json has no FP64 entry",
                         "flops_per_unit": F, "unit_of_work": "particle-step",
                         "traffic": traffic},
            "gpu_launches": launches,
            "clocks": clocks,
        }
        if world == 1 and not args.no_cpu_baseline:
            try:
                v, cores, sample = cpu_reference_sample(spec, steps_per_eval)
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


def _ncu_traffic():
    """DRAM bytes per K1 launch from the committed ncu --set full capture."""
    caps = sorted(PROFILES.glob("r*_k1_c2.json"))
    if caps:
        try:
            d = json.loads(caps[-1].read_text())
            return {"dram_bytes_per_launch": d.get("dram_bytes_per_launch"), "source": f"profiles/{caps[-1].name}"}
        except Exception:  # noqa: BLE001
            return None
    return None


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import copy

    import paper_1808_10580_b200 as S
    import specs
    from oracle.oracle import Reference

    R = Reference()
    cores = os.cpu_count() or 1
    # same workload as ours; the reference's input recipe, with the reference's
    # own prior_draw (inference.cpp:55-61) so no GPU is needed on this arm
    if args.config == "c2":
        u = R.prior_draw(specs.C2_PRIOR, 808, 0xBE9C4, 0)
        spec = specs.c2_spec(u, n_particles=100_000)
        desc = {"workload": "C2: AD forward map, K=8 Fourier velocity (M=98, N_u=197), 9 obs, 1e5 particles/obs, "
                            "1000 EM steps, FP64", "K": 8, "modes": 98, "n_obs": 9, "particles_per_obs": 100_000,
                "em_steps": 1000, "seed": 808}
    else:
        spec = specs.c1_two_mode()
        desc = {"workload": "C1: shipped forward_ad_two_mode.json", "K": 1, "modes": 2}
    steps_per_eval = sum(int(math.ceil(o.t / spec.dt)) for o in spec.observations) * spec.n_particles
    per_particle = steps_per_eval // spec.n_particles
    sample = copy.copy(spec)
    n = int(max(64, min(spec.n_particles, 4.0 * 1.5e6 * cores / per_particle)))  # ~4 s per step
    sample.n_particles = n
    for _ in range(args.warmup):
        R.observe_ad(sample, 808, cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        R.observe_ad(sample, 808, cores)
    el = time.perf_counter() - t0
    value = per_particle * n * args.steps / el
    line = {"metric": METRIC, "impl": "reference", "value": value, "unit": "particle-steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (prior-draw velocity, reference recipe)",
            "config": dict(desc, parallelism=f"std::thread x{cores} (reference executor)"),
            "evals_per_sec": value / steps_per_eval,
            "cpu_baseline": {"value": value, "unit": "particle-steps/s", "cores": cores, "kind": "reference",
                             "sample": f"observe_ad with {n} particles/obs (of {spec.n_particles}) per step, "
                                       f"workers={cores}"},
            "e2e": {"value": value, "unit": "particle-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
