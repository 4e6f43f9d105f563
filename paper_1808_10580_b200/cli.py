"""Command-line front end with the reference CLI's commands, options, output
files and exit codes (src/cli.cpp:1-306; tools/main.cpp), running the
forward maps and the callers above them on the B200 path.

    python -m paper_1808_10580_b200.cli forward-ad  --config C --out F [--seed S] [--workers W] [--format csv|jsonl]
    python -m paper_1808_10580_b200.cli forward-bvp --config C --out F ...
    python -m paper_1808_10580_b200.cli sample      --config C --out DIR [--steps N] [--beta B] ...
    python -m paper_1808_10580_b200.cli optimize    --config C --out F ...

Exit codes: 0 ok, 2 ConfigError ("config error: ..."), 1 any other error
("error: ..."), argument errors as the parser reports them (2).
`reference --method galerkin` runs the device spectral solver; `reference
--method fd` (finite-difference Dirichlet solver) and `benchmark` (the CPU
cost-scaling harness) are not part of what this repository rebuilds
(SURVEY.md §8, §2): they exit 1 with an explanation.  `--workers` /
SCALARMC_WORKERS are resolved and validated as in the reference
(cli.cpp:40-50) and otherwise ignored: the device is the worker pool.
"""
from __future__ import annotations

import argparse
import os
import sys
from pathlib import Path

from . import api as S
from .config import ConfigError, McmcSection, load_config, make_ad_spec, make_bvp_spec, make_forcing_control, \
    make_likelihood
from .records import RecordWriter, format_double, parse_record_format


def _effective_workers(opts, cfg) -> int:
    """cli.cpp:40-50 precedence (flag, SCALARMC_WORKERS, config)."""
    if opts.workers >= 0:
        return opts.workers
    env = os.environ.get("SCALARMC_WORKERS")
    if env is not None:
        try:
            return int(env)
        except ValueError:
            raise ConfigError("SCALARMC_WORKERS", "not an integer") from None
    return cfg.workers


def _effective_seed(opts, cfg) -> int:
    return opts.seed if opts.seed >= 0 else cfg.seed


def _open_output(path: str):
    parent = Path(path).parent
    if str(parent) not in ("", "."):
        parent.mkdir(parents=True, exist_ok=True)
    try:
        return open(path, "w", encoding="utf-8", newline="")
    except OSError:
        raise RuntimeError("cannot open output file: " + path) from None


def cmd_forward_ad(opts) -> int:
    """cli.cpp:63-78."""
    cfg = load_config(opts.config)
    spec = make_ad_spec(cfg)
    seed, _ = _effective_seed(opts, cfg), _effective_workers(opts, cfg)
    est = S.observe_ad(spec, seed)
    with _open_output(opts.out) as out:
        w = RecordWriter(out, opts.format, ["t", "x1", "x2", "mean", "std_error", "n_particles", "n_failed"])
        for o, e in zip(spec.observations, est):
            w.write_row([o.t, o.x[0], o.x[1], e.mean, e.std_error, float(e.n_particles), float(e.n_failed)])
    return 0


def cmd_forward_bvp(opts) -> int:
    """cli.cpp:80-96."""
    cfg = load_config(opts.config)
    spec = make_bvp_spec(cfg)
    seed, _ = _effective_seed(opts, cfg), _effective_workers(opts, cfg)
    est = S.observe_bvp(spec, seed)
    with _open_output(opts.out) as out:
        w = RecordWriter(out, opts.format, ["x1", "x2", "mean", "std_error", "mean_exit_time", "n_failed"])
        for x, e in zip(spec.observations, est):
            w.write_row([x[0], x[1], e.mean, e.std_error, e.aux_mean, float(e.n_failed)])
    return 0


def cmd_sample(opts) -> int:
    """cli.cpp:140-199: one pCN chain (the device multi-chain driver with one
    chain is the reference's run_chain for that seed)."""
    cfg = load_config(opts.config)
    if cfg.prior is None:
        raise ConfigError("prior", "section required by `sample`")
    prior = cfg.prior
    likelihood = make_likelihood(cfg)
    likelihood.workers = _effective_workers(opts, cfg)
    mc = cfg.mcmc or McmcSection()
    if opts.steps >= 0:
        mc.steps = opts.steps
    if opts.beta > 0.0:
        mc.beta = opts.beta
    chain = S.ChainConfig(n_steps=mc.steps, beta=mc.beta, burn_in=mc.burn_in, thin=mc.thin,
                          seed=_effective_seed(opts, cfg))
    res = S.run_chains(chain, prior, likelihood, [chain.seed])
    samples = res["samples"][0] if res["samples"] is not None else []
    phi_trace = res["phi_trace"][0]
    Path(opts.out).mkdir(parents=True, exist_ok=True)
    dim = prior.dimension()
    ucols = [f"u{c}" for c in range(dim)]
    with _open_output(f"{opts.out}/archive.{opts.format}") as out:
        w = RecordWriter(out, opts.format, ["iteration", "phi"] + ucols)
        for s, u in enumerate(samples):
            it = chain.burn_in + s * chain.thin + 1
            w.write_row([float(it), phi_trace[it - 1]] + list(u))
    with _open_output(f"{opts.out}/map.{opts.format}") as out:
        RecordWriter(out, opts.format, ucols).write_row(list(res["map_u"][0]))
    acceptance = float(res["acceptance_rate"][0])
    with _open_output(f"{opts.out}/summary.{opts.format}") as out:
        w = RecordWriter(out, opts.format, ["steps", "acceptance_rate", "map_objective", "final_phi",
                                            "flagged_failures", "samples"])
        # an AD forward map cannot fail (no exit condition), so no step is ever flagged
        w.write_row([float(mc.steps), acceptance, float(res["map_objective"][0]), float(res["final_phi"][0]), 0.0,
                     float(len(samples))])
    print(f"acceptance_rate {format_double(acceptance)}")
    print(f"map_objective {format_double(float(res['map_objective'][0]))}")
    print(f"samples {len(samples)}")
    return 0


def cmd_optimize(opts) -> int:
    """cli.cpp:201-228."""
    cfg = load_config(opts.config)
    base = make_bvp_spec(cfg)
    control = make_forcing_control(cfg)
    seed, _ = _effective_seed(opts, cfg), _effective_workers(opts, cfg)
    res = S.optimize_forcing(control, base, cfg.optimize.options, seed)
    cols = ["iteration", "best_cost"] + [f"f{c}" for c in range(len(control.centers))]
    with _open_output(opts.out) as out:
        w = RecordWriter(out, opts.format, cols)
        for it, best, point in res["trace"]:
            w.write_row([float(it), best] + list(point))
    print(f"best_cost {format_double(res['min_value'])}")
    print(f"iterations {res['iterations']} ({res['stop_reason']})")
    print("amplitudes" + "".join(" " + format_double(f) for f in res["argmin"]))
    return 0


def cmd_reference(opts) -> int:
    """cli.cpp:98-138, `--method galerkin` (the spectral reference solver on
    the device; `fd` — the finite-difference Dirichlet solver — is not
    rebuilt here)."""
    cfg = load_config(opts.config)
    from .config import ReferenceSection
    ref = cfg.reference or ReferenceSection()
    with _open_output(opts.out) as out:
        grid_writer = RecordWriter(out, opts.format, ["x1", "x2", "value"])
        obs_writer = RecordWriter(sys.stdout, opts.format, ["obs", "x1", "x2", "value"])
        if opts.method == "galerkin":
            spec = make_ad_spec(cfg)
            dt_ref = ref.dt_ref if ref.dt_ref > 0.0 else spec.resolved_dt() / 10.0
            result = S.galerkin_solve_ad(spec, ref.galerkin_cutoff, dt_ref)
            n = ref.field_grid
            field = S.galerkin_field_grid(result, n)
            for i in range(n):
                for j in range(n):
                    grid_writer.write_row([i / n, j / n, field[i * n + j]])
            for j, v in enumerate(result.observation_values):
                o = spec.observations[j]
                obs_writer.write_row([float(j), o.x[0], o.x[1], v])
            return 0
        raise RuntimeError("`reference --method fd` (finite-difference Dirichlet solver) is not part of the B200 "
                           "path; it stays in scalarmc")


def _not_on_path(name: str):
    def run(opts) -> int:
        raise RuntimeError(f"`{name}` is not part of the B200 forward-map path (the Galerkin/FD reference solvers "
                           "and the CPU cost-scaling harness stay in scalarmc)")
    return run


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="scalarmc-b200",
                                 description="Backward-particle evaluation of sparse advection-diffusion "
                                             "observations (B200 path)")
    sub = ap.add_subparsers(dest="command", required=True)

    def common(p, needs_out=True):
        p.add_argument("--config", required=True, help="run configuration file (JSON)")
        p.add_argument("--out", required=needs_out, default="", help="output file")
        p.add_argument("--seed", type=int, default=-1, help="seed override")
        p.add_argument("--workers", type=int, default=-1, help="worker thread count (0 = hardware)")
        p.add_argument("--format", default="csv", choices=["csv", "jsonl"], help="record format: csv or jsonl")
        return p

    common(sub.add_parser("forward-ad", help="particle forward map, time-dependent problem")).set_defaults(
        run=cmd_forward_ad)
    common(sub.add_parser("forward-bvp", help="particle forward map, Dirichlet problem")).set_defaults(
        run=cmd_forward_bvp)
    ref = common(sub.add_parser("reference", help="reference solver (full field + observations)"))
    ref.add_argument("--method", required=True, choices=["galerkin", "fd"])
    ref.set_defaults(run=cmd_reference)
    smp = common(sub.add_parser("sample", help="pCN MCMC sampling of the posterior"))
    smp.add_argument("--steps", type=int, default=-1, help="chain length override")
    smp.add_argument("--beta", type=float, default=-1.0, help="pCN step size override")
    smp.set_defaults(run=cmd_sample)
    common(sub.add_parser("optimize", help="Nelder-Mead forcing optimization")).set_defaults(run=cmd_optimize)
    common(sub.add_parser("benchmark", help="particle vs reference cost scaling")).set_defaults(
        run=_not_on_path("benchmark"))
    return ap


def main(argv=None) -> int:
    opts = build_parser().parse_args(argv)
    parse_record_format(opts.format)
    try:
        return opts.run(opts)
    except ConfigError as e:
        print(f"config error: {e}", file=sys.stderr)
        return 2
    except Exception as e:  # cli.cpp:296-302
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
