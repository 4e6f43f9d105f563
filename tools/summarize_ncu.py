"""Summarise ncu outputs into profiles/ (committed evidence).

    python tools/summarize_ncu.py launches gpurun_out/launches.csv profiles/r01_launches.md
    python tools/summarize_ncu.py full gpurun_out/k1_c2_full.ncu-rep profiles/r01_k1_c2 [--units N]

`launches` turns the `--metrics gpu__time_duration.sum` launch list into a
per-kernel table (count, total, share of device time).  `full` extracts the
key metrics of a `--set full` capture (duration, FP64 pipe, issue, occupancy,
registers, DRAM bytes, instruction mix, stall reasons) into <out>.json and
<out>.md; the JSON's dram_bytes_per_launch is what bench.py reports as
roofline.traffic.
"""
from __future__ import annotations

import collections
import csv
import json
import subprocess
import sys
from pathlib import Path


def launches(src: Path, out: Path) -> None:
    rows = [r for r in csv.reader(l for l in src.read_text().splitlines() if l.startswith('"'))]
    hdr, data = rows[0], rows[1:]
    iN, iV = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in data:
        name = r[iN].split("(")[0]
        tot[name] += float(r[iV].replace(",", "")) / 1e6
        cnt[name] += 1
    total = sum(tot.values())
    lines = [f"# Launch list: `{src.name}` (ncu --metrics gpu__time_duration.sum --clock-control none)", "",
             "Cold-cache, serialised per-launch times; compare shares, not absolutes.", "",
             "| kernel | launches | total ms | share |", "|---|---:|---:|---:|"]
    for name, t in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"| `{name}` | {cnt[name]} | {t:.3f} | {100 * t / total:.1f}% |")
    lines.append(f"| **all** | {sum(cnt.values())} | {total:.3f} | 100% |")
    out.write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


WANT = {
    "gpu__time_duration.sum": "duration",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_inst_pct_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pipe_pct_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pipe_pct_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid_size",
    "launch__block_size": "block_size",
    "dram__bytes_read.sum": "dram_bytes_read",
    "dram__bytes_write.sum": "dram_bytes_write",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__cycles_elapsed.avg": "sm_cycles_elapsed",
    "smsp__cycles_active.avg": "smsp_cycles_active",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum": "thread_dfma",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum": "thread_dadd",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum": "thread_dmul",
    "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum": "thread_ffma",
    "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum": "thread_fadd",
    "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum": "thread_fmul",
    "smsp__thread_inst_executed.sum": "thread_instructions",
}


def _num(v: str) -> float:
    return float(v.replace(",", ""))


def full(rep: Path, out: Path, units: float | None) -> None:
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, unit_row, vals = rows[0], rows[1], rows[2]
    res: dict = {"report": rep.name, "kernel": vals[hdr.index("Kernel Name")]}
    for k, name in WANT.items():
        if k in hdr:
            i = hdr.index(k)
            res[name] = _num(vals[i]) if vals[i] else None
            res[name + "_unit"] = unit_row[i]
    # normalise units
    def to_bytes(v, u):
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    dr = to_bytes(res.get("dram_bytes_read", 0) or 0, res.get("dram_bytes_read_unit", "byte"))
    dw = to_bytes(res.get("dram_bytes_write", 0) or 0, res.get("dram_bytes_write_unit", "byte"))
    res["dram_bytes_per_launch"] = dr + dw
    dur = res.get("duration")
    if dur is not None and res.get("duration_unit") == "ms":
        res["duration_ms"] = dur
    elif dur is not None:
        res["duration_ms"] = dur / {"ns": 1e6, "us": 1e3, "msecond": 1, "s": 1e-3}.get(res.get("duration_unit"), 1e6)
    stalls = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
            try:
                stalls.append((_num(vals[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in stalls) or 1.0
    res["stall_samples_pct"] = {n: round(100 * v / tot, 1) for v, n in sorted(stalls, reverse=True)[:8]}
    if units:
        res["units_per_launch"] = units
        res["dram_bytes_per_unit"] = res["dram_bytes_per_launch"] / units
        # the FP64 (FP32) flops the kernel actually executes per unit: 2 per
        # FMA, 1 per add / mul thread-instruction (predicated-on)
        if res.get("thread_dfma") is not None:
            res["executed_fp64_flops_per_unit"] = (2 * res["thread_dfma"] + (res.get("thread_dadd") or 0) +
                                                   (res.get("thread_dmul") or 0)) / units
        if res.get("thread_ffma") is not None:
            res["executed_fp32_flops_per_unit"] = (2 * res["thread_ffma"] + (res.get("thread_fadd") or 0) +
                                                   (res.get("thread_fmul") or 0)) / units
        if res.get("thread_instructions") is not None:
            res["thread_instructions_per_unit"] = res["thread_instructions"] / units
    out.with_suffix(".json").write_text(json.dumps(res, indent=1) + "\n")
    md = [f"# ncu --set full: {res['kernel'][:120]}", "", f"report `{rep.name}`", "", "| metric | value |", "|---|---|"]
    for k, v in res.items():
        if k.endswith("_unit") or k in ("kernel", "report"):
            continue
        md.append(f"| {k} | {v} {res.get(k + '_unit', '')} |")
    out.with_suffix(".md").write_text("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    mode, src, dst = sys.argv[1], Path(sys.argv[2]), Path(sys.argv[3])
    if mode == "launches":
        launches(src, dst)
    else:
        u = float(sys.argv[sys.argv.index("--units") + 1]) if "--units" in sys.argv else None
        full(src, dst, u)
