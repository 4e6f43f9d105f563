"""SASS opcode summary of the hot kernels (committed evidence, profiles/):
per kernel the instruction count of the function, its FP64 / integer /
load mix, DFMAs with a uniform-register operand (coefficients from the
constant bank), spills (ptxas) and registers.

    python tools/sass_summary.py > profiles/r02_sass_summary.md
"""
from __future__ import annotations

import collections
import re
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OBJ = ROOT / "paper_1808_10580_b200" / "lib" / "obj"

# (label, object, mangled-name regex)
KERNELS = [
    ("K1 disk, parameter coefficients, K=8 FP64 (C2)", "ad_disk", r"ad_particles_disk_paramILi8EdLi5E"),
    ("K1 tiled disk, shared memory, K=25 FP64 batched (C4)", "ad_disk", r"17ad_particles_diskILi25EdLi1ELi4E"),
    ("K1 generic tiled lattice, 512 threads FP64 (C5)", "ad_kernels", r"ad_particlesIdLb1ELi512ELb0ELb0E"),
    ("K1 disk, packed FFMA2, K=8 FP32 (C2 FP32)", "ad_disk", r"ad_particles_disk_paramILi8EfLi4E"),
    ("K2 walkers, 3 bumps, constant velocity, box FP64 (C3)", "bvp_kernels", r"bvp_walkersIdLb0ELi0ELi3ELi1ELb0ELi0ELi1E"),
    ("K3 tree pass", "reduce_kernels", r"tree_pass"),
]


def functions(obj: Path) -> dict[str, str]:
    out = subprocess.run(["cuobjdump", "-sass", str(obj)], capture_output=True, text=True).stdout
    funcs, cur, buf = {}, None, []
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if cur:
                funcs[cur] = "\n".join(buf)
            cur, buf = m.group(1), []
        elif cur:
            buf.append(line)
    if cur:
        funcs[cur] = "\n".join(buf)
    return funcs


def ptxas(obj: str, name: str) -> tuple[str, str]:
    log = (OBJ / f"{obj}.ptxas.log").read_text().splitlines()
    for i, l in enumerate(log):
        if name in l and "Compiling entry" in l:
            spill = next((x for x in log[i + 1:i + 4] if "spill" in x), "")
            regs = next((x for x in log[i + 1:i + 5] if "registers" in x), "")
            s = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", spill)
            r = re.search(r"Used (\d+) registers", regs)
            return (f"{s.group(1)}/{s.group(2)} B" if s else "?", r.group(1) if r else "?")
    return "?", "?"


def main() -> None:
    rows = ["# SASS opcode summary (sm_100a, `cuobjdump -sass` of the in-tree build)", "",
            "Whole-function static counts (prologue, step loop and epilogue together); "
            "`DFMA.UR` = DFMAs taking an operand from a uniform register (constant-bank "
            "coefficients); spills = ptxas spill stores/loads.", "",
            "| kernel | instructions | DFMA | DFMA.UR | DMUL+DADD | FFMA/FFMA2 | IMAD+LOP3 | LDS | LDCU/LDC | LDG | registers | spills |",
            "|---|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|---|"]
    cache: dict[str, dict[str, str]] = {}
    for label, obj, pat in KERNELS:
        funcs = cache.setdefault(obj, functions(OBJ / f"{obj}.o"))
        name = next((n for n in funcs if re.search(pat, n)), None)
        if not name:
            rows.append(f"| {label} | (not found) |")
            continue
        ins = [l for l in funcs[name].splitlines() if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l)]
        ops = collections.Counter()
        dfma_ur = 0
        for l in ins:
            m = re.search(r"\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", l)
            if not m:
                continue
            op = m.group(1)
            base = op.split(".")[0]
            ops[base] += 1
            if base == "DFMA" and re.search(r"\bUR\d+", l):
                dfma_ur += 1
        spills, regs = ptxas(obj, name)
        rows.append(f"| {label} | {len(ins)} | {ops['DFMA']} | {dfma_ur} | {ops['DMUL'] + ops['DADD']} | "
                    f"{ops['FFMA'] + ops['FFMA2']} | {ops['IMAD'] + ops['LOP3']} | {ops['LDS']} | "
                    f"{ops['LDCU'] + ops['LDC']} | {ops['LDG']} | {regs} | {spills} |")
    print("\n".join(rows))


if __name__ == "__main__":
    main()
