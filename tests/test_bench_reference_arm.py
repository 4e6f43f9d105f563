"""bench.py --impl reference (CPU, no GPU needed): the reference's own CPU
path (oracle/_ref, compiled from the reference's sources) timed on this
host's cores, printing the contract's JSON line with impl = "reference"."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("config", ["c1", "c2", "c3", "c4", "c5"])
def test_reference_arm_line(config):
    """Every config runs on the reference with no product code in the process
    (bench.py exits non-zero if paper_1808_10580_b200 was imported or
    libscalarmc_b200.so mapped), with the same config dict as our arm."""
    if not (ROOT / "oracle" / "_ref").exists():
        pytest.skip("oracle/_ref not built (build() compiles it where /root/reference is present)")
    steps = "3" if config == "c1" else "1"
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", config, "--steps", steps,
                        "--warmup", "1"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "particle-steps/s"
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    sys.path.insert(0, str(ROOT))
    import bench
    assert d["config"] == bench.CONFIGS[config]
    assert d["native_libraries"] and all("/oracle/" in p for p in d["native_libraries"])
    assert not any("libscalarmc_b200" in p for p in d["native_libraries"])
