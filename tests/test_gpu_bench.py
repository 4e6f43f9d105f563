"""bench.py's contract on the GPU: the N=1 JSON line (keys, units, a live
roofline and clocks) and the N>1 code path under torchrun (2 ranks sharing
the one GPU through a gloo group — plumbing only: the driver's scaling run
uses one GPU per rank over NCCL)."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu

KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "e2e", "roofline", "gpu_launches", "clocks"}


def _last_json(out: str) -> dict:
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


def test_bench_single_gpu_line():
    r = subprocess.run([sys.executable, "bench.py", "--config", "c1", "--steps", "3", "--warmup", "3",
                        "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    assert KEYS <= set(d)
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["unit"] == "particle-steps/s"
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert 0 < d["roofline"]["achieved"] and d["roofline"]["peak"] > 20  # FP64 DFMA peak measured in the run
    assert d["gpu_launches"] > 0


@pytest.mark.parametrize("config,shard", [("c1", "particle chunks"), ("c3", "walker ranges"),
                                          ("c4", "parameter samples")])
def test_bench_two_ranks_self_launch(config, shard):
    """`bench.py --gpus 2` launches its own two ranks (torch.distributed.run);
    with --dist-backend gloo --device 0 both share the one GPU and the library
    stages its exchange through torch.distributed (NCCL refuses two ranks on
    one GPU) — the plumbing of the driver's 1/2/4/8-GPU runs, which use one
    GPU per rank over NCCL."""
    args = ["--config", config, "--steps", "2", "--warmup", "3"]
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", *args, "--dist-backend", "gloo", "--device", "0"],
                       cwd=ROOT, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _last_json(r.stdout)
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["parallelism"].startswith(shard + " sharded over 2 ranks")
    sys.path.insert(0, str(ROOT))
    import bench
    assert d["config"] == bench.CONFIGS[config]


def test_bench_world_size_mismatch_fails():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--config", "c1"], cwd=ROOT, capture_output=True,
                       text=True, timeout=300, env=env)
    assert r.returncode != 0 and "WORLD_SIZE=1 but --gpus 2" in r.stderr
