"""Device-buffer overrun checks (the GPU pool refuses compute-sanitizer).

With SMC_GUARD=1 every device buffer of the library carries 4 KB guard zones
of a fixed byte pattern before and after it, and every C-ABI call ends by
synchronising and verifying every live buffer's zones (capi.cu guard_check):
a kernel or copy writing past either end of its buffer fails that call.

  * positive control: smc_guard_selftest writes into the zones on purpose and
    must be caught on either side, while a write that fills the buffer exactly
    passes;
  * the GPU parity, group (multi-device), pCN, forcing-basis, Galerkin,
    full-size, acceptance, CLI and rank suites run again in a child process
    under SMC_GUARD=1 — every C-ABI call they make (K1 disk/tiled/strict/FP32,
    batched, K2 + compaction, K3 trees, pCN graphs, group exchanges, Galerkin)
    is checked for overruns.
"""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

SELFTEST = r"""
import ctypes as C, json, sys
sys.path.insert(0, sys.argv[1])
import paper_1808_10580_b200 as S
from paper_1808_10580_b200 import _abi as A
ctx = S.Context(0)
lib = ctx.lib
out = {}
for off, n in [(0, 1024), (1024, 1), (1020, 8), (-1, 1), (-4096, 4096), (100, 0)]:
    rc = lib.smc_guard_selftest(ctx.handle, off, n)
    out[f"{off},{n}"] = [rc, lib.smc_last_error().decode() if rc else ""]
print(json.dumps(out))
"""


def _run(code_or_args, env_extra, timeout):
    env = dict(os.environ, **env_extra)
    return subprocess.run([sys.executable, *code_or_args], env=env, cwd=ROOT, capture_output=True, text=True,
                          timeout=timeout)


def test_guard_zones_catch_overruns():
    import json
    r = _run(["-c", SELFTEST, str(ROOT)], {"SMC_GUARD": "1"}, 300)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["0,1024"][0] == 0 and res["100,0"][0] == 0, res  # in bounds
    for k in ("1024,1", "1020,8", "-1,1", "-4096,4096"):
        rc, msg = res[k]
        assert rc != 0 and "overrun" in msg, (k, res[k])
    assert "after" in res["1024,1"][1] and "before" in res["-1,1"][1]


def test_guard_mode_off_refuses_selftest():
    code = SELFTEST
    r = _run(["-c", code, str(ROOT)], {"SMC_GUARD": "0"}, 300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert '"1024,1": [' in r.stdout and "guard mode is off" in r.stdout


@pytest.mark.skipif(os.environ.get("SMC_GUARD") == "1", reason="already the child run")
def test_gpu_suites_under_guard_zones():
    suites = ["tests/test_gpu_parity.py", "tests/test_gpu_group.py", "tests/test_gpu_pcn.py",
              "tests/test_gpu_forcing.py", "tests/test_gpu_galerkin.py", "tests/test_gpu_fullsize.py",
              "tests/test_gpu_acceptance.py", "tests/test_gpu_cli.py", "tests/test_gpu_ranks.py"]
    r = _run(["-m", "pytest", *suites, "-m", "gpu", "-x", "-q", "-p", "no:cacheprovider"], {"SMC_GUARD": "1"}, 1500)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, tail
    assert "overrun" not in r.stdout, tail
    print(r.stdout.strip().splitlines()[-1])
