"""The C++ drop-in (paper_1808_10580_b200/host/scalarmc_forward_gpu.cpp) under
the reference's unchanged callers, on the GPU.

tests/cpp/test_dropin.cpp is linked with the reference's own inference.cpp /
optimize.cpp (compiled in place into oracle/_ref by build()) and the drop-in
instead of forward_ad.cpp / forward_bvp.cpp, so LikelihoodSpec::misfit,
run_chain and forcing_cost call the GPU forward map exactly as they would in a
scalarmc build.  The numbers must match the golden fixtures of the real
reference within the FP64 parity gate."""
import json
import os
import subprocess
from pathlib import Path

import pytest

from conftest import est_from

BIN = Path(__file__).resolve().parent / "cpp" / "_bin" / "test_dropin"


def run_dropin(env=None):
    if not BIN.exists():
        pytest.skip("tests/cpp/_bin/test_dropin not built (needs the reference headers at build time)")
    out = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600,
                         env=dict(os.environ, **(env or {})))
    assert out.returncode == 0, out.stderr
    checks = {}
    for line in out.stdout.splitlines():
        rec = json.loads(line)
        checks[rec["check"]] = rec
    return checks


@pytest.mark.gpu
def test_cpp_dropin_multi_device_bit_identical():
    """SCALARMC_DEVICES puts the unchanged reference callers (misfit,
    run_chain, forcing_cost, the CLI bodies) on a multi-device context; with
    the one B200 the list repeats device 0 (emulated exchange, same shard
    plans).  Every number must equal the one-device run bit for bit."""
    one = run_dropin()
    for devs in ("0,0", "0,0,0,0,0,0,0,0"):
        many = run_dropin({"SCALARMC_DEVICES": devs})
        assert many == one, devs


@pytest.mark.gpu
def test_cpp_dropin_under_reference_callers(golden):
    checks = run_dropin()
    bad = [k for k, v in checks.items() if v.get("ok") is False]
    assert not bad, {k: checks[k] for k in bad}

    def close(a, b, rel=1e-10, floor=1.0):
        return abs(a - b) <= rel * max(abs(b), floor)

    for name, key in (("c1", "c1"), ("bvp_box", "bvp_box")):
        for got, want in zip(checks[name]["estimates"], golden[key]["estimates"]):
            g, w = est_from(got), est_from(want)
            assert close(g["mean"], w["mean"], floor=2.0), (name, g, w)
            assert close(g["std_error"], w["std_error"], rel=1e-8, floor=0.0)
            assert g["n_failed"] == w["n_failed"]
    assert close(float.fromhex(checks["misfit"]["value"]), float.fromhex(golden["misfit"]["phi"]), rel=1e-9)
    fc = [r for r in golden["forcing_cost"] if r["F"] == [1.0, -0.5, 2.0]][0]
    assert close(float.fromhex(checks["forcing_cost"]["value"]), float.fromhex(fc["cost"]), rel=1e-9)
