"""SURVEY §5 sanitizers, GPU side: every librepops.so kernel on tiny shapes
(tools/sanitize_driver.py: all R-GEMM configurations, row operators, elementwise
kernels, commit plans with multi-pass reduces, the fused attention, the tiny GPT-2
step with its aux and commit side streams, the MLP step, the tiny Llama prefill, and
the peer-memory combine with device signal / wait flags) under NVIDIA
compute-sanitizer: memcheck (out-of-bounds / misaligned accesses, leaks of device
allocations), racecheck (shared-memory hazards) and synccheck (barrier misuse).
Any reported error fails the test (--error-exitcode)."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


def _run(tool, sections, extra=()):
    cmd = [SAN, "--tool", tool, "--error-exitcode", "99", "--print-limit", "20", *extra, sys.executable,
           os.path.join(ROOT, "tools", "sanitize_driver.py"), sections]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=3000)
    out = r.stdout + r.stderr
    if "compute-sanitizer is closed on this pool" in out:
        # the GPU pool's wrapper refuses sanitizer runs (they have left GPUs needing a reset);
        # the recorded clean runs are listed in DESIGN.md §5 (sanitizers)
        pytest.skip("compute-sanitizer refused by the GPU pool")
    assert r.returncode == 0, f"{tool} on {sections}: rc {r.returncode}\n{out[-6000:]}"
    assert "ERROR SUMMARY: 0 errors" in out or "(0 errors, 0 warnings)" in out, out[-6000:]
    for s in sections.split(","):
        assert f"section {s}: ok" in out


@pytest.mark.parametrize("sections", ["gemm", "rowops,elem,commit,attn", "steps", "p2p"])
def test_memcheck(sections):
    _run("memcheck", sections)


@pytest.mark.parametrize("sections", ["gemm", "rowops,commit,attn"])
def test_racecheck(sections):
    _run("racecheck", sections, ("--racecheck-report", "hazard"))


@pytest.mark.parametrize("sections", ["gemm,rowops,commit,attn"])
def test_synccheck(sections):
    _run("synccheck", sections)
