"""SURVEY §5 sanitizers, CPU side: the oracle (oracle/repops_oracle.c) built with
AddressSanitizer + UndefinedBehaviorSanitizer (-fno-sanitize-recover=all) runs the
oracle's own pin suites; any out-of-bounds access, use-after-free, signed overflow,
misaligned load or invalid shift aborts the run.  (The CUDA side runs under
compute-sanitizer: tests/test_gpu_sanitizers.py.)"""
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _libasan():
    try:
        p = subprocess.check_output(["gcc", "-print-file-name=libasan.so"], text=True).strip()
    except (OSError, subprocess.CalledProcessError):
        return None
    return p if os.path.isabs(p) and os.path.exists(p) else None


@pytest.mark.skipif(shutil.which("gcc") is None or _libasan() is None, reason="gcc / libasan not available")
def test_oracle_suites_clean_under_asan_ubsan():
    env = dict(os.environ)
    env.update(REPOPS_ORACLE_SANITIZE="1", LD_PRELOAD=_libasan(),
               ASAN_OPTIONS="detect_leaks=0:verify_asan_link_order=0:abort_on_error=1",
               UBSAN_OPTIONS="print_stacktrace=1:halt_on_error=1")
    suites = ["tests/test_oracle_gemm.py", "tests/test_oracle_reduce.py", "tests/test_oracle_math.py",
              "tests/test_oracle_rowops.py", "tests/test_oracle_hash.py", "tests/test_oracle_lowp.py",
              "tests/test_oracle_rand.py", "tests/test_oracle_mlp.py", "tests/test_oracle_llama.py",
              "tests/test_oracle_definitional.py"]
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", *suites],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    out = r.stdout + r.stderr
    assert "AddressSanitizer" not in out and "runtime error" not in out, out[-4000:]
    assert r.returncode == 0, out[-4000:]
    assert os.path.exists(os.path.join(ROOT, "oracle", "liboracle_san.so"))
