"""The GPU suites that exercise every kernel, re-run against a -DTLC_DEVICE_CHECKS build of
libtlc (device-side bounds assertions on every data-dependent store index: K3's emission and
stage, K6/K6c's payload and stage, K5m's scatter; a violation traps), selected with TLC_LIB.
compute-sanitizer is closed on the GPU pool, so this and the guard-band tests
(test_gpu_guards.py) stand in for memcheck."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_suites_under_device_checks():
    import importlib.util

    spec = importlib.util.spec_from_file_location("_b", os.path.join(ROOT, "paper_1802_07389_b200", "build.py"))
    B = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(B)
    lib = B.build(out=os.path.join(ROOT, "paper_1802_07389_b200", "libtlc_checks.so"), defines=["TLC_DEVICE_CHECKS"])
    for coop in ("0", "1"):
        env = dict(os.environ, TLC_LIB=lib, TLC_COOP=coop)
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "tests/test_gpu_guards.py",
                            "tests/test_gpu_parity.py::test_parity_sizes", "tests/test_gpu_parity.py::test_parity_runs_many_tiles",
                            "tests/test_gpu_parity.py::test_corrupt_payloads_raise_format",
                            "tests/test_gpu_batched.py", "tests/test_gpu_exchange_loopback.py::test_loopback_matches_oracle",
                            "tests/test_gpu_codecs.py"],
                           cwd=ROOT, env=env, capture_output=True, text=True, timeout=1800)
        assert r.returncode == 0, (coop, r.stdout[-3000:] + r.stderr[-2000:])
        assert "TLC_CHECK failed" not in r.stdout + r.stderr
