"""Small tensors normally take the fused one-CTA kernels (csrc/small.cu); with TLC_NO_SMALL=1
they go through the streaming K1-K5 path instead.  Both must give the oracle's bytes: rerun
the small-size parity and batch suites in a subprocess with the fused path switched off."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_streaming_path_on_small_sizes():
    env = dict(os.environ, TLC_NO_SMALL="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        "tests/test_gpu_parity.py::test_parity_sizes", "tests/test_gpu_parity.py::test_parity_misaligned",
                        "tests/test_gpu_parity.py::test_special_values", "tests/test_gpu_batched.py"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_cooperative_small_table_path():
    """TLC_COOP=1 routes small tables through the cooperative K6c (slices over all SMs, two
    grid barriers) instead of K6 (one CTA per tensor); the batch suites and the loopback
    exchange must give the oracle's bytes on that path too."""
    env = dict(os.environ, TLC_COOP="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "tests/test_gpu_batched.py",
                        "tests/test_gpu_exchange_loopback.py::test_loopback_matches_oracle"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
