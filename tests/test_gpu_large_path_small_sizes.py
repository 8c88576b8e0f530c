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


@pytest.mark.parametrize("env", [{"TLC_K6G": "0"}, {"TLC_K6G_BULK": "1"}, {"TLC_K6G": "8"}, {"TLC_K6G_SYNC": "1"},
                                 {"TLC_K7_REC": "0"}])
def test_small_table_compressor_variants(env):
    """K6g (clusters of 4 CTAs per tensor group, st.async + mbarriers) is the small-table
    compressor and K7 takes per-CTA records; K6 (one CTA per tensor, TLC_K6G=0), K6g with
    bulk-copy staging (TLC_K6G_BULK=1), clusters of 8 with one-row slices (TLC_K6G=8), K6g with
    two cluster barriers (TLC_K6G_SYNC=1) and the table-walking K7 (TLC_K7_REC=0) stay
    selectable and must give the oracle's bytes too (test_gpu_batched: ResNet-110 and mixed
    small tables, corrupt payloads, graphs)."""
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "tests/test_gpu_batched.py",
                        "tests/test_gpu_exchange_loopback.py::test_loopback_graph_replay"],
                       cwd=ROOT, env=dict(os.environ, **env), capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_fused_max_quantize_table_path():
    """TLC_K12=1: K1 and K2 fused over L2-sized windows of tensors (compress.cu K12, opt-in) --
    batches, the loopback exchange with contexts above the small-table bound (aligned and
    unaligned partitions) and the full-size BERT-large sample must give the oracle's bytes."""
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "tests/test_gpu_batched.py",
                        "tests/test_gpu_exchange_loopback.py::test_loopback_large_contexts",
                        "tests/test_gpu_exchange_loopback.py::test_loopback_bert_large_full_size_sampled"],
                       cwd=ROOT, env=dict(os.environ, TLC_K12="1"), capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_unkeyed_pull_compress():
    """TLC_NO_KEYED=1: the owner's pull compress runs its own K1 instead of taking the max keys
    the parallel K5m folds while writing the means; both must give the oracle's bytes."""
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        "tests/test_gpu_exchange_loopback.py::test_loopback_matches_oracle",
                        "tests/test_gpu_exchange_loopback.py::test_loopback_large_contexts",
                        "tests/test_gpu_exchange_loopback.py::test_loopback_failed_push_poisons_context"],
                       cwd=ROOT, env=dict(os.environ, TLC_NO_KEYED="1"), capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
