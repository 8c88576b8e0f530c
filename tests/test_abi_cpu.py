"""CPU-only checks of the boundary: libtlc.so loads and exports every symbol
declared in include/*.h; size queries and argument validation (no GPU compute)."""
import ctypes
import glob
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    syms = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"\b(tlc_[a-z0-9_]+)\s*\(", src):
            syms.add(m.group(1))
    return syms


@pytest.fixture(scope="module")
def T():
    import __graft_entry__

    __graft_entry__.build()        # builds libtlc.so on a fresh checkout (no package import first)
    import paper_1802_07389_b200 as T

    return T


def test_exports_every_declared_symbol(T):
    syms = declared_symbols()
    assert {"tlc_compress", "tlc_decompress"} <= syms
    lib = ctypes.CDLL(T.LIB_PATH)
    missing = [s for s in sorted(syms) if not hasattr(lib, s)]
    assert not missing, missing


def test_size_queries(T):
    for n in (1, 4, 5, 6, 1000, 1 << 28, (1 << 28) + 1):
        assert T.tlc_quartic_bytes(n) == -(-n // 5)
        assert T.tlc_max_payload_bytes(n) == -(-n // 5)
        assert T.tlc_compress_workspace_bytes(n) >= 256
        assert T.tlc_decompress_workspace_bytes(n) >= 256
    assert T.tlc_status_string(0) == "TLC_OK"
    assert T.tlc_status_string(4) == "TLC_ERR_FORMAT"
    assert T.tlc_version() >= 100


def test_argument_validation_without_gpu(T):
    lib = T.lib()
    # null pointers / n == 0 / bad s are rejected synchronously, before any CUDA call
    assert lib.tlc_compress(None, None, 10, 1.0, 1, None, 2, None, None, 0, None) == T.TLC_ERR_ARG
    fake = 1 << 20
    assert lib.tlc_compress(fake, fake + 4096, 0, 1.0, 1, fake, 2, fake, fake, 1 << 20, None) == T.TLC_ERR_ARG
    assert lib.tlc_compress(fake, fake + 4096, 10, 2.0, 1, fake, 2, fake, fake, 1 << 20, None) == T.TLC_ERR_ARG
    assert lib.tlc_compress(fake, fake + 4096, 10, 0.99, 1, fake, 2, fake, fake, 1 << 20, None) == T.TLC_ERR_ARG
    pay, hdr = fake + 8192, fake + 12288
    assert lib.tlc_compress(fake, fake + 4096, 10, 1.0, 1, pay, 1, hdr, fake, 1 << 20, None) == T.TLC_ERR_CAPACITY
    assert lib.tlc_compress(fake, fake + 4096, 10, 1.0, 1, pay, 2, hdr, fake, 8, None) == T.TLC_ERR_CAPACITY
    assert lib.tlc_decompress(fake, fake, 10, fake, 7, fake, 1 << 20, None) == T.TLC_ERR_ARG


def test_build_id_matches_sources(T):
    """The loaded libtlc.so was built from this tree: its embedded id is the hash of the
    current csrc/, include/ and flags (build.py rebuilds on any difference)."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("_b", os.path.join(ROOT, "paper_1802_07389_b200", "build.py"))
    B = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(B)
    assert T.tlc_build_id() == B.source_id()
    assert not B.stale()


def test_overlapping_ranges_rejected_without_gpu(T):
    lib = T.lib()
    n = 1000
    t, err, pay, hdr, ws = 1 << 24, 2 << 24, 3 << 24, 4 << 24, 5 << 24
    ok = [t, err, n, 1.5, 1, pay, 200, hdr, ws, 1 << 24, None]
    for k, v in [(1, t + 4 * 999), (1, t - 4 * 999), (5, t + 16), (5, err + 3996), (7, t + 64), (7, pay + 100),
                 (7, err)]:
        a = list(ok)
        a[k] = v
        assert lib.tlc_compress(*a) == T.TLC_ERR_ARG, (k, v)
