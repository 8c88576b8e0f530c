"""3LC1 blobs (tlc_blob_write / tlc_blob_read, host-only C ABI) on CPU:
the library's bytes equal a blob packed here field by field from the SPEC's layout, for
payloads made by the CPU oracle; round trips; malformed blobs are FORMAT errors."""
import struct

import numpy as np
import pytest

import oracle as O
import synth


@pytest.fixture(scope="module")
def T():
    import __graft_entry__

    __graft_entry__.build()
    import paper_1802_07389_b200 as T

    return T


def _spec_blob(codec, flags, dims, m, payload):
    # "3LC1", version 1, codec_id, flags, rank, rank x u64 dims, f32 m, u64 payload_len, payload
    return (b"3LC1" + bytes([1, codec, flags, len(dims)]) + b"".join(struct.pack("<Q", d) for d in dims)
            + struct.pack("<f", m) + struct.pack("<Q", len(payload)) + bytes(payload))


@pytest.mark.parametrize("dims,s,zre", [([5], 1.0, True), ([70], 1.0, True), ([7, 11, 13], 1.75, True),
                                        ([1000], 1.9, False), ([3, 3, 64, 64], 1.5, True)])
def test_blob_bytes_match_spec_layout(T, dims, s, zre):
    n = int(np.prod(dims))
    t = synth.gaussian(n, 61, n) if n != 70 else synth.zeros(n)
    buf = np.zeros(n, np.float32)
    c = O.compress(t, buf, s, zre)
    hdr = {"M": float(c.M), "flags": 1 if zre else 0, "n": n, "payload_len": c.payload_len, "status": 0}
    blob = T.tlc_blob_write(hdr, dims, c.payload.tobytes())
    assert blob == _spec_blob(0, 1 if zre else 0, dims, float(c.M), c.payload.tobytes())
    assert len(blob) == T.lib().tlc_blob_size(len(dims), c.payload_len)
    h2, d2, p2 = T.tlc_blob_read(blob)
    assert d2 == list(dims) and p2 == c.payload.tobytes()
    assert h2["n"] == n and h2["payload_len"] == c.payload_len and h2["flags"] == hdr["flags"]
    assert np.float32(h2["M"]) == c.M
    st, out = O.decompress(np.frombuffer(p2, np.uint8), bool(h2["flags"] & 1), np.float32(h2["M"]), h2["n"])
    assert st == 0


def test_blob_examples_from_spec(T):
    # S:288 70 zeros -> payload [255], m = 0 (ratio 280x, header excluded); S:289 [175], m 0.4
    b70 = T.tlc_blob_write({"M": 0.0, "flags": 1, "n": 70, "payload_len": 1, "status": 0}, [70], bytes([255]))
    assert b70 == _spec_blob(0, 1, [70], 0.0, [255])
    b5 = T.tlc_blob_write({"M": np.float32(0.4), "flags": 1, "n": 5, "payload_len": 1, "status": 0}, [5], bytes([175]))
    h, d, p = T.tlc_blob_read(b5)
    assert p == bytes([175]) and d == [5] and np.float32(h["M"]) == np.float32(0.4)
    assert 4 * h["n"] / h["payload_len"] == 20.0          # S:310 blob_ratio of a 5-element blob


def test_blob_rejects_malformed(T):
    good = _spec_blob(0, 1, [10], 0.5, [121, 243][:1] + [1])
    T.tlc_blob_read(good)
    bad = [b"3LC2" + good[4:],                    # magic (S:296 corrupted magic -> FormatError)
           good[:4] + bytes([2]) + good[5:],     # version
           good[:5] + bytes([7]) + good[6:],     # unknown codec
           good[:6] + bytes([2]) + good[7:],     # unknown flag
           good[:-1],                            # truncated payload
           good + bytes([0]),                    # trailing byte
           _spec_blob(0, 0, [10], 0.5, [1]),     # no ZRE but payload != ceil(n/5)
           _spec_blob(0, 1, [10], 0.5, [1, 2, 3]),   # longer than ceil(n/5): ZRE never expands
           _spec_blob(0, 1, [0], 0.5, [1]),      # no elements
           good[:10]]
    for b in bad:
        with pytest.raises(T.TlcError) as e:
            T.tlc_blob_read(b)
        assert e.value.code == T.TLC_ERR_FORMAT, b
    with pytest.raises(T.TlcError):             # header n must equal the product of dims
        T.tlc_blob_write({"M": 1.0, "flags": 0, "n": 11, "payload_len": 2, "status": 0}, [10], bytes([1, 2]))
    with pytest.raises(T.TlcError):             # only successful compressions are written
        T.tlc_blob_write({"M": 0.0, "flags": 0, "n": 10, "payload_len": 0, "status": 2}, [10], b"")
