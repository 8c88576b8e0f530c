"""B200-native 3LC state-change compression (arXiv 1802.07389) -- Python binding.

Thin ctypes marshalling over the C ABI of ``include/tlc.h`` (``libtlc.so``, built
in-tree from ``csrc/`` for sm_100a).  Functions keep the C names
(``tlc_compress``, ``tlc_decompress``, ...); torch is used only to own device
memory and to supply the CUDA stream.  Every step of the method runs in the
CUDA kernels; there is no CPU fallback -- importing this package without the
built library raises.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# TLC_LIB: a development build of the same sources (tools/, e.g. a -DTLC_K6C_TRACE variant)
LIB_PATH = os.environ.get("TLC_LIB") or os.path.join(_HERE, "libtlc.so")

TLC_OK, TLC_ERR_ARG, TLC_ERR_NONFINITE, TLC_ERR_RANGE, TLC_ERR_FORMAT, TLC_ERR_CAPACITY, \
    TLC_ERR_CUDA, TLC_ERR_NCCL = range(8)
TLC_FLAG_ZRE = 1
TLC_FLAG_INT8 = 2
TLC_MODE_OVERWRITE, TLC_MODE_ACCUMULATE = 0, 1
HEADER_BYTES = 32


class TlcError(RuntimeError):
    def __init__(self, code: int, where: str):
        super().__init__(f"{where}: {tlc_status_string(code)} ({code})")
        self.code = code


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(nvcc, sm_100a). There is no CPU fallback.")
    L = ctypes.CDLL(LIB_PATH)
    P, U64, SZ, F, I = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_size_t, ctypes.c_float, ctypes.c_int
    sig = {
        "tlc_version": (I, []),
        "tlc_build_id": (ctypes.c_char_p, []),
        "tlc_status_string": (ctypes.c_char_p, [I]),
        "tlc_quartic_bytes": (U64, [U64]),
        "tlc_max_payload_bytes": (U64, [U64]),
        "tlc_compress_workspace_bytes": (SZ, [U64]),
        "tlc_decompress_workspace_bytes": (SZ, [U64]),
        "tlc_compress": (I, [P, P, U64, F, I, P, U64, P, P, SZ, P]),
        "tlc_decompress": (I, [P, P, U64, P, I, P, SZ, P]),
        "tlc_batch_create": (I, [P, I, P]),
        "tlc_batch_update": (I, [P, P]),
        "tlc_batch_destroy": (I, [P]),
        "tlc_batch_workspace_bytes": (SZ, [P]),
        "tlc_batch_compress": (I, [P, F, I, P]),
        "tlc_batch_decompress": (I, [P, I, P]),
        "tlc_comm_unique_id": (I, [P]),
        "tlc_comm_init": (I, [P, P, I, I, I]),
        "tlc_comm_destroy": (I, [P]),
        "tlc_plan_count": (I, [I, P, I]),
        "tlc_plan_compute": (I, [I, P, I, I, P, P, P, P]),
        "tlc_exchange_create": (I, [P, P, I, P]),
        "tlc_exchange_destroy": (I, [P]),
        "tlc_exchange_num_contexts": (I, [P]),
        "tlc_exchange_context": (I, [P, I, P, P, P, P, P, P]),
        "tlc_exchange_owned_elements": (U64, [P]),
        "tlc_exchange_owned_buffer": (P, [P]),
        "tlc_exchange_push_error": (P, [P]),
        "tlc_exchange_pull_error": (P, [P]),
        "tlc_exchange_wire_bytes": (U64, [P, I]),
        "tlc_exchange_bind_error_buffers": (I, [P, P, P]),
        "tlc_exchange_set_transport": (I, [P, I]),
        "tlc_exchange_push": (I, [P, P, F, I, P]),
        "tlc_exchange_pull": (I, [P, P, F, I, P]),
        "tlc_exchange_status": (I, [P, P, P]),
        "tlc_exchange_status_async": (I, [P, P, P]),
        "tlc_exchange_ipc_handles": (I, [P, P]),
        "tlc_exchange_ipc_open": (I, [P, P]),
        "tlc_exchange_traffic": (I, [P, P]),
        "tlc_loopback_create": (I, [P, I, I, P, I]),
        "tlc_loopback_destroy": (I, [P]),
        "tlc_loopback_rank": (P, [P, I]),
        "tlc_loopback_push": (I, [P, P, F, I, P]),
        "tlc_loopback_pull": (I, [P, P, F, I, P]),
        "tlc_stoch_compress": (I, [P, U64, U64, U64, I, P, U64, P, P, SZ, P]),
        "tlc_int8_workspace_bytes": (SZ, [U64]),
        "tlc_int8_compress": (I, [P, U64, P, P, P, SZ, P]),
        "tlc_int8_decompress": (I, [P, P, U64, P, I, P]),
        "tlc_aggregate_create": (I, [P, I, I, P, P]),
        "tlc_aggregate_run": (I, [P, P]),
        "tlc_aggregate_destroy": (I, [P]),
        "tlc_blob_size": (U64, [I, U64]),
        "tlc_blob_write": (I, [P, I, P, P, P, U64, P]),
        "tlc_blob_read": (I, [P, U64, P, P, P, I, P]),
        "tlc_launch_count": (ctypes.c_ulonglong, []),
        "tlc_prof_enable": (None, [I]),
        "tlc_prof_collect": (I, [P, I]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype, fn.argtypes = res, args
    return L


_lib = _load()


def lib():
    return _lib


# ------------------------------------------------------------------ sizes / strings
def tlc_version() -> int:
    return _lib.tlc_version()


def tlc_build_id() -> str:
    return _lib.tlc_build_id().decode()


def tlc_status_string(code: int) -> str:
    return _lib.tlc_status_string(int(code)).decode()


def tlc_quartic_bytes(n: int) -> int:
    return int(_lib.tlc_quartic_bytes(n))


def tlc_max_payload_bytes(n: int) -> int:
    return int(_lib.tlc_max_payload_bytes(n))


def tlc_compress_workspace_bytes(n: int) -> int:
    return int(_lib.tlc_compress_workspace_bytes(n))


def tlc_decompress_workspace_bytes(n: int) -> int:
    return int(_lib.tlc_decompress_workspace_bytes(n))


# ------------------------------------------------------------------ helpers
def _stream_ptr(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream)


def _check_dev(name, x, dtype):
    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if x.dtype != dtype or not x.is_contiguous():
        raise TypeError(f"{name} must be contiguous {dtype}")


_ws_cache: dict = {}


def workspace(nbytes: int, device=None, tag: str = "default") -> torch.Tensor:
    """A cached device workspace of at least ``nbytes`` (torch allocations are
    >= 512-byte aligned, the ABI needs 256)."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    key = (dev, tag)
    w = _ws_cache.get(key)
    if w is None or w.numel() < nbytes:
        w = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=dev)
        _ws_cache[key] = w
    return w


def new_header(device=None) -> torch.Tensor:
    return torch.zeros(HEADER_BYTES, dtype=torch.uint8, device=device or "cuda")


def parse_header(hdr: torch.Tensor) -> dict:
    """Copy a device header to the host (synchronizes) and decode its fields."""
    import struct

    raw = bytes(hdr.detach().to("cpu").numpy().tobytes())
    M, flags, n, plen, status, _ = struct.unpack("<fIQQII", raw)
    return {"M": M, "flags": flags, "n": n, "payload_len": plen, "status": status}


class Header(ctypes.Structure):
    """struct tlc_header (include/tlc.h), host copy."""
    _fields_ = [("M", ctypes.c_float), ("flags", ctypes.c_uint32), ("n", ctypes.c_uint64),
                ("payload_len", ctypes.c_uint64), ("status", ctypes.c_uint32), ("reserved", ctypes.c_uint32)]


def tlc_blob_write(hdr: dict, dims, payload: bytes) -> bytes:
    """3LC1 blob of a compressed tensor: `hdr` as parse_header() returns it,
    `payload` its payload_len bytes (host).  Marshalling only: the C ABI writes the bytes."""
    h = Header(float(hdr["M"]), int(hdr["flags"]), int(hdr["n"]), int(hdr["payload_len"]), int(hdr["status"]), 0)
    d = (ctypes.c_uint64 * max(1, len(dims)))(*[int(x) for x in dims])
    pb = bytes(payload)
    cap = int(_lib.tlc_blob_size(len(dims), len(pb)))
    out = (ctypes.c_uint8 * max(cap, 1))()
    wr = ctypes.c_uint64()
    src = ctypes.create_string_buffer(pb, max(1, len(pb)))
    rc = _lib.tlc_blob_write(ctypes.byref(h), len(dims), ctypes.cast(d, ctypes.c_void_p), src, out, cap,
                             ctypes.byref(wr))
    if rc != TLC_OK:
        raise TlcError(rc, "tlc_blob_write")
    return bytes(out)[: wr.value]


def tlc_blob_read(blob: bytes):
    """(header dict, dims, payload bytes) of a 3LC1 blob; TlcError(FORMAT) if malformed."""
    b = bytes(blob)
    h = Header()
    rank = ctypes.c_int()
    dims = (ctypes.c_uint64 * 255)()
    off = ctypes.c_uint64()
    src = ctypes.create_string_buffer(b, max(1, len(b)))
    rc = _lib.tlc_blob_read(src, len(b), ctypes.byref(h), ctypes.byref(rank), dims, 255, ctypes.byref(off))
    if rc != TLC_OK:
        raise TlcError(rc, "tlc_blob_read")
    hd = {"M": h.M, "flags": h.flags, "n": h.n, "payload_len": h.payload_len, "status": h.status}
    return hd, [int(dims[i]) for i in range(rank.value)], b[off.value: off.value + h.payload_len]


# ------------------------------------------------------------------ the ABI calls
def tlc_compress(t: torch.Tensor, err: torch.Tensor, s: float, use_zre: bool = True,
                 payload: torch.Tensor | None = None, hdr: torch.Tensor | None = None,
                 ws: torch.Tensor | None = None, stream=None):
    """Enqueue 3LC compression of ``t`` with error buffer ``err`` (updated in place).
    Returns (payload, hdr) device tensors; read lengths/status with parse_header()."""
    _check_dev("t", t, torch.float32)
    _check_dev("err", err, torch.float32)
    n = t.numel()
    if err.numel() != n:
        raise ValueError("err must have as many elements as t")
    cap = tlc_max_payload_bytes(n)
    if payload is None:
        payload = torch.empty(max(cap, 1), dtype=torch.uint8, device=t.device)
    if hdr is None:
        hdr = new_header(t.device)
    need = tlc_compress_workspace_bytes(n)
    if ws is None:
        ws = workspace(need, t.device, "compress")
    rc = _lib.tlc_compress(t.data_ptr(), err.data_ptr(), n, ctypes.c_float(s), int(bool(use_zre)),
                           payload.data_ptr(), payload.numel(), hdr.data_ptr(), ws.data_ptr(),
                           ws.numel(), _stream_ptr(stream))
    if rc != TLC_OK:
        raise TlcError(rc, "tlc_compress")
    return payload, hdr


def tlc_decompress(payload: torch.Tensor, hdr: torch.Tensor, n: int, out: torch.Tensor | None = None,
                   mode: int = TLC_MODE_OVERWRITE, ws: torch.Tensor | None = None, stream=None):
    """Enqueue decompression into ``out`` (fp32[n]); mode ACCUMULATE adds M*q where q != 0."""
    if out is None:
        out = torch.empty(n, dtype=torch.float32, device=payload.device)
    _check_dev("out", out, torch.float32)
    _check_dev("payload", payload, torch.uint8)
    _check_dev("hdr", hdr, torch.uint8)
    if out.numel() < n:
        raise ValueError(f"out holds {out.numel()} elements, n = {n}")
    if hdr.numel() < HEADER_BYTES:
        raise ValueError("hdr must hold 32 bytes")
    need = tlc_decompress_workspace_bytes(n)
    if ws is None:
        ws = workspace(need, out.device, "decompress")
    rc = _lib.tlc_decompress(payload.data_ptr(), hdr.data_ptr(), n, out.data_ptr(), int(mode),
                             ws.data_ptr(), ws.numel(), _stream_ptr(stream))
    if rc != TLC_OK:
        raise TlcError(rc, "tlc_decompress")
    return out


# ------------------------------------------------------------------ batches of tensors
class TensorDesc(ctypes.Structure):
    """struct tlc_tensor_desc (include/tlc.h)."""
    _fields_ = [("t", ctypes.c_void_p), ("err", ctypes.c_void_p), ("out", ctypes.c_void_p),
                ("payload", ctypes.c_void_p), ("hdr", ctypes.c_void_p), ("n", ctypes.c_uint64)]


def _descs(rows):
    arr = (TensorDesc * len(rows))()
    for k, (t, e, o, pl, h, n) in enumerate(rows):
        arr[k] = TensorDesc(*[x.data_ptr() if isinstance(x, torch.Tensor) else (x or None) for x in (t, e, o, pl, h)],
                            int(n))
    return arr


class Batch:
    """tlc_batch: a fixed list of tensors compressed / decompressed by one set of
    kernel launches (device-resident table and workspace)."""

    def __init__(self, rows):
        self.rows = list(rows)
        self._b = ctypes.c_void_p()
        arr = _descs(self.rows)
        rc = _lib.tlc_batch_create(ctypes.byref(self._b), len(self.rows), ctypes.cast(arr, ctypes.c_void_p))
        if rc != TLC_OK:
            raise TlcError(rc, "tlc_batch_create")

    def update(self, rows):
        self.rows = list(rows)
        arr = _descs(self.rows)
        rc = _lib.tlc_batch_update(self._b, ctypes.cast(arr, ctypes.c_void_p))
        if rc != TLC_OK:
            raise TlcError(rc, "tlc_batch_update")

    def compress(self, s: float, use_zre: bool = True, stream=None):
        rc = _lib.tlc_batch_compress(self._b, ctypes.c_float(s), int(bool(use_zre)), _stream_ptr(stream))
        if rc != TLC_OK:
            raise TlcError(rc, "tlc_batch_compress")

    def decompress(self, mode: int = TLC_MODE_OVERWRITE, stream=None):
        rc = _lib.tlc_batch_decompress(self._b, int(mode), _stream_ptr(stream))
        if rc != TLC_OK:
            raise TlcError(rc, "tlc_batch_decompress")

    def close(self):
        if self._b:
            _lib.tlc_batch_destroy(self._b)
            self._b = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class TensorSet:
    """Compression contexts for a list of tensors (one error buffer, payload and
    header each -- the paper's per-tensor contexts), compressed and
    decompressed through tlc_batch objects.  Marshalling only."""

    def __init__(self, sizes, device=None):
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.device, self.sizes = dev, [int(n) for n in sizes]
        self.errs = [torch.zeros(n, dtype=torch.float32, device=dev) for n in self.sizes]
        self.payloads = [torch.empty(max(1, tlc_max_payload_bytes(n)), dtype=torch.uint8, device=dev)
                         for n in self.sizes]
        self.hdrs = torch.zeros(len(self.sizes), HEADER_BYTES, dtype=torch.uint8, device=dev)
        self._cb = self._db = None
        self._ckey = self._dkey = None

    def compress_batch(self, ts) -> Batch:
        return Batch([(ts[i], self.errs[i], None, self.payloads[i], self.hdrs[i], n) for i, n in enumerate(self.sizes)])

    def decompress_batch(self, outs, payloads=None, hdrs=None) -> Batch:
        payloads = self.payloads if payloads is None else payloads
        hdrs = self.hdrs if hdrs is None else hdrs
        return Batch([(None, None, outs[i], payloads[i], hdrs[i], n) for i, n in enumerate(self.sizes)])

    def compress(self, ts, s: float, use_zre: bool = True, stream=None, batch: Batch | None = None):
        if batch is None:
            key = tuple(t.data_ptr() for t in ts)
            if self._ckey != key:
                self._cb, self._ckey = self.compress_batch(ts), key
            batch = self._cb
        batch.compress(s, use_zre, stream)

    def decompress(self, outs, mode: int = TLC_MODE_OVERWRITE, stream=None, batch: Batch | None = None):
        if batch is None:
            key = tuple(o.data_ptr() for o in outs)
            if self._dkey != key:
                self._db, self._dkey = self.decompress_batch(outs), key
            batch = self._db
        batch.decompress(mode, stream)

    def headers(self):
        import struct

        raw = self.hdrs.cpu().numpy().tobytes()
        out = []
        for k in range(len(self.sizes)):
            M, flags, n, plen, status, _ = struct.unpack("<fIQQII", raw[32 * k: 32 * k + 32])
            out.append({"M": M, "flags": flags, "n": n, "payload_len": plen, "status": status})
        return out


# ------------------------------------------------------------------ parameter-server exchange
def tlc_plan(sizes, world: int):
    """The exchange plan (R17) computed by the library on the host:
    list of (tensor, lo, hi, owner)."""
    import numpy as np

    sz = np.ascontiguousarray(np.asarray(sizes, dtype=np.uint64))
    k = _lib.tlc_plan_count(len(sz), sz.ctypes.data, int(world))
    if k < 0:
        raise TlcError(TLC_ERR_ARG, "tlc_plan_count")
    t = np.zeros(max(k, 1), np.int32)
    lo = np.zeros(max(k, 1), np.uint64)
    hi = np.zeros(max(k, 1), np.uint64)
    ow = np.zeros(max(k, 1), np.int32)
    rc = _lib.tlc_plan_compute(len(sz), sz.ctypes.data, int(world), k, t.ctypes.data, lo.ctypes.data,
                               hi.ctypes.data, ow.ctypes.data)
    if rc != TLC_OK:
        raise TlcError(rc, "tlc_plan_compute")
    return [(int(t[i]), int(lo[i]), int(hi[i]), int(ow[i])) for i in range(k)]


class _DevArray:
    """__cuda_array_interface__ view of library-owned device memory (fp32)."""

    def __init__(self, ptr, n, device):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f4", "data": (int(ptr), False),
                                         "version": 3, "strides": None}
        self.device = device


def _as_tensor(ptr, n, device):
    if n == 0:
        return torch.zeros(0, dtype=torch.float32, device=device)
    return torch.as_tensor(_DevArray(ptr, n, device), device=device)


class Comm:
    """The library's NCCL communicator.  The 128-byte unique id is created on rank 0
    and broadcast through torch.distributed (plumbing only)."""

    def __init__(self, rank: int = 0, world: int = 1, device=None, group=None):
        import torch.distributed as dist

        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        uid = (ctypes.c_ubyte * 128)()
        if rank == 0:
            rc = _lib.tlc_comm_unique_id(ctypes.cast(uid, ctypes.c_void_p))
            if rc != TLC_OK:
                raise TlcError(rc, "tlc_comm_unique_id")
        if world > 1:
            backend = dist.get_backend(group)
            t = torch.tensor(list(bytes(uid)), dtype=torch.uint8, device=dev if backend == "nccl" else "cpu")
            dist.broadcast(t, src=0, group=group)
            ctypes.memmove(uid, bytes(t.cpu().tolist()), 128)
        self._c = ctypes.c_void_p()
        rc = _lib.tlc_comm_init(ctypes.byref(self._c), ctypes.cast(uid, ctypes.c_void_p), int(rank), int(world),
                                int(dev.index))
        if rc != TLC_OK:
            raise TlcError(rc, "tlc_comm_init")
        self.rank, self.world, self.device = rank, world, dev

    def close(self):
        if self._c:
            _lib.tlc_comm_destroy(self._c)
            self._c = ctypes.c_void_p()


def _check_list(name, ts, sizes, device):
    """The C ABI reads one pointer per configured tensor and that many elements through
    it: check the list length, each tensor's dtype / contiguity / numel and device."""
    if len(ts) != len(sizes):
        raise ValueError(f"{name}: {len(ts)} tensors given, the exchange was created for {len(sizes)}")
    for i, (x, n) in enumerate(zip(ts, sizes)):
        _check_dev(f"{name}[{i}]", x, torch.float32)
        if x.numel() != n:
            raise ValueError(f"{name}[{i}] has {x.numel()} elements, expected {n}")
        if x.device != device:
            raise ValueError(f"{name}[{i}] is on {x.device}, the exchange on {device}")


class Exchange:
    """3LC parameter-server push/pull for a fixed tensor list (include/tlc.h)."""

    def __init__(self, comm: Comm | None, sizes, p2p: bool = False, group=None, _handle=None, _device=None,
                 exact: bool = False):
        """p2p=True: peer-memory mode -- the compressed payloads are read by the consuming
        kernels straight from the producing GPU over NVLink (CUDA IPC mappings set up
        here through torch.distributed); otherwise NCCL send/recv moves them: whole capacity
        regions, or with exact=True the payload bytes after a sizes all-gather.
        (_handle: a virtual rank of a Loopback group, owned by the group.)"""
        import numpy as np

        self.comm, self.sizes = comm, [int(n) for n in sizes]
        self._owned_handle = _handle is None
        if _handle is None:
            sz = np.ascontiguousarray(np.asarray(self.sizes, dtype=np.uint64))
            self._x = ctypes.c_void_p()
            rc = _lib.tlc_exchange_create(ctypes.byref(self._x), comm._c, len(sz), sz.ctypes.data)
            if rc != TLC_OK:
                raise TlcError(rc, "tlc_exchange_create")
            self.device = comm.device
        else:
            self._x = ctypes.c_void_p(_handle)
            self.device = _device
            p2p = False                   # the group has already mapped its peers
        self.num_contexts = _lib.tlc_exchange_num_contexts(self._x)
        self.owned_elements = int(_lib.tlc_exchange_owned_elements(self._x))
        self.owned = _as_tensor(_lib.tlc_exchange_owned_buffer(self._x), self.owned_elements, self.device)
        self.pull_err = _as_tensor(_lib.tlc_exchange_pull_error(self._x), self.owned_elements, self.device)
        self.push_err = _as_tensor(_lib.tlc_exchange_push_error(self._x), sum(self.sizes), self.device)
        self.p2p = bool(p2p) or _handle is not None
        if exact and not self.p2p:
            rc = _lib.tlc_exchange_set_transport(self._x, 1)
            if rc != TLC_OK:
                raise TlcError(rc, "tlc_exchange_set_transport")
        if p2p:
            mine = (ctypes.c_ubyte * 320)()
            rc = _lib.tlc_exchange_ipc_handles(self._x, ctypes.cast(mine, ctypes.c_void_p))
            if rc != TLC_OK:
                raise TlcError(rc, "tlc_exchange_ipc_handles")
            blobs = [bytes(mine)]
            if comm.world > 1:
                import torch.distributed as dist

                blobs = [None] * comm.world
                dist.all_gather_object(blobs, bytes(mine), group=group)
            allh = (ctypes.c_ubyte * (320 * comm.world)).from_buffer_copy(b"".join(blobs))
            rc = _lib.tlc_exchange_ipc_open(self._x, ctypes.cast(allh, ctypes.c_void_p))
            if rc != TLC_OK:
                raise TlcError(rc, "tlc_exchange_ipc_open")

    def contexts(self):
        out = []
        t, o = ctypes.c_int32(), ctypes.c_int32()
        lo, hi, eo, oo = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        for k in range(self.num_contexts):
            _lib.tlc_exchange_context(self._x, k, ctypes.byref(t), ctypes.byref(lo), ctypes.byref(hi),
                                      ctypes.byref(o), ctypes.byref(eo), ctypes.byref(oo))
            out.append({"tensor": t.value, "lo": lo.value, "hi": hi.value, "owner": o.value,
                        "elem_off": eo.value, "owned_off": None if oo.value == 2 ** 64 - 1 else oo.value})
        return out

    def traffic(self):
        """(push bytes, pull bytes) this rank received from other ranks in the last step."""
        out = (ctypes.c_uint64 * 2)()
        rc = _lib.tlc_exchange_traffic(self._x, ctypes.cast(out, ctypes.c_void_p))
        if rc != TLC_OK:
            raise TlcError(rc, "tlc_exchange_traffic")
        return int(out[0]), int(out[1])

    def bind_error_buffers(self, push_err: torch.Tensor | None = None, pull_err: torch.Tensor | None = None):
        """Use caller-owned fp32 device tensors as the push / pull error buffers (checkpointable
        training state; contents used as they are).  The exchange keeps references to them."""
        if push_err is not None:
            _check_dev("push_err", push_err, torch.float32)
            if push_err.numel() != self.push_err.numel() or push_err.device != self.device:
                raise ValueError(f"push_err must hold {self.push_err.numel()} values on {self.device}")
        if pull_err is not None:
            _check_dev("pull_err", pull_err, torch.float32)
            if pull_err.numel() != self.owned_elements or pull_err.device != self.device:
                raise ValueError(f"pull_err must hold {self.owned_elements} values on {self.device}")
        rc = _lib.tlc_exchange_bind_error_buffers(self._x, push_err.data_ptr() if push_err is not None else None,
                                                  pull_err.data_ptr() if pull_err is not None else None)
        if rc != TLC_OK:
            raise TlcError(rc, "tlc_exchange_bind_error_buffers")
        if push_err is not None:
            self.push_err = push_err
        if pull_err is not None and self.owned_elements:
            self.pull_err = pull_err

    def wire_bytes(self, direction: int) -> int:
        return int(_lib.tlc_exchange_wire_bytes(self._x, int(direction)))

    @staticmethod
    def _ptrs(ts):
        return (ctypes.c_void_p * len(ts))(*[x.data_ptr() for x in ts])

    def push(self, grads, s: float, use_zre: bool = True, stream=None):
        _check_list("grads", grads, self.sizes, self.device)
        self._g = self._ptrs(grads)
        rc = _lib.tlc_exchange_push(self._x, ctypes.cast(self._g, ctypes.c_void_p), ctypes.c_float(s),
                                    int(bool(use_zre)), _stream_ptr(stream))
        if rc != TLC_OK:
            raise TlcError(rc, "tlc_exchange_push")

    def pull(self, outs, s: float, use_zre: bool = True, stream=None):
        _check_list("outs", outs, self.sizes, self.device)
        self._o = self._ptrs(outs)
        rc = _lib.tlc_exchange_pull(self._x, ctypes.cast(self._o, ctypes.c_void_p), ctypes.c_float(s),
                                    int(bool(use_zre)), _stream_ptr(stream))
        if rc != TLC_OK:
            raise TlcError(rc, "tlc_exchange_pull")

    def status(self, stream=None) -> int:
        st = ctypes.c_uint()
        rc = _lib.tlc_exchange_status(self._x, ctypes.byref(st), _stream_ptr(stream))
        if rc != TLC_OK:
            raise TlcError(rc, "tlc_exchange_status")
        return int(st.value)

    def status_async(self, dst, stream=None):
        """Enqueue the worst status into `dst` (a 1-element uint32/int32 tensor, pinned
        host or device) without synchronizing."""
        rc = _lib.tlc_exchange_status_async(self._x, ctypes.c_void_p(dst.data_ptr()), _stream_ptr(stream))
        if rc != TLC_OK:
            raise TlcError(rc, "tlc_exchange_status_async")

    def close(self):
        if self._x and self._owned_handle:
            _lib.tlc_exchange_destroy(self._x)
        self._x = ctypes.c_void_p()


class Loopback:
    """W virtual ranks of one exchange on one GPU (tlc_loopback_*): the multi-source push /
    aggregate / pull kernels run exactly as across W GPUs, with plain device pointers for
    the peers' buffers and stream order for the barriers.  ``ranks[r]`` is rank r's view
    (an Exchange: push_err, pull_err, owned, contexts(), status())."""

    def __init__(self, world: int, sizes, device=None):
        import numpy as np

        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.world, self.sizes, self.device = int(world), [int(n) for n in sizes], dev
        sz = np.ascontiguousarray(np.asarray(self.sizes, dtype=np.uint64))
        self._g = ctypes.c_void_p()
        rc = _lib.tlc_loopback_create(ctypes.byref(self._g), self.world, len(sz), sz.ctypes.data, int(dev.index))
        if rc != TLC_OK:
            raise TlcError(rc, "tlc_loopback_create")
        self.ranks = [Exchange(None, self.sizes, _handle=_lib.tlc_loopback_rank(self._g, r), _device=dev)
                      for r in range(self.world)]

    def _ptrs(self, name, per_rank):
        if len(per_rank) != self.world:
            raise ValueError(f"{name}: {len(per_rank)} ranks given, the group has {self.world}")
        flat = []
        for r, ts in enumerate(per_rank):
            _check_list(f"{name}[{r}]", ts, self.sizes, self.device)
            flat.extend(ts)
        return (ctypes.c_void_p * len(flat))(*[x.data_ptr() for x in flat])

    def push(self, grads, s: float, use_zre: bool = True, stream=None):
        """grads[r][i]: rank r's state change of tensor i."""
        self._gp = self._ptrs("grads", grads)
        rc = _lib.tlc_loopback_push(self._g, ctypes.cast(self._gp, ctypes.c_void_p), ctypes.c_float(s),
                                    int(bool(use_zre)), _stream_ptr(stream))
        if rc != TLC_OK:
            raise TlcError(rc, "tlc_loopback_push")

    def pull(self, outs, s: float, use_zre: bool = True, stream=None):
        """outs[r][i]: rank r's full-size output of tensor i (accumulated)."""
        self._op = self._ptrs("outs", outs)
        rc = _lib.tlc_loopback_pull(self._g, ctypes.cast(self._op, ctypes.c_void_p), ctypes.c_float(s),
                                    int(bool(use_zre)), _stream_ptr(stream))
        if rc != TLC_OK:
            raise TlcError(rc, "tlc_loopback_pull")

    def close(self):
        for x in getattr(self, "ranks", []):
            x.close()
        if self._g:
            _lib.tlc_loopback_destroy(self._g)
            self._g = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Aggregate:
    """tlc_aggregate: outs[i] <- mean over W ranks of the decompressed sources[w][i] (rank-
    ordered fp32 fold of the nonzero trits, then IEEE / W; R15), one fused launch pair.
    sources[w] = (payloads, headers) of rank w, as TensorSet keeps them."""

    def __init__(self, outs, sources):
        self.W, self.outs = len(sources), list(outs)
        rows_o = [(None, None, o, None, None, o.numel()) for o in self.outs]
        rows_s = []
        for pays, hdrs in sources:
            if len(pays) != len(self.outs) or len(hdrs) != len(self.outs):
                raise ValueError("every rank needs one payload and header per output")
            rows_s += [(None, None, None, p, h, o.numel()) for p, h, o in zip(pays, hdrs, self.outs)]
        ao, asrc = _descs(rows_o), _descs(rows_s)
        self._a = ctypes.c_void_p()
        rc = _lib.tlc_aggregate_create(ctypes.byref(self._a), self.W, len(self.outs), ctypes.cast(ao, ctypes.c_void_p),
                                       ctypes.cast(asrc, ctypes.c_void_p))
        if rc != TLC_OK:
            raise TlcError(rc, "tlc_aggregate_create")

    def run(self, stream=None):
        rc = _lib.tlc_aggregate_run(self._a, _stream_ptr(stream))
        if rc != TLC_OK:
            raise TlcError(rc, "tlc_aggregate_run")

    def close(self):
        if self._a:
            _lib.tlc_aggregate_destroy(self._a)
            self._a = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------ instrumentation
class _ProfEntry(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char_p), ("launches", ctypes.c_ulonglong), ("total_ms", ctypes.c_double)]


def tlc_launch_count() -> int:
    return int(_lib.tlc_launch_count())


def tlc_prof_enable(on: bool = True) -> None:
    _lib.tlc_prof_enable(int(bool(on)))


def tlc_prof_collect() -> dict:
    """{kernel name: (launches, total device ms)} since the last collect (synchronizes)."""
    arr = (_ProfEntry * 16)()
    k = _lib.tlc_prof_collect(ctypes.cast(arr, ctypes.c_void_p), 16)
    return {arr[i].name.decode(): (int(arr[i].launches), float(arr[i].total_ms)) for i in range(min(k, 16))}


compress = tlc_compress
decompress = tlc_decompress


# ------------------------------------------------------------------ compared designs (Sec. 5.1)
def tlc_stoch_compress(t: torch.Tensor, seed: int, step: int, use_zre: bool = False,
                       payload: torch.Tensor | None = None, hdr: torch.Tensor | None = None,
                       ws: torch.Tensor | None = None, stream=None):
    """"Stoch 3-value + QE": stochastic trits (draws keyed by seed, step and
    element index; reading R22), quartic encoding, optional ZRE.  Decode with tlc_decompress."""
    _check_dev("t", t, torch.float32)
    n = t.numel()
    cap = tlc_max_payload_bytes(n)
    if payload is None:
        payload = torch.empty(max(cap, 1), dtype=torch.uint8, device=t.device)
    if hdr is None:
        hdr = new_header(t.device)
    if ws is None:
        ws = workspace(tlc_compress_workspace_bytes(n), t.device, "compress")
    rc = _lib.tlc_stoch_compress(t.data_ptr(), n, int(seed) & (2 ** 64 - 1), int(step) & (2 ** 64 - 1),
                                 int(bool(use_zre)), payload.data_ptr(), payload.numel(), hdr.data_ptr(),
                                 ws.data_ptr(), ws.numel(), _stream_ptr(stream))
    if rc != TLC_OK:
        raise TlcError(rc, "tlc_stoch_compress")
    return payload, hdr


def tlc_int8_workspace_bytes(n: int) -> int:
    return int(_lib.tlc_int8_workspace_bytes(n))


def tlc_int8_compress(t: torch.Tensor, codes: torch.Tensor | None = None, hdr: torch.Tensor | None = None,
                      ws: torch.Tensor | None = None, stream=None):
    """"8-bit int": codes in [-127,127], hdr M = scale (reading R23)."""
    _check_dev("t", t, torch.float32)
    n = t.numel()
    if codes is None:
        codes = torch.empty(n, dtype=torch.int8, device=t.device)
    _check_dev("codes", codes, torch.int8)
    if codes.numel() < n:
        raise ValueError("codes must hold n elements")
    if hdr is None:
        hdr = new_header(t.device)
    if ws is None:
        ws = workspace(tlc_int8_workspace_bytes(n), t.device, "int8")
    rc = _lib.tlc_int8_compress(t.data_ptr(), n, codes.data_ptr(), hdr.data_ptr(), ws.data_ptr(), ws.numel(),
                                _stream_ptr(stream))
    if rc != TLC_OK:
        raise TlcError(rc, "tlc_int8_compress")
    return codes, hdr


def tlc_int8_decompress(codes: torch.Tensor, hdr: torch.Tensor, n: int, out: torch.Tensor | None = None,
                        mode: int = TLC_MODE_OVERWRITE, stream=None):
    if out is None:
        out = torch.empty(n, dtype=torch.float32, device=codes.device)
    _check_dev("out", out, torch.float32)
    _check_dev("codes", codes, torch.int8)
    _check_dev("hdr", hdr, torch.uint8)
    if out.numel() < n or codes.numel() < n:
        raise ValueError(f"out / codes must hold n = {n} elements")
    rc = _lib.tlc_int8_decompress(codes.data_ptr(), hdr.data_ptr(), n, out.data_ptr(), int(mode),
                                  _stream_ptr(stream))
    if rc != TLC_OK:
        raise TlcError(rc, "tlc_int8_decompress")
    return out
