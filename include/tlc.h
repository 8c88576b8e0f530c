/*
 * tlc.h -- C ABI of the B200-native 3LC state-change compression library
 * (libtlc.so, built from paper_1802_07389_b200/csrc/).
 *
 * The operation is 3LC's compressor (arXiv 1802.07389, Sec. 3, Fig.
 * "fig:compression"; PAPER.md lines cited as P:n, SPEC.md lines as S:n):
 *
 *   (1)  u = err + t                                  P:406-408 (Fig. step 1)
 *   Eq.1 M = fl(max|u| * s),  1 <= s < 2
 *   Eq.2 q = round(u / M) in {-1,0,1}, half away       P:379, reading R1
 *   (a,b) err = u - M*q   (exact, Sterbenz)
 *   (3)  quartic: B[j] = sum_i 3^(4-i) * (q[iP+j]+1)   P:495-510, P = ceil(n/5)
 *   (4)  zero-run: runs of 121 -> 243+(k-2), k<=14
 *
 * and its inverse (ZRE expand, base-3 decode, Eq.3 T_out = M*q).
 * The readings R1..R20 the implementation takes where the paper is silent are
 * listed in DESIGN.md section 3.
 *
 * Conventions for every call below:
 *  - Pointers named t, err, payload, hdr, out, ws are DEVICE pointers (cudaMalloc
 *    / torch CUDA storage) owned by the caller; the library allocates nothing on
 *    the hot path.  `stream` is a cudaStream_t (NULL = legacy default stream).
 *  - Calls enqueue work on `stream` and return without synchronizing.
 *  - Argument errors are returned synchronously (TLC_ERR_ARG / TLC_ERR_CAPACITY /
 *    TLC_ERR_CUDA).  Data errors are raised ON THE DEVICE into hdr->status
 *    (NONFINITE, RANGE, FORMAT); the caller reads them after synchronizing.
 *  - Results are bit-identical to the CPU oracle (oracle/tlc_oracle.c) for
 *    the same inputs: payload bytes, err, and decompressed values (0 ulp).
 */
#ifndef TLC_H
#define TLC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  S:164 (s out of range is a hard error), S:33/S:70 (NaN/Inf
 * rejected), S:214/S:235 (malformed payload), reading R6 (M overflow). */
typedef enum tlc_status {
    TLC_OK = 0,
    TLC_ERR_ARG = 1,        /* null pointer, n == 0, s not in [1,2), bad mode      */
    TLC_ERR_NONFINITE = 2,  /* device: some u = err + t is NaN or +-Inf             */
    TLC_ERR_RANGE = 3,      /* device: max|u| * s overflows fp32                    */
    TLC_ERR_FORMAT = 4,     /* device: payload does not decode to exactly P bytes,  */
                            /*   a literal > 242 without ZRE, or hdr->n != n         */
    TLC_ERR_CAPACITY = 5,   /* payload_cap < ceil(n/5) or workspace too small       */
    TLC_ERR_CUDA = 6,       /* a CUDA runtime call failed (launch, memset)          */
    TLC_ERR_NCCL = 7        /* an NCCL call failed (exchange)                       */
} tlc_status;

/* Device-resident header of one compressed tensor (32 bytes, naturally
 * aligned).  Written by tlc_compress, read by tlc_decompress.  This is the
 * scalar M "sent next to the payload". */
typedef struct tlc_header {
    float M;               /* fl(max|u| * s); 0 for an all-zero u (R5)               */
    uint32_t flags;        /* bit 0: payload is zero-run encoded (TLC_FLAG_ZRE)       */
    uint64_t n;            /* element count of the state-change tensor               */
    uint64_t payload_len;  /* payload bytes: Z with ZRE, P = ceil(n/5) without       */
    uint32_t status;       /* tlc_status raised on the device (0 = OK)               */
    uint32_t reserved;
} tlc_header;

#define TLC_FLAG_ZRE 1u
#define TLC_FLAG_INT8 2u       /* payload is 8-bit int codes (tlc_int8_compress)  */
#define TLC_MODE_OVERWRITE 0   /* out  = M*q                     (Eq. 3)     */
#define TLC_MODE_ACCUMULATE 1  /* out += M*q where q != 0        (reading R16)      */

/* Library version (major*10000 + minor*100 + patch). */
int tlc_version(void);

/* 16 hex digits: sha256 of the csrc/ and include/ sources and the nvcc flags this
 * library was built from (build.py rebuilds whenever it differs from the tree). */
const char *tlc_build_id(void);

/* Human-readable name of a tlc_status value; never NULL. */
const char *tlc_status_string(int status);

/* P = ceil(n/5): quartic bytes of an n-element tensor (step 4).   */
uint64_t tlc_quartic_bytes(uint64_t n);

/* Payload capacity the caller must provide: P (ZRE never expands).    */
uint64_t tlc_max_payload_bytes(uint64_t n);

/* Workspace bytes (device memory, 256-byte aligned) for one compress /
 * decompress of n elements.  A workspace may be reused by consecutive calls on
 * the same stream, never by concurrent calls. */
size_t tlc_compress_workspace_bytes(uint64_t n);
size_t tlc_decompress_workspace_bytes(uint64_t n);

/*
 * tlc_compress -- Fig. "fig:compression" steps (1),(2),(a),(b),(3),(4).
 *
 *  t        [in]  fp32[n], the state change T_in (gradient or model delta).
 *  err      [in/out] fp32[n], the error-accumulation buffer of this tensor's
 *                 compression context.  Zero-initialised by the
 *                 caller before the first call (R20); one writer at a time
 *                 (S:167).  Left unmodified when a data error is raised.
 *                 Must not overlap t, payload or hdr (TLC_ERR_ARG: any two of
 *                 the ranges t[n], err[n], payload[payload_cap], hdr share a byte).
 *  n        number of elements, >= 1.
 *  s        sparsity multiplier, fp32, 1 <= s < 2.
 *  use_zre  nonzero: apply zero-run encoding (step 4); 0: payload = quartic bytes.
 *  payload  [out] u8[payload_cap], payload_cap >= tlc_max_payload_bytes(n).
 *  hdr      [out] device header: M, flags, n, payload_len, status.
 *  ws       device workspace of >= tlc_compress_workspace_bytes(n) bytes.
 *  stream   cudaStream_t.
 *
 * Returns TLC_OK once enqueued; TLC_ERR_ARG / TLC_ERR_CAPACITY / TLC_ERR_CUDA
 * synchronously.  Device-side: hdr->status = NONFINITE / RANGE (R6).
 * Layout: t, err flat row-major fp32; payload bytes in stream order.
 */
int tlc_compress(const float *t, float *err, uint64_t n, float s, int use_zre,
                 uint8_t *payload, uint64_t payload_cap, tlc_header *hdr,
                 void *ws, size_t ws_bytes, void *stream);

/*
 * tlc_decompress -- the reverse path: ZRE expand, quartic decode
 * (P:512-522), dequantize T_out = M*q (Eq. 3).
 *
 *  payload  [in] u8[hdr->payload_len] as written by tlc_compress (or received).
 *  hdr      [in/out] header of that payload; hdr->status is set to
 *           TLC_ERR_FORMAT on a malformed payload.  If hdr->status is already
 *           nonzero the call does nothing on the device.
 *  n        element count; must equal hdr->n (checked on the device).
 *  out      [out or in/out] fp32[n].  mode TLC_MODE_OVERWRITE writes M*q;
 *           TLC_MODE_ACCUMULATE adds M*q only where q != 0 (R16), leaving the
 *           other elements untouched (used to apply pulled model deltas and
 *           to aggregate pushes in rank order, R15).
 *  ws       device workspace of >= tlc_decompress_workspace_bytes(n) bytes.
 *
 * On FORMAT no byte outside out[0, n) is written; the contents of out are
 * then unspecified.
 */
int tlc_decompress(const uint8_t *payload, tlc_header *hdr, uint64_t n, float *out,
                   int mode, void *ws, size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------------
 * Compared designs of the paper's evaluation (Sec. 5.1) that share
 * the 3LC kernels.  Same conventions as above.
 *
 * tlc_stoch_compress -- "Stoch 3-value + QE": stochastic 3-value
 *   quantization "similar to TernGrad (but without gradient clipping)" -- each
 *   element x becomes sign(x) with probability |x|/m, m = max|t| (P:412-416,
 *   expectation = input), no sparsity multiplier, no error buffer -- then the
 *   3LC quartic encoding (1.6 bits/value) and, if use_zre, zero-run encoding.
 *   The draws are a pure function of (seed, step, element index): reading R22
 *   of DESIGN.md (Philox4x32-10, counter (e/4, step), key seed, word e%4;
 *   q = sign(x) iff (w>>8)*2^-24 < fl(|x|/m)).  Decode with tlc_decompress
 *   (hdr->M = m).  t: fp32[n] in; payload: u8[payload_cap >= ceil(n/5)] out;
 *   hdr out (status NONFINITE on NaN/Inf in t); ws >= tlc_compress_workspace_bytes(n).
 *
 * tlc_int8_compress -- "8-bit int": 255 values [-127,127], -128
 *   unused.  scale = fl(max|t|/127), code = clamp(round_half_away(fl(t/scale)))
 *   (reading R23).  codes: int8[n] out; hdr->M = scale, hdr->flags =
 *   TLC_FLAG_INT8, hdr->payload_len = n; ws >= tlc_int8_workspace_bytes(n).
 * tlc_int8_decompress -- out = scale*code (mode OVERWRITE) or out += scale*code
 *   where code != 0 (mode ACCUMULATE).  FORMAT in hdr->status if the header is
 *   not an int8 header of n elements with a finite scale >= +0.
 */
int tlc_stoch_compress(const float *t, uint64_t n, uint64_t seed, uint64_t step, int use_zre,
                       uint8_t *payload, uint64_t payload_cap, tlc_header *hdr,
                       void *ws, size_t ws_bytes, void *stream);
size_t tlc_int8_workspace_bytes(uint64_t n);
int tlc_int8_compress(const float *t, uint64_t n, int8_t *codes, tlc_header *hdr,
                      void *ws, size_t ws_bytes, void *stream);
int tlc_int8_decompress(const int8_t *codes, tlc_header *hdr, uint64_t n, float *out, int mode,
                        void *stream);

/* ---------------------------------------------------------------------------
 * Batches of tensors (SURVEY 8(a) "small-tensor regime"; BASELINE configs[1]
 * and [4]: the per-layer gradient tensors of ResNet-110 / ResNet-50 /
 * BERT-large).  A batch is a fixed list of independent tensors, each with its
 * own error buffer, payload and header -- the per-tensor compression contexts
 * of the paper -- compressed (decompressed) by one set of kernel
 * launches over all of them, with results identical to one tlc_compress /
 * tlc_decompress call per tensor.
 *
 * tlc_batch_create    `descs` is a HOST array of `count` descriptors (device
 *                     pointers inside); the batch uploads its tensor table and
 *                     allocates its own device workspace once.  Fields used by
 *                     compress: t, err, payload (capacity >= ceil(n/5)), hdr,
 *                     n; by decompress: payload, hdr, out, n.  1 <= n < 2^42.
 * tlc_batch_update    replaces the pointers (same n's); synchronous upload.
 * tlc_batch_compress  / tlc_batch_decompress enqueue on `stream`, no host
 *                     traffic, no allocation (CUDA-graph capturable); per-tensor
 *                     data errors land in each tensor's hdr->status.
 */
typedef struct tlc_tensor_desc {
    const float *t;
    float *err;
    float *out;
    uint8_t *payload;
    tlc_header *hdr;
    uint64_t n;
} tlc_tensor_desc;

typedef struct tlc_batch tlc_batch;

int tlc_batch_create(tlc_batch **batch, int count, const tlc_tensor_desc *descs);
int tlc_batch_update(tlc_batch *batch, const tlc_tensor_desc *descs);
int tlc_batch_destroy(tlc_batch *batch);
size_t tlc_batch_workspace_bytes(const tlc_batch *batch);
int tlc_batch_compress(tlc_batch *batch, float s, int use_zre, void *stream);
int tlc_batch_decompress(tlc_batch *batch, int mode, void *stream);

/* ---------------------------------------------------------------------------
 * Parameter-server exchange over NCCL.
 *
 * The paper's data-parallel architecture: workers push compressed
 * state changes, servers aggregate ("average the gradients") and
 * update, workers pull compressed model deltas which the server compresses ONCE
 * and shares.  Here every rank is a worker and the owner (server)
 * of a shard of the compression contexts given by the plan (reading R17).
 *
 * tlc_comm_unique_id  writes a 128-byte NCCL unique id to `out` (host memory);
 *                     rank 0 creates it and the caller broadcasts it (e.g. with
 *                     torch.distributed).
 * tlc_comm_init       creates the library's NCCL communicator on `device`.
 * tlc_plan_count / tlc_plan_compute  the deterministic plan (R17) for `world`
 *                     ranks over host `sizes[num_tensors]`: context k covers
 *                     elements [lo[k], hi[k]) of tensor[k] and is owned by
 *                     owner[k].  Pure host computation (no GPU).
 * tlc_exchange_create (world <= 8) allocates every buffer of the exchange for the tensor
 *                     list (error buffers zeroed, R20): push error buffers for
 *                     all contexts, the owned (aggregate / delta) buffer and
 *                     pull error buffers for this rank's contexts, send/receive
 *                     regions in capacity layout (ceil(n/5) bytes per context).
 * tlc_exchange_push   grads: host array of num_tensors DEVICE pointers (fp32,
 *                     the local state changes).  Compresses every context with
 *                     its push error buffer, sends each owner its payloads and
 *                     headers, and leaves in the owned buffer (see
 *                     tlc_exchange_owned_buffer) the mean over ranks of the
 *                     decompressed pushes: rank-ordered sum from +0, zero trits
 *                     skipped, then / world in fp32 (R15) -- one fused
 *                     decompress-aggregate pass over the W received payloads.  The caller may turn
 *                     that mean into a model delta in place (R18) before pull.
 * tlc_exchange_pull   compresses this rank's owned buffer once with its pull
 *                     error buffers, all-gathers every owner's payloads, and
 *                     adds the decompressed delta (where q != 0, R16) into
 *                     outs: host array of num_tensors DEVICE pointers to
 *                     full-size fp32 tensors.
 * tlc_exchange_status synchronizes `stream` and returns the worst device status
 *                     of the last step: this rank's own pushes and every
 *                     context's shared pull (which carries any rank's push
 *                     failure, R24); with NCCL also the received pushes.
 * tlc_exchange_status_async  the same worst status, written by an async copy
 *                     enqueued on `stream` to `dst` (pinned host or device
 *                     memory, 4 bytes, owned by the caller); no host sync.
 * Push/pull enqueue on `stream`, allocate nothing and do not synchronize the
 * host (a descriptor upload happens when the grads/outs pointers change).
 * Ordering: push and pull strictly alternate (push, pull, push, ...); a call out
 * of turn returns TLC_ERR_ARG.  Every rank must issue its pushes and pulls on
 * one stream: in peer-memory mode the two flag barriers of a step order both the
 * reads of a rank's send/pull buffers by the other ranks and that rank's next
 * overwrite of them, which holds only if nothing of the next phase can start
 * before this rank's barrier kernel (stream order).
 * Failed pushes (reading R24): if any rank's push of a context fails (NaN/Inf
 * in u, M overflow, malformed payload), the owner's mean of that context is NaN
 * (owned buffer), its pull compression then raises NONFINITE, and every rank's
 * apply leaves that context's outputs untouched; tlc_exchange_status on every
 * rank reports it.
 * CUDA graphs: in peer-memory mode a push or pull may be captured (stream
 * capture) once the grads/outs pointers have been seen by an eager call; the
 * flag-barrier epochs are counted on the device, so replays stay ordered.  The
 * NCCL transport returns TLC_ERR_ARG when called on a capturing stream.
 */
typedef struct tlc_comm tlc_comm;
typedef struct tlc_exchange tlc_exchange;

int tlc_comm_unique_id(void *out);
int tlc_comm_init(tlc_comm **comm, const void *unique_id, int rank, int world, int device);
int tlc_comm_destroy(tlc_comm *comm);
int tlc_plan_count(int num_tensors, const uint64_t *sizes, int world);
int tlc_plan_compute(int num_tensors, const uint64_t *sizes, int world, int cap, int32_t *tensor,
                     uint64_t *lo, uint64_t *hi, int32_t *owner);
int tlc_exchange_create(tlc_exchange **x, tlc_comm *comm, int num_tensors, const uint64_t *sizes);
int tlc_exchange_destroy(tlc_exchange *x);
int tlc_exchange_num_contexts(const tlc_exchange *x);
int tlc_exchange_context(const tlc_exchange *x, int k, int32_t *tensor, uint64_t *lo, uint64_t *hi,
                         int32_t *owner, uint64_t *elem_off, uint64_t *owned_off);
uint64_t tlc_exchange_owned_elements(const tlc_exchange *x);
float *tlc_exchange_owned_buffer(tlc_exchange *x);
float *tlc_exchange_push_error(tlc_exchange *x);
float *tlc_exchange_pull_error(tlc_exchange *x);
uint64_t tlc_exchange_wire_bytes(const tlc_exchange *x, int direction /* 0 push, 1 pull */);
/* tlc_exchange_bind_error_buffers: make caller-owned DEVICE buffers the exchange's
 * error-accumulation state (the contexts of P:400-404 are training state to
 * checkpoint): push_err[tlc_exchange_push_error's length = every context] and
 * pull_err[tlc_exchange_owned_elements] (either may be NULL: unchanged).  Their
 * contents are used as they are (zero them for a fresh start, R20, or restore a
 * checkpoint); the caller keeps them alive and unaliased until the exchange is
 * destroyed.  Synchronizes the device. */
int tlc_exchange_bind_error_buffers(tlc_exchange *x, float *push_err, float *pull_err);
/* tlc_exchange_set_transport: the NCCL transport's mode (between steps, not in peer-memory
 * or loopback mode).  0 (default): every owner's whole capacity region (ceil(n/5) bytes
 * per context) and the headers move each direction, no host synchronization.  1 (exact,
 * "sizes first"): each rank packs its payloads, the packing offsets are all-gathered
 * (ncclAllGather), the host waits for them once per direction, then grouped
 * ncclSend/ncclRecv move exactly the payload bytes, unpacked on the receiver.  Same
 * results bit for bit.  Push/pull in mode 1 synchronize `stream` once each. */
int tlc_exchange_set_transport(tlc_exchange *x, int mode);
int tlc_exchange_push(tlc_exchange *x, const float *const *grads, float s, int use_zre, void *stream);
int tlc_exchange_pull(tlc_exchange *x, float *const *outs, float s, int use_zre, void *stream);
int tlc_exchange_status(tlc_exchange *x, unsigned int *status, void *stream);
int tlc_exchange_status_async(tlc_exchange *x, unsigned int *dst, void *stream);

/* Peer-memory mode (one rank per GPU on an NVLink/NVSwitch box).  After
 * tlc_exchange_create, every rank calls tlc_exchange_ipc_handles (writes 5 x 64
 * bytes of CUDA IPC handles of its send / pull buffers and flag slots to host
 * memory `out`), the caller all-gathers them in rank order (W x 320 bytes) and
 * every rank calls tlc_exchange_ipc_open.  From then on push/pull move no data
 * with NCCL: a flag barrier over peer memory orders the phases, and the owner's
 * fused aggregation kernels (and every rank's apply kernels) read the compressed
 * payloads -- exactly their payload_len bytes -- straight from the producing GPU
 * over NVLink, with the seek entries (8 bytes per 4096 quartic positions) the
 * producer's zero-run encoder wrote behind its buffers, so no consumer rescans a
 * payload (env TLC_NO_PRODSEEK=1: the consumers scan).  Results are identical to
 * the NCCL mode. */
int tlc_exchange_ipc_handles(tlc_exchange *x, void *out);
int tlc_exchange_ipc_open(tlc_exchange *x, const void *all);

/* Loopback group (single GPU): `world` (1..8) virtual ranks of one exchange in
 * one process on `device`, for testing and profiling the multi-source path on
 * one B200.  Each virtual rank is a full tlc_exchange (tlc_loopback_rank: its
 * error buffers, owned buffer and contexts through the tlc_exchange_* queries;
 * tlc_exchange_push/pull on it return TLC_ERR_ARG) whose peers' buffers are
 * plain device pointers.  tlc_loopback_push takes `grads`, a host array of
 * world x num_tensors DEVICE pointers (rank-major: grads[r*num_tensors + i]),
 * and runs every rank's push compression, then every owner's K4 + fused
 * aggregation reading all ranks' payloads; tlc_loopback_pull likewise takes
 * outs[r*num_tensors + i] and runs every owner's pull compression, then every
 * rank's apply reading all owners' payloads.  Stream order replaces the flag
 * barriers; results are those of a world-GPU exchange, bit for bit.  Push and
 * pull alternate (TLC_ERR_ARG otherwise).  The group owns its ranks; destroy
 * the group, not the ranks. */
typedef struct tlc_loopback tlc_loopback;
int tlc_loopback_create(tlc_loopback **group, int world, int num_tensors, const uint64_t *sizes, int device);
int tlc_loopback_destroy(tlc_loopback *group);
tlc_exchange *tlc_loopback_rank(tlc_loopback *group, int rank);
int tlc_loopback_push(tlc_loopback *group, const float *const *grads, float s, int use_zre, void *stream);
int tlc_loopback_pull(tlc_loopback *group, float *const *outs, float s, int use_zre, void *stream);

/* Standalone aggregation: the server's "average the gradients" over
 * `world` (1..8) compressed copies of a list of `count` tensors, for callers that
 * move the payloads themselves (e.g. a single-server simulator).  outs: HOST
 * array of count descriptors (out = fp32[n] DEVICE output, n); srcs: HOST array
 * of world x count descriptors, rank-major (srcs[w*count + i]: payload and hdr
 * of rank w's compression of tensor i, n).  tlc_aggregate_run overwrites every
 * out with fl(fold_w M_w q_w / world): the rank-ordered fp32 sum from +0 of the
 * nonzero dequantized trits, then the IEEE quotient (R15), in one fused pass
 * (K4 scan + K5m); a tensor with any source whose header is not OK gets NaN
 * (R24).  Enqueues on `stream`; the descriptors are fixed at create. */
typedef struct tlc_aggregate tlc_aggregate;
int tlc_aggregate_create(tlc_aggregate **agg, int world, int count, const tlc_tensor_desc *outs,
                         const tlc_tensor_desc *srcs);
int tlc_aggregate_run(tlc_aggregate *agg, void *stream);
int tlc_aggregate_destroy(tlc_aggregate *agg);

/* Bytes this rank received from other ranks in the last push (out[0]) and pull
 * (out[1]): capacity regions + headers with NCCL; exactly the payload_len (+
 * header) bytes read over NVLink in peer-memory mode.  Synchronizes the device. */
int tlc_exchange_traffic(tlc_exchange *x, uint64_t *out);

/* ---------------------------------------------------------------------------
 * 3LC1 blobs (host memory only): one compressed tensor as
 * "3LC1" | version 1 | codec (0 = 3LC pipeline incl. Stoch 3-value + QE, 2 =
 * 8-bit int) | flags (bit 0 = ZRE) | rank | rank x u64 dims | f32 M |
 * u64 payload_len | payload, little-endian -- the file format of oracle-parity
 * dumps.  Bits/value counts the payload only (R14).
 *
 * tlc_blob_size   bytes of a blob with `rank` dims and payload_len payload bytes
 *                 (0 if rank is outside 0..255).
 * tlc_blob_write  hdr: a HOST copy of a successful compression's header
 *                 (status OK, n = product of dims); payload: host, hdr->
 *                 payload_len bytes; writes tlc_blob_size(...) bytes to `out`
 *                 (TLC_ERR_CAPACITY if out_cap is short) and their count to
 *                 *written.
 * tlc_blob_read   parses `len` bytes: fills *hdr (M, flags, n = product of dims,
 *                 payload_len, status 0), *rank and dims[0..rank) (dims_cap
 *                 entries available, else TLC_ERR_CAPACITY), and the payload's
 *                 offset in the blob.  TLC_ERR_FORMAT for a bad magic / version
 *                 / codec / flags, a truncated or overlong blob, or a payload
 *                 length impossible for n ("malformed header").
 */
uint64_t tlc_blob_size(int rank, uint64_t payload_len);
int tlc_blob_write(const tlc_header *hdr, int rank, const uint64_t *dims, const uint8_t *payload,
                   uint8_t *out, uint64_t out_cap, uint64_t *written);
int tlc_blob_read(const uint8_t *blob, uint64_t len, tlc_header *hdr, int *rank, uint64_t *dims,
                  int dims_cap, uint64_t *payload_offset);

/* ---------------------------------------------------------------------------
 * Instrumentation (host-side, not part of the method).
 *
 * tlc_launch_count: number of kernels this library has launched in the
 *   process so far (bench.py reports the difference over the timed region).
 * tlc_prof_enable: when on, every library kernel launch is bracketed by a pair
 *   of CUDA events on its stream.
 * tlc_prof_collect: synchronizes the recorded events and writes up to `cap`
 *   entries {kernel name (static string), launches, summed device ms} to
 *   `out` (host memory); returns the number of distinct kernels seen and
 *   resets the record.
 */
typedef struct tlc_prof_entry {
    const char *name;
    unsigned long long launches;
    double total_ms;
} tlc_prof_entry;

unsigned long long tlc_launch_count(void);
void tlc_prof_enable(int on);
int tlc_prof_collect(tlc_prof_entry *out, int cap);

#ifdef __cplusplus
}
#endif

#endif /* TLC_H */
