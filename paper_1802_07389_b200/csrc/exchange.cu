// exchange.cu -- the parameter-server push/pull of 3LC over NCCL.
//
// The paper's data-parallel architecture (fig. push-and-pull): workers
// push compressed state changes, the servers aggregate ("average the gradients",
// P:184-185) and update, and workers pull compressed model deltas, which the
// server compresses ONCE and shares with every worker.  On an
// NVSwitch box every rank is both a worker and the server ("owner") of a shard
// of the compression contexts (plan R17):
//
//   push   compress every context with this rank's push error buffer (one
//          segment-table launch of K1-K3 for all contexts) straight into a send
//          buffer laid out by owner; one grouped ncclSend/ncclRecv per peer moves
//          each owner's region (capacity layout: ceil(n/5) bytes per context, so
//          no host-side size exchange is needed) plus the headers; the owner
//          decompresses the W payloads of each owned context in rank order into a
//          zeroed sum (ACCUMULATE, R15) and divides by W in fp32.
//   pull   the owner compresses its shard of the (caller-updated) mean once with
//          its pull error buffer into its region of the pull buffer; a grouped
//          send/recv gives every rank every owner's region; every rank applies all
//          contexts to its full-size output (ACCUMULATE, R16).
//
// Buffers are allocated once by tlc_exchange_create; push/pull allocate nothing
// and never synchronize the host.
#include <algorithm>
#include <cstring>
#include <nccl.h>
#include <vector>

#include "tlc_device.cuh"
#include "tlc_launch.h"

struct tlc_comm {
    ncclComm_t nccl;
    int rank, world, device;
};

namespace tlc {

namespace {
constexpr size_t kAlign = 16;
size_t a16(size_t x) { return (x + kAlign - 1) & ~(kAlign - 1); }

struct Ctx {
    int tensor;
    uint64_t lo, hi, n, cap;
    int owner;
    int slot;           // index among the owner's contexts
    size_t region_off;  // byte offset inside the owner's region
    size_t elem_off;    // offset in the flat push error buffer
    size_t owned_off;   // offset in the owner's flat owned buffer (valid on the owner)
};

// worst (largest) status over a header array -> *out (atomicMax)
__global__ void tlc_status_kernel(const tlc_header *__restrict__ h, int count, unsigned int *out) {
    unsigned int m = 0;
    for (int i = threadIdx.x; i < count; i += blockDim.x) m = max(m, h[i].status);
    m = __reduce_max_sync(0xffffffffu, m);
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}
}  // namespace

// ------------------------------------------------------------------ the plan (R17)
// Whole tensors go to owners, largest first, each to the least-loaded rank (ties:
// lower tensor id first, lower rank wins); a tensor larger than ceil(N/W) is cut
// into ceil(n/ceil(N/W)) contiguous shards whose sizes differ by at most one
// (the first n mod m shards get the extra element).
static std::vector<Ctx> make_plan(int T, const uint64_t *sizes, int W) {
    uint64_t N = 0;
    for (int i = 0; i < T; i++) N += sizes[i];
    const uint64_t cap = std::max<uint64_t>(1, (N + W - 1) / W);
    std::vector<Ctx> ctx;
    for (int i = 0; i < T; i++) {
        const uint64_t n = sizes[i];
        if (n == 0) continue;
        const uint64_t m = n > cap ? (n + cap - 1) / cap : 1;
        const uint64_t base = n / m, rem = n % m;
        uint64_t lo = 0;
        for (uint64_t k = 0; k < m; k++) {
            const uint64_t len = base + (k < rem ? 1 : 0);
            Ctx c{};
            c.tensor = i;
            c.lo = lo;
            c.hi = lo + len;
            c.n = len;
            c.cap = (len + 4) / 5;
            ctx.push_back(c);
            lo += len;
        }
    }
    std::vector<int> order(ctx.size());
    for (size_t k = 0; k < ctx.size(); k++) order[k] = (int)k;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return ctx[a].n > ctx[b].n; });
    std::vector<uint64_t> load(W, 0);
    for (int k : order) {
        int best = 0;
        for (int r = 1; r < W; r++)
            if (load[r] < load[best]) best = r;
        ctx[k].owner = best;
        load[best] += ctx[k].n;
    }
    return ctx;
}

}  // namespace tlc

using namespace tlc;

struct tlc_exchange {
    tlc_comm *comm = nullptr;
    int W = 1, me = 0;
    std::vector<Ctx> ctx;
    std::vector<std::vector<int>> owned;      // per owner: its contexts in context order
    std::vector<size_t> region_start, region_bytes, hdr_start;
    size_t total_region = 0;
    uint64_t owned_elems = 0, total_elems = 0;
    std::vector<uint64_t> tensor_sizes;
    // device memory
    float *push_err = nullptr, *owned_buf = nullptr, *pull_err = nullptr;
    uint8_t *push_send = nullptr, *push_recv = nullptr, *pull_buf = nullptr;
    tlc_header *push_hdr_send = nullptr, *push_hdr_recv = nullptr, *pull_hdr = nullptr;
    unsigned int *d_status = nullptr;
    // segment tables: push compress (all contexts), aggregation (owned contexts A and
    // the W x |A| received payloads X), pull compress (owned), apply (all contexts)
    Table push_tab, pullc_tab, apply_tab, a_tab, x_tab;
    std::vector<const float *> last_grads;
    std::vector<float *> last_outs;
};

static int cuda_ok(cudaError_t e) { return e == cudaSuccess ? TLC_OK : TLC_ERR_CUDA; }
static int nccl_ok(ncclResult_t r) { return r == ncclSuccess ? TLC_OK : TLC_ERR_NCCL; }

extern "C" {

int tlc_comm_unique_id(void *out) {
    if (!out) return TLC_ERR_ARG;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return TLC_ERR_NCCL;
    std::memcpy(out, &id, sizeof(id));
    return TLC_OK;
}

int tlc_comm_init(tlc_comm **c, const void *unique_id, int rank, int world, int device) {
    if (!c || !unique_id || world < 1 || rank < 0 || rank >= world) return TLC_ERR_ARG;
    if (cudaSetDevice(device) != cudaSuccess) return TLC_ERR_CUDA;
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    auto *cm = new tlc_comm{};
    cm->rank = rank;
    cm->world = world;
    cm->device = device;
    if (ncclCommInitRank(&cm->nccl, world, id, rank) != ncclSuccess) {
        delete cm;
        return TLC_ERR_NCCL;
    }
    *c = cm;
    return TLC_OK;
}

int tlc_comm_destroy(tlc_comm *c) {
    if (!c) return TLC_ERR_ARG;
    const int rc = nccl_ok(ncclCommDestroy(c->nccl));
    delete c;
    return rc;
}

int tlc_plan_count(int num_tensors, const uint64_t *sizes, int world) {
    if (num_tensors < 0 || (num_tensors && !sizes) || world < 1) return -1;
    return (int)make_plan(num_tensors, sizes, world).size();
}

int tlc_plan_compute(int num_tensors, const uint64_t *sizes, int world, int cap, int32_t *tensor,
                     uint64_t *lo, uint64_t *hi, int32_t *owner) {
    if (num_tensors < 0 || (num_tensors && !sizes) || world < 1) return TLC_ERR_ARG;
    const std::vector<Ctx> ctx = make_plan(num_tensors, sizes, world);
    if ((int)ctx.size() > cap || !tensor || !lo || !hi || !owner) return TLC_ERR_CAPACITY;
    for (size_t k = 0; k < ctx.size(); k++) {
        tensor[k] = ctx[k].tensor;
        lo[k] = ctx[k].lo;
        hi[k] = ctx[k].hi;
        owner[k] = ctx[k].owner;
    }
    return TLC_OK;
}

int tlc_exchange_destroy(tlc_exchange *x) {
    if (!x) return TLC_ERR_ARG;
    void *dev[] = {x->push_err, x->owned_buf, x->pull_err, x->push_send, x->push_recv, x->pull_buf,
                   x->push_hdr_send, x->push_hdr_recv, x->pull_hdr, x->d_status};
    for (void *p : dev)
        if (p) cudaFree(p);
    x->push_tab.release();
    x->pullc_tab.release();
    x->apply_tab.release();
    x->a_tab.release();
    x->x_tab.release();
    delete x;
    return TLC_OK;
}

int tlc_exchange_create(tlc_exchange **out, tlc_comm *comm, int num_tensors, const uint64_t *sizes) {
    if (!out || !comm || num_tensors < 1 || !sizes) return TLC_ERR_ARG;
    if (comm->world > 8) return TLC_ERR_ARG;   // the fused aggregation holds <= 8 sources per tile
    auto *x = new tlc_exchange{};
    x->comm = comm;
    x->W = comm->world;
    x->me = comm->rank;
    x->tensor_sizes.assign(sizes, sizes + num_tensors);
    x->ctx = make_plan(num_tensors, sizes, x->W);
    const int C = (int)x->ctx.size();
    x->owned.assign(x->W, {});
    for (int k = 0; k < C; k++) x->owned[x->ctx[k].owner].push_back(k);
    x->region_start.assign(x->W, 0);
    x->region_bytes.assign(x->W, 0);
    x->hdr_start.assign(x->W, 0);
    size_t pos = 0, hpos = 0, elem = 0;
    for (int o = 0; o < x->W; o++) {
        x->region_start[o] = pos;
        x->hdr_start[o] = hpos;
        size_t off = 0;
        int slot = 0;
        for (int k : x->owned[o]) {
            x->ctx[k].region_off = off;
            x->ctx[k].slot = slot++;
            off += a16(x->ctx[k].cap);
        }
        x->region_bytes[o] = off;
        pos += off;
        hpos += x->owned[o].size();
    }
    x->total_region = pos;
    for (int k = 0; k < C; k++) {
        x->ctx[k].elem_off = elem;
        elem += x->ctx[k].n;
    }
    x->total_elems = elem;
    uint64_t oe = 0;
    for (int k : x->owned[x->me]) {
        x->ctx[k].owned_off = oe;
        oe += x->ctx[k].n;
    }
    x->owned_elems = oe;
    const int nown = (int)x->owned[x->me].size();
    const size_t own_region = x->region_bytes[x->me];
    int rc = TLC_OK;
    auto alloc = [&](void **p, size_t bytes) {
        if (rc == TLC_OK && cudaMalloc(p, std::max<size_t>(bytes, 256)) != cudaSuccess) rc = TLC_ERR_CUDA;
    };
    alloc((void **)&x->push_err, x->total_elems * sizeof(float));
    alloc((void **)&x->owned_buf, x->owned_elems * sizeof(float));
    alloc((void **)&x->pull_err, x->owned_elems * sizeof(float));
    alloc((void **)&x->push_send, x->total_region);
    alloc((void **)&x->push_recv, (size_t)x->W * own_region);
    alloc((void **)&x->pull_buf, x->total_region);
    alloc((void **)&x->push_hdr_send, (size_t)C * sizeof(tlc_header));
    alloc((void **)&x->push_hdr_recv, (size_t)x->W * nown * sizeof(tlc_header));
    alloc((void **)&x->pull_hdr, (size_t)C * sizeof(tlc_header));
    alloc((void **)&x->d_status, 256);
    if (rc == TLC_OK) {
        // error buffers start at zero (R20)
        rc = cuda_ok(cudaMemset(x->push_err, 0, std::max<size_t>(x->total_elems * sizeof(float), 256)));
        if (rc == TLC_OK) rc = cuda_ok(cudaMemset(x->pull_err, 0, std::max<size_t>(x->owned_elems * sizeof(float), 256)));
    }
    if (rc == TLC_OK && nown) {
        // tables that only point at exchange-owned memory are built once
        std::vector<tlc_tensor_desc> agg(nown), pullc(nown);
        for (int q = 0; q < nown; q++) {
            const Ctx &c = x->ctx[x->owned[x->me][q]];
            tlc_tensor_desc &d = pullc[q];
            d = tlc_tensor_desc{};
            d.t = x->owned_buf + c.owned_off;
            d.err = x->pull_err + c.owned_off;
            d.payload = x->pull_buf + x->region_start[x->me] + c.region_off;
            d.hdr = x->pull_hdr + x->hdr_start[x->me] + c.slot;
            d.n = c.n;
        }
        rc = x->pullc_tab.create(pullc.data(), nown, true, nullptr);
        std::vector<tlc_tensor_desc> xs((size_t)x->W * nown);
        for (int q = 0; q < nown; q++) {
            const Ctx &c = x->ctx[x->owned[x->me][q]];
            tlc_tensor_desc &d = agg[q];
            d = tlc_tensor_desc{};
            d.out = x->owned_buf + c.owned_off;
            d.hdr = x->push_hdr_recv + c.slot;      // only n / out are used through A
            d.n = c.n;
            for (int w = 0; w < x->W; w++) {
                tlc_tensor_desc &e = xs[(size_t)w * nown + q];
                e = tlc_tensor_desc{};
                e.payload = x->push_recv + (size_t)w * own_region + c.region_off;
                e.hdr = x->push_hdr_recv + (size_t)w * nown + c.slot;
                e.n = c.n;
            }
        }
        if (rc == TLC_OK) rc = x->a_tab.create(agg.data(), nown, false, nullptr);
        if (rc == TLC_OK) rc = x->x_tab.create(xs.data(), x->W * nown, false, nullptr);
    }
    if (rc != TLC_OK) {
        tlc_exchange_destroy(x);
        return rc;
    }
    *out = x;
    return TLC_OK;
}

int tlc_exchange_num_contexts(const tlc_exchange *x) { return x ? (int)x->ctx.size() : -1; }

uint64_t tlc_exchange_owned_elements(const tlc_exchange *x) { return x ? x->owned_elems : 0; }

float *tlc_exchange_owned_buffer(tlc_exchange *x) { return x ? x->owned_buf : nullptr; }

float *tlc_exchange_push_error(tlc_exchange *x) { return x ? x->push_err : nullptr; }

float *tlc_exchange_pull_error(tlc_exchange *x) { return x ? x->pull_err : nullptr; }

int tlc_exchange_context(const tlc_exchange *x, int k, int32_t *tensor, uint64_t *lo, uint64_t *hi,
                         int32_t *owner, uint64_t *elem_off, uint64_t *owned_off) {
    if (!x || k < 0 || k >= (int)x->ctx.size()) return TLC_ERR_ARG;
    const Ctx &c = x->ctx[k];
    if (tensor) *tensor = c.tensor;
    if (lo) *lo = c.lo;
    if (hi) *hi = c.hi;
    if (owner) *owner = c.owner;
    if (elem_off) *elem_off = c.elem_off;
    if (owned_off) *owned_off = c.owner == x->me ? c.owned_off : ~0ull;
    return TLC_OK;
}

uint64_t tlc_exchange_wire_bytes(const tlc_exchange *x, int direction) {
    // bytes this rank sends per call (capacity layout, payload + headers)
    if (!x) return 0;
    uint64_t b = 0;
    if (direction == 0) {
        for (int o = 0; o < x->W; o++)
            if (o != x->me) b += x->region_bytes[o] + x->owned[o].size() * sizeof(tlc_header);
    } else {
        b = (uint64_t)(x->W - 1) * (x->region_bytes[x->me] + x->owned[x->me].size() * sizeof(tlc_header));
    }
    return b;
}

int tlc_exchange_push(tlc_exchange *x, const float *const *grads, float s, int use_zre, void *stream) {
    if (!x || !grads || !(s >= 1.0f && s < 2.0f)) return TLC_ERR_ARG;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int T = (int)x->tensor_sizes.size(), C = (int)x->ctx.size();
    for (int i = 0; i < T; i++)
        if (!grads[i] && x->tensor_sizes[i]) return TLC_ERR_ARG;
    int rc = TLC_OK;
    // (1) compress every context with this rank's push error buffer into the send layout
    bool same = x->last_grads.size() == (size_t)T;
    for (int i = 0; same && i < T; i++) same = x->last_grads[i] == grads[i];
    if (!same) {
        std::vector<tlc_tensor_desc> d(C);
        for (int k = 0; k < C; k++) {
            const Ctx &c = x->ctx[k];
            d[k] = tlc_tensor_desc{};
            d[k].t = grads[c.tensor] + c.lo;
            d[k].err = x->push_err + c.elem_off;
            d[k].payload = x->push_send + x->region_start[c.owner] + c.region_off;
            d[k].hdr = x->push_hdr_send + x->hdr_start[c.owner] + c.slot;
            d[k].n = c.n;
        }
        if (cudaStreamSynchronize(st) != cudaSuccess) return TLC_ERR_CUDA;   // table may be in use
        rc = x->push_tab.d ? x->push_tab.update(d.data()) : x->push_tab.create(d.data(), C, true, nullptr);
        if (rc != TLC_OK) return rc;
        x->last_grads.assign(grads, grads + T);
    }
    if ((rc = launch_compress_table(x->push_tab.T, s, use_zre ? 1 : 0, x->push_tab.ws, st)) != TLC_OK) return rc;
    // (2) every owner receives its contexts' payloads and headers from every rank
    const int nown = (int)x->owned[x->me].size();
    const size_t own_region = x->region_bytes[x->me];
    ncclComm_t nc = x->comm->nccl;
    if ((rc = nccl_ok(ncclGroupStart())) != TLC_OK) return rc;
    for (int o = 0; o < x->W; o++) {
        if (x->region_bytes[o] == 0) continue;
        ncclSend(x->push_send + x->region_start[o], x->region_bytes[o], ncclUint8, o, nc, st);
        ncclSend(x->push_hdr_send + x->hdr_start[o], x->owned[o].size() * sizeof(tlc_header), ncclUint8, o, nc, st);
    }
    if (own_region)
        for (int w = 0; w < x->W; w++) {
            ncclRecv(x->push_recv + (size_t)w * own_region, own_region, ncclUint8, w, nc, st);
            ncclRecv(x->push_hdr_recv + (size_t)w * nown, nown * sizeof(tlc_header), ncclUint8, w, nc, st);
        }
    if ((rc = nccl_ok(ncclGroupEnd())) != TLC_OK) return rc;
    // (3) owner: fused decompress-aggregate of the W pushes of every owned context,
    //     rank-ordered sum from +0 of the nonzero trits, then / W (R15), written once
    if (x->owned_elems &&
        (rc = launch_aggregate(x->a_tab.T, x->x_tab.T, x->W, x->x_tab.ws, st)) != TLC_OK)
        return rc;
    return TLC_OK;
}

int tlc_exchange_pull(tlc_exchange *x, float *const *outs, float s, int use_zre, void *stream) {
    if (!x || !outs || !(s >= 1.0f && s < 2.0f)) return TLC_ERR_ARG;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int T = (int)x->tensor_sizes.size(), C = (int)x->ctx.size();
    for (int i = 0; i < T; i++)
        if (!outs[i] && x->tensor_sizes[i]) return TLC_ERR_ARG;
    int rc = TLC_OK;
    // (1) the owner compresses its shard of the model delta ONCE (shared pull)
    if (x->owned_elems &&
        (rc = launch_compress_table(x->pullc_tab.T, s, use_zre ? 1 : 0, x->pullc_tab.ws, st)) != TLC_OK)
        return rc;
    // (2) all-gather of the owners' regions (grouped send/recv, sizes differ per owner)
    ncclComm_t nc = x->comm->nccl;
    if ((rc = nccl_ok(ncclGroupStart())) != TLC_OK) return rc;
    for (int o = 0; o < x->W; o++) {
        if (o == x->me) continue;
        if (x->region_bytes[x->me]) {
            ncclSend(x->pull_buf + x->region_start[x->me], x->region_bytes[x->me], ncclUint8, o, nc, st);
            ncclSend(x->pull_hdr + x->hdr_start[x->me], x->owned[x->me].size() * sizeof(tlc_header), ncclUint8, o, nc, st);
        }
        if (x->region_bytes[o]) {
            ncclRecv(x->pull_buf + x->region_start[o], x->region_bytes[o], ncclUint8, o, nc, st);
            ncclRecv(x->pull_hdr + x->hdr_start[o], x->owned[o].size() * sizeof(tlc_header), ncclUint8, o, nc, st);
        }
    }
    if ((rc = nccl_ok(ncclGroupEnd())) != TLC_OK) return rc;
    // (3) every rank applies every context to its full-size output (ACCUMULATE, R16)
    bool same = x->last_outs.size() == (size_t)T;
    for (int i = 0; same && i < T; i++) same = x->last_outs[i] == outs[i];
    if (!same) {
        std::vector<tlc_tensor_desc> d(C);
        for (int k = 0; k < C; k++) {
            const Ctx &c = x->ctx[k];
            d[k] = tlc_tensor_desc{};
            d[k].out = outs[c.tensor] + c.lo;
            d[k].payload = x->pull_buf + x->region_start[c.owner] + c.region_off;
            d[k].hdr = x->pull_hdr + x->hdr_start[c.owner] + c.slot;
            d[k].n = c.n;
        }
        if (cudaStreamSynchronize(st) != cudaSuccess) return TLC_ERR_CUDA;
        rc = x->apply_tab.d ? x->apply_tab.update(d.data()) : x->apply_tab.create(d.data(), C, false, nullptr);
        if (rc != TLC_OK) return rc;
        x->last_outs.assign(outs, outs + T);
    }
    return launch_decompress_table(x->apply_tab.T, TLC_MODE_ACCUMULATE, x->apply_tab.ws, st);
}

int tlc_exchange_status(tlc_exchange *x, unsigned int *status_out, void *stream) {
    // worst device status over every received header (push and pull); synchronizes `stream`
    if (!x || !status_out) return TLC_ERR_ARG;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    int rc = cuda_ok(cudaMemsetAsync(x->d_status, 0, sizeof(unsigned int), st));
    const int nown = (int)x->owned[x->me].size();
    if (rc == TLC_OK && nown) tlc_status_kernel<<<1, 256, 0, st>>>(x->push_hdr_recv, x->W * nown, x->d_status);
    if (rc == TLC_OK && !x->ctx.empty()) tlc_status_kernel<<<1, 256, 0, st>>>(x->pull_hdr, (int)x->ctx.size(), x->d_status);
    if (rc == TLC_OK) rc = cuda_ok(cudaMemcpyAsync(status_out, x->d_status, sizeof(unsigned int), cudaMemcpyDeviceToHost, st));
    if (rc == TLC_OK) rc = cuda_ok(cudaStreamSynchronize(st));
    return rc;
}

}  // extern "C"
