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
#include <array>
#include <cstring>
#include <nccl.h>
#include <vector>

#include "tlc_device.cuh"
#include "tlc_launch.h"

struct tlc_comm {
    ncclComm_t nccl;
    int rank, world, device;
    int loopback;      // a virtual rank of a tlc_loopback group: no NCCL, no other process
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

// Exact transport.  Packing: the payloads of `count` contexts whose headers are the
// consecutive hdr[0..count) (a region's contexts in slot order: the layout of the header
// arrays) are laid end to end; off[k] = packed offset, off[count] = total, len[k] = bytes
// (payload_len, 0 for a failed compression).  Tiny: one thread.
__global__ void tlc_pack_offsets_kernel(const tlc_header *hdr, int count, uint64_t *off, uint64_t *len) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        uint64_t o = 0;
        for (int k = 0; k < count; k++) {
            const uint64_t l = hdr[k].status == TLC_OK ? hdr[k].payload_len : 0;
            off[k] = o;
            len[k] = l;
            o += l;
        }
        off[count] = o;
    }
}
// copy len[k] bytes src_base + src_off[k] -> dst_base + dst_off[k] for every item k (one
// block per item; 16-byte steps where both ends are aligned)
__global__ void tlc_copy_items_kernel(const uint8_t *src_base, const uint64_t *src_off, uint8_t *dst_base,
                                      const uint64_t *dst_off, const uint64_t *len, int count) {
    for (int k = blockIdx.x; k < count; k += gridDim.x) {
        const uint8_t *src = src_base + src_off[k];
        uint8_t *dst = dst_base + dst_off[k];
        const uint64_t n = len[k];
        if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15u) == 0) {
            for (uint64_t i = 16 * threadIdx.x; i + 16 <= n; i += 16 * blockDim.x)
                *reinterpret_cast<uint4 *>(dst + i) = *reinterpret_cast<const uint4 *>(src + i);
            for (uint64_t i = (n & ~15ull) + threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
        } else {
            for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
        }
    }
}

// worst status over a list of header pointers (peer-memory mode: the headers live on
// the producing ranks)
__global__ void tlc_status_list_kernel(const tlc_header *const *__restrict__ h, int count, unsigned int *out) {
    unsigned int m = 0;
    for (int i = threadIdx.x; i < count; i += blockDim.x) m = max(m, h[i]->status);
    m = __reduce_max_sync(0xffffffffu, m);
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}
// Cross-GPU flag barrier over peer memory (one rank per GPU): after a system
// fence, write `epoch` into this rank's slot on every rank, then wait until every
// rank has written it here.  Ordered after the kernels that produced the data.
__global__ void tlc_flag_barrier_kernel(unsigned long long *const *peer_flags, unsigned long long *mine, int me,
                                        int W, int slot, unsigned long long *epoch_ctr) {
    // the epoch is counted on the device (every rank runs the same barrier sequence),
    // so a captured CUDA graph replays with fresh epochs
    __shared__ unsigned long long s_epoch;
    if (threadIdx.x == 0) {
        s_epoch = *epoch_ctr + 1;
        *epoch_ctr = s_epoch;
    }
    __syncthreads();
    const unsigned long long epoch = s_epoch;
    const int w = threadIdx.x;
    if (w < W) {
        __threadfence_system();
        unsigned long long *dst = peer_flags[w] + (size_t)slot * W + me;
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(dst), "l"(epoch) : "memory");
        unsigned long long v;
        do {
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine + (size_t)slot * W + w) : "memory");
        } while (v < epoch);
    }
    __syncthreads();
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
    // push / apply tables cached for the two most recent pointer sets (a caller that
    // double-buffers its gradients or outputs alternates between two without re-uploads)
    Table push_tab[2], pullc_tab, apply_tab[2], a_tab, x_tab;
    bool keyed = false;                // this step's K5m folded the pull compress's max keys
    // peer-memory mode (tlc_exchange_ipc_*): the owner's kernels read the pushed
    // payloads and every rank reads the pulled payloads straight from the producing
    // rank's buffers over NVLink; two flag barriers per step order the phases
    int p2p = 0;
    unsigned long long *flags = nullptr;             // 2 x W epoch slots (local)
    unsigned long long **d_peer_flags = nullptr;     // device array: every rank's flag slots
    std::vector<void *> opened;                      // peer mappings to close
    std::vector<std::array<void *, 5>> peer;         // per rank: push_send, push_hdr, pull_buf, pull_hdr, flags
    unsigned long long *d_epoch = nullptr;           // barrier epochs issued (device counter)
    std::vector<const float *> push_key[2];
    std::vector<float *> apply_key[2];
    int push_mru = 0, apply_mru = 0;
    float *own_push_err = nullptr, *own_pull_err = nullptr;   // library-allocated (freed at destroy)
    // every header whose status the exchange reports: the pushes this rank aggregates
    // (from every rank) and the pulls it applies (from every owner)
    const tlc_header **d_status_list = nullptr;
    int status_count = 0;
    int phase = 0;                                   // 0: next call is push, 1: pull
    // NCCL "exact" transport (tlc_exchange_set_transport): payloads packed per owner, the
    // byte counts all-gathered first (one host sync per direction), then only those bytes sent
    int exact = 0;
    uint8_t *pack = nullptr;                         // packed send (push: by owner; pull: own region)
    uint8_t *pack_recv = nullptr;                    // packed receive, W slots of the larger region
    // device: [0, C+1) packed offsets, [C+1, 2C+1) lengths, [2C+1, 2C+1+C) capacity offsets of
    // the contexts in owner-major order; then the W x (C+1) all-gathered offsets; then the
    // unpack items (src, dst, len: 3 x W x C)
    uint64_t *d_pk = nullptr, *d_all = nullptr, *d_items = nullptr;
    uint64_t *h_all = nullptr;                       // pinned host copy of the all-gathered offsets
    std::vector<uint64_t> h_items;
    size_t max_region = 0;
    uint64_t last_recv[2] = {0, 0};                  // bytes received in the last push / pull (exact mode)
    // producer seek entries: behind the payload regions of push_send and pull_buf (at
    // seek_base), tile_off[k] entries in for context k; written by the producing K3, read by
    // the consumers' K5m / K5 over peer memory instead of running K4 (TLC_NO_PRODSEEK=1: off)
    size_t seek_base = 0;
    std::vector<uint64_t> tile_off;
    bool push_seeks = false;                         // the push compress runs K3 (not K6g)
    std::vector<char> pull_seeks;                    // per owner: its pull compress runs K3
};

static bool prodseek_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("TLC_NO_PRODSEEK");
        v = (e && e[0] == '1') ? 0 : 1;
    }
    return v == 1;
}

// Seg::seek pointers of a table over contexts ks: base + tile_off[k] (base == nullptr: none)
static std::vector<unsigned long long *> seek_ptrs(const tlc_exchange *x, const std::vector<int> &ks,
                                                   const std::vector<uint8_t *> &bases) {
    std::vector<unsigned long long *> v(ks.size(), nullptr);
    for (size_t i = 0; i < ks.size(); i++)
        if (bases[i]) v[i] = reinterpret_cast<unsigned long long *>(bases[i] + x->seek_base) + x->tile_off[ks[i]];
    return v;
}

static int cuda_ok(cudaError_t e) { return e == cudaSuccess ? TLC_OK : TLC_ERR_CUDA; }
static int nccl_ok(ncclResult_t r) { return r == ncclSuccess ? TLC_OK : TLC_ERR_NCCL; }

// The headers tlc_exchange_status reports on: this rank's own push headers, and the
// pull header of every context (on its owner in peer-memory mode, the received copy with
// NCCL), which by reading R24 carries every rank's push failure as NONFINITE -- so every
// rank reports the same worst status for a step.  With NCCL the received push headers
// of the owned contexts are added (FORMAT from the owner's scan lands there).  Peer
// mode reads no other rank's push header: after pull that rank may already be writing
// the next step's.
static int upload_status_list(tlc_exchange *x) {
    const int W = x->W, me = x->me, C = (int)x->ctx.size(), nown = (int)x->owned[me].size();
    std::vector<const tlc_header *> h;
    h.reserve((size_t)W * nown + 2 * C);
    for (int k = 0; k < C; k++) {
        const Ctx &c = x->ctx[k];
        h.push_back(x->push_hdr_send + x->hdr_start[c.owner] + c.slot);
        h.push_back((x->p2p ? static_cast<const tlc_header *>(x->peer[c.owner][3]) : x->pull_hdr) +
                    x->hdr_start[c.owner] + c.slot);
    }
    if (!x->p2p)
        for (int i = 0; i < W * nown; i++) h.push_back(x->push_hdr_recv + i);
    x->status_count = (int)h.size();
    if (h.empty()) return TLC_OK;
    return cuda_ok(cudaMemcpy(x->d_status_list, h.data(), h.size() * sizeof(void *), cudaMemcpyHostToDevice));
}

// Peer-memory mode: `peer[w]` = rank w's {push_send, push headers, pull buffer, pull
// headers, flag slots} as addressable from this device (CUDA IPC mappings of other
// processes' buffers, or plain device pointers for the virtual ranks of a loopback
// group).  The owner's aggregation then reads row w*|A|+q straight from rank w's send
// buffer, and the apply table is rebuilt on the next pull with the owners' pull buffers.
static int set_peers(tlc_exchange *x, const std::vector<std::array<void *, 5>> &peer) {
    const int W = x->W, me = x->me;
    x->peer = peer;
    std::vector<unsigned long long *> pf(W);
    for (int w = 0; w < W; w++) pf[w] = static_cast<unsigned long long *>(x->peer[w][4]);
    int rc = cuda_ok(cudaMemcpy(x->d_peer_flags, pf.data(), W * sizeof(void *), cudaMemcpyHostToDevice));
    const int nown = (int)x->owned[me].size();
    if (rc == TLC_OK && nown) {
        std::vector<tlc_tensor_desc> xs((size_t)W * nown);
        for (int q = 0; q < nown; q++) {
            const Ctx &c = x->ctx[x->owned[me][q]];
            for (int w = 0; w < W; w++) {
                tlc_tensor_desc &e = xs[(size_t)w * nown + q];
                e = tlc_tensor_desc{};
                e.payload = static_cast<uint8_t *>(x->peer[w][0]) + x->region_start[me] + c.region_off;
                e.hdr = static_cast<tlc_header *>(x->peer[w][1]) + x->hdr_start[me] + c.slot;
                e.n = c.n;
            }
        }
        // rank w's K3 wrote the seek entries of its pushes behind its send buffer
        std::vector<int> ks((size_t)W * nown);
        std::vector<uint8_t *> bases((size_t)W * nown, nullptr);
        for (int w = 0; w < W; w++)
            for (int q = 0; q < nown; q++) {
                ks[(size_t)w * nown + q] = x->owned[me][q];
                if (x->push_seeks) bases[(size_t)w * nown + q] = static_cast<uint8_t *>(x->peer[w][0]);
            }
        x->x_tab.seekp = seek_ptrs(x, ks, bases);
        rc = x->x_tab.update(xs.data());
    }
    if (rc == TLC_OK) {
        x->p2p = 1;
        x->apply_key[0].clear();   // the apply tables are rebuilt with peer pointers
        x->apply_key[1].clear();
        rc = upload_status_list(x);
    }
    return rc;
}

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
    if (!c || c->loopback) return TLC_ERR_ARG;     // a loopback group owns its virtual comms
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
    for (void *p : x->opened) cudaIpcCloseMemHandle(p);
    if (x->h_all) cudaFreeHost(x->h_all);
    void *dev2[] = {x->pack, x->pack_recv, x->d_pk, x->d_all, x->d_items};
    for (void *p : dev2)
        if (p) cudaFree(p);
    void *dev[] = {x->own_push_err, x->owned_buf, x->own_pull_err, x->push_send, x->push_recv, x->pull_buf,
                   x->push_hdr_send, x->push_hdr_recv, x->pull_hdr, x->d_status, x->flags, x->d_peer_flags,
                   x->d_epoch, (void *)x->d_status_list};
    for (void *p : dev)
        if (p) cudaFree(p);
    x->push_tab[0].release();
    x->push_tab[1].release();
    x->pullc_tab.release();
    x->apply_tab[0].release();
    x->apply_tab[1].release();
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
    alloc((void **)&x->own_push_err, x->total_elems * sizeof(float));
    alloc((void **)&x->owned_buf, x->owned_elems * sizeof(float));
    alloc((void **)&x->own_pull_err, x->owned_elems * sizeof(float));
    x->push_err = x->own_push_err;
    x->pull_err = x->own_pull_err;
    x->tile_off.assign(C + 1, 0);
    for (int k = 0; k < C; k++) x->tile_off[k + 1] = x->tile_off[k] + ((x->ctx[k].n + 4) / 5 + kT5 - 1) / kT5;
    x->seek_base = align256(x->total_region);
    const size_t seek_bytes = x->tile_off[C] * sizeof(unsigned long long);
    {
        // a table whose tensors are all small takes K6g (no K3, no seek entries)
        auto runs_k3 = [&](const std::vector<int> &ks) {
            uint64_t mx = 0;
            for (int k : ks) mx = tmax<uint64_t>(mx, x->ctx[k].n);
            return prodseek_enabled() && !ks.empty() && (mx > kSmallMaxN || !small_enabled());
        };
        std::vector<int> all(C);
        for (int k = 0; k < C; k++) all[k] = k;
        x->push_seeks = runs_k3(all);
        x->pull_seeks.assign(x->W, 0);
        for (int o = 0; o < x->W; o++) x->pull_seeks[o] = runs_k3(x->owned[o]) ? 1 : 0;
    }
    alloc((void **)&x->push_send, x->seek_base + seek_bytes);
    alloc((void **)&x->push_recv, (size_t)x->W * own_region);
    alloc((void **)&x->pull_buf, x->seek_base + seek_bytes);
    alloc((void **)&x->push_hdr_send, (size_t)C * sizeof(tlc_header));
    alloc((void **)&x->push_hdr_recv, (size_t)x->W * nown * sizeof(tlc_header));
    alloc((void **)&x->pull_hdr, (size_t)C * sizeof(tlc_header));
    alloc((void **)&x->d_status, 256);
    alloc((void **)&x->flags, 2 * x->W * sizeof(unsigned long long));
    alloc((void **)&x->d_epoch, sizeof(unsigned long long));
    if (rc == TLC_OK) rc = cuda_ok(cudaMemset(x->d_epoch, 0, sizeof(unsigned long long)));
    alloc((void **)&x->d_peer_flags, x->W * sizeof(unsigned long long *));
    alloc((void **)&x->d_status_list, ((size_t)x->W * nown + 2 * C) * sizeof(tlc_header *));
    if (rc == TLC_OK) rc = cuda_ok(cudaMemset(x->flags, 0, 2 * x->W * sizeof(unsigned long long)));
    // headers start zeroed (status OK, length 0): a header is only ever read after the
    // phase that writes it, but the status report must never see stale allocator bytes
    if (rc == TLC_OK) rc = cuda_ok(cudaMemset(x->push_hdr_send, 0, std::max<size_t>((size_t)C * sizeof(tlc_header), 256)));
    if (rc == TLC_OK)
        rc = cuda_ok(cudaMemset(x->push_hdr_recv, 0, std::max<size_t>((size_t)x->W * nown * sizeof(tlc_header), 256)));
    if (rc == TLC_OK) rc = cuda_ok(cudaMemset(x->pull_hdr, 0, std::max<size_t>((size_t)C * sizeof(tlc_header), 256)));
    if (rc == TLC_OK) rc = upload_status_list(x);
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
        x->pullc_tab.seekp = seek_ptrs(x, x->owned[x->me], std::vector<uint8_t *>(nown, x->pull_buf));
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

int tlc_exchange_bind_error_buffers(tlc_exchange *x, float *push_err, float *pull_err) {
    // caller-owned error buffers (training state to checkpoint): push_err holds
    // tlc_exchange_push_error's layout (every context, fp32), pull_err this rank's owned
    // contexts; NULL keeps the current buffer.  Synchronizes the device.
    if (!x || (!push_err && !pull_err)) return TLC_ERR_ARG;
    if (cudaDeviceSynchronize() != cudaSuccess) return TLC_ERR_CUDA;
    if (push_err) {
        x->push_err = push_err;
        x->push_key[0].clear();                       // push tables are rebuilt on the next push
        x->push_key[1].clear();
    }
    if (pull_err && x->owned_elems) {
        x->pull_err = pull_err;
        const int nown = (int)x->owned[x->me].size();
        std::vector<tlc_tensor_desc> pullc(nown);
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
        return x->pullc_tab.update(pullc.data());
    }
    return TLC_OK;
}

// ------------------------------------------------------------------ peer-memory mode
int tlc_exchange_ipc_handles(tlc_exchange *x, void *out) {
    // five cudaIpcMemHandle_t (64 bytes each): push_send, push headers, pull buffer,
    // pull headers, flag slots
    if (!x || !out) return TLC_ERR_ARG;
    void *bufs[5] = {x->push_send, x->push_hdr_send, x->pull_buf, x->pull_hdr, x->flags};
    for (int k = 0; k < 5; k++) {
        cudaIpcMemHandle_t h;
        if (cudaIpcGetMemHandle(&h, bufs[k]) != cudaSuccess) return TLC_ERR_CUDA;
        std::memcpy(static_cast<char *>(out) + 64 * k, &h, 64);
    }
    return TLC_OK;
}

int tlc_exchange_ipc_open(tlc_exchange *x, const void *all) {
    // all: W x 5 handles in rank order (the all-gather of tlc_exchange_ipc_handles)
    if (!x || !all || x->p2p || x->comm->loopback) return TLC_ERR_ARG;
    const int W = x->W, me = x->me;
    std::vector<std::array<void *, 5>> peer(W);
    void *mine[5] = {x->push_send, x->push_hdr_send, x->pull_buf, x->pull_hdr, x->flags};
    for (int w = 0; w < W; w++)
        for (int k = 0; k < 5; k++) {
            if (w == me) { peer[w][k] = mine[k]; continue; }
            cudaIpcMemHandle_t h;
            std::memcpy(&h, static_cast<const char *>(all) + 64 * (5 * w + k), 64);
            void *p = nullptr;
            if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return TLC_ERR_CUDA;
            x->opened.push_back(p);
            peer[w][k] = p;
        }
    return set_peers(x, peer);
}

// Stream capture (CUDA graphs) is supported by the peer-memory transport only;
// the NCCL transport refuses it instead of hanging in capture.
static int capture_ok(const tlc_exchange *x, cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) return TLC_ERR_CUDA;
    return (cs != cudaStreamCaptureStatusNone && !x->p2p) ? TLC_ERR_ARG : TLC_OK;
}

static int flag_barrier(tlc_exchange *x, int slot, cudaStream_t st) {
    KernelScope ks(kK7, st);
    tlc_flag_barrier_kernel<<<1, 32 * ((x->W + 31) / 32), 0, st>>>(x->d_peer_flags, x->flags, x->me, x->W, slot,
                                                                    x->d_epoch);
    return cuda_ok(cudaPeekAtLastError());
}

int tlc_exchange_traffic(tlc_exchange *x, uint64_t *out) {
    // bytes this rank received in the last push (out[0]) and pull (out[1]) from other
    // ranks: capacity regions with NCCL, exactly the payload (+ header) bytes the
    // consuming kernels read in peer-memory mode.  Synchronizes the device.
    if (!x || !out) return TLC_ERR_ARG;
    if (cudaDeviceSynchronize() != cudaSuccess) return TLC_ERR_CUDA;
    const int W = x->W, me = x->me;
    const int nown = (int)x->owned[me].size();
    if (x->exact) {
        out[0] = x->last_recv[0];
        out[1] = x->last_recv[1];
        return TLC_OK;
    }
    if (!x->p2p) {
        out[0] = (uint64_t)(W - 1) * (x->region_bytes[me] + nown * sizeof(tlc_header));
        uint64_t b = 0;
        for (int o = 0; o < W; o++)
            if (o != me) b += x->region_bytes[o] + x->owned[o].size() * sizeof(tlc_header);
        out[1] = b;
        return TLC_OK;
    }
    uint64_t push = 0, pull = 0;
    std::vector<tlc_header> h;
    for (int w = 0; w < W; w++) {
        if (w == me) continue;
        h.resize(nown);
        if (nown && cudaMemcpy(h.data(), static_cast<tlc_header *>(x->peer[w][1]) + x->hdr_start[me],
                               nown * sizeof(tlc_header), cudaMemcpyDefault) != cudaSuccess) return TLC_ERR_CUDA;
        for (auto &e : h) push += e.payload_len + sizeof(tlc_header);
        const int no = (int)x->owned[w].size();
        h.resize(no);
        if (no && cudaMemcpy(h.data(), static_cast<tlc_header *>(x->peer[w][3]) + x->hdr_start[w],
                             no * sizeof(tlc_header), cudaMemcpyDefault) != cudaSuccess) return TLC_ERR_CUDA;
        for (auto &e : h) pull += e.payload_len + sizeof(tlc_header);
    }
    out[0] = push;
    out[1] = pull;
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

}  // extern "C"

// ------------------------------------------------------------------ the four phases
// push = (1) compress + transport + (2) owner aggregate; pull = (3) owner compress +
// transport + (4) apply.  The loopback group runs each phase for every virtual rank
// before the next phase, which is the order the flag barriers enforce across GPUs.
static int check_ptrs(const tlc_exchange *x, const void *const *p) {
    for (size_t i = 0; i < x->tensor_sizes.size(); i++)
        if (!p[i] && x->tensor_sizes[i]) return TLC_ERR_ARG;
    return TLC_OK;
}

// (1) compress every context with this rank's push error buffer into the send layout
static int phase_push_compress(tlc_exchange *x, const float *const *grads, float s, int use_zre, cudaStream_t st) {
    const int T = (int)x->tensor_sizes.size(), C = (int)x->ctx.size();
    int slot = -1;
    for (int k = 0; k < 2 && slot < 0; k++)
        if (x->push_key[k].size() == (size_t)T && std::equal(grads, grads + T, x->push_key[k].begin())) slot = k;
    if (slot < 0) {
        slot = x->push_key[x->push_mru].empty() ? x->push_mru : 1 - x->push_mru;   // the least recently used
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
        Table &tb = x->push_tab[slot];
        std::vector<int> ks(C);
        for (int k = 0; k < C; k++) ks[k] = k;
        tb.seekp = seek_ptrs(x, ks, std::vector<uint8_t *>(C, x->push_seeks ? x->push_send : nullptr));
        const int rc = tb.d ? tb.update(d.data()) : tb.create(d.data(), C, true, nullptr);
        if (rc != TLC_OK) return rc;
        x->push_key[slot].assign(grads, grads + T);
    }
    x->push_mru = slot;
    return launch_compress_table(x->push_tab[slot].T, s, use_zre ? 1 : 0, x->push_tab[slot].ws, st);
}

// (2) owner: fused decompress-aggregate of the W pushes of every owned context,
//     rank-ordered sum from +0 of the nonzero trits, then / W (R15), written once
// TLC_NO_KEYED=1: the pull compress runs its own K1 instead of taking the keys the fused
// aggregate folded while it wrote the means (A/B)
static bool keyed_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("TLC_NO_KEYED");
        v = (e && e[0] == '1') ? 0 : 1;
    }
    return v == 1;
}

static int phase_aggregate(tlc_exchange *x, cudaStream_t st) {
    x->keyed = false;
    if (!x->owned_elems) return TLC_OK;
    // the pull compress's K1 (max |pull_err + mean| per owned context) folded into K5m, which
    // has the means in registers as it writes them: one launch and 8 n_own bytes less
    if (keyed_enabled() && aggregate_keyable(x->W) && compress_runs_k1(x->pullc_tab.T) &&
        x->pullc_tab.count == x->a_tab.count) {
        unsigned int *keys = nullptr;
        int rc = prepare_keyed_compress(x->pullc_tab.T, x->pullc_tab.ws, st, &keys);
        if (rc == TLC_OK) rc = launch_aggregate(x->a_tab.T, x->x_tab.T, x->W, x->x_tab.ws, st, &x->pullc_tab.T, keys);
        x->keyed = rc == TLC_OK;
        return rc;
    }
    return launch_aggregate(x->a_tab.T, x->x_tab.T, x->W, x->x_tab.ws, st);
}

// (3) the owner compresses its shard of the model delta ONCE (shared pull)
static int phase_pull_compress(tlc_exchange *x, float s, int use_zre, cudaStream_t st) {
    if (!x->owned_elems) return TLC_OK;
    if (x->keyed) return launch_compress_table_keyed(x->pullc_tab.T, s, use_zre ? 1 : 0, x->pullc_tab.ws, st);
    return launch_compress_table(x->pullc_tab.T, s, use_zre ? 1 : 0, x->pullc_tab.ws, st);
}

// (4) every rank applies every context to its full-size output (ACCUMULATE, R16)
static int phase_apply(tlc_exchange *x, float *const *outs, cudaStream_t st) {
    const int T = (int)x->tensor_sizes.size(), C = (int)x->ctx.size();
    int slot = -1;
    for (int k = 0; k < 2 && slot < 0; k++)
        if (x->apply_key[k].size() == (size_t)T && std::equal(outs, outs + T, x->apply_key[k].begin())) slot = k;
    if (slot < 0) {
        slot = x->apply_key[x->apply_mru].empty() ? x->apply_mru : 1 - x->apply_mru;
        std::vector<tlc_tensor_desc> d(C);
        for (int k = 0; k < C; k++) {
            const Ctx &c = x->ctx[k];
            d[k] = tlc_tensor_desc{};
            d[k].out = outs[c.tensor] + c.lo;
            uint8_t *pb = x->p2p ? static_cast<uint8_t *>(x->peer[c.owner][2]) : x->pull_buf;
            tlc_header *ph = x->p2p ? static_cast<tlc_header *>(x->peer[c.owner][3]) : x->pull_hdr;
            d[k].payload = pb + x->region_start[c.owner] + c.region_off;
            d[k].hdr = ph + x->hdr_start[c.owner] + c.slot;
            d[k].n = c.n;
        }
        if (cudaStreamSynchronize(st) != cudaSuccess) return TLC_ERR_CUDA;
        Table &tb = x->apply_tab[slot];
        // peer memory: every owner's K3 wrote its pulls' seek entries behind its pull buffer
        std::vector<int> ks(C);
        std::vector<uint8_t *> bases(C, nullptr);
        for (int k = 0; k < C; k++) {
            ks[k] = k;
            const int o = x->ctx[k].owner;
            if (x->p2p && x->pull_seeks[o]) bases[k] = static_cast<uint8_t *>(x->peer[o][2]);
        }
        tb.seekp = seek_ptrs(x, ks, bases);
        const int rc = tb.d ? tb.update(d.data()) : tb.create(d.data(), C, false, nullptr);
        if (rc != TLC_OK) return rc;
        x->apply_key[slot].assign(outs, outs + T);
    }
    x->apply_mru = slot;
    return launch_decompress_table(x->apply_tab[slot].T, TLC_MODE_ACCUMULATE, x->apply_tab[slot].ws, st);
}

// ------------------------------------------------------------------ NCCL exact transport
// Sizes first: pack the payloads, all-gather the packing offsets, one host
// sync, then grouped send/recv of exactly the payload bytes, and unpack into the capacity
// layout the aggregation / apply tables read.
static int exact_alloc(tlc_exchange *x) {
    const int W = x->W, C = (int)x->ctx.size();
    for (int o = 0; o < W; o++) x->max_region = std::max(x->max_region, x->region_bytes[o]);
    int rc = TLC_OK;
    auto alloc = [&](void **p, size_t bytes) {
        if (rc == TLC_OK && cudaMalloc(p, std::max<size_t>(bytes, 256)) != cudaSuccess) rc = TLC_ERR_CUDA;
    };
    alloc((void **)&x->pack, x->total_region);
    alloc((void **)&x->pack_recv, (size_t)W * x->max_region);
    alloc((void **)&x->d_pk, (3 * (size_t)C + 1) * sizeof(uint64_t));
    alloc((void **)&x->d_all, (size_t)W * (C + 1) * sizeof(uint64_t));
    alloc((void **)&x->d_items, 3 * (size_t)W * C * sizeof(uint64_t));
    if (rc == TLC_OK && cudaMallocHost((void **)&x->h_all, (size_t)W * (C + 1) * sizeof(uint64_t)) != cudaSuccess)
        rc = TLC_ERR_CUDA;
    if (rc != TLC_OK) return rc;
    // capacity offsets of the contexts in owner-major (header) order
    std::vector<uint64_t> cap(C);
    for (int o = 0; o < W; o++)
        for (int q = 0; q < (int)x->owned[o].size(); q++) {
            const Ctx &c = x->ctx[x->owned[o][q]];
            cap[x->hdr_start[o] + q] = x->region_start[o] + c.region_off;
        }
    if (C) rc = cuda_ok(cudaMemcpy(x->d_pk + 2 * C + 1, cap.data(), C * sizeof(uint64_t), cudaMemcpyHostToDevice));
    return rc;
}

// pack `count` contexts whose headers are hdr[0..count) and whose capacity offsets in `src`
// are cap[0..count); all-gather the offsets; wait for them on the host (h_all)
static int exact_pack_gather(tlc_exchange *x, const tlc_header *hdr, const uint64_t *cap, const uint8_t *src,
                             int count, cudaStream_t st) {
    const int C = (int)x->ctx.size();
    uint64_t *off = x->d_pk, *len = x->d_pk + C + 1;
    tlc_pack_offsets_kernel<<<1, 32, 0, st>>>(hdr, count, off, len);
    if (count)
        tlc_copy_items_kernel<<<std::min(count, num_sms() * 4), 256, 0, st>>>(src, cap, x->pack, off, len, count);
    int rc = cuda_ok(cudaPeekAtLastError());
    if (rc == TLC_OK) rc = nccl_ok(ncclAllGather(off, x->d_all, C + 1, ncclUint64, x->comm->nccl, st));
    if (rc == TLC_OK)
        rc = cuda_ok(cudaMemcpyAsync(x->h_all, x->d_all, (size_t)x->W * (C + 1) * sizeof(uint64_t),
                                     cudaMemcpyDeviceToHost, st));
    if (rc == TLC_OK) rc = cuda_ok(cudaStreamSynchronize(st));   // the counts are host arguments
    return rc;
}

// unpack items: (src offset in pack_recv, dst offset in dst_base, length)
static int exact_unpack(tlc_exchange *x, uint8_t *dst_base, cudaStream_t st) {
    const int k = (int)(x->h_items.size() / 3);
    if (!k) return TLC_OK;
    int rc = cuda_ok(cudaMemcpyAsync(x->d_items, x->h_items.data(), x->h_items.size() * sizeof(uint64_t),
                                     cudaMemcpyHostToDevice, st));
    if (rc != TLC_OK) return rc;
    tlc_copy_items_kernel<<<std::min(k, num_sms() * 4), 256, 0, st>>>(x->pack_recv, x->d_items, dst_base,
                                                                      x->d_items + k, x->d_items + 2 * k, k);
    return cuda_ok(cudaPeekAtLastError());
}

static int exact_push(tlc_exchange *x, cudaStream_t st) {
    const int W = x->W, C = (int)x->ctx.size(), me = x->me, nown = (int)x->owned[me].size();
    int rc = exact_pack_gather(x, x->push_hdr_send, x->d_pk + 2 * C + 1, x->push_send, C, st);
    if (rc != TLC_OK) return rc;
    const uint64_t *mine = x->h_all + (size_t)me * (C + 1);
    ncclComm_t nc = x->comm->nccl;
    uint64_t recvd = 0;
    if ((rc = nccl_ok(ncclGroupStart())) != TLC_OK) return rc;
    for (int o = 0; o < W; o++) {
        const int f = (int)x->hdr_start[o], no = (int)x->owned[o].size();
        if (!no) continue;
        const uint64_t b = mine[f + no] - mine[f];
        if (b) ncclSend(x->pack + mine[f], b, ncclUint8, o, nc, st);
        ncclSend(x->push_hdr_send + f, no * sizeof(tlc_header), ncclUint8, o, nc, st);
    }
    if (nown) {
        const int f = (int)x->hdr_start[me];
        for (int w = 0; w < W; w++) {
            const uint64_t *ow = x->h_all + (size_t)w * (C + 1);
            const uint64_t b = ow[f + nown] - ow[f];
            if (b) ncclRecv(x->pack_recv + (size_t)w * x->max_region, b, ncclUint8, w, nc, st);
            ncclRecv(x->push_hdr_recv + (size_t)w * nown, nown * sizeof(tlc_header), ncclUint8, w, nc, st);
            if (w != me) recvd += b + nown * sizeof(tlc_header);
        }
    }
    if ((rc = nccl_ok(ncclGroupEnd())) != TLC_OK) return rc;
    x->last_recv[0] = recvd;
    // unpack every sender's payloads of my contexts into the capacity layout of push_recv
    x->h_items.clear();
    if (nown) {
        const int f = (int)x->hdr_start[me];
        std::vector<uint64_t> so, dof, ln;
        for (int w = 0; w < W; w++) {
            const uint64_t *ow = x->h_all + (size_t)w * (C + 1);
            for (int q = 0; q < nown; q++) {
                const uint64_t l = ow[f + q + 1] - ow[f + q];
                if (!l) continue;
                so.push_back((size_t)w * x->max_region + (ow[f + q] - ow[f]));
                dof.push_back((size_t)w * x->region_bytes[me] + x->ctx[x->owned[me][q]].region_off);
                ln.push_back(l);
            }
        }
        x->h_items = so;
        x->h_items.insert(x->h_items.end(), dof.begin(), dof.end());
        x->h_items.insert(x->h_items.end(), ln.begin(), ln.end());
    }
    return exact_unpack(x, x->push_recv, st);
}

static int exact_pull(tlc_exchange *x, cudaStream_t st) {
    const int W = x->W, C = (int)x->ctx.size(), me = x->me, nown = (int)x->owned[me].size();
    const int fme = (int)x->hdr_start[me];
    int rc = exact_pack_gather(x, x->pull_hdr + fme, x->d_pk + 2 * C + 1 + fme, x->pull_buf, nown, st);
    if (rc != TLC_OK) return rc;
    ncclComm_t nc = x->comm->nccl;
    const uint64_t mine = x->h_all[(size_t)me * (C + 1) + nown];
    uint64_t recvd = 0;
    if ((rc = nccl_ok(ncclGroupStart())) != TLC_OK) return rc;
    for (int o = 0; o < W; o++) {
        if (o == me) continue;
        const int no = (int)x->owned[o].size();
        if (nown) {
            if (mine) ncclSend(x->pack, mine, ncclUint8, o, nc, st);
            ncclSend(x->pull_hdr + fme, nown * sizeof(tlc_header), ncclUint8, o, nc, st);
        }
        if (no) {
            const uint64_t b = x->h_all[(size_t)o * (C + 1) + no];
            if (b) ncclRecv(x->pack_recv + (size_t)o * x->max_region, b, ncclUint8, o, nc, st);
            ncclRecv(x->pull_hdr + x->hdr_start[o], no * sizeof(tlc_header), ncclUint8, o, nc, st);
            recvd += b + no * sizeof(tlc_header);
        }
    }
    if ((rc = nccl_ok(ncclGroupEnd())) != TLC_OK) return rc;
    x->last_recv[1] = recvd;
    // unpack every owner's shared pull payloads into the capacity layout of pull_buf
    std::vector<uint64_t> so, dof, ln;
    for (int o = 0; o < W; o++) {
        if (o == me) continue;
        const uint64_t *oo = x->h_all + (size_t)o * (C + 1);
        for (int q = 0; q < (int)x->owned[o].size(); q++) {
            const uint64_t l = oo[q + 1] - oo[q];
            if (!l) continue;
            so.push_back((size_t)o * x->max_region + oo[q]);
            dof.push_back(x->region_start[o] + x->ctx[x->owned[o][q]].region_off);
            ln.push_back(l);
        }
    }
    x->h_items = so;
    x->h_items.insert(x->h_items.end(), dof.begin(), dof.end());
    x->h_items.insert(x->h_items.end(), ln.begin(), ln.end());
    return exact_unpack(x, x->pull_buf, st);
}

extern "C" {

int tlc_exchange_set_transport(tlc_exchange *x, int mode) {
    // NCCL transports: 0 = capacity regions (no host sync), 1 = exact payload bytes after a
    // sizes all-gather (one host sync per direction).  Not for peer-memory or loopback.
    if (!x || x->p2p || x->comm->loopback || (mode != 0 && mode != 1) || x->phase != 0) return TLC_ERR_ARG;
    if (mode == 1 && !x->pack) {
        const int rc = exact_alloc(x);
        if (rc != TLC_OK) return rc;
    }
    x->exact = mode;
    return TLC_OK;
}

int tlc_exchange_push(tlc_exchange *x, const float *const *grads, float s, int use_zre, void *stream) {
    if (!x || !grads || !(s >= 1.0f && s < 2.0f) || x->comm->loopback) return TLC_ERR_ARG;
    if (x->phase != 0) return TLC_ERR_ARG;        // push and pull alternate (buffer reuse, see tlc.h)
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (int rc0 = capture_ok(x, st)) return rc0;
    int rc = check_ptrs(x, reinterpret_cast<const void *const *>(grads));
    if (rc == TLC_OK) rc = phase_push_compress(x, grads, s, use_zre, st);
    if (rc != TLC_OK) return rc;
    // every owner receives its contexts' payloads and headers from every rank
    if (x->p2p) {
        // peer memory: no copy -- once every rank's pushes are written, the owner's
        // scan and aggregation kernels read them from the producing GPU over NVLink
        if ((rc = flag_barrier(x, 0, st)) != TLC_OK) return rc;
    } else if (x->exact) {
        if ((rc = exact_push(x, st)) != TLC_OK) return rc;
    } else {
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
    }
    if ((rc = phase_aggregate(x, st)) != TLC_OK) return rc;
    x->phase = 1;
    return TLC_OK;
}

int tlc_exchange_pull(tlc_exchange *x, float *const *outs, float s, int use_zre, void *stream) {
    if (!x || !outs || !(s >= 1.0f && s < 2.0f) || x->comm->loopback) return TLC_ERR_ARG;
    if (x->phase != 1) return TLC_ERR_ARG;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (int rc0 = capture_ok(x, st)) return rc0;
    int rc = check_ptrs(x, reinterpret_cast<const void *const *>(outs));
    if (rc == TLC_OK) rc = phase_pull_compress(x, s, use_zre, st);
    if (rc != TLC_OK) return rc;
    // all-gather of the owners' regions (grouped send/recv, sizes differ per owner);
    // in peer-memory mode a barrier, then the apply kernels read the owners' regions
    if (x->p2p) {
        if ((rc = flag_barrier(x, 1, st)) != TLC_OK) return rc;
    } else if (x->exact) {
        if ((rc = exact_pull(x, st)) != TLC_OK) return rc;
    } else {
        ncclComm_t nc = x->comm->nccl;
        if ((rc = nccl_ok(ncclGroupStart())) != TLC_OK) return rc;
        for (int o = 0; o < x->W; o++) {
            if (o == x->me) continue;
            if (x->region_bytes[x->me]) {
                ncclSend(x->pull_buf + x->region_start[x->me], x->region_bytes[x->me], ncclUint8, o, nc, st);
                ncclSend(x->pull_hdr + x->hdr_start[x->me], x->owned[x->me].size() * sizeof(tlc_header), ncclUint8,
                         o, nc, st);
            }
            if (x->region_bytes[o]) {
                ncclRecv(x->pull_buf + x->region_start[o], x->region_bytes[o], ncclUint8, o, nc, st);
                ncclRecv(x->pull_hdr + x->hdr_start[o], x->owned[o].size() * sizeof(tlc_header), ncclUint8, o, nc, st);
            }
        }
        if ((rc = nccl_ok(ncclGroupEnd())) != TLC_OK) return rc;
    }
    if ((rc = phase_apply(x, outs, st)) != TLC_OK) return rc;
    x->phase = 0;
    return TLC_OK;
}

}  // extern "C"

static int exchange_status_enqueue(tlc_exchange *x, unsigned int *dst, cudaStream_t st) {
    // worst device status over every header this rank consumed (push and pull)
    int rc = cuda_ok(cudaMemsetAsync(x->d_status, 0, sizeof(unsigned int), st));
    if (rc == TLC_OK && x->status_count)
        tlc_status_list_kernel<<<1, 256, 0, st>>>(x->d_status_list, x->status_count, x->d_status);
    if (rc == TLC_OK) rc = cuda_ok(cudaPeekAtLastError());
    if (rc == TLC_OK) rc = cuda_ok(cudaMemcpyAsync(dst, x->d_status, sizeof(unsigned int), cudaMemcpyDefault, st));
    return rc;
}

extern "C" {

int tlc_exchange_status(tlc_exchange *x, unsigned int *status_out, void *stream) {
    // synchronizes `stream`
    if (!x || !status_out) return TLC_ERR_ARG;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    int rc = exchange_status_enqueue(x, status_out, st);
    if (rc == TLC_OK) rc = cuda_ok(cudaStreamSynchronize(st));
    return rc;
}

int tlc_exchange_status_async(tlc_exchange *x, unsigned int *dst, void *stream) {
    if (!x || !dst) return TLC_ERR_ARG;
    return exchange_status_enqueue(x, dst, reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"

// ------------------------------------------------------------------ loopback group
// W virtual ranks in one process on one device: each has its own tlc_exchange (own
// push / pull error buffers, owned buffer, send and pull regions) and sees the others'
// buffers as plain device pointers (peer-memory mode without IPC); stream order
// replaces the flag barriers.  Push and pull run the same kernels as the multi-GPU
// transports -- K1-K3 per rank, K4 + K5m per owner reading every rank's payloads,
// K1-K3 per owner, K4 + K5 per rank reading every owner's payloads.
struct tlc_loopback {
    int W = 0;
    std::vector<tlc_comm *> comms;
    std::vector<tlc_exchange *> xs;
    int phase = 0;
};

extern "C" {

int tlc_loopback_destroy(tlc_loopback *g) {
    if (!g) return TLC_ERR_ARG;
    for (tlc_exchange *x : g->xs)
        if (x) tlc_exchange_destroy(x);
    for (tlc_comm *c : g->comms) delete c;
    delete g;
    return TLC_OK;
}

int tlc_loopback_create(tlc_loopback **out, int world, int num_tensors, const uint64_t *sizes, int device) {
    if (!out || world < 1 || world > 8 || num_tensors < 1 || !sizes) return TLC_ERR_ARG;
    if (cudaSetDevice(device) != cudaSuccess) return TLC_ERR_CUDA;
    auto *g = new tlc_loopback{};
    g->W = world;
    int rc = TLC_OK;
    for (int r = 0; r < world && rc == TLC_OK; r++) {
        auto *c = new tlc_comm{};
        c->nccl = nullptr;
        c->rank = r;
        c->world = world;
        c->device = device;
        c->loopback = 1;
        g->comms.push_back(c);
        tlc_exchange *x = nullptr;
        rc = tlc_exchange_create(&x, c, num_tensors, sizes);
        if (rc == TLC_OK) g->xs.push_back(x);
    }
    if (rc == TLC_OK) {
        std::vector<std::array<void *, 5>> peer(world);
        for (int w = 0; w < world; w++) {
            tlc_exchange *y = g->xs[w];
            peer[w] = {y->push_send, y->push_hdr_send, y->pull_buf, y->pull_hdr, y->flags};
        }
        for (int r = 0; r < world && rc == TLC_OK; r++) rc = set_peers(g->xs[r], peer);
    }
    if (rc != TLC_OK) {
        tlc_loopback_destroy(g);
        return rc;
    }
    *out = g;
    return TLC_OK;
}

tlc_exchange *tlc_loopback_rank(tlc_loopback *g, int rank) {
    return (g && rank >= 0 && rank < g->W) ? g->xs[rank] : nullptr;
}

int tlc_loopback_push(tlc_loopback *g, const float *const *grads, float s, int use_zre, void *stream) {
    if (!g || !grads || !(s >= 1.0f && s < 2.0f) || g->phase != 0) return TLC_ERR_ARG;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const size_t T = g->xs[0]->tensor_sizes.size();
    int rc = TLC_OK;
    for (int r = 0; r < g->W && rc == TLC_OK; r++) rc = check_ptrs(g->xs[r], reinterpret_cast<const void *const *>(grads + r * T));
    for (int r = 0; r < g->W && rc == TLC_OK; r++) rc = phase_push_compress(g->xs[r], grads + r * T, s, use_zre, st);
    for (int r = 0; r < g->W && rc == TLC_OK; r++) rc = phase_aggregate(g->xs[r], st);
    if (rc == TLC_OK) g->phase = 1;
    return rc;
}

int tlc_loopback_pull(tlc_loopback *g, float *const *outs, float s, int use_zre, void *stream) {
    if (!g || !outs || !(s >= 1.0f && s < 2.0f) || g->phase != 1) return TLC_ERR_ARG;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const size_t T = g->xs[0]->tensor_sizes.size();
    int rc = TLC_OK;
    for (int r = 0; r < g->W && rc == TLC_OK; r++) rc = check_ptrs(g->xs[r], reinterpret_cast<const void *const *>(outs + r * T));
    for (int r = 0; r < g->W && rc == TLC_OK; r++) rc = phase_pull_compress(g->xs[r], s, use_zre, st);
    for (int r = 0; r < g->W && rc == TLC_OK; r++) rc = phase_apply(g->xs[r], outs + r * T, st);
    if (rc == TLC_OK) g->phase = 0;
    return rc;
}

}  // extern "C"

// ------------------------------------------------------------------ standalone aggregation
// The server's "average the gradients" (reading R15; R24 for failed sources) over
// W compressed copies of a tensor list, outside any exchange: the owner-side fused
// decompress-aggregate (K4 + K5m) of the parameter server, for callers that move the
// payloads themselves (the desk-scale simulator's single server, psim.py).
struct tlc_aggregate {
    int W = 0;
    Table a_tab, x_tab;
};

extern "C" {

int tlc_aggregate_destroy(tlc_aggregate *g) {
    if (!g) return TLC_ERR_ARG;
    g->a_tab.release();
    g->x_tab.release();
    delete g;
    return TLC_OK;
}

int tlc_aggregate_create(tlc_aggregate **out, int world, int count, const tlc_tensor_desc *outs,
                         const tlc_tensor_desc *srcs) {
    if (!out || world < 1 || world > 8 || count < 1 || !outs || !srcs) return TLC_ERR_ARG;
    for (int i = 0; i < count; i++) {
        if (!outs[i].out || outs[i].n == 0) return TLC_ERR_ARG;
        for (int w = 0; w < world; w++) {
            const tlc_tensor_desc &d = srcs[(size_t)w * count + i];
            if (!d.payload || !d.hdr || d.n != outs[i].n) return TLC_ERR_ARG;
        }
    }
    auto *g = new tlc_aggregate{};
    g->W = world;
    std::vector<tlc_tensor_desc> a(outs, outs + count);
    for (int i = 0; i < count; i++) a[i].hdr = srcs[i].hdr;      // only n / out are used through A
    int rc = g->a_tab.create(a.data(), count, false, nullptr);
    if (rc == TLC_OK) rc = g->x_tab.create(srcs, world * count, false, nullptr);
    if (rc != TLC_OK) {
        tlc_aggregate_destroy(g);
        return rc;
    }
    *out = g;
    return TLC_OK;
}

int tlc_aggregate_run(tlc_aggregate *g, void *stream) {
    if (!g) return TLC_ERR_ARG;
    return launch_aggregate(g->a_tab.T, g->x_tab.T, g->W, g->x_tab.ws, reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
