// segments.cu -- host side of the segment tables (tlc_launch.h) and the batch
// objects of the C ABI (tlc_batch_*): a fixed list of independent tensors whose
// table and workspace live on the device, so compressing or decompressing the
// whole list is 4 (3) kernel launches and no host-to-device traffic.
#include <algorithm>
#include <vector>

#include "tlc_device.cuh"
#include "tlc_launch.h"

namespace tlc {

void seg_items(Seg &s, const ItemSizes &z, uint64_t &c1, uint64_t &c2, uint64_t &c3, uint64_t &c4, uint64_t &c5) {
    s.P = (s.n + 4) / 5;
    s.k1 = c1; c1 += (s.n + z.t1 - 1) / z.t1;
    s.k2 = c2; c2 += (s.P + z.t2 - 1) / z.t2;
    s.k3 = c3; c3 += (s.P + z.c3 - 1) / z.c3;
    s.k4 = c4; c4 += (s.P + z.c4 - 1) / z.c4;
    s.k5 = c5; c5 += (s.P + kT5 - 1) / kT5;
}

uint32_t seg_flags(const Seg &s) {
    uint32_t f = 0;
    if (aligned16(s.t) && aligned16(s.err)) f |= kSegVec1;
    if (s.P % 4 == 0 && aligned16(s.t) && aligned16(s.err) && aligned4(s.payload)) f |= kSegVec2;
    if (s.P % 4 == 0 && aligned16(s.out)) f |= kSegVec5;
    return f;
}

SegTable single_table(const float *t, float *err, float *out, uint8_t *payload, tlc_header *hdr, uint64_t n,
                      uint64_t &scratch) {
    SegTable T{};
    T.count = 1;
    Seg &s = T.one;
    s = Seg{};
    s.t = t; s.err = err; s.out = out; s.payload = payload; s.hdr = hdr; s.n = n;
    T.sz = item_sizes(n);
    T.max_n = n;
    seg_items(s, T.sz, T.n1, T.n2, T.n3, T.n4, T.n5);
    s.bytes_off = 0;
    s.flags = seg_flags(s);
    scratch = (s.P + 15) & ~uint64_t(15);
    return T;
}

WsLayout ws_layout(const SegTable &T, uint64_t scratch_bytes) {
    WsLayout L{};
    size_t p = 0;
    L.ctrl = p;   p += sizeof(Ctrl);
    L.maxkey = p; p += align256((size_t)T.count * sizeof(unsigned int));
    L.k12done = p; p += T.k12 ? align256((size_t)T.count * sizeof(unsigned int)) : 0;
    L.k3st = p;   p += align256(T.n3 * sizeof(unsigned long long));
    L.memset_c = p;                                   // ctrl + max keys + K12 counts + K3 states
    L.k4st = p;   p += align256(T.n4 * sizeof(unsigned long long));
    L.memset_d = T.n4 * sizeof(unsigned long long);   // K4 states (ctrl separately)
    L.seek = p;   p += align256(T.n5 * sizeof(unsigned long long));
    L.bytes = p;  p += align256(scratch_bytes);
    L.total = p;
    return L;
}

// ---------------------------------------------------------------- Table
int Table::create(const tlc_tensor_desc *descs, int cnt, bool with_scratch, void *shared_ws) {
    count = cnt;
    host.assign(cnt, Seg{});
    uint64_t c1 = 0, c2 = 0, c3 = 0, c4 = 0, c5 = 0, scratch = 0, total = 0;
    for (int i = 0; i < cnt; i++) total += descs[i].n;
    const ItemSizes z = item_sizes(total);
    for (int i = 0; i < cnt; i++) {
        const tlc_tensor_desc &d = descs[i];
        if (d.n == 0 || d.n >= (1ull << 42) || !d.hdr) return TLC_ERR_ARG;
        Seg &s = host[i];
        s.t = d.t; s.err = d.err; s.out = d.out; s.payload = d.payload; s.hdr = d.hdr; s.n = d.n;
        seg_items(s, z, c1, c2, c3, c4, c5);
        s.bytes_off = scratch;
        scratch += (s.P + 15) & ~uint64_t(15);
    }
    T = SegTable{};
    T.sz = z;
    T.count = cnt;
    T.n1 = c1; T.n2 = c2; T.n3 = c3; T.n4 = c4; T.n5 = c5;
    for (int i = 0; i < cnt; i++) T.max_n = tmax<uint64_t>(T.max_n, host[i].n);
    if (with_scratch && T.max_n > kSmallMaxN) {                     // compress tables
        const int rc = k12_plan_build(T, host, &d_k12);
        if (rc != TLC_OK) return rc;
    }
    ws_bytes = ws_layout(T, with_scratch ? scratch : 0).total;
    if (cudaMalloc((void **)&d, cnt * sizeof(Seg)) != cudaSuccess) return TLC_ERR_CUDA;
    if (cudaMalloc((void **)&d_first, 5 * (size_t)cnt * sizeof(uint64_t)) != cudaSuccess) return TLC_ERR_CUDA;
    {
        std::vector<uint64_t> f(5 * (size_t)cnt);
        for (int i = 0; i < cnt; i++) {
            f[0 * cnt + i] = host[i].k1; f[1 * cnt + i] = host[i].k2; f[2 * cnt + i] = host[i].k3;
            f[3 * cnt + i] = host[i].k4; f[4 * cnt + i] = host[i].k5;
        }
        if (cudaMemcpy(d_first, f.data(), f.size() * sizeof(uint64_t), cudaMemcpyHostToDevice) != cudaSuccess)
            return TLC_ERR_CUDA;
        for (int k = 0; k < 5; k++) T.first[k] = d_first + (size_t)k * cnt;
    }
    if (T.max_n <= kSmallMaxN) {
        int rc = small_group_plan_build(T, host, &d_grp, grp_layout);
        if (rc == TLC_OK) rc = small_dec_plan_build(T, host, &d_dec, dec_layout);
        if (rc != TLC_OK) return rc;
    }
    if (with_scratch && cnt > 1 && T.max_n <= kSmallMaxN && small_coop_enabled()) {
        const int rc = small_plan_build(T, host, &d_small, sl_layout);
        if (rc != TLC_OK) return rc;
    }
    if (shared_ws) {
        ws = shared_ws;
    } else {
        if (cudaMalloc(&ws, ws_bytes) != cudaSuccess) return TLC_ERR_CUDA;
        own_ws = true;
    }
    return upload();
}

int Table::upload() {
    for (Seg &s : host) s.flags = seg_flags(s);
    bool all = !host.empty();
    for (size_t i = 0; i < host.size(); i++) {
        host[i].seek = i < seekp.size() ? seekp[i] : nullptr;
        all = all && host[i].seek;
    }
    T.all_seek = all ? 1 : 0;
    T.d = d;
    if (count == 1) T.one = host[0];
    // the K2 tiles the bulk-copy kernel takes (count > 1; one tensor uses a tile range)
    std::vector<uint64_t> list, rest;
    bool nozre_ok = true;
    if (count > 1) {
        for (const Seg &s : host) {
            const uint64_t nt = (s.P + T.sz.t2 - 1) / T.sz.t2;
            bool any = false;
            for (uint64_t lt = 0; lt < nt; lt++) {
                if (bulk_tile_ok(s, lt, T.sz.t2)) { list.push_back(s.k2 + lt); any = true; }
                else rest.push_back(s.k2 + lt);
            }
            if (any && !aligned4(s.payload)) nozre_ok = false;
        }
    }
    if (d_bulk) { cudaFree(d_bulk); d_bulk = nullptr; }
    if (!list.empty()) {
        list.insert(list.end(), rest.begin(), rest.end());
        if (cudaMalloc((void **)&d_bulk, list.size() * sizeof(uint64_t)) != cudaSuccess) return TLC_ERR_CUDA;
        if (cudaMemcpy(d_bulk, list.data(), list.size() * sizeof(uint64_t), cudaMemcpyHostToDevice) != cudaSuccess)
            return TLC_ERR_CUDA;
    }
    T.bulk_list = d_bulk;
    T.n_bulk = list.size() - rest.size();
    T.rest_list = d_bulk ? d_bulk + T.n_bulk : nullptr;
    T.n_rest = d_bulk ? rest.size() : 0;
    T.bulk_nozre_ok = nozre_ok ? 1 : 0;
    if (T.sl) {
        const int rc = small_plan_refresh(T, host, sl_layout);   // the slices carry the pointers
        if (rc != TLC_OK) return rc;
    }
    if (T.grp) {
        const int rc = small_group_plan_refresh(T, host, grp_layout);
        if (rc != TLC_OK) return rc;
    }
    if (T.dec) {
        const int rc = small_dec_plan_refresh(T, host, dec_layout);
        if (rc != TLC_OK) return rc;
    }
    return cudaMemcpy(d, host.data(), host.size() * sizeof(Seg), cudaMemcpyHostToDevice) == cudaSuccess
               ? TLC_OK : TLC_ERR_CUDA;
}

int Table::update(const tlc_tensor_desc *descs) {
    for (int i = 0; i < count; i++)
        if (descs[i].n != host[i].n || !descs[i].hdr) return TLC_ERR_ARG;
    for (int i = 0; i < count; i++) {
        Seg &s = host[i];
        s.t = descs[i].t; s.err = descs[i].err; s.out = descs[i].out;
        s.payload = descs[i].payload; s.hdr = descs[i].hdr;
    }
    return upload();
}

void Table::release() {
    if (d) cudaFree(d);
    if (d_first) cudaFree(d_first);
    d_first = nullptr;
    if (d_bulk) cudaFree(d_bulk);
    d_bulk = nullptr;
    if (own_ws && ws) cudaFree(ws);
    if (d_small) cudaFree(d_small);
    d_small = nullptr;
    if (d_grp) cudaFree(d_grp);
    d_grp = nullptr;
    if (d_k12) cudaFree(d_k12);
    d_k12 = nullptr;
    if (d_dec) cudaFree(d_dec);
    d_dec = nullptr;
    d = nullptr;
    ws = nullptr;
}

}  // namespace tlc

using namespace tlc;

struct tlc_batch {
    Table tab;
};

extern "C" {

int tlc_batch_create(tlc_batch **out, int count, const tlc_tensor_desc *descs) {
    if (!out || count < 1 || !descs) return TLC_ERR_ARG;
    auto *b = new tlc_batch{};
    const int rc = b->tab.create(descs, count, true, nullptr);
    if (rc != TLC_OK) {
        b->tab.release();
        delete b;
        return rc;
    }
    *out = b;
    return TLC_OK;
}

int tlc_batch_update(tlc_batch *b, const tlc_tensor_desc *descs) {
    if (!b || !descs) return TLC_ERR_ARG;
    return b->tab.update(descs);
}

int tlc_batch_destroy(tlc_batch *b) {
    if (!b) return TLC_ERR_ARG;
    b->tab.release();
    delete b;
    return TLC_OK;
}

size_t tlc_batch_workspace_bytes(const tlc_batch *b) { return b ? b->tab.ws_bytes : 0; }

int tlc_batch_compress(tlc_batch *b, float s, int use_zre, void *stream) {
    if (!b || !(s >= 1.0f && s < 2.0f)) return TLC_ERR_ARG;
    for (const Seg &g : b->tab.host)
        if (!g.t || !g.err || !g.payload || g.t == g.err) return TLC_ERR_ARG;
    return launch_compress_table(b->tab.T, s, use_zre ? 1 : 0, b->tab.ws, reinterpret_cast<cudaStream_t>(stream));
}

int tlc_batch_decompress(tlc_batch *b, int mode, void *stream) {
    if (!b || (mode != TLC_MODE_OVERWRITE && mode != TLC_MODE_ACCUMULATE)) return TLC_ERR_ARG;
    for (const Seg &g : b->tab.host)
        if (!g.out || !g.payload) return TLC_ERR_ARG;
    return launch_decompress_table(b->tab.T, mode, b->tab.ws, reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
