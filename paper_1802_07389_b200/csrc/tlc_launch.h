// tlc_launch.h -- host-side helpers shared by the kernel launchers.
#pragma once

#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#include "../../include/tlc.h"

namespace tlc {

constexpr int kMaxSms = 256;          // workspace sizing bound (B200 has 148)
constexpr int kK1BlocksPerSm = 2;     // K1 grid = SMs x 2 x 512 threads (2 waves of 1 CTA/SM)

template <class T> __host__ __device__ inline T tmin(T a, T b) { return a < b ? a : b; }
template <class T> __host__ __device__ inline T tmax(T a, T b) { return a < b ? b : a; }

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
__host__ __device__ inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
__host__ __device__ inline bool aligned4(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 3u) == 0; }

inline int num_sms() {
    static int sms[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!sms[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        sms[dev] = v > 0 ? (v > kMaxSms ? kMaxSms : v) : 1;
    }
    return sms[dev];
}

// Programmatic dependent launch: the kernel may be scheduled while its stream
// predecessor drains; it must execute pdl_wait() (griddepcontrol.wait) before
// touching the predecessor's results.  Launch overhead of the chain overlaps.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// Once per device: a kernel's attributes (cudaFuncSetAttribute, e.g. its dynamic shared
// memory limit) belong to the current device's context, so a process driving several GPUs
// sets them on each.
inline int cur_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d & 63;
}
struct PerDevice {
    bool done[64] = {};
    bool first() {
        const int d = cur_device();
        if (done[d]) return false;
        done[d] = true;
        return true;
    }
};

// Kernel ids for launch counting / profiling (prof.cu).
enum KernelId { kK1 = 0, kK2 = 1, kK3 = 2, kK4 = 3, kK5 = 4, kK6 = 5, kK7 = 6, kK8 = 7,
                kK2s = 8, kKq8 = 9, kKd8 = 10, kK6s = 11, kK7s = 12, kK12 = 13, kNumKernelIds = 14 };

struct Ctrl;

// RAII bracket around one kernel launch: counts it and, when profiling is on,
// records CUDA events before and after it on `st`.
class KernelScope {
  public:
    KernelScope(int id, cudaStream_t st);
    ~KernelScope();
  private:
    int id_;
    cudaStream_t st_;
    void *a_;
    int dev_ = 0;
};

// ---------------------------------------------------------------- segments
// Every kernel works on a table of independent tensors ("segments"): a single
// tlc_compress call is a one-segment table passed by value (no upload), a batch
// (tlc_batch_*) is a device-resident table.  Work items of each kernel are
// numbered globally, segment after segment; a CTA maps an item to its segment by
// a binary search over the per-segment first-item numbers.
// Work-item sizes of a table: large tables favour long streams per item, small ones
// (e.g. the 1.7M values of ResNet-110) more items so that every SM gets work.
struct ItemSizes {
    uint64_t t1;    // K1 tile: elements
    uint64_t t2;    // K2 tile: quartic positions
    uint64_t c3;    // K3 chunk: quartic bytes (8 warps x rows of 1 KiB)
    uint64_t c4;    // K4 chunk: payload bytes (capacity based)
};
#ifndef TLC_K4_CHUNK
#define TLC_K4_CHUNK 16384                 // K4 chunk of large tables (A/B builds: 32768, 65536)
#endif
constexpr ItemSizes kLargeItems{65536, 4096, 32768, TLC_K4_CHUNK};
constexpr ItemSizes kSmallItems{8192, 1024, 8192, 4096};
constexpr uint64_t kSmallTableElems = 32ull << 20;   // tables below 32M values use kSmallItems
constexpr uint64_t kT5 = 4096;      // K5 tile: quartic positions per output tile
// Tables whose tensors all have at most kSmallMaxN values (P <= 8192 quartic bytes) take
// the fused one-CTA-per-tensor kernels of small.cu (u staged in 160 KiB of shared memory).
constexpr uint64_t kSmallMaxN = 40960;

enum SegFlags : uint32_t { kSegVec2 = 1u, kSegVec5 = 2u, kSegVec1 = 4u };

struct Seg {
    const float *t;
    float *err;
    float *out;
    uint8_t *payload;
    tlc_header *hdr;
    uint64_t n, P;
    uint64_t k1, k2, k3, k4, k5;    // first global item of each kernel
    uint64_t bytes_off;             // quartic scratch offset (compress with ZRE)
    uint32_t flags, pad;
    // seek entries of the segment's K5 tiles written by the producer (nullptr: none).  A
    // compress table's K3 writes them as it emits the payload; a decompress table whose
    // segments all carry them (payloads produced by this library's K3 in the same exchange,
    // read over peer memory) skips K4 and K5 reads them instead of the workspace's.
    unsigned long long *seek;
};

// A slice of a small tensor (K6c): quartic positions [j0, j0+len) of segment `seg` with
// the segment's pointers and sizes, its index k among the segment's slices (the first at
// global slice id `first`), last = 1 for the segment's last slice.
struct SliceRec {
    const float *t;
    float *err;
    uint8_t *payload;
    tlc_header *hdr;
    uint32_t n, P, j0, len;
    uint32_t first, k, last, seg;
};
static_assert(sizeof(SliceRec) == 64, "slice records are 64 bytes");

// A CTA of the K6g cluster launch (small.cu): quartic positions [j0, j0+len) of segment `seg`
// (~0u: an idle CTA) with the segment's pointers and sizes; the tensor's slices sit at cluster
// ranks g0 .. g0+gcnt-1, this one at g0+grank.
struct GrpRec {
    const float *t;
    float *err;
    uint8_t *payload;
    tlc_header *hdr;
    uint32_t n, P, j0, len;
    uint32_t g0, gcnt, grank, seg;
};
static_assert(sizeof(GrpRec) == 64, "group records are 64 bytes");

// A CTA of the K7 record launch (small.cu): quartic positions [jr0, jr0+pl) of a segment's
// decode, with the segment's pointers and sizes; first = 1 for the segment's first part.
struct DecRec {
    const uint8_t *payload;
    tlc_header *hdr;
    float *out;
    uint32_t n, P, jr0, pl;
    uint32_t first, seg;
};
static_assert(sizeof(DecRec) == 48, "decode records are 48 bytes");

struct SegTable {
    const Seg *d;                   // device table when count > 1
    Seg one;                        // the segment when count == 1
    int count;
    uint64_t n1, n2, n3, n4, n5;    // total items per kernel
    ItemSizes sz;
    const uint64_t *first[5];       // device: first item of every segment, per kernel (count > 1)
    uint64_t max_n;                 // largest segment
    const uint64_t *bulk_list;      // device: K2 tiles taken by the bulk (TMA) kernel (count > 1)
    uint64_t n_bulk;                // entries of bulk_list
    const uint64_t *rest_list;      // device: the other K2 tiles (the register kernel's, when bulk runs)
    uint64_t n_rest;
    int bulk_nozre_ok;              // every listed segment's payload is 4-byte aligned
    // small tables (K6c, small.cu): slices of <= kSlice quartic positions of the segments,
    // contiguous runs of them per CTA of one cooperative launch (sl == nullptr: no plan)
    const struct SliceRec *sl;      // every slice with its tensor's pointers (refreshed at upload)
    const uint32_t *sl_cta;         // first slice of every CTA (sl_grid + 1 entries)
    unsigned int *sl_key;           // per segment max key, zero between launches
    unsigned long long *sl_sum;     // per slice ZRE run summary
    unsigned long long *sl_bar;     // grid barrier counter (monotonic)
    int sl_grid;
    uint32_t sl_smem;               // dynamic shared memory of the launch
    // small tables (K6g, small.cu): one record per CTA of a cluster launch (refreshed at
    // upload: the records carry the pointers); grp == nullptr: no plan
    // tables of several tensors (K12, compress.cu): the fused K1/K2 work list, K1 and K2 tiles
    // of consecutive L2-sized windows of tensors interleaved (k12 == nullptr: no plan)
    const uint32_t *k12;            // item = K2 tile index << 1 | (1: quantize, 0: max)
    uint32_t k12_n;
    const DecRec *dec;              // K7 records (small tables; nullptr: K7 walks the table)
    int dec_grid;
    const GrpRec *grp;
    int grp_grid;                   // CTAs (a multiple of grp_cl)
    int grp_cl;                     // cluster size
    uint32_t grp_maxlen;            // longest slice (quartic positions)
    int all_seek;                   // every segment carries producer seek entries (Seg::seek)
};

// Workspace layout of one table: control block, per-segment max keys, K3 / K4
// chunk states, K5 seek entries, quartic scratch.
struct WsLayout {
    size_t ctrl, maxkey, k12done, k3st, k4st, seek, bytes, memset_c, memset_d, total;
};

WsLayout ws_layout(const SegTable &T, uint64_t scratch_bytes);
void seg_items(Seg &s, const ItemSizes &z, uint64_t &c1, uint64_t &c2, uint64_t &c3, uint64_t &c4, uint64_t &c5);
inline ItemSizes item_sizes(uint64_t total_elems) { return total_elems < kSmallTableElems ? kSmallItems : kLargeItems; }
SegTable single_table(const float *t, float *err, float *out, uint8_t *payload, tlc_header *hdr, uint64_t n,
                      uint64_t &scratch);
int launch_compress_table(const SegTable &T, float s, int use_zre, void *ws, cudaStream_t st);
// K12 work list of a table of several tensors (sizes only); no-op when K12 is off or the
// table is small or a single tensor
int k12_plan_build(SegTable &T, const std::vector<Seg> &host, uint32_t **d_k12);
int launch_compress(const float *t, float *err, uint64_t n, float s, int use_zre, uint8_t *payload,
                    tlc_header *hdr, void *ws, cudaStream_t st);
size_t compress_workspace_bytes(uint64_t n);
int launch_decompress(const uint8_t *payload, tlc_header *hdr, uint64_t n, float *out, int mode,
                      void *ws, cudaStream_t st);
size_t decompress_workspace_bytes(uint64_t n);
uint32_t seg_flags(const Seg &s);
// K2 tile lt (t2 positions) of segment s can go through the bulk-copy kernel: t and err
// 16-byte aligned, and all positions of the tile have their five elements with 4 elements
// of slack at the end (unaligned partitions are fetched as aligned supersets).
__host__ __device__ inline bool bulk_tile_ok(const Seg &s, uint64_t lt, uint64_t t2) {
    if (!aligned16(s.t) || !aligned16(s.err)) return false;
    const uint64_t complete = s.n >= 4 * s.P + 4 ? (s.P < s.n - 4 * s.P - 4 ? s.P : s.n - 4 * s.P - 4) : 0;
    return (lt + 1) * t2 <= complete;
}

// A device-resident segment table with its workspace (batches, exchange).
struct Table {
    int count = 0;
    std::vector<Seg> host;
    Seg *d = nullptr;
    uint64_t *d_first = nullptr;    // 5 x count first-item arrays
    uint64_t *d_bulk = nullptr;     // eligible K2 tiles of the bulk kernel, then the rest
    SegTable T{};
    void *ws = nullptr;
    size_t ws_bytes = 0;
    bool own_ws = false;
    void *d_small = nullptr;        // the K6c plan and its state (small tables only)
    GrpRec *d_grp = nullptr;        // the K6g plan (small tables only)
    uint32_t *d_k12 = nullptr;      // the K12 work list (tables of several tensors)
    std::vector<uint4> grp_layout;  // K6g CTAs on the host: (seg, j0, len, g0 | gcnt << 8 | grank << 16)
    DecRec *d_dec = nullptr;        // the K7 records (small tables only)
    std::vector<uint4> dec_layout;  // K7 CTAs on the host: (seg, jr0, pl, first)
    std::vector<uint4> sl_layout;   // K6c slices on the host: (seg, j0, len, k | last << 16)
    std::vector<unsigned long long *> seekp;   // per segment Seg::seek (empty: none), kept across update()
    int create(const tlc_tensor_desc *descs, int cnt, bool with_scratch, void *shared_ws);
    int update(const tlc_tensor_desc *descs);
    int upload();
    void release();
};
int launch_decompress_table(const SegTable &T, int mode, void *ws, cudaStream_t st);

// Small tensors (small.cu): one CTA per tensor, one launch per direction.
bool small_enabled();
bool small_coop_enabled();   // TLC_COOP=1: small tables take K6c (its plan is only built then)
bool small_table(const SegTable &T);
// K6c plan of a small table (slices, CTA runs, state); leaves T.sl null when the table does
// not fit one cooperative wave (K6, one CTA per tensor, then runs instead)
int small_plan_build(SegTable &T, const std::vector<Seg> &host, void **d_small, std::vector<uint4> &layout);
int small_plan_refresh(const SegTable &T, const std::vector<Seg> &host, const std::vector<uint4> &layout);
int launch_small_compress(const SegTable &T, float s, int use_zre, cudaStream_t st);
// K6g plan of a small table: every tensor cut into up to `cl` slices of whole 1 KiB ZRE rows,
// the slices of one tensor in one thread-block cluster, clusters packed best-fit; depends on
// the sizes only (the kernel takes the pointers from the table).  No-op when K6g is off.
int small_group_plan_build(SegTable &T, const std::vector<Seg> &host, GrpRec **d_grp, std::vector<uint4> &layout);
int small_group_plan_refresh(const SegTable &T, const std::vector<Seg> &host, const std::vector<uint4> &layout);
int small_dec_plan_build(SegTable &T, const std::vector<Seg> &host, DecRec **d_dec, std::vector<uint4> &layout);
int small_dec_plan_refresh(const SegTable &T, const std::vector<Seg> &host, const std::vector<uint4> &layout);
int launch_small_decompress(const SegTable &T, int mode, cudaStream_t st);

// K1 alone: per-segment max key of |err + t| (has_err) or |t| into maxkey[].
void launch_absmax(const SegTable &T, unsigned int *maxkey, bool has_err, cudaStream_t st);
// Compared designs of Sec. 5.1 (stoch.cu, int8.cu).
void launch_stoch_qe(const SegTable &T, const unsigned int *maxkey, uint64_t seed, uint64_t step, int use_zre,
                     uint8_t *scratch, cudaStream_t st);
int launch_stoch_compress_table(const SegTable &T, uint64_t seed, uint64_t step, int use_zre, void *ws,
                                cudaStream_t st);
int launch_int8_compress(const float *t, uint64_t n, int8_t *codes, tlc_header *hdr, void *ws, cudaStream_t st);
int launch_int8_decompress(const int8_t *codes, tlc_header *hdr, uint64_t n, float *out, int mode, cudaStream_t st);
// keys (optional, W >= 2): K1's max keys of u = K.err + mean per context of A (K = the
// owner's pull compress table, same context order), folded by atomicMax into `keys`
int launch_aggregate(const SegTable &A, const SegTable &X, int W, void *xws, cudaStream_t st,
                     const SegTable *K = nullptr, unsigned int *keys = nullptr);
// the compress path of a table takes its max keys from elsewhere (K1 skipped, workspace
// control block, keys and scan states zeroed by prepare_keyed_compress beforehand)
int prepare_keyed_compress(const SegTable &T, void *ws, cudaStream_t st, unsigned int **keys);
int launch_compress_table_keyed(const SegTable &T, float s, int use_zre, void *ws, cudaStream_t st);
bool compress_runs_k1(const SegTable &T);
bool aggregate_keyable(int W);                 // the parallel K5m (W >= 2) can fold the keys

}  // namespace tlc
