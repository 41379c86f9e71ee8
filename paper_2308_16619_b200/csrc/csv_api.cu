// csv_api.cu -- C-ABI of libcsvgpu.so (declared in include/csvgpu.h).
//
// Owns the per-volume device state: directory unpacked to SoA, the three
// blobs (+16 B tail padding), packed decode tables, and a grow-only decode
// workspace.  All entry points are extern "C" with plain pointers; see the
// header for the reference function each one replaces.
#include <cstdio>
#include <cstring>
#include <cstdarg>
#include <string>
#include <vector>
#include <algorithm>
#include <mutex>
#include <cstdlib>
#include "csv_device.cuh"

namespace csv {
cudaError_t run_decode(const VolView& V, Plan P, int mode, uint64_t* sizes_tmp, uint64_t* scan_tmp,
                       unsigned long long* counter, uint32_t* gws, uint64_t gws_stride, int gws_ctas,
                       int nsm, int min_t, cudaStream_t st, cudaEvent_t* ev, const Overlap* ov);
cudaError_t run_root_raster(const VolView& V, Plan P, cudaStream_t st);
cudaError_t run_streams_only(const VolView& V, Plan P, uint64_t* sizes_tmp, uint64_t* scan_tmp,
                             unsigned long long* counter, int nsm, cudaStream_t st);
size_t k2_smem_bytes(int L);
cudaError_t run_op_counts(const VolView& V, Plan P, unsigned long long* counter, int nsm, cudaStream_t st);
uint64_t k2_gws_words(int L);
}  // namespace csv

using namespace csv;

static thread_local std::string g_err;
namespace csv { void set_error(const char* msg) { g_err = msg; } }

static int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}
#define CUDA_TRY(x)                                                                         \
    do {                                                                                    \
        cudaError_t e_ = (x);                                                               \
        if (e_ != cudaSuccess) return fail(CSV_E_CUDA, "%s: %s", #x, cudaGetErrorString(e_)); \
    } while (0)

struct csv_volume {
    int device = 0;
    VolView V{};
    void* d_soa = nullptr;          // directory SoA columns
    uint8_t* d_blob = nullptr;      // owned blobs (host upload) or nullptr (borrowed)
    uint32_t* d_dtab = nullptr;
    // workspace (grow-only)
    uint64_t plan_cap = 0;          // requests
    uint64_t* d_sizes = nullptr;    // 2*cap
    uint64_t* d_eoff = nullptr;     // 2*cap + 1
    uint64_t* d_scan = nullptr;     // 4097
    csv_stream_result* d_sres = nullptr;
    unsigned long long* d_counter = nullptr;
    uint8_t* d_entries = nullptr;
    uint64_t entries_cap = 0;
    uint32_t* d_gws = nullptr;
    uint16_t* d_wscratch = nullptr;  // K2w per-warp palette bases (nsm x 64 warps x 4096)
    uint16_t* d_wscratch6 = nullptr; // K2w<6> per-warp slots (nsm x 8 warps x kWScratch6Stride), N >= 6 only
    uint64_t gws_stride = 0;
    int gws_ctas = 0;
    uint64_t gws_words_cap = 0;
    int nsm = 148;
    uint64_t region_total_t0 = 0;   // sum over bricks of entry regions at t=0 (bytes)
    uint64_t region_max_t0 = 0;     // max over bricks
    int64_t dims[3]{}, grid[3]{};
    uint64_t blob_cap[3]{};         // bytes of the palette / coarse / detail slices held
    bool timing = false;
    cudaEvent_t ev[4]{};            // plan start, K1 start, K1 end / K2 start, K2 end
    Overlap ovl{};                  // K1 -> K2w overlap side stream (run_decode)
    // csv_decode_bricks_host: pinned request staging + device requests / pool / results (grow-only)
    uint64_t hreq_cap = 0, hpool_cap = 0;
    uint8_t* h_req = nullptr;       // pinned: brick u32[cap] | lod u8[cap] (16-aligned) | dst u64[cap]
    uint8_t* d_req = nullptr;       // same layout on the device
    csv_result* d_hres = nullptr;
    uint32_t* d_hpool = nullptr;
    // per-brick calls (n <= kBrickGraphMax): the request copy and the decode launches (storing
    // labels and results into mapped pinned staging) replayed as ONE CUDA graph, keyed by (n, voxels) and the
    // workspace pointers; captured on the second call with a key (the first one sizes the
    // workspace and loads the kernels), on a private stream
    struct BrickGraph {
        cudaGraphExec_t exec = nullptr;
        uint64_t n = 0, total = 0, seen = 0, wide = 0;
        const void* ptrs[8]{};
    } bgraph[8];
    uint32_t bg_next = 0;
    cudaStream_t cap_stream = nullptr;
    std::mutex host_mu;             // csv_decode_bricks_host: staging buffers and graphs are per volume
    uint8_t* h_bout = nullptr;      // pinned + mapped: labels then results of a graph replay (the kernels store
                                    // into it over PCIe: no copy-back nodes)
    std::vector<uint32_t> h_paln;   // palette length per brick (host directory only): per-brick plans skip
                                    // the u16 replay pass when no request needs it
    uint64_t h_bout_cap = 0;
};
constexpr uint64_t kBrickGraphMax = 16;

// ---------------------------------------------------------------------------- kernels local to the API
// Unpack 44-byte directory rows (container.py:53-64) into SoA, rebasing global
// blob offsets to the uploaded slices and clamping lengths like numpy slicing.
__global__ void k_unpack_dir(const uint8_t* dir44, uint64_t n, uint64_t pal_base, uint64_t pal_len,
                             uint64_t c_base, uint64_t c_len, uint64_t d_base, uint64_t d_len,
                             uint64_t* pal_off, uint32_t* pal_n, uint64_t* c_off, uint32_t* c_bytes,
                             uint32_t* c_nib, uint64_t* d_off, uint32_t* d_bytes, uint32_t* d_nib) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint8_t* p = dir44 + 44 * i;
    auto u64 = [&](int o) { uint64_t v = 0; for (int k = 7; k >= 0; --k) v = (v << 8) | p[o + k]; return v; };
    auto u32 = [&](int o) { uint32_t v = 0; for (int k = 3; k >= 0; --k) v = (v << 8) | p[o + k]; return v; };
    auto clamp = [](uint64_t off, uint64_t len, uint64_t base, uint64_t avail, uint64_t* ooff) -> uint64_t {
        // slice blob[off : off+len] of the global blob, of which [base, base+avail) was uploaded
        if (off < base || off >= base + avail) { *ooff = 0; return 0; }
        uint64_t rel = off - base;
        uint64_t l = avail - rel;
        *ooff = rel;
        return len < l ? len : l;
    };
    uint64_t o;
    pal_n[i] = (uint32_t)clamp(u64(0), u32(8), pal_base, pal_len, &o);
    pal_off[i] = o;
    c_bytes[i] = (uint32_t)clamp(u64(12), u32(20), c_base, c_len, &o);
    c_off[i] = o;
    c_nib[i] = u32(24);
    d_bytes[i] = (uint32_t)clamp(u64(28), u32(36), d_base, d_len, &o);
    d_off[i] = o;
    d_nib[i] = u32(40);
}

__global__ void k_region_stats(VolView V, unsigned long long* total, unsigned long long* mx) {
    uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (b < V.nb) atomicMax(mx + 1, (unsigned long long)V.pal_len[b]);
    unsigned long long s = 0;
    if (b < V.nb && V.N > 0) s = round32(stream_limit(V, b, 0, 0)) + round32(stream_limit(V, b, 0, 1));
    unsigned long long m = s;
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        unsigned long long u = __shfl_xor_sync(0xffffffffu, m, o);
        m = m > u ? m : u;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(total, s);
        atomicMax(mx, m);
    }
}

// Cold detail (render.py:782-832): point the staged bricks' detail streams at
// the frame's staging buffer; every other brick has no detail until staged.
__global__ void k_stage_detail(uint64_t* d_off, uint32_t* d_bytes, uint64_t brick_begin, uint64_t nb,
                               const uint32_t* bricks, const uint64_t* offs, const uint32_t* lens, uint64_t n) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint64_t b = (uint64_t)bricks[i] - brick_begin;
    if (b < nb) {
        d_off[b] = offs[i];
        d_bytes[b] = lens[i];
    }
}

// One-brick scratch volume (csv_decode_brick_streams): brick 0's directory row, set per call.
__global__ void k_set_brick0(uint64_t* pal_off, uint32_t* pal_n, uint64_t* c_off, uint32_t* c_bytes, uint32_t* c_nib,
                             uint64_t* d_off, uint32_t* d_bytes, uint32_t* d_nib, uint32_t np, uint32_t cb, uint32_t cn,
                             uint32_t db, uint32_t dn) {
    pal_off[0] = 0; pal_n[0] = np;
    c_off[0] = 0; c_bytes[0] = cb; c_nib[0] = cn;
    d_off[0] = 0; d_bytes[0] = db; d_nib[0] = dn;
}

// ---------------------------------------------------------------------------- helpers
static int parse_head(const uint8_t* h, csv_volume* v, uint32_t* dtab_host) {
    if (memcmp(h, "CSV1", 4) != 0) return fail(CSV_E_FORMAT, "bad magic");
    uint16_t version; memcpy(&version, h + 4, 2);
    if (version != 1) return fail(CSV_E_FORMAT, "unsupported container version %u", version);
    uint8_t flags = h[6];
    uint16_t bl2; memcpy(&bl2, h + 10, 2);
    uint32_t d3[3]; memcpy(d3, h + 12, 12);
    if (bl2 < 1 || bl2 > 7) return fail(CSV_E_FORMAT, "brick_log2 must be in [1, 7], got %u", bl2);
    v->V.N = bl2;
    v->V.entropy = flags & 1;
    int64_t b = 1ll << bl2;
    for (int k = 0; k < 3; ++k) {
        v->dims[k] = d3[k];
        v->grid[k] = (d3[k] + b - 1) / b;
    }
    v->V.X = d3[0]; v->V.Y = d3[1]; v->V.Z = d3[2];
    v->V.gx = v->grid[0]; v->V.gy = v->grid[1]; v->V.gz = v->grid[2];
    // packed decode tables {freq:16 | (slot-cum):12 | sym:4} (rans.py:31-62, codec.py:290-300)
    v->V.fast_tab = 1;
    for (int tb = 0; tb < 2; ++tb) {
        uint16_t cnt[16];
        memcpy(cnt, h + 32 + 32 * tb, 32);
        for (int s = 0; s < 16; ++s)
            if (cnt[s] > 4095) v->V.fast_tab = 0;
        uint32_t sum = 0;
        for (int s = 0; s < 16; ++s) sum += cnt[s];
        if (sum != kTotalFreq && v->V.entropy) return fail(CSV_E_FORMAT, "counts must sum to 4096, got %u", sum);
        uint32_t slot = 0;
        for (int s = 0; s < 16 && slot < kTotalFreq; ++s)
            for (uint32_t j = 0; j < cnt[s] && slot < kTotalFreq; ++j, ++slot)
                dtab_host[tb * 4096 + slot] = ((uint32_t)cnt[s] << 16) | (j << 4) | (uint32_t)s;
        for (; slot < kTotalFreq; ++slot) dtab_host[tb * 4096 + slot] = (1u << 16) | 0u;
    }
    return CSV_OK;
}

// Volume memory comes from the device's default stream-ordered pool, which keeps up
// to kPoolKeep bytes (env CSVGPU_POOL_KEEP_GB overrides) of freed blocks mapped for
// the next volume: a host-in/host-out
// decompress_volume creates and frees a ~2 GB volume per call, and plain
// cudaMalloc/cudaFree of that made every call pay 10-850 ms of driver page mapping.
// Frees follow a device synchronisation (the cudaFree semantics the callers rely on).
constexpr uint64_t kPoolKeep = 8ull << 30;
constexpr int kPoolDevices = 64;
static std::once_flag g_pool_once[kPoolDevices];

static void pool_init(int device) {
    if (device < 0 || device >= kPoolDevices) return;
    std::call_once(g_pool_once[device], [device] {
        cudaMemPool_t mp;
        if (cudaDeviceGetDefaultMemPool(&mp, device) == cudaSuccess) {
            uint64_t keep = kPoolKeep;
            if (const char* g = std::getenv("CSVGPU_POOL_KEEP_GB")) keep = (uint64_t)(std::atof(g) * (1ull << 30));
            cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    });
}

template <typename T>
static cudaError_t dalloc(T** p, size_t bytes, cudaStream_t st) {
    return cudaMallocAsync(reinterpret_cast<void**>(p), bytes ? bytes : 16, st);
}

template <typename T>
static void dfree(T*& p) {   // caller has synchronised the device (or the pointer's stream)
    if (p) cudaFreeAsync(reinterpret_cast<void*>(p), 0);
    p = nullptr;
}

static void vol_release(csv_volume* v) {
    if (!v) return;
    cudaSetDevice(v->device);
    cudaDeviceSynchronize();
    dfree(v->d_soa); dfree(v->d_blob); dfree(v->d_dtab);
    dfree(v->d_sizes); dfree(v->d_eoff); dfree(v->d_scan); dfree(v->d_sres);
    dfree(v->d_counter); dfree(v->d_entries); dfree(v->d_gws); dfree(v->d_wscratch); dfree(v->d_wscratch6);
    dfree(v->d_req); dfree(v->d_hres); dfree(v->d_hpool);
    if (v->h_req) cudaFreeHost(v->h_req);
    for (auto& g : v->bgraph) if (g.exec) cudaGraphExecDestroy(g.exec);
    if (v->cap_stream) cudaStreamDestroy(v->cap_stream);
    if (v->h_bout) cudaFreeHost(v->h_bout);
    cudaStreamSynchronize(0);
    for (auto& e : v->ev) if (e) cudaEventDestroy(e);
    if (v->ovl.fork) cudaEventDestroy(v->ovl.fork);
    if (v->ovl.join) cudaEventDestroy(v->ovl.join);
    if (v->ovl.side) cudaStreamDestroy(v->ovl.side);
    delete v;
}

static int ensure_plan(csv_volume* v, uint64_t n, uint64_t entries_need, int Lg, cudaStream_t st) {
    if (n > v->plan_cap) {
        uint64_t cap = std::max<uint64_t>(n, 1024);
        if (v->d_sizes) CUDA_TRY(cudaDeviceSynchronize());
        dfree(v->d_sizes); dfree(v->d_eoff); dfree(v->d_sres);
        v->plan_cap = 0;
        CUDA_TRY(dalloc(&v->d_sizes, 2 * cap * sizeof(uint64_t), st));
        CUDA_TRY(dalloc(&v->d_eoff, (2 * cap + 1) * sizeof(uint64_t), st));
        CUDA_TRY(dalloc(&v->d_sres, 2 * cap * sizeof(csv_stream_result), st));
        v->plan_cap = cap;
    }
    if (!v->d_wscratch) CUDA_TRY(dalloc(&v->d_wscratch, (size_t)v->nsm * 64 * kWScratchStride * sizeof(uint16_t), st));
    if (!v->d_wscratch6 && v->V.N >= 6)
        CUDA_TRY(dalloc(&v->d_wscratch6, (size_t)v->nsm * kK2W6MaxWarpsPerSM * kWScratch6Stride * sizeof(uint16_t), st));
    if (!v->d_scan) {
        CUDA_TRY(dalloc(&v->d_scan, (kScanTmpSlots + 512) * sizeof(uint64_t), st));
        CUDA_TRY(dalloc(&v->d_counter, kCounterSlots * sizeof(unsigned long long), st));
    }
    if (!v->ovl.side) {
        CUDA_TRY(cudaStreamCreateWithFlags(&v->ovl.side, cudaStreamNonBlocking));
        CUDA_TRY(cudaEventCreateWithFlags(&v->ovl.fork, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&v->ovl.join, cudaEventDisableTiming));
    }
    if (entries_need + 64 > v->entries_cap) {
        if (v->d_entries) CUDA_TRY(cudaDeviceSynchronize());
        dfree(v->d_entries);
        v->entries_cap = 0;
        uint64_t cap = entries_need + 64;
        CUDA_TRY(dalloc(&v->d_entries, cap, st));
        v->entries_cap = cap;
    }
    if (Lg > 5) {
        uint64_t words = k2_gws_words(Lg);
        words = (words + 31) & ~31ull;
        int ctas = v->nsm * 2;
        if (words * ctas > v->gws_words_cap) {
            if (v->d_gws) CUDA_TRY(cudaDeviceSynchronize());
            dfree(v->d_gws);
            CUDA_TRY(dalloc(&v->d_gws, words * ctas * 4, st));
            v->gws_words_cap = words * ctas;
        }
        v->gws_stride = words;
        v->gws_ctas = ctas;
    }
    return CSV_OK;
}

static int vol_create(int device, const uint8_t* head120, const uint8_t* dir44, bool dir_on_device,
                      uint64_t brick_begin, uint64_t brick_end,
                      const uint32_t* palette, uint64_t palette_base, uint64_t palette_len,
                      const uint8_t* coarse, uint64_t coarse_base, uint64_t coarse_len,
                      const uint8_t* detail, uint64_t detail_base, uint64_t detail_len,
                      bool blobs_on_device, uintptr_t stream, csv_volume** out, bool deferred = false) {
    if (!head120 || !out) return fail(CSV_E_ARG, "null argument");
    if (brick_end < brick_begin) return fail(CSV_E_ARG, "brick_end < brick_begin");
    CUDA_TRY(cudaSetDevice(device));
    pool_init(device);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    csv_volume* v = new csv_volume();
    v->device = device;
    std::vector<uint32_t> dtab(8192);
    int rc = parse_head(head120, v, dtab.data());
    if (rc != CSV_OK) { delete v; return rc; }
    uint64_t ntot = (uint64_t)(v->grid[0] * v->grid[1] * v->grid[2]);
    if (brick_end > ntot) { delete v; return fail(CSV_E_ARG, "brick range [%llu, %llu) exceeds %llu bricks",
                                                  (unsigned long long)brick_begin, (unsigned long long)brick_end,
                                                  (unsigned long long)ntot); }
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    v->nsm = nsm;
    uint64_t n = brick_end - brick_begin;
    v->V.brick_begin = brick_begin;
    v->V.nb = n;
    // directory SoA
    size_t soa_bytes = n * (8 + 4 + 8 + 4 + 4 + 8 + 4 + 4) + 64;
    cudaError_t ce = dalloc(&v->d_soa, soa_bytes, st);
    if (ce != cudaSuccess) { vol_release(v); return fail(CSV_E_NOMEM, "directory: %s", cudaGetErrorString(ce)); }
    uint8_t* p = (uint8_t*)v->d_soa;
    uint64_t* pal_off = (uint64_t*)p; p += 8 * n;
    uint64_t* c_off = (uint64_t*)p; p += 8 * n;
    uint64_t* d_off = (uint64_t*)p; p += 8 * n;
    uint32_t* pal_n = (uint32_t*)p; p += 4 * n;
    uint32_t* c_bytes = (uint32_t*)p; p += 4 * n;
    uint32_t* c_nib = (uint32_t*)p; p += 4 * n;
    uint32_t* d_bytes = (uint32_t*)p; p += 4 * n;
    uint32_t* d_nib = (uint32_t*)p; p += 4 * n;
    v->V.pal_off = pal_off; v->V.pal_len = pal_n; v->V.c_off = c_off; v->V.c_bytes = c_bytes;
    v->V.c_nib = c_nib; v->V.d_off = d_off; v->V.d_bytes = d_bytes; v->V.d_nib = d_nib;
    // blobs
    if (blobs_on_device) {
        v->V.palette = palette;
        v->V.coarse = coarse;
        v->V.detail = detail;
    } else {
        uint64_t pb = ((palette_len * 4 + 15) & ~15ull) + kBlobPad;
        uint64_t cb = ((coarse_len + 15) & ~15ull) + kBlobPad;
        uint64_t db = ((detail_len + 15) & ~15ull) + kBlobPad;
        ce = dalloc(&v->d_blob, pb + cb + db, st);
        if (ce != cudaSuccess) { vol_release(v); return fail(CSV_E_NOMEM, "blobs: %s", cudaGetErrorString(ce)); }
        cudaMemsetAsync(v->d_blob, 0, pb + cb + db, st);
        if (!deferred) {
            if (palette_len) cudaMemcpyAsync(v->d_blob, palette, palette_len * 4, cudaMemcpyHostToDevice, st);
            if (coarse_len) cudaMemcpyAsync(v->d_blob + pb, coarse, coarse_len, cudaMemcpyHostToDevice, st);
            if (detail_len) cudaMemcpyAsync(v->d_blob + pb + cb, detail, detail_len, cudaMemcpyHostToDevice, st);
        }
        v->blob_cap[0] = palette_len * 4; v->blob_cap[1] = coarse_len; v->blob_cap[2] = detail_len;
        v->V.palette = (const uint32_t*)v->d_blob;
        v->V.coarse = v->d_blob + pb;
        v->V.detail = v->d_blob + pb + cb;
    }
    ce = dalloc(&v->d_dtab, 8192 * 4, st);
    if (ce != cudaSuccess) { vol_release(v); return fail(CSV_E_NOMEM, "tables"); }
    cudaMemcpyAsync(v->d_dtab, dtab.data(), 8192 * 4, cudaMemcpyHostToDevice, st);
    v->V.dtab = v->d_dtab;
    if (n) {
        const uint8_t* ddir = dir44;
        uint8_t* tmp = nullptr;
        if (!dir_on_device) {
            v->h_paln.resize(n);
            for (uint64_t i = 0; i < n; ++i) {
                const uint8_t* r = dir44 + 44 * i + 8;
                v->h_paln[i] = (uint32_t)r[0] | ((uint32_t)r[1] << 8) | ((uint32_t)r[2] << 16) | ((uint32_t)r[3] << 24);
            }
            ce = dalloc(&tmp, n * 44, st);
            if (ce != cudaSuccess) { vol_release(v); return fail(CSV_E_NOMEM, "directory staging"); }
            cudaMemcpyAsync(tmp, dir44, n * 44, cudaMemcpyHostToDevice, st);
            ddir = tmp;
        }
        k_unpack_dir<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(ddir, n, palette_base, palette_len, coarse_base,
                                                               coarse_len, detail_base, detail_len, pal_off, pal_n,
                                                               c_off, c_bytes, c_nib, d_off, d_bytes, d_nib);
        unsigned long long* stats = nullptr;
        dalloc(&stats, 24, st);
        cudaMemsetAsync(stats, 0, 24, st);
        k_region_stats<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(v->V, stats, stats + 1);
        unsigned long long hs[3] = {0, 0, 0};
        cudaMemcpyAsync(hs, stats, 24, cudaMemcpyDeviceToHost, st);
        cudaFreeAsync(stats, st);
        if (tmp) cudaFreeAsync(tmp, st);
        ce = cudaStreamSynchronize(st);
        if (ce != cudaSuccess) { vol_release(v); return fail(CSV_E_CUDA, "create: %s", cudaGetErrorString(ce)); }
        v->region_total_t0 = hs[0];
        v->region_max_t0 = hs[1];
        v->V.max_pal = (uint32_t)(hs[2] < 0xffffffffull ? hs[2] : 0xffffffffull);
    }
    // pool allocations, the zero fill and the uploads must land before other streams use them
    ce = cudaStreamSynchronize(st);
    if (ce != cudaSuccess) { vol_release(v); return fail(CSV_E_CUDA, "create: %s", cudaGetErrorString(ce)); }
    *out = v;
    return CSV_OK;
}

namespace csv {
const VolView& volume_view(const csv_volume* v) { return v->V; }
int volume_device(const csv_volume* v) { return v->device; }
}  // namespace csv

// ---------------------------------------------------------------------------- exported API
extern "C" {

int csv_version(void) { return 1; }
const char* csv_last_error(void) { return g_err.c_str(); }

int csv_volume_create(int device, const uint8_t* head120, const uint8_t* dir44, uint64_t brick_begin,
                      uint64_t brick_end, const uint32_t* palette, uint64_t palette_base, uint64_t palette_len,
                      const uint8_t* coarse, uint64_t coarse_base, uint64_t coarse_len, const uint8_t* detail,
                      uint64_t detail_base, uint64_t detail_len, uintptr_t stream, csv_volume** vol) {
    return vol_create(device, head120, dir44, false, brick_begin, brick_end, palette, palette_base, palette_len,
                      coarse, coarse_base, coarse_len, detail, detail_base, detail_len, false, stream, vol);
}

int csv_volume_create_device(int device, const uint8_t* head120, const uint8_t* d_dir44, uint64_t brick_begin,
                             uint64_t brick_end, const uint32_t* d_palette, uint64_t palette_base,
                             uint64_t palette_len, const uint8_t* d_coarse, uint64_t coarse_base,
                             uint64_t coarse_len, const uint8_t* d_detail, uint64_t detail_base,
                             uint64_t detail_len, uintptr_t stream, csv_volume** vol) {
    return vol_create(device, head120, d_dir44, true, brick_begin, brick_end, d_palette, palette_base, palette_len,
                      d_coarse, coarse_base, coarse_len, d_detail, detail_base, detail_len, true, stream, vol);
}

int csv_volume_create_deferred(int device, const uint8_t* head120, const uint8_t* dir44, uint64_t brick_begin,
                               uint64_t brick_end, uint64_t palette_base, uint64_t palette_len, uint64_t coarse_base,
                               uint64_t coarse_len, uint64_t detail_base, uint64_t detail_len, uintptr_t stream,
                               csv_volume** vol) {
    return vol_create(device, head120, dir44, false, brick_begin, brick_end, nullptr, palette_base, palette_len,
                      nullptr, coarse_base, coarse_len, nullptr, detail_base, detail_len, false, stream, vol, true);
}

int csv_volume_upload(csv_volume* vol, int blob, const void* host, uint64_t offset, uint64_t nbytes, uintptr_t stream) {
    if (!vol || blob < 0 || blob > 2 || (nbytes && !host)) return fail(CSV_E_ARG, "bad upload arguments");
    if (!vol->d_blob) return fail(CSV_E_ARG, "volume does not own its blobs");
    if (offset + nbytes > vol->blob_cap[blob]) return fail(CSV_E_ARG, "upload beyond the blob slice");
    if (nbytes == 0) return CSV_OK;
    CUDA_TRY(cudaSetDevice(vol->device));
    uint8_t* base = blob == 0 ? (uint8_t*)vol->V.palette : (blob == 1 ? (uint8_t*)vol->V.coarse : (uint8_t*)vol->V.detail);
    CUDA_TRY(cudaMemcpyAsync(base + offset, host, nbytes, cudaMemcpyHostToDevice, reinterpret_cast<cudaStream_t>(stream)));
    return CSV_OK;
}

int csv_volume_stage_detail(csv_volume* vol, const uint32_t* d_bricks, const uint64_t* d_offs, const uint32_t* d_lens,
                            uint64_t n, const uint8_t* d_stage, uint64_t stage_len, uintptr_t stream) {
    if (!vol || (n && (!d_bricks || !d_offs || !d_lens || !d_stage))) return fail(CSV_E_ARG, "null argument");
    CUDA_TRY(cudaSetDevice(vol->device));
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    uint32_t* dbytes = const_cast<uint32_t*>(vol->V.d_bytes);
    uint64_t* doff = const_cast<uint64_t*>(vol->V.d_off);
    if (vol->V.nb) {
        CUDA_TRY(cudaMemsetAsync(dbytes, 0, vol->V.nb * 4, st));
        CUDA_TRY(cudaMemsetAsync(doff, 0, vol->V.nb * 8, st));
    }
    vol->V.detail = d_stage;
    vol->blob_cap[2] = stage_len;
    if (n) {
        k_stage_detail<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(doff, dbytes, vol->V.brick_begin, vol->V.nb, d_bricks,
                                                                   d_offs, d_lens, n);
        CUDA_TRY(cudaGetLastError());
    }
    if (!vol->V.entropy && vol->V.nb) {   // raw streams: entry regions depend on the stream bytes
        unsigned long long* stats = nullptr;
        CUDA_TRY(dalloc(&stats, 24, st));
        cudaMemsetAsync(stats, 0, 24, st);
        k_region_stats<<<(unsigned)((vol->V.nb + 255) / 256), 256, 0, st>>>(vol->V, stats, stats + 1);
        unsigned long long hs[3] = {0, 0, 0};
        cudaMemcpyAsync(hs, stats, 24, cudaMemcpyDeviceToHost, st);
        cudaFreeAsync(stats, st);
        cudaError_t ce = cudaStreamSynchronize(st);
        if (ce != cudaSuccess) return fail(CSV_E_CUDA, "stage: %s", cudaGetErrorString(ce));
        vol->region_total_t0 = std::max<uint64_t>(vol->region_total_t0, hs[0]);
        vol->region_max_t0 = std::max<uint64_t>(vol->region_max_t0, hs[1]);
    }
    return CSV_OK;
}

// DetailStore.plan's budget scan (render.py:808-823), host-side: candidates in
// request order are fetched while the running total stays within the budget;
// a candidate that does not fit is deferred and the scan continues.
int csv_detail_plan_greedy(const uint64_t* sizes, uint64_t n, uint64_t budget, uint8_t* accept, uint64_t* spent) {
    if ((n && (!sizes || !accept)) || !spent) return fail(CSV_E_ARG, "null argument");
    uint64_t sp = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const bool ok = sp + sizes[i] <= budget;
        accept[i] = ok ? 1 : 0;
        if (ok) sp += sizes[i];
    }
    *spent = sp;
    return CSV_OK;
}

int csv_volume_free(csv_volume* vol) {
    vol_release(vol);
    return CSV_OK;
}

int csv_volume_info(csv_volume* vol, int64_t* dims3, int64_t* grid3, int* brick_log2, int* entropy) {
    if (!vol) return fail(CSV_E_ARG, "null volume");
    if (dims3) memcpy(dims3, vol->dims, 24);
    if (grid3) memcpy(grid3, vol->grid, 24);
    if (brick_log2) *brick_log2 = vol->V.N;
    if (entropy) *entropy = vol->V.entropy;
    return CSV_OK;
}

int csv_decode_volume_range(csv_volume* vol, int t, uint64_t brick_first, uint64_t brick_last, uint32_t* d_out,
                            int64_t z_begin, int64_t z_end, csv_result* d_res, uintptr_t stream) {
    if (!vol || !d_out) return fail(CSV_E_ARG, "null argument");
    if (t < 0 || t > vol->V.N) return fail(CSV_E_ARG, "LOD %d outside [0, %d]", t, vol->V.N);
    if (brick_first < vol->V.brick_begin || brick_last > vol->V.brick_begin + vol->V.nb || brick_last < brick_first)
        return fail(CSV_E_ARG, "brick range outside the volume");
    if (z_begin < 0 || z_end < z_begin || z_begin % (1ll << (vol->V.N - t)) != 0)
        return fail(CSV_E_ARG, "z range [%lld, %lld) must start on a brick boundary (multiple of %lld)",
                    (long long)z_begin, (long long)z_end, 1ll << (vol->V.N - t));
    CUDA_TRY(cudaSetDevice(vol->device));
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    Plan P{};
    P.n = brick_last - brick_first;
    P.first = brick_first - vol->V.brick_begin;
    P.t_uniform = t;
    P.out = d_out;
    P.z_begin = z_begin;
    P.z_end = z_end;
    P.cx = (vol->dims[0] + (1ll << t) - 1) >> t;
    P.cy = (vol->dims[1] + (1ll << t) - 1) >> t;
    P.res = d_res;
    if (P.n == 0) return CSV_OK;
    if (t == vol->V.N) {
        CUDA_TRY(csv::run_root_raster(vol->V, P, st));
        return CSV_OK;
    }
    int rc = ensure_plan(vol, P.n, vol->region_total_t0, vol->V.N - t, st);
    if (rc) return rc;
    P.eoff = vol->d_eoff;
    P.sres = vol->d_sres;
    P.entries = vol->d_entries;
    P.wscratch = vol->d_wscratch;
    P.wscratch_stride = kWScratchStride;
    P.wscratch6 = vol->d_wscratch6;
    CUDA_TRY(run_decode(vol->V, P, 0, vol->d_sizes, vol->d_scan, vol->d_counter, vol->d_gws, vol->gws_stride,
                        vol->gws_ctas, vol->nsm, t, st, vol->timing ? vol->ev : nullptr, &vol->ovl));
    return CSV_OK;
}

int csv_decode_volume(csv_volume* vol, int t, uint32_t* d_out, int64_t z_begin, int64_t z_end, csv_result* d_res,
                      uintptr_t stream) {
    if (!vol) return fail(CSV_E_ARG, "null volume");
    return csv_decode_volume_range(vol, t, vol->V.brick_begin, vol->V.brick_begin + vol->V.nb, d_out, z_begin, z_end,
                                   d_res, stream);
}

int csv_decode_bricks(csv_volume* vol, uint64_t n, const uint32_t* d_brick, const uint8_t* d_lod,
                      const uint64_t* d_dst, uint32_t* d_pool, csv_result* d_res, uintptr_t stream) {
    if (!vol || (n && (!d_brick || !d_lod || !d_dst || !d_pool))) return fail(CSV_E_ARG, "null argument");
    if (n == 0) return CSV_OK;
    CUDA_TRY(cudaSetDevice(vol->device));
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    Plan P{};
    P.n = n;
    P.brick = d_brick;
    P.lod = d_lod;
    P.dst = d_dst;
    P.out = d_pool;
    P.res = d_res;
    uint64_t need = n * vol->region_max_t0;
    int rc = ensure_plan(vol, n, need, vol->V.N, st);
    if (rc) return rc;
    P.eoff = vol->d_eoff;
    P.sres = vol->d_sres;
    P.entries = vol->d_entries;
    P.wscratch = vol->d_wscratch;
    P.wscratch_stride = kWScratchStride;
    P.wscratch6 = vol->d_wscratch6;
    CUDA_TRY(run_decode(vol->V, P, 1, vol->d_sizes, vol->d_scan, vol->d_counter, vol->d_gws, vol->gws_stride,
                        vol->gws_ctas, vol->nsm, 0, st, vol->timing ? vol->ev : nullptr, &vol->ovl));
    return CSV_OK;
}

// Per-brick host API: requests and labels in host memory, one call per batch
// (CsvContainer.decode_brick's device-resident path).  Requests go through a
// pinned staging buffer in one copy; outputs land contiguously in request order.
static bool brick_graph_enabled() {   // CSVGPU_BRICK_GRAPH=0: per-brick calls launch directly
    static int v = -1;
    if (v < 0) { const char* e = getenv("CSVGPU_BRICK_GRAPH"); v = (e && strcmp(e, "0") == 0) ? 0 : 1; }
    return v == 1;
}

int csv_decode_bricks_host(csv_volume* vol, uint64_t n, const uint32_t* h_brick, const uint8_t* h_lod,
                           uint32_t* h_out, csv_result* h_res, uintptr_t stream) {
    if (!vol || (n && (!h_brick || !h_lod || !h_out || !h_res))) return fail(CSV_E_ARG, "null argument");
    if (n == 0) return CSV_OK;
    std::lock_guard<std::mutex> lk(vol->host_mu);   // ctypes drops the GIL: calls from two threads share the staging
    CUDA_TRY(cudaSetDevice(vol->device));
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const uint64_t lod_off = (4 * n + 15) & ~15ull, dst_off = (lod_off + n + 15) & ~15ull, req_bytes = dst_off + 8 * n;
    if (n > vol->hreq_cap) {
        CUDA_TRY(cudaStreamSynchronize(st));
        if (vol->h_req) cudaFreeHost(vol->h_req);
        vol->h_req = nullptr;
        dfree(vol->d_req); dfree(vol->d_hres);
        vol->hreq_cap = 0;
        const uint64_t cap = std::max<uint64_t>(n, 64);
        const uint64_t bytes = ((4 * cap + 15) & ~15ull) + ((cap + 15) & ~15ull) + 8 * cap + 32;
        CUDA_TRY(cudaMallocHost(&vol->h_req, bytes));
        CUDA_TRY(dalloc(&vol->d_req, bytes, st));
        CUDA_TRY(dalloc(&vol->d_hres, cap * sizeof(csv_result), st));
        vol->hreq_cap = cap;
    }
    uint8_t* h = vol->h_req;
    uint64_t* dst = reinterpret_cast<uint64_t*>(h + dst_off);
    uint64_t total = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const int t = h_lod[i];
        if (t > vol->V.N) return fail(CSV_E_ARG, "LOD %d outside [0, %d]", t, vol->V.N);
        dst[i] = total;
        total += 1ull << (3 * (vol->V.N - t));
    }
    if (total > vol->hpool_cap) {
        CUDA_TRY(cudaStreamSynchronize(st));
        dfree(vol->d_hpool);
        vol->hpool_cap = 0;
        CUDA_TRY(dalloc(&vol->d_hpool, total * sizeof(uint32_t), st));
        vol->hpool_cap = total;
    }
    memcpy(h, h_brick, 4 * n);
    memcpy(h + lod_off, h_lod, n);
    if (n <= kBrickGraphMax && !vol->timing && brick_graph_enabled()) {
        // graph replay: same launches and copies as below, labels and results through pinned staging
        const uint64_t out_bytes = total * sizeof(uint32_t), res_off = (out_bytes + 15) & ~15ull;
        const uint64_t stage = res_off + n * sizeof(csv_result);
        if (stage > vol->h_bout_cap) {
            CUDA_TRY(cudaStreamSynchronize(st));
            if (vol->h_bout) cudaFreeHost(vol->h_bout);
            vol->h_bout = nullptr;
            vol->h_bout_cap = 0;
            CUDA_TRY(cudaHostAlloc(&vol->h_bout, std::max<uint64_t>(stage, 4096), cudaHostAllocMapped));
            vol->h_bout_cap = std::max<uint64_t>(stage, 4096);
        }
        void* d_bout = nullptr;   // the device's address of the mapped staging (== h_bout under UVA)
        CUDA_TRY(cudaHostGetDevicePointer(&d_bout, vol->h_bout, 0));
        uint32_t* const g_pool = reinterpret_cast<uint32_t*>(d_bout);
        csv_result* const g_res = reinterpret_cast<csv_result*>(reinterpret_cast<uint8_t*>(d_bout) + res_off);
        // u16 replay pass only if a request's palette exceeds the u8 pass's 253 labels (unknown: keep it)
        uint64_t wide = 1;
        if (!vol->h_paln.empty()) {
            wide = 0;
            for (uint64_t i = 0; i < n; ++i) {
                const uint64_t b = (uint64_t)h_brick[i] - vol->V.brick_begin;
                if (b >= vol->h_paln.size() || vol->h_paln[b] > 253u) wide = 1;
            }
        }
        struct PalScope {   // the plan's palette bound for the launches issued below, restored after
            csv_volume* v; uint32_t keep;
            PalScope(csv_volume* v_, bool narrow) : v(v_), keep(v_->V.max_pal) { if (narrow && v->V.max_pal > 253u) v->V.max_pal = 253u; }
            ~PalScope() { v->V.max_pal = keep; }
        } pal_scope(vol, wide == 0);
        const void* ptrs[8] = {vol->h_req, vol->d_req, vol->d_hpool, vol->d_hres, vol->h_bout, vol->d_eoff,
                               vol->d_entries, vol->d_sizes};
        csv_volume::BrickGraph* g = nullptr;
        for (auto& c : vol->bgraph)
            if (c.seen && c.n == n && c.total == total && c.wide == wide && memcmp(c.ptrs, ptrs, sizeof(ptrs)) == 0) g = &c;
        if (g && g->exec) {
            CUDA_TRY(cudaGraphLaunch(g->exec, st));
            CUDA_TRY(cudaStreamSynchronize(st));
            memcpy(h_out, vol->h_bout, out_bytes);
            memcpy(h_res, vol->h_bout + res_off, n * sizeof(csv_result));
            return CSV_OK;
        }
        if (g) {   // second call with this key: capture
            if (!vol->cap_stream) CUDA_TRY(cudaStreamCreateWithFlags(&vol->cap_stream, cudaStreamNonBlocking));
            cudaStream_t cs = vol->cap_stream;
            cudaGraph_t graph = nullptr;
            CUDA_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
            cudaMemcpyAsync(vol->d_req, h, req_bytes, cudaMemcpyHostToDevice, cs);
            const int rc = csv_decode_bricks(vol, n, reinterpret_cast<const uint32_t*>(vol->d_req), vol->d_req + lod_off,
                                             reinterpret_cast<const uint64_t*>(vol->d_req + dst_off), g_pool, g_res,
                                             reinterpret_cast<uintptr_t>(cs));
            const cudaError_t ce = cudaStreamEndCapture(cs, &graph);
            if (rc) { if (graph) cudaGraphDestroy(graph); return rc; }
            CUDA_TRY(ce);
            const void* now[8] = {vol->h_req, vol->d_req, vol->d_hpool, vol->d_hres, vol->h_bout, vol->d_eoff,
                                  vol->d_entries, vol->d_sizes};
            if (memcmp(now, ptrs, sizeof(ptrs)) != 0) {   // the decode grew a workspace during capture: not replayable
                cudaGraphDestroy(graph);
                g->seen = 0;
                return fail(CSV_E_CUDA, "per-brick graph capture reallocated a workspace");
            }
            const cudaError_t ie = cudaGraphInstantiate(&g->exec, graph, 0);
            cudaGraphDestroy(graph);
            CUDA_TRY(ie);
            CUDA_TRY(cudaGraphLaunch(g->exec, st));
            CUDA_TRY(cudaStreamSynchronize(st));
            memcpy(h_out, vol->h_bout, out_bytes);
            memcpy(h_res, vol->h_bout + res_off, n * sizeof(csv_result));
            return CSV_OK;
        }
        // first call with this key: run directly (sizes the workspace), remember the key
        CUDA_TRY(cudaMemcpyAsync(vol->d_req, h, req_bytes, cudaMemcpyHostToDevice, st));
        const int rc = csv_decode_bricks(vol, n, reinterpret_cast<const uint32_t*>(vol->d_req), vol->d_req + lod_off,
                                         reinterpret_cast<const uint64_t*>(vol->d_req + dst_off), g_pool, g_res, stream);
        if (rc) return rc;
        CUDA_TRY(cudaStreamSynchronize(st));
        memcpy(h_out, vol->h_bout, out_bytes);
        memcpy(h_res, vol->h_bout + res_off, n * sizeof(csv_result));
        const void* now[8] = {vol->h_req, vol->d_req, vol->d_hpool, vol->d_hres, vol->h_bout, vol->d_eoff,
                              vol->d_entries, vol->d_sizes};
        csv_volume::BrickGraph& c = vol->bgraph[vol->bg_next++ % 8];
        if (c.exec) cudaGraphExecDestroy(c.exec);
        c.exec = nullptr;
        c.n = n;
        c.total = total;
        c.wide = wide;
        c.seen = 1;
        memcpy(c.ptrs, now, sizeof(now));
        return CSV_OK;
    }
    CUDA_TRY(cudaMemcpyAsync(vol->d_req, h, req_bytes, cudaMemcpyHostToDevice, st));
    const int rc = csv_decode_bricks(vol, n, reinterpret_cast<const uint32_t*>(vol->d_req), vol->d_req + lod_off,
                                     reinterpret_cast<const uint64_t*>(vol->d_req + dst_off), vol->d_hpool, vol->d_hres,
                                     stream);
    if (rc) return rc;
    CUDA_TRY(cudaMemcpyAsync(h_res, vol->d_hres, n * sizeof(csv_result), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(h_out, vol->d_hpool, total * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return CSV_OK;
}

// Streams passed per call (decode_brick_entropy / decode_brick): one cached one-brick
// volume per device, re-created only when the head's tables / brick size / entropy flag
// change or a stream outgrows its capacity; per call the streams go through pinned
// staging into the volume's blobs, one tiny kernel sets brick 0's directory row, and
// csv_decode_bricks_host decodes it (graph replay from the third call of a shape).
namespace {
struct BrickScratch {
    uint8_t key[68]{};              // flags, brick_log2, the two count tables
    csv_volume* vol = nullptr;
    uint64_t cap_pal = 0, cap_c = 0, cap_d = 0;
    uint8_t* h_stage = nullptr;     // pinned: palette | coarse | detail
    uint64_t h_cap = 0;
};
BrickScratch g_scratch[64];
std::mutex g_scratch_mu;
}  // namespace

int csv_decode_brick_streams(int device, const uint8_t* head120, const uint32_t* palette, uint64_t n_pal,
                             const uint8_t* coarse, uint64_t coarse_bytes, uint32_t coarse_nibbles,
                             const uint8_t* detail, uint64_t detail_bytes, uint32_t detail_nibbles, int t,
                             uint32_t* h_out, csv_result* h_res, uintptr_t stream) {
    if (!head120 || !h_out || !h_res || (n_pal && !palette) || (coarse_bytes && !coarse) || (detail_bytes && !detail))
        return fail(CSV_E_ARG, "null argument");
    if (device < 0 || device >= 64) return fail(CSV_E_ARG, "device %d out of range", device);
    if (n_pal == 0) return fail(CSV_E_ARG, "empty palette");
    if (n_pal > 0xffffffffull || coarse_bytes > 0xffffffffull || detail_bytes > 0xffffffffull)
        return fail(CSV_E_ARG, "stream too long");
    std::lock_guard<std::mutex> lk(g_scratch_mu);
    CUDA_TRY(cudaSetDevice(device));
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    BrickScratch& S = g_scratch[device];
    uint8_t key[68];
    key[0] = head120[6]; key[1] = head120[10]; key[2] = head120[11]; key[3] = 0;
    memcpy(key + 4, head120 + 32, 64);
    auto grow = [](uint64_t need, uint64_t have) { uint64_t c = have ? have : 1024; while (c < need) c *= 2; return c; };
    if (!S.vol || memcmp(key, S.key, sizeof key) != 0 || n_pal > S.cap_pal || coarse_bytes > S.cap_c ||
        detail_bytes > S.cap_d) {
        const bool same = S.vol && memcmp(key, S.key, sizeof key) == 0;
        const uint64_t cp = grow(n_pal, same ? S.cap_pal : 0), cc = grow(coarse_bytes, same ? S.cap_c : 0),
                       cd = grow(detail_bytes, same ? S.cap_d : 0);
        if (S.vol) { vol_release(S.vol); S.vol = nullptr; }
        uint8_t row[44] = {};
        const uint32_t ucp = (uint32_t)cp, ucc = (uint32_t)cc, ucd = (uint32_t)cd;
        memcpy(row + 8, &ucp, 4);
        memcpy(row + 20, &ucc, 4);
        memcpy(row + 36, &ucd, 4);
        csv_volume* v = nullptr;
        const int rc = vol_create(device, head120, row, false, 0, 1, nullptr, 0, cp, nullptr, 0, cc, nullptr, 0, cd, false,
                                  stream, &v, true);
        if (rc) return rc;
        if (v->V.nb != 1) { vol_release(v); return fail(CSV_E_ARG, "head must describe a one-brick volume"); }
        // entry regions: bounded by the format (<= 2 nibbles per entry of each stream)
        v->region_max_t0 = round32(2ull * max_entries(v->V.N, 0, 0)) + round32(2ull * max_entries(v->V.N, 0, 1));
        v->region_total_t0 = v->region_max_t0;
        S.vol = v;
        memcpy(S.key, key, sizeof key);
        S.cap_pal = cp; S.cap_c = cc; S.cap_d = cd;
    }
    csv_volume* v = S.vol;
    if (t < 0 || t > v->V.N) return fail(CSV_E_ARG, "LOD %d outside [0, %d]", t, v->V.N);
    const uint64_t pb = 4 * n_pal, need = pb + coarse_bytes + detail_bytes;
    if (need > S.h_cap) {
        CUDA_TRY(cudaStreamSynchronize(st));
        if (S.h_stage) cudaFreeHost(S.h_stage);
        S.h_stage = nullptr;
        S.h_cap = 0;
        const uint64_t cap = grow(need, 0);
        CUDA_TRY(cudaMallocHost(&S.h_stage, cap));
        S.h_cap = cap;
    }
    memcpy(S.h_stage, palette, pb);
    if (coarse_bytes) memcpy(S.h_stage + pb, coarse, coarse_bytes);
    if (detail_bytes) memcpy(S.h_stage + pb + coarse_bytes, detail, detail_bytes);
    CUDA_TRY(cudaMemcpyAsync(const_cast<uint32_t*>(v->V.palette), S.h_stage, pb, cudaMemcpyHostToDevice, st));
    if (coarse_bytes)
        CUDA_TRY(cudaMemcpyAsync(const_cast<uint8_t*>(v->V.coarse), S.h_stage + pb, coarse_bytes, cudaMemcpyHostToDevice, st));
    if (detail_bytes)
        CUDA_TRY(cudaMemcpyAsync(const_cast<uint8_t*>(v->V.detail), S.h_stage + pb + coarse_bytes, detail_bytes,
                                 cudaMemcpyHostToDevice, st));
    k_set_brick0<<<1, 1, 0, st>>>(const_cast<uint64_t*>(v->V.pal_off), const_cast<uint32_t*>(v->V.pal_len),
                                  const_cast<uint64_t*>(v->V.c_off), const_cast<uint32_t*>(v->V.c_bytes),
                                  const_cast<uint32_t*>(v->V.c_nib), const_cast<uint64_t*>(v->V.d_off),
                                  const_cast<uint32_t*>(v->V.d_bytes), const_cast<uint32_t*>(v->V.d_nib), (uint32_t)n_pal,
                                  (uint32_t)coarse_bytes, coarse_nibbles, (uint32_t)detail_bytes, detail_nibbles);
    CUDA_TRY(cudaGetLastError());
    v->V.max_pal = (uint32_t)n_pal;
    if (!v->h_paln.empty()) v->h_paln[0] = (uint32_t)n_pal;
    const uint32_t b0 = 0;
    const uint8_t t8 = (uint8_t)t;
    if (t == v->V.N) {   // coarsest LOD: palette[0], no decode (codec.py:514-516)
        h_out[0] = palette[0];
        memset(h_res, 0, sizeof(csv_result));
        return CSV_OK;
    }
    return csv_decode_bricks_host(v, 1, &b0, &t8, h_out, h_res, stream);
}

int csv_streams_capacity(csv_volume* vol, uint64_t n, int t, uint64_t* cap) {
    if (!vol || !cap) return fail(CSV_E_ARG, "null argument");
    (void)t;
    *cap = n * vol->region_max_t0 + 64;
    return CSV_OK;
}

int csv_decode_streams(csv_volume* vol, uint64_t n, const uint32_t* d_brick, int t, uint8_t* d_entries,
                       uint64_t entries_cap, uint64_t* d_entry_off, csv_stream_result* d_sres, uintptr_t stream) {
    if (!vol || (n && (!d_entries || !d_entry_off || !d_sres))) return fail(CSV_E_ARG, "null argument");
    if (t < 0 || t > vol->V.N) return fail(CSV_E_ARG, "LOD %d outside [0, %d]", t, vol->V.N);
    if (n == 0) return CSV_OK;
    if (entries_cap < n * vol->region_max_t0) return fail(CSV_E_ARG, "entries_cap too small (need %llu)",
                                                          (unsigned long long)(n * vol->region_max_t0));
    CUDA_TRY(cudaSetDevice(vol->device));
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    int rc = ensure_plan(vol, n, 0, 0, st);
    if (rc) return rc;
    Plan P{};
    P.n = n;
    P.brick = d_brick;
    P.t_uniform = t;
    P.eoff = d_entry_off;
    P.sres = d_sres;
    P.entries = d_entries;
    CUDA_TRY(run_streams_only(vol->V, P, vol->d_sizes, vol->d_scan, vol->d_counter, vol->nsm, st));
    return CSV_OK;
}

int csv_volume_set_timing(csv_volume* vol, int enable) {
    if (!vol) return fail(CSV_E_ARG, "null volume");
    CUDA_TRY(cudaSetDevice(vol->device));
    if (enable && !vol->ev[0])
        for (auto& e : vol->ev) CUDA_TRY(cudaEventCreate(&e));
    vol->timing = enable != 0;
    return CSV_OK;
}

int csv_volume_get_timing(csv_volume* vol, float* ms3) {
    if (!vol || !ms3) return fail(CSV_E_ARG, "null argument");
    if (!vol->timing) return fail(CSV_E_ARG, "timing not enabled");
    CUDA_TRY(cudaEventSynchronize(vol->ev[3]));
    CUDA_TRY(cudaEventElapsedTime(&ms3[0], vol->ev[0], vol->ev[1]));
    CUDA_TRY(cudaEventElapsedTime(&ms3[1], vol->ev[1], vol->ev[2]));
    CUDA_TRY(cudaEventElapsedTime(&ms3[2], vol->ev[2], vol->ev[3]));
    return CSV_OK;
}

int csv_volume_op_counts(csv_volume* vol, uint64_t* d_counts8, csv_stream_result* d_sres, uintptr_t stream) {
    if (!vol || !d_counts8 || !d_sres) return fail(CSV_E_ARG, "null argument");
    CUDA_TRY(cudaSetDevice(vol->device));
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    int rc = ensure_plan(vol, vol->V.nb, 0, 0, st);
    if (rc) return rc;
    Plan P{};
    P.n = vol->V.nb;
    P.t_uniform = 0;
    P.sres = d_sres;
    P.op_counts = reinterpret_cast<unsigned long long*>(d_counts8);
    CUDA_TRY(cudaMemsetAsync(d_counts8, 0, 8 * sizeof(uint64_t), st));
    CUDA_TRY(run_op_counts(vol->V, P, vol->d_counter, vol->nsm, st));
    return CSV_OK;
}

}  // extern "C"
