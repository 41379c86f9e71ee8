// csv_cache.cu -- device-side frame bookkeeping around the batched brick decode
// (SURVEY.md §8f.2): per-brick LOD selection, palette visibility, and the
// brick-cache residency manager with per-size-class free stacks.
//
// Reference (host, serial): desired_lods (render.py:145-158), visibility_mask
// (render.py:174-187), BrickCache.end_frame_assign / _allocate / _free_block /
// _rebuild (cache.py:108-195).  On the GPU the frame's assignment is four
// bulk kernels instead of one Python loop over requests:
//   want   : requests -> per-brick wanted LOD (a brick requested twice ends at
//            the larger LOD, as the sorted reference loop leaves it)
//   free   : evict bricks not marked used this frame, free re-LOD'd blocks
//            (pushes onto the size class's stack, atomics)
//   alloc  : pop a block of the class or carve from the shared top (atomics,
//            the SAS-style allocator of the paper); exhaustion -> rebuild
//   decode : the fill list goes straight into csv_decode_bricks (K1 + K2w)
// A rebuild is deterministic: every wanted brick (requests, plus bricks marked
// used, the coarsest LOD excluded) gets a block carved in brick order, exactly
// the reference's _rebuild.  Outside rebuilds the resident set and every
// resident brick's labels match the reference; block positions are the
// allocator's own (they are not observable through lookup/brick_view semantics).
#include <cstdio>
#include <cstring>
#include <cstdarg>
#include <cmath>
#include <string>
#include "csv_device.cuh"

namespace csv {
cudaError_t run_scan(const uint64_t* sizes, uint64_t* out, uint64_t n, uint64_t* tmp, cudaStream_t st);
const VolView& volume_view(const csv_volume* v);
int volume_device(const csv_volume* v);
}  // namespace csv

using namespace csv;

namespace {

int cfail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    set_error(buf);
    return code;
}
#define CTRY(x)                                                                              \
    do {                                                                                     \
        cudaError_t e_ = (x);                                                                \
        if (e_ != cudaSuccess) return cfail(CSV_E_CUDA, "%s: %s", #x, cudaGetErrorString(e_)); \
    } while (0)

enum { C_TOP = 0, C_NFILL, C_FAILED, C_BAD, C_EVICT, C_FBYTES, C_COUNT };   // C_FBYTES: this frame's fills

// ------------------------------------------------------------------ LOD selection
// desired_lods (render.py:145-158): distance of the brick centre to the camera,
// ratio = max(1, d * 2 tan(fov/2) / H), lod = clip(ceil(log2(ratio)), 0, N).
// Same float64 operation order as the numpy restatement; tan(fov/2) comes from the host.
__global__ void k_desired_lods(VolView V, double px, double py, double pz, double tanh2, double height,
                               uint8_t* lod) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= V.nb) return;
    const uint64_t g = V.brick_begin + i;
    const double b = (double)(1ll << V.N);
    const double cx = ((double)(g % V.gx) + 0.5) * b;
    const double cy = ((double)((g / V.gx) % V.gy) + 0.5) * b;
    const double cz = ((double)(g / (V.gx * V.gy)) + 0.5) * b;
    const double dx = cx - px, dy = cy - py, dz = cz - pz;
    const double d = sqrt(dx * dx + dy * dy + dz * dz);
    double ratio = d * 2.0 * tanh2 / height;
    ratio = ratio > 1.0 ? ratio : 1.0;
    double l = ceil(log2(ratio));
    l = l < 0.0 ? 0.0 : (l > (double)V.N ? (double)V.N : l);
    lod[i] = (uint8_t)l;
}

// ------------------------------------------------------------------ visibility
// visibility_mask (render.py:174-187): alpha of each palette entry from the
// sorted transfer-function labels (default alpha otherwise), then numpy's
// add.reduceat over the directory's palette offsets: brick i sums entries
// [off_i, off_{i+1}) -- or takes entry off_i alone when off_i >= off_{i+1}.
__global__ void k_visibility(VolView V, uint64_t pal_total, const uint32_t* tf_labels, const double* tf_alpha,
                             uint32_t n_tf, double default_alpha, uint8_t* vis) {
    const uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= V.nb) return;
    const uint64_t lo = V.pal_off[i];
    const uint64_t hi = i + 1 < V.nb ? V.pal_off[i + 1] : pal_total;
    const uint64_t a = lo, e = lo < hi ? hi : lo + 1;
    bool any = false;
    for (uint64_t k = a + lane; k < e && k < pal_total; k += 32) {
        const uint32_t lab = V.palette[k];
        double alpha = default_alpha;
        if (n_tf) {   // searchsorted(labels, lab) (left), clamped, hit test
            uint32_t l = 0, r = n_tf;
            while (l < r) {
                const uint32_t m = (l + r) >> 1;
                if (tf_labels[m] < lab) l = m + 1; else r = m;
            }
            const uint32_t c = l < n_tf ? l : n_tf - 1;
            if (tf_labels[c] == lab) alpha = tf_alpha[c];
        }
        any |= alpha > 0.0;
    }
    any = __any_sync(0xffffffffu, any);
    if (lane == 0) vis[i] = any ? 1 : 0;
}

// ------------------------------------------------------------------ residency
struct CacheView {
    uint64_t nb;
    int N;
    uint64_t capacity;          // base elements (8 voxels each)
    int64_t* block_start;
    int8_t* resident;
    int8_t* usage;
    int32_t* want;
    uint64_t* stacks;           // N stacks of nb entries
    long long* counts;          // N stack heights
    unsigned long long* ctr;    // C_*
    uint32_t* fill_brick;
    uint8_t* fill_lod;
    uint64_t* fill_dst;         // voxel offsets
};

__device__ __forceinline__ uint64_t class_elems(int c) { return 1ull << (3 * c); }

__global__ void k_mark_used(CacheView C, const uint32_t* bricks, const uint8_t* lods, uint64_t n) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t b = bricks[i];
    if (b < C.nb) C.usage[b] = (int8_t)lods[i];   // idempotent (cache.py:82-89)
}

// requests -> wanted LOD per brick; out-of-range LODs/bricks flag the call (cache.py:157-159)
__global__ void k_want(CacheView C, const uint32_t* bricks, const uint8_t* lods, uint64_t n) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t b = bricks[i];
    const int l = lods[i];
    if (b >= C.nb || l >= C.N) { atomicOr(C.ctr + C_BAD, 1ull); return; }
    atomicMax(C.want + b, l);
}

// evict unused bricks and free blocks of bricks re-requested at another LOD (cache.py:108-112, :160-166)
__global__ void k_free(CacheView C) {
    const uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (b >= C.nb) return;
    const int res = C.resident[b];
    if (res < 0) return;
    const bool evict = C.usage[b] < 0;
    const int w = C.want[b];
    if (!evict && !(w >= 0 && w != res)) return;
    const int c = C.N - res - 1;
    const long long slot = atomicAdd(reinterpret_cast<unsigned long long*>(C.counts + c), 1ull);
    C.stacks[(uint64_t)c * C.nb + (uint64_t)slot] = (uint64_t)C.block_start[b];
    C.block_start[b] = -1;
    C.resident[b] = -1;
    if (evict) atomicAdd(C.ctr + C_EVICT, 1ull);
}

// pop a block of the size class or carve from the top (cache.py:114-123)
__global__ void k_alloc(CacheView C) {
    const uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (b >= C.nb) return;
    const int w = C.want[b];
    if (w < 0 || C.resident[b] == w) return;
    const int c = C.N - w - 1;
    const long long old = (long long)atomicAdd(reinterpret_cast<unsigned long long*>(C.counts + c),
                                               (unsigned long long)-1ll);
    uint64_t start;
    if (old > 0) {
        start = C.stacks[(uint64_t)c * C.nb + (uint64_t)(old - 1)];
    } else {
        const uint64_t size = class_elems(c);
        start = atomicAdd(C.ctr + C_TOP, size);
        if (start + size > C.capacity) { atomicOr(C.ctr + C_FAILED, 1ull); return; }
    }
    C.block_start[b] = (int64_t)start;
    C.resident[b] = (int8_t)w;
    const unsigned long long k = atomicAdd(C.ctr + C_NFILL, 1ull);
    C.fill_brick[k] = (uint32_t)b;
    C.fill_lod[k] = (uint8_t)w;
    C.fill_dst[k] = start * 8;
    atomicAdd(C.ctr + C_FBYTES, 32ull * class_elems(c));
}

__global__ void k_fix_counts(CacheView C) {
    const int c = threadIdx.x;
    if (c < C.N && C.counts[c] < 0) C.counts[c] = 0;
}

// rebuild (cache.py:172-195): wanted = requests + bricks marked used (not the coarsest LOD)
__global__ void k_rebuild_sizes(CacheView C, uint64_t* sizes) {
    const uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (b >= C.nb) return;
    int w = C.want[b];
    if (w < 0) {
        const int u = C.usage[b];
        w = (u >= 0 && u < C.N) ? u : -1;
    }
    C.want[b] = w;
    sizes[b] = w >= 0 ? class_elems(C.N - w - 1) : 0ull;
}
__global__ void k_rebuild_apply(CacheView C, const uint64_t* starts) {
    const uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (b >= C.nb) return;
    const int w = C.want[b];
    C.resident[b] = (int8_t)w;
    C.block_start[b] = w >= 0 ? (int64_t)starts[b] : -1;
    if (w < 0) return;
    const unsigned long long k = atomicAdd(C.ctr + C_NFILL, 1ull);
    C.fill_brick[k] = (uint32_t)b;
    C.fill_lod[k] = (uint8_t)w;
    C.fill_dst[k] = starts[b] * 8;
    atomicAdd(C.ctr + C_FBYTES, 32ull * class_elems(C.N - w - 1));
}

unsigned grid_of(uint64_t n, unsigned bs = 256) { return (unsigned)((n + bs - 1) / bs ? (n + bs - 1) / bs : 1); }

}  // namespace

struct csv_cache {
    int device = 0;
    CacheView C{};
    uint64_t* scan_sizes = nullptr;   // nb + 1
    uint64_t* scan_out = nullptr;     // nb + 1
    uint64_t* scan_tmp = nullptr;     // 4104
    unsigned long long* h_ctr = nullptr;   // pinned mirror of the counters
    uint64_t rebuilds = 0, decodes = 0, decoded_bytes = 0, last_placed = 0;
};

static void cache_release(csv_cache* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaFree(c->C.block_start); cudaFree(c->C.resident); cudaFree(c->C.usage); cudaFree(c->C.want);
    cudaFree(c->C.stacks); cudaFree(c->C.counts); cudaFree(c->C.ctr); cudaFree(c->C.fill_brick);
    cudaFree(c->C.fill_lod); cudaFree(c->C.fill_dst); cudaFree(c->scan_sizes); cudaFree(c->scan_out);
    cudaFree(c->scan_tmp);
    if (c->h_ctr) cudaFreeHost(c->h_ctr);
    delete c;
}

extern "C" {

int csv_desired_lods(csv_volume* vol, double px, double py, double pz, double tan_half_fov, double height,
                     uint8_t* d_lod, uintptr_t stream) {
    if (!vol || !d_lod) return cfail(CSV_E_ARG, "null argument");
    CTRY(cudaSetDevice(volume_device(vol)));
    const VolView& V = volume_view(vol);
    if (V.nb == 0) return CSV_OK;
    k_desired_lods<<<grid_of(V.nb), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(V, px, py, pz, tan_half_fov,
                                                                                    height, d_lod);
    CTRY(cudaGetLastError());
    return CSV_OK;
}

int csv_visibility_mask(csv_volume* vol, uint64_t palette_total, const uint32_t* d_tf_labels, const double* d_tf_alpha,
                        uint32_t n_tf, double default_alpha, uint8_t* d_vis, uintptr_t stream) {
    if (!vol || !d_vis || (n_tf && (!d_tf_labels || !d_tf_alpha))) return cfail(CSV_E_ARG, "null argument");
    CTRY(cudaSetDevice(volume_device(vol)));
    const VolView& V = volume_view(vol);
    if (V.nb == 0) return CSV_OK;
    k_visibility<<<grid_of(V.nb * 32), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        V, palette_total, d_tf_labels, d_tf_alpha, n_tf, default_alpha, d_vis);
    CTRY(cudaGetLastError());
    return CSV_OK;
}

int csv_cache_create(int device, uint64_t num_bricks, int brick_log2, uint64_t pool_elements, csv_cache** out) {
    if (!out) return cfail(CSV_E_ARG, "null argument");
    if (brick_log2 < 1 || brick_log2 > 7) return cfail(CSV_E_ARG, "bricks must span at least 2 voxels per axis");
    CTRY(cudaSetDevice(device));
    csv_cache* c = new csv_cache();
    c->device = device;
    CacheView& C = c->C;
    C.nb = num_bricks;
    C.N = brick_log2;
    C.capacity = pool_elements ? pool_elements : 1;
    const uint64_t n = num_bricks ? num_bricks : 1;
    cudaError_t e = cudaSuccess;
    auto A = [&](void** p, size_t bytes) { if (e == cudaSuccess) e = cudaMalloc(p, bytes); };
    A((void**)&C.block_start, n * 8);
    A((void**)&C.resident, n);
    A((void**)&C.usage, n);
    A((void**)&C.want, n * 4);
    A((void**)&C.stacks, (size_t)brick_log2 * n * 8);
    A((void**)&C.counts, 8 * 8);
    A((void**)&C.ctr, C_COUNT * 8);
    A((void**)&C.fill_brick, n * 4);
    A((void**)&C.fill_lod, n);
    A((void**)&C.fill_dst, n * 8);
    A((void**)&c->scan_sizes, (n + 1) * 8);
    A((void**)&c->scan_out, (n + 1) * 8);
    A((void**)&c->scan_tmp, 4104 * 8);
    if (e == cudaSuccess) e = cudaMallocHost((void**)&c->h_ctr, C_COUNT * 8);
    if (e != cudaSuccess) { cache_release(c); return cfail(CSV_E_NOMEM, "cache: %s", cudaGetErrorString(e)); }
    cudaMemset(C.block_start, 0xFF, n * 8);
    cudaMemset(C.resident, 0xFF, n);
    cudaMemset(C.usage, 0xFF, n);
    cudaMemset(C.counts, 0, 64);
    cudaMemset(C.ctr, 0, C_COUNT * 8);
    e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { cache_release(c); return cfail(CSV_E_CUDA, "cache: %s", cudaGetErrorString(e)); }
    *out = c;
    return CSV_OK;
}

int csv_cache_free(csv_cache* c) {
    cache_release(c);
    return CSV_OK;
}

int csv_cache_begin_frame(csv_cache* c, uintptr_t stream) {
    if (!c) return cfail(CSV_E_ARG, "null cache");
    CTRY(cudaSetDevice(c->device));
    CTRY(cudaMemsetAsync(c->C.usage, 0xFF, c->C.nb, reinterpret_cast<cudaStream_t>(stream)));
    return CSV_OK;
}

int csv_cache_mark_used(csv_cache* c, const uint32_t* d_bricks, const uint8_t* d_lods, uint64_t n, uintptr_t stream) {
    if (!c || (n && (!d_bricks || !d_lods))) return cfail(CSV_E_ARG, "null argument");
    if (!n) return CSV_OK;
    CTRY(cudaSetDevice(c->device));
    k_mark_used<<<grid_of(n), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(c->C, d_bricks, d_lods, n);
    CTRY(cudaGetLastError());
    return CSV_OK;
}

int csv_cache_plan(csv_cache* c, const uint32_t* d_bricks, const uint8_t* d_lods, uint64_t n, uint64_t* placed,
                   int* rebuilt, uintptr_t stream);
int csv_cache_decode_fills(csv_cache* c, csv_volume* vol, uint32_t* d_pool, csv_result* d_res, uintptr_t stream);

// One frame's assignment + batched decode into d_pool.  *placed receives the
// number of bricks decoded; *rebuilt is 1 when the pool was rebuilt.
int csv_decode_bricks(csv_volume* vol, uint64_t n, const uint32_t* d_brick, const uint8_t* d_lod,
                      const uint64_t* d_dst, uint32_t* d_pool, csv_result* d_res, uintptr_t stream);

int csv_cache_assign(csv_cache* c, csv_volume* vol, const uint32_t* d_bricks, const uint8_t* d_lods, uint64_t n,
                     uint32_t* d_pool, csv_result* d_res, uint64_t* placed, int* rebuilt, uintptr_t stream) {
    const int rc = csv_cache_plan(c, d_bricks, d_lods, n, placed, rebuilt, stream);
    if (rc) return rc;
    return csv_cache_decode_fills(c, vol, d_pool, d_res, stream);
}

int csv_cache_decode_fills(csv_cache* c, csv_volume* vol, uint32_t* d_pool, csv_result* d_res, uintptr_t stream) {
    if (!c || !vol || !d_pool) return cfail(CSV_E_ARG, "null argument");
    const uint64_t nfill = c->last_placed;
    if (nfill) {
        const int rc = csv_decode_bricks(vol, nfill, c->C.fill_brick, c->C.fill_lod, c->C.fill_dst, d_pool, d_res, stream);
        if (rc) return rc;
        c->decodes += nfill;
        c->decoded_bytes += c->h_ctr[C_FBYTES];
    }
    return CSV_OK;
}

int csv_cache_plan(csv_cache* c, const uint32_t* d_bricks, const uint8_t* d_lods, uint64_t n, uint64_t* placed,
                   int* rebuilt, uintptr_t stream) {
    if (!c || (n && (!d_bricks || !d_lods))) return cfail(CSV_E_ARG, "null argument");
    CTRY(cudaSetDevice(c->device));
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    CacheView& C = c->C;
    if (placed) *placed = 0;
    if (rebuilt) *rebuilt = 0;
    CTRY(cudaMemsetAsync(C.want, 0xFF, C.nb * 4, st));
    CTRY(cudaMemsetAsync(C.ctr + C_NFILL, 0, 3 * 8, st));   // nfill, failed, bad
    CTRY(cudaMemsetAsync(C.ctr + C_FBYTES, 0, 8, st));
    if (n) k_want<<<grid_of(n), 256, 0, st>>>(C, d_bricks, d_lods, n);
    CTRY(cudaMemcpyAsync(c->h_ctr, C.ctr, C_COUNT * 8, cudaMemcpyDeviceToHost, st));
    CTRY(cudaStreamSynchronize(st));
    if (c->h_ctr[C_BAD]) return cfail(CSV_E_ARG, "cannot cache LOD outside [0, %d] (or brick outside the volume)", C.N - 1);
    k_free<<<grid_of(C.nb), 256, 0, st>>>(C);
    k_alloc<<<grid_of(C.nb), 256, 0, st>>>(C);
    k_fix_counts<<<1, 32, 0, st>>>(C);
    CTRY(cudaMemcpyAsync(c->h_ctr, C.ctr, C_COUNT * 8, cudaMemcpyDeviceToHost, st));
    CTRY(cudaStreamSynchronize(st));
    if (c->h_ctr[C_FAILED]) {   // pool exhausted: rebuild in brick order (also defragments)
        k_rebuild_sizes<<<grid_of(C.nb), 256, 0, st>>>(C, c->scan_sizes);
        CTRY(run_scan(c->scan_sizes, c->scan_out, C.nb, c->scan_tmp, st));
        uint64_t total = 0;
        CTRY(cudaMemcpyAsync(&total, c->scan_out + C.nb, 8, cudaMemcpyDeviceToHost, st));
        CTRY(cudaStreamSynchronize(st));
        CTRY(cudaMemsetAsync(C.counts, 0, 64, st));
        CTRY(cudaMemsetAsync(C.ctr + C_NFILL, 0, 2 * 8, st));
        CTRY(cudaMemsetAsync(C.ctr + C_FBYTES, 0, 8, st));   // the discarded placements do not count
        if (total > C.capacity) {
            CTRY(cudaMemsetAsync(C.block_start, 0xFF, C.nb * 8, st));
            CTRY(cudaMemsetAsync(C.resident, 0xFF, C.nb, st));
            CTRY(cudaMemsetAsync(C.ctr + C_TOP, 0, 8, st));
            CTRY(cudaStreamSynchronize(st));
            return cfail(CSV_E_CAPACITY, "visible set needs %llu base elements, pool holds %llu",
                         (unsigned long long)total, (unsigned long long)C.capacity);
        }
        k_rebuild_apply<<<grid_of(C.nb), 256, 0, st>>>(C, c->scan_out);
        CTRY(cudaMemcpyAsync(C.ctr + C_TOP, c->scan_out + C.nb, 8, cudaMemcpyDeviceToDevice, st));
        c->rebuilds += 1;
        CTRY(cudaMemcpyAsync(c->h_ctr, C.ctr, C_COUNT * 8, cudaMemcpyDeviceToHost, st));
        CTRY(cudaStreamSynchronize(st));
        if (rebuilt) *rebuilt = 1;
    }
    const uint64_t nfill = c->h_ctr[C_NFILL];
    if (placed) *placed = nfill;
    c->last_placed = nfill;
    return CSV_OK;
}

// Device pointers of the residency state (block_start i64, resident_lod i8,
// usage i8, fill list) and the counters (top, evictions, rebuilds, decodes,
// decoded bytes) -- for the host mirror's lookup/occupancy and for tests.
int csv_cache_state(csv_cache* c, int64_t** d_block_start, int8_t** d_resident, int8_t** d_usage,
                    uint32_t** d_fill_brick, uint8_t** d_fill_lod, uint64_t** d_fill_dst) {
    if (!c) return cfail(CSV_E_ARG, "null cache");
    if (d_block_start) *d_block_start = c->C.block_start;
    if (d_resident) *d_resident = c->C.resident;
    if (d_usage) *d_usage = c->C.usage;
    if (d_fill_brick) *d_fill_brick = c->C.fill_brick;
    if (d_fill_lod) *d_fill_lod = c->C.fill_lod;
    if (d_fill_dst) *d_fill_dst = c->C.fill_dst;
    return CSV_OK;
}

// Host copy of the last plan's fill list (brick, lod), up to cap entries; returns the count in *n.
int csv_cache_read_fills(csv_cache* c, uint32_t* bricks, uint8_t* lods, uint64_t cap, uint64_t* n) {
    if (!c || !n || (cap && (!bricks || !lods))) return cfail(CSV_E_ARG, "null argument");
    CTRY(cudaSetDevice(c->device));
    CTRY(cudaDeviceSynchronize());
    const uint64_t k = c->last_placed < cap ? c->last_placed : cap;
    if (k) {
        CTRY(cudaMemcpy(bricks, c->C.fill_brick, k * 4, cudaMemcpyDeviceToHost));
        CTRY(cudaMemcpy(lods, c->C.fill_lod, k, cudaMemcpyDeviceToHost));
    }
    *n = c->last_placed;
    return CSV_OK;
}

// Host copies of block_start (i64) and resident LOD (i8), num_bricks each.
int csv_cache_read_state(csv_cache* c, int64_t* block_start, int8_t* resident) {
    if (!c || !block_start || !resident) return cfail(CSV_E_ARG, "null argument");
    CTRY(cudaSetDevice(c->device));
    CTRY(cudaDeviceSynchronize());
    CTRY(cudaMemcpy(block_start, c->C.block_start, c->C.nb * 8, cudaMemcpyDeviceToHost));
    CTRY(cudaMemcpy(resident, c->C.resident, c->C.nb, cudaMemcpyDeviceToHost));
    return CSV_OK;
}

int csv_cache_counters(csv_cache* c, uint64_t* out8) {
    if (!c || !out8) return cfail(CSV_E_ARG, "null argument");
    CTRY(cudaSetDevice(c->device));
    unsigned long long h[C_COUNT];
    CTRY(cudaMemcpy(h, c->C.ctr, C_COUNT * 8, cudaMemcpyDeviceToHost));
    out8[0] = h[C_TOP] < c->C.capacity ? h[C_TOP] : c->C.capacity;
    out8[1] = h[C_EVICT];
    out8[2] = c->rebuilds;
    out8[3] = c->decodes;
    out8[4] = c->decoded_bytes;
    out8[5] = c->last_placed;
    out8[6] = 0;
    out8[7] = 0;
    return CSV_OK;
}

int csv_cache_stack_heights(csv_cache* c, int64_t* out_n) {
    if (!c || !out_n) return cfail(CSV_E_ARG, "null argument");
    CTRY(cudaSetDevice(c->device));
    long long counts[8];
    CTRY(cudaMemcpy(counts, c->C.counts, 64, cudaMemcpyDeviceToHost));
    for (int k = 0; k < c->C.N; ++k) out_n[k] = counts[k];
    return CSV_OK;
}

}  // extern "C"
