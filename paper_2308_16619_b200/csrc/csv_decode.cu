// csv_decode.cu -- B200 (sm_100a) decode kernels for CSV compressed segmentation volumes.
//
// Hot path: per-brick decompression = rANS entropy decode +
// coarse-to-fine operation replay, reference _decode_kernel
// (/root/reference/pkg/src/csvol/codec.py:303-471).  Restructured for the GPU:
//
//  K1 k1_streams   -- entropy stage.  One LANE per (brick, stream): a lane owns
//                     one single-state rANS chain (codec.py:290-300), decodes it
//                     with the packed 4096-entry decode table in shared memory,
//                     parses op/payload nibbles into one entry byte per
//                     operation and stores them 8 at a time.  Lanes refill
//                     work dynamically from a global counter (warp-aggregated
//                     atomics), detail streams (long) first.
//  K2 k2_replay    -- replay stage.  One CTA per brick, level-synchronous:
//                     per level a popcount rank of active parents locates each
//                     parent's 8 entries, a block scan of palette-advance
//                     counts gives i_p, every child is evaluated independently
//                     (same-level neighbour chains resolved directly, <=3
//                     hops), and the final level streams straight to HBM in
//                     raster (K3, decompress_volume) or Morton pool order (K4,
//                     brick cache).
#include <cstdio>
#include <cstring>
#include <type_traits>
#include "csv_device.cuh"

namespace csv {

constexpr int K1_THREADS = 256;
constexpr int K2_THREADS = 256;
constexpr int K2_WARPS = K2_THREADS / 32;

// ============================================================================ planning
// Entry-region sizes per (request, stream) -> sizes[2r+s]; then exclusive scan.
__global__ void k_region_sizes(VolView V, Plan P, uint64_t* sizes) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= 2 * P.n) return;
    uint64_t r = i >> 1;
    int s = (int)(i & 1);
    uint64_t b = req_local(V, P, r);
    int t = req_lod(P, r);
    uint32_t lim = (b < V.nb && t < V.N) ? stream_limit(V, b, t, s) : 0;
    sizes[i] = round16(lim);
}

// Simple 3-phase exclusive scan of u64 (n <= 4096 * 4096).
constexpr int SCAN_ITEMS = 4096;
__device__ __forceinline__ uint64_t warp_incl_scan(uint64_t v) {
    for (int o = 1; o < 32; o <<= 1) {
        uint64_t u = __shfl_up_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) >= o) v += u;
    }
    return v;
}
// Block-wide exclusive scan of one value per thread (blockDim multiple of 32, <= 1024).
__device__ uint64_t block_excl_scan(uint64_t v, uint64_t* sh, uint64_t* total) {
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint64_t inc = warp_incl_scan(v);
    if (lane == 31) sh[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        uint64_t w = lane < nw ? sh[lane] : 0;
        uint64_t wi = warp_incl_scan(w);
        if (lane < nw) sh[lane] = wi - w;
        if (lane == nw - 1) sh[32] = wi;
    }
    __syncthreads();
    uint64_t r = sh[wid] + inc - v;
    if (total) *total = sh[32];
    __syncthreads();
    return r;
}

__global__ void k_scan_blocks(const uint64_t* in, uint64_t* out, uint64_t n, uint64_t* block_sums) {
    __shared__ uint64_t sh[33];
    uint64_t base = (uint64_t)blockIdx.x * SCAN_ITEMS;
    constexpr int PER = SCAN_ITEMS / 256;
    uint64_t loc[PER];
    uint64_t sum = 0;
    for (int k = 0; k < PER; ++k) {
        uint64_t i = base + threadIdx.x * PER + k;
        loc[k] = i < n ? in[i] : 0;
        sum += loc[k];
    }
    uint64_t tot;
    uint64_t pre = block_excl_scan(sum, sh, &tot);
    for (int k = 0; k < PER; ++k) {
        uint64_t i = base + threadIdx.x * PER + k;
        if (i < n) out[i] = pre;
        pre += loc[k];
    }
    if (threadIdx.x == 0) block_sums[blockIdx.x] = tot;
}
__global__ void k_scan_sums(uint64_t* block_sums, int nblocks, uint64_t* out_total) {
    __shared__ uint64_t sh[33];
    // nblocks <= 4096; 1024 threads x 4
    uint64_t loc[4];
    uint64_t sum = 0;
    for (int k = 0; k < 4; ++k) {
        int i = threadIdx.x * 4 + k;
        loc[k] = i < nblocks ? block_sums[i] : 0;
        sum += loc[k];
    }
    uint64_t tot;
    uint64_t pre = block_excl_scan(sum, sh, &tot);
    for (int k = 0; k < 4; ++k) {
        int i = threadIdx.x * 4 + k;
        if (i < nblocks) block_sums[i] = pre;
        pre += loc[k];
    }
    if (threadIdx.x == 0) *out_total = tot;
}
__global__ void k_scan_add(uint64_t* out, uint64_t n, const uint64_t* block_sums) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] += block_sums[i / SCAN_ITEMS];
}

// ============================================================================ K1: entropy lanes
// Per-lane stream state.  The byte reader keeps a 64-bit MSB-first bit buffer
// (renorm bytes are consumed in stream order, rans.py:9-11) plus one aligned
// 32-bit word in flight, so each refill's load latency overlaps ~6 symbols.
struct Lane {
    const uint32_t* wp;     // next aligned word to prefetch
    uint64_t buf;           // upcoming stream bits, MSB first
    uint64_t acc;           // pending entry bytes (<= 8)
    uint64_t* outp;         // entry region (8-byte groups)
    const uint8_t* rawp;    // raw mode: packed nibble bytes
    uint32_t nxt;           // prefetched word
    uint32_t x;             // rANS state (fits 32 bits: f*(x>>12) < 2^32)
    uint32_t pos, len;      // bytes consumed (incl. 4 state bytes) / stream bytes
    uint32_t i, lim, n;     // nibble index, nibble limit, stored count
    uint32_t g;             // groups stored
    uint32_t cur;           // current entry byte
    uint64_t item;
    int nb;                 // valid bits in buf
    int k;                  // entries in acc
    int tsel;               // decode table (0 interior, 1 leaf)
    bool pend;              // next nibble is a P_delta payload
    bool slow;              // first step from a state < 2^23 (corrupt streams only)
};

__device__ __forceinline__ uint32_t bswap32(uint32_t v) { return __byte_perm(v, 0, 0x0123); }

__device__ __forceinline__ void lane_refill(Lane& L) {
    L.buf |= (uint64_t)bswap32(L.nxt) << (32 - L.nb);
    L.nb += 32;
    L.nxt = __ldg(L.wp);
    ++L.wp;
}

__device__ __forceinline__ void lane_emit(Lane& L, uint32_t s) {
    bool pay = L.pend;
    L.pend = !pay && ((s & 7u) == 5u);
    L.cur = pay ? (L.cur | (s << 4)) : s;
    if (!L.pend) {
        L.acc |= (uint64_t)L.cur << (8 * L.k);
        if (++L.k == 8) {
            L.outp[L.g++] = L.acc;
            L.acc = 0;
            L.k = 0;
        }
    }
}

__device__ __forceinline__ void lane_finish(Lane& L, const Plan& P, bool failed, bool entropy) {
    if (L.k > 0) L.outp[L.g] = L.acc;
    csv_stream_result r;
    r.n_entries = L.g * 8 + L.k;
    r.flags = 0;
    r.fail_nibble = 0xffffffffu;
    r.partial_op = 0;
    if (failed) {
        r.flags |= CSV_SF_FAILED;
        r.fail_nibble = L.i;
    } else if (L.i == L.n) {
        r.flags |= CSV_SF_FAILED | CSV_SF_COMPLETE;
        r.fail_nibble = L.n;
        if (entropy && L.n > 0 && (L.x != kStateLower || L.pos != L.len)) r.flags |= CSV_SF_DESYNC;
    }
    if (L.pend) {
        r.flags |= CSV_SF_PARTIAL;
        r.partial_op = L.cur;
    }
    P.sres[L.item] = r;
}

// Initialise lane for work item `item`; returns false if the item finished at once.
template <bool ENTROPY>
__device__ bool lane_init(Lane& L, const VolView& V, const Plan& P, uint64_t item) {
    uint64_t r = item < P.n ? item : item - P.n;
    int s = item < P.n ? 1 : 0;           // detail streams first (longest chains)
    uint64_t w = 2 * r + s;               // result / region index
    L.item = w;
    L.acc = 0; L.k = 0; L.g = 0; L.pend = false; L.cur = 0; L.i = 0; L.slow = false;
    L.x = 0; L.pos = 0; L.len = 0; L.nb = 0; L.buf = 0;
    uint64_t b = req_local(V, P, r);
    int t = req_lod(P, r);
    L.outp = reinterpret_cast<uint64_t*>(P.entries + P.eoff[w]);
    bool ok = b < V.nb && t < V.N && !(s == 1 && t != 0);
    L.n = ok ? eff_nibbles(V, b, s) : 0;
    L.lim = ok ? stream_limit(V, b, t, s) : 0;
    L.tsel = s;
    if (!ok) {
        L.n = 0; L.lim = 0;
        P.sres[w] = csv_stream_result{0, 0xffffffffu, 0, 0};
        return false;
    }
    const uint8_t* base = s ? V.detail + V.d_off[b] : V.coarse + V.c_off[b];
    L.len = s ? V.d_bytes[b] : V.c_bytes[b];
    if (L.lim == 0) {
        if (L.n == 0) P.sres[w] = csv_stream_result{0, 0, CSV_SF_FAILED | CSV_SF_COMPLETE, 0};
        else P.sres[w] = csv_stream_result{0, 0xffffffffu, 0, 0};
        return false;
    }
    if (!ENTROPY) {
        L.rawp = base;
        return true;
    }
    if (L.len < 4) {   // entropy stream shorter than its state word (codec.py:333-334)
        P.sres[w] = csv_stream_result{0, 0, CSV_SF_FAILED, 0};
        return false;
    }
    L.x = (uint32_t)base[0] | ((uint32_t)base[1] << 8) | ((uint32_t)base[2] << 16) | ((uint32_t)base[3] << 24);
    L.pos = 4;
    uintptr_t q = reinterpret_cast<uintptr_t>(base) + 4;
    const uint32_t* aq = reinterpret_cast<const uint32_t*>(q & ~uintptr_t(3));
    int sh = (int)(q & 3);
    L.buf = (uint64_t)bswap32(__ldg(aq)) << (32 + 8 * sh);
    L.nb = 32 - 8 * sh;
    L.wp = aq + 1;
    L.nxt = __ldg(L.wp);
    ++L.wp;
    L.slow = L.x < kStateLower;
    return true;
}

// One symbol; returns false when the lane's item is finished.
template <bool ENTROPY>
__device__ __forceinline__ bool lane_step(Lane& L, const Plan& P, const uint32_t* tab) {
    uint32_t s;
    if (ENTROPY) {
        if (L.nb < 16) lane_refill(L);
        uint32_t e = tab[(L.tsel << 12) | (L.x & (kTotalFreq - 1))];
        s = e & 15u;
        uint32_t xn = (e >> 16) * (L.x >> kPrecision) + ((e >> 4) & 0xFFFu);
        if (!L.slow) {
            // after a step from x >= 2^23, x >= 2^11: at most two renorm bytes
            uint32_t r = (xn < kStateLower) + (xn < (1u << 15));
            if (L.pos + r > L.len) {           // underrun (codec.py:295-297)
                lane_finish(L, P, true, true);
                return false;
            }
            uint32_t top = (uint32_t)(L.buf >> 48);
            L.x = (xn << (8 * r)) | (top >> (16 - 8 * r));
            L.buf <<= 8 * r;
            L.nb -= 8 * r;
            L.pos += r;
        } else {
            L.slow = false;
            while (xn < kStateLower) {
                if (L.pos >= L.len) {
                    lane_finish(L, P, true, true);
                    return false;
                }
                if (L.nb < 8) lane_refill(L);
                xn = (xn << 8) | (uint32_t)(L.buf >> 56);
                L.buf <<= 8;
                L.nb -= 8;
                ++L.pos;
            }
            L.x = xn;
        }
    } else {
        s = (L.rawp[L.i >> 1] >> (4 * (L.i & 1))) & 15u;
    }
    lane_emit(L, s);
    if (++L.i == L.lim) {
        lane_finish(L, P, false, ENTROPY);
        return false;
    }
    return true;
}

template <bool ENTROPY>
__global__ void __launch_bounds__(K1_THREADS) k1_streams(VolView V, Plan P, unsigned long long* counter) {
    __shared__ uint32_t tab[2 * 4096];
    if (ENTROPY) {
        for (int i = threadIdx.x; i < 2 * 4096; i += blockDim.x) tab[i] = V.dtab[i];
        __syncthreads();
    }
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const uint64_t total = 2 * P.n;
    Lane L;
    bool has = false, done = false;
    while (true) {
        bool need = !has && !done;
        unsigned m = __ballot_sync(FULL, need);
        if (m) {
            int leader = __ffs(m) - 1;
            unsigned long long base = 0;
            if (lane == leader) base = atomicAdd(counter, (unsigned long long)__popc(m));
            base = __shfl_sync(FULL, base, leader);
            if (need) {
                uint64_t my = base + __popc(m & ((1u << lane) - 1u));
                if (my < total) has = lane_init<ENTROPY>(L, V, P, my);
                else done = true;
            }
        }
        if (__all_sync(FULL, done)) break;
        if (has) {
#pragma unroll 4
            for (int u = 0; u < 32; ++u) {
                if (!lane_step<ENTROPY>(L, P, tab)) { has = false; break; }
            }
        }
    }
}

// ============================================================================ K2: replay
// Shared (or global-workspace) layout for one brick, sized for L = N - t levels:
//   lev  : values of levels t+1..N in Morton order; level N-j at levoffA(j)
//          (16-byte aligned for j >= 1)
//   mask : 2 x W words, active-parent bitmask ping-pong
//   wpre : W+1 words, exclusive popcount prefix of the parent mask
//   ipb  : per active parent (by rank) palette-advance prefix, level-relative
//   list : per active parent (by rank) its Morton index
//   pend : one bit per child of the level: "same-level chain not resolved yet"
// IdxT is u16 in the shared-memory variant (L <= 5: <= 4096 parents, <= 32768
// entries per level) and u32 in the global-workspace variant (L = 6, 7).
__host__ __device__ __forceinline__ uint32_t levoffA(int j) {
    return j == 0 ? 0u : 4u + ((1u << (3 * j)) - 8u) / 7u;
}
struct Layout {
    uint32_t lev, mask, wpre, ipb, list, pend, words, W;   // offsets in u32 units
};
__host__ __device__ inline Layout make_layout(int L, int idx_bytes) {
    Layout Y;
    uint32_t nlev = levoffA(L);
    uint32_t maxP = 1u << (3 * (L - 1));
    Y.W = (maxP + 31) / 32;
    Y.lev = 0;
    Y.mask = (nlev + 3) & ~3u;
    Y.wpre = Y.mask + 2 * Y.W;
    Y.ipb = (Y.wpre + Y.W + 1 + 3) & ~3u;
    uint32_t idx_words = (maxP * idx_bytes + 15) / 16 * 4;
    Y.list = Y.ipb + idx_words;
    Y.pend = Y.list + idx_words;
    Y.words = Y.pend + (8 * maxP + 31) / 32;
    return Y;
}

enum { OUT_RASTER = 0, OUT_MORTON = 1 };

// error key = entry << 8 | priority << 4 | status; per entry BAD_OP beats
// LEAF_STOP beats the op-specific check (codec.py:396-457 order).
__device__ __forceinline__ unsigned long long ekey(uint32_t ent, int prio, int st) {
    return ((unsigned long long)ent << 8) | (unsigned)(prio << 4) | (unsigned)st;
}
enum { EK_UNDERRUN_NV = 15 };   // status placeholder: entry == K1's n_entries

struct K2Shared {
    unsigned long long errkey;
    uint32_t scan[K2_WARPS + 1];
    uint64_t red64[2][K2_WARPS];
};

// Block-wide in-place exclusive scan of arr[0..n); returns the total.
template <typename T>
__device__ uint32_t block_scan_inplace(T* arr, uint32_t n, K2Shared& S) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t per = (n + K2_WARPS - 1) / K2_WARPS;
    uint32_t lo = wid * per, hi = min(n, lo + per);
    uint32_t sum = 0;
    for (uint32_t i = lo + lane; i < hi; i += 32) sum += arr[i];
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) S.scan[wid] = sum;
    __syncthreads();
    if (threadIdx.x < 32) {
        uint32_t v = lane < K2_WARPS ? S.scan[lane] : 0, inc = v;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += u;
        }
        if (lane < K2_WARPS) S.scan[lane] = inc - v;
        if (lane == K2_WARPS - 1) S.scan[K2_WARPS] = inc;
    }
    __syncthreads();
    uint32_t carry = S.scan[wid];
    for (uint32_t c0 = lo; c0 < hi; c0 += 32) {
        uint32_t i = c0 + lane;
        uint32_t v = i < hi ? (uint32_t)arr[i] : 0, inc = v;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += u;
        }
        if (i < hi) arr[i] = (T)(carry + inc - v);
        carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    uint32_t total = S.scan[K2_WARPS];
    __syncthreads();
    return total;
}

__device__ __forceinline__ uint64_t block_sum64(uint64_t v, int slot, K2Shared& S) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) S.red64[slot][threadIdx.x >> 5] = v;
    __syncthreads();
    uint64_t t = 0;
    for (int w = 0; w < K2_WARPS; ++w) t += S.red64[slot][w];
    __syncthreads();
    return t;
}

struct RasterCtx {
    uint32_t* base;     // voxel (ox, oy, oz) of the slab (valid when fast)
    int64_t ox, oy, oz; // brick origin (LOD-t voxels)
    int64_t cx, cy;     // row pitch / plane
    int64_t zb, ze;
    bool fast;          // brick fully inside crop and slab, 8-byte aligned rows
};

// Address of brick-local voxel (x, y, z) in the raster slab, or nullptr if cropped away.
__device__ __forceinline__ uint32_t* raster_ptr(const RasterCtx& R, const Plan& P, int64_t x, int64_t y, int64_t z) {
    if (R.fast) return R.base + (z * R.cy + y) * R.cx + x;
    int64_t gz = R.oz + z, gy = R.oy + y, gx = R.ox + x;
    if (gz < R.zb || gz >= R.ze || gy >= R.cy || gx >= R.cx) return nullptr;
    return P.out + ((gz - R.zb) * R.cy + gy) * R.cx + gx;
}

__device__ __forceinline__ void store_pair(const RasterCtx& R, const Plan& P, int64_t x, int64_t y, int64_t z,
                                           uint32_t a, uint32_t b) {
    if (R.fast) {
        *reinterpret_cast<uint2*>(R.base + (z * R.cy + y) * R.cx + x) = make_uint2(a, b);
        return;
    }
    uint32_t* p = raster_ptr(R, P, x, y, z);
    if (!p) return;
    if (R.ox + x + 1 < R.cx) {
        if ((reinterpret_cast<uintptr_t>(p) & 7) == 0) *reinterpret_cast<uint2*>(p) = make_uint2(a, b);
        else { p[0] = a; p[1] = b; }
    } else {
        p[0] = a;
    }
}

__device__ __forceinline__ void write_result(const Plan& P, uint64_t r, int st, int stream, int64_t pos,
                                             int64_t ci, int64_t di) {
    if (P.res && threadIdx.x == 0) {
        csv_result o;
        o.status = st; o.stream = stream; o.pos = pos; o.ci = ci; o.di = di;
        P.res[r] = o;
    }
}

// Fill the whole output of request r with one value (relevant == 0, codec.py:353-358).
template <int MODE>
__device__ void fill_output(const VolView& V, const Plan& P, const RasterCtx& R, int t, uint32_t* out_m, uint32_t val) {
    const int lb = V.N - t;
    const uint64_t n = 1ull << (3 * lb);
    if (MODE == OUT_MORTON) {
        for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) out_m[i] = val;
    } else if (lb == 0) {
        if (threadIdx.x == 0) {
            uint32_t* p = raster_ptr(R, P, 0, 0, 0);
            if (p) *p = val;
        }
    } else {
        const int side = 1 << lb;
        for (uint64_t i = threadIdx.x; i < n / 2; i += blockDim.x) {
            int64_t x = (2 * i) & (side - 1), y = ((2 * i) >> lb) & (side - 1), z = (2 * i) >> (2 * lb);
            store_pair(R, P, x, y, z, val, val);
        }
    }
}

// Storage slot of child j of the current level: shared level array, raster
// voxel or Morton pool entry.  nullptr when the voxel is cropped away.
template <int MODE>
__device__ __forceinline__ uint32_t* child_slot(bool final_level, uint32_t* clev, uint32_t* out_m, const RasterCtx& R,
                                                const Plan& P, uint32_t j) {
    if (!final_level) return clev + j;
    if (MODE == OUT_MORTON) return out_m + j;
    return raster_ptr(R, P, compact3(j), compact3(j >> 1), compact3(j >> 2));
}

template <int MODE, bool SMEM>
__global__ void __launch_bounds__(K2_THREADS, SMEM ? 5 : 1)
k2_replay(VolView V, Plan P, int Lmax, uint32_t* gws, uint64_t ws_stride) {
    using IdxT = typename std::conditional<SMEM, uint16_t, uint32_t>::type;
    extern __shared__ __align__(16) uint32_t dsm[];
    __shared__ K2Shared S;
    const Layout Y = make_layout(Lmax, sizeof(IdxT));
    uint32_t* ws = SMEM ? dsm : gws + blockIdx.x * ws_stride;
    uint32_t* lev = ws + Y.lev;
    uint32_t* mask0 = ws + Y.mask;
    uint32_t* wpre = ws + Y.wpre;
    IdxT* ipb = reinterpret_cast<IdxT*>(ws + Y.ipb);
    IdxT* list = reinterpret_cast<IdxT*>(ws + Y.list);
    uint32_t* pend = ws + Y.pend;
    const int N = V.N;
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    for (uint64_t r = blockIdx.x; r < P.n; r += gridDim.x) {
        const uint64_t b = req_local(V, P, r);
        const int t = req_lod(P, r);
        if (b >= V.nb || t > N) { write_result(P, r, -1, 0, 0, 0, 0); continue; }
        if (t < N && N - t > Lmax) continue;           // belongs to the other variant
        if (!SMEM && N - t <= 5) continue;
        uint32_t* out_m = MODE == OUT_MORTON ? P.out + P.dst[r] : nullptr;
        const uint32_t plen = V.pal_len[b];
        const uint32_t* pal = V.palette + V.pal_off[b];
        RasterCtx R{};
        if (MODE == OUT_RASTER) {
            const uint64_t gb = V.brick_begin + b;
            const int64_t side = 1ll << (N - t);
            R.ox = (int64_t)(gb % V.gx) * side;
            R.oy = (int64_t)((gb / V.gx) % V.gy) * side;
            R.oz = (int64_t)(gb / (V.gx * V.gy)) * side;
            R.cx = P.cx; R.cy = P.cy; R.zb = P.z_begin; R.ze = P.z_end;
            R.base = P.out + ((R.oz - R.zb) * R.cy + R.oy) * R.cx + R.ox;
            R.fast = side >= 2 && R.ox + side <= R.cx && R.oy + side <= R.cy && R.oz >= R.zb && R.oz + side <= R.ze &&
                     (R.cx & 1) == 0 && ((reinterpret_cast<uintptr_t>(P.out) & 7) == 0);
        }
        if (plen == 0) { write_result(P, r, CSV_ST_EMPTY_PALETTE, 0, 0, 0, 0); continue; }
        if (t == N) {   // coarsest LOD: palette[0] (codec.py:514-516, container.py:178-182)
            if (MODE == OUT_MORTON) { if (threadIdx.x == 0) out_m[0] = __ldg(pal); }
            else fill_output<MODE>(V, P, R, t, nullptr, __ldg(pal));
            write_result(P, r, 0, 0, 0, 0, 0);
            continue;
        }
        const uint32_t nc_raw = V.c_nib[b], nd_raw = t == 0 ? V.d_nib[b] : 0;
        const uint32_t nc = eff_nibbles(V, b, 0), nd = t == 0 ? eff_nibbles(V, b, 1) : 0;
        if (V.entropy) {   // state-word checks come first (codec.py:331-351)
            if (nc_raw > 0 && V.c_bytes[b] < 4) { write_result(P, r, CSV_ST_UNDERRUN, 0, 0, 0, 0); continue; }
            if (t == 0 && nd_raw > 0 && V.d_bytes[b] < 4) { write_result(P, r, CSV_ST_UNDERRUN, 1, 0, 0, 0); continue; }
        }
        if ((uint64_t)nc + nd == 0) {
            fill_output<MODE>(V, P, R, t, out_m, __ldg(pal));
            write_result(P, r, 0, 0, 0, 0, 0);
            continue;
        }
        const csv_stream_result src = P.sres[2 * r], srd = P.sres[2 * r + 1];
        const uint64_t eo0 = P.eoff[2 * r], eo1 = P.eoff[2 * r + 1], eo2 = P.eoff[2 * r + 2];
        if (threadIdx.x == 0) {
            lev[0] = __ldg(pal);      // root (codec.py:353)
            mask0[0] = 1u;
            S.errkey = ~0ull;
        }
        __syncthreads();
        uint32_t cur_c = 0, cur_d = 0;
        uint64_t pd_c = 0, pd_d = 0;
        int64_t ipbase = 0;
        int cur = 0;
        bool failed = false;
        for (int l = N; l > t; --l) {
            const bool leaf = l == 1;
            const bool final_level = (l - 1 == t);
            const uint32_t Pn = 1u << (3 * (N - l));
            const uint32_t W = (Pn + 31) >> 5;
            const uint32_t PW = (8 * Pn + 31) >> 5;      // pending words (children)
            uint32_t* pmask = mask0 + cur * Y.W;
            uint32_t* cmask = mask0 + (cur ^ 1) * Y.W;
            const csv_stream_result& sr = leaf ? srd : src;
            const uint32_t e0 = leaf ? cur_d : cur_c;
            const uint8_t* Eb = P.entries + (leaf ? eo1 : eo0);          // this stream's entry bytes
            const uint32_t ecap = (uint32_t)((leaf ? eo2 : eo1) - (leaf ? eo1 : eo0));
            const uint32_t* plev = lev + levoffA(N - l);
            uint32_t* clev = final_level ? nullptr : lev + levoffA(N - l + 1);
            const int cbits = N - l + 1;
            // (A) rank prefix of active parents; clear pending bits
            for (uint32_t i = threadIdx.x; i < W; i += blockDim.x) {
                uint32_t mw = pmask[i];
                if (Pn < 32) mw &= (1u << Pn) - 1u;
                pmask[i] = mw;
                wpre[i] = __popc(mw);
            }
            for (uint32_t i = threadIdx.x; i < PW; i += blockDim.x) pend[i] = 0;
            __syncthreads();
            const uint32_t nact = block_scan_inplace(wpre, W, S);
            // (B) active list + palette-advance counts per active parent
            for (uint32_t i = threadIdx.x; i < W; i += blockDim.x) {
                uint32_t mw = pmask[i], rk = wpre[i];
                while (mw) {
                    int bit = __ffs(mw) - 1;
                    mw &= mw - 1;
                    list[rk++] = (IdxT)(32 * i + bit);
                }
            }
            uint64_t pdl = 0;
            for (uint32_t i = threadIdx.x; i < nact; i += blockDim.x) {
                const uint32_t off = e0 + 8 * i;
                uint64_t w = off + 8 <= ecap ? __ldg(reinterpret_cast<const uint64_t*>(Eb + off)) : 0ull;
                ipb[i] = (IdxT)__popcll(op_eq(w, 6));
                pdl += __popcll(op_eq(w, 5));
            }
            if (leaf) pd_d += pdl; else pd_c += pdl;
            __syncthreads();
            const uint32_t tot_pa = block_scan_inplace(ipb, nact, S);
            const uint32_t nvalid = sr.n_entries;
            // (C1) one lane per child of an active parent (8 consecutive lanes = one parent)
            const uint32_t nch = 8 * nact;
            unsigned long long myerr = ~0ull;
            for (uint32_t kb = threadIdx.x - lane; kb < nch; kb += blockDim.x) {
                const uint32_t k = kb + lane;
                const bool valid = k < nch;
                const uint32_t rk = k >> 3;
                const int c = k & 7;
                const uint32_t q = valid ? (uint32_t)list[rk] : 0u;
                const uint32_t ent = e0 + k;
                const uint32_t e = (valid && ent < ecap) ? (uint32_t)__ldg(Eb + ent) : 0u;
                const uint32_t op = e & 7u;
                const uint32_t pv = plev[q];
                const uint32_t seg = 0xFFu << (lane & 24);
                const uint32_t pam = __ballot_sync(FULL, valid && op == 6u);
                const uint32_t nstop = __ballot_sync(FULL, valid && !(e & 8u));
                uint32_t val = pv;
                int st = 0;
                bool chain = false;
                const uint32_t j = (q << 3) | c;
                if (op >= 1 && op <= 3) {
                    const int a = op - 1;
                    const uint32_t M = axis_mask(a, cbits);
                    const uint32_t part = j & M;
                    if ((c >> a) & 1) {      // odd: the +1 neighbour is decoded later -> its parent's value
                        if (part == M) st = CSV_ST_BAD_NEIGHBOR;
                        else val = plev[((((part | ~M) + 1u) & M) | (j & ~M)) >> 3];
                    } else {                 // even: the -1 neighbour at this level (resolved in rounds)
                        if (part == 0) st = CSV_ST_BAD_NEIGHBOR;
                        else chain = true;
                    }
                } else if (op >= 4 && op <= 6) {
                    const int64_t ip = ipbase + (int64_t)ipb[valid ? rk : 0] + __popc(pam & seg & ((1u << lane) - 1u));
                    int64_t idx;
                    if (op == 4) idx = ip;
                    else if (op == 5) { idx = ip - (int64_t)(e >> 4) - 1; if (idx < 0) st = CSV_ST_DELTA_RANGE; }
                    else { idx = ip + 1; if (idx >= (int64_t)plen) st = CSV_ST_PALETTE_RANGE; }
                    idx = idx < 0 ? 0 : (idx >= (int64_t)plen ? (int64_t)plen - 1 : idx);
                    val = __ldg(pal + idx);
                }
                if (valid && ent < nvalid) {
                    unsigned long long kk = ~0ull;
                    if (op == 7) kk = ekey(ent, 0, CSV_ST_BAD_OP);
                    else if (leaf && (e & 8u)) kk = ekey(ent, 1, CSV_ST_LEAF_STOP);
                    else if (st) kk = ekey(ent, 2, st);
                    myerr = kk < myerr ? kk : myerr;
                }
                if (!final_level && valid && c == 0)
                    reinterpret_cast<uint8_t*>(cmask)[q] = (uint8_t)(nstop >> (lane & 24));
                if (valid) {
                    if (chain) {
                        atomicOr(&pend[j >> 5], 1u << (j & 31));
                    } else {
                        uint32_t* slot = child_slot<MODE>(final_level, clev, out_m, R, P, j);
                        if (slot) *slot = val;
                    }
                }
            }
            if (myerr != ~0ull) atomicMin(&S.errkey, myerr);
            // (C2) inactive parents: their children repeat the parent value
            if (final_level && MODE == OUT_RASTER) {
                const int pb = N - l;
                const uint32_t pm = (1u << pb) - 1u;
                for (uint32_t i = threadIdx.x; i < Pn; i += blockDim.x) {
                    const uint32_t qx = i & pm, qy = (i >> pb) & pm, qz = i >> (2 * pb);
                    const uint32_t q = spread3_u32(qx) | (spread3_u32(qy) << 1) | (spread3_u32(qz) << 2);
                    if ((pmask[q >> 5] >> (q & 31)) & 1u) continue;
                    const uint32_t pv = plev[q];
#pragma unroll
                    for (int row = 0; row < 4; ++row)
                        store_pair(R, P, 2 * qx, 2 * qy + (row & 1), 2 * qz + (row >> 1), pv, pv);
                }
            } else {
                for (uint32_t q = threadIdx.x; q < Pn; q += blockDim.x) {
                    if ((pmask[q >> 5] >> (q & 31)) & 1u) continue;
                    const uint32_t pv = plev[q];
                    uint32_t* dstp = final_level ? out_m + 8ull * q : clev + 8 * q;
                    if (!final_level || ((reinterpret_cast<uintptr_t>(dstp) & 15) == 0)) {
                        reinterpret_cast<uint4*>(dstp)[0] = make_uint4(pv, pv, pv, pv);
                        reinterpret_cast<uint4*>(dstp)[1] = make_uint4(pv, pv, pv, pv);
                    } else {
#pragma unroll
                        for (int c = 0; c < 8; ++c) dstp[c] = pv;
                    }
                    if (!final_level) reinterpret_cast<uint8_t*>(cmask)[q] = 0;
                }
            }
            if (threadIdx.x == 0 && (uint64_t)e0 + 8ull * nact > nvalid)
                atomicMin(&S.errkey, ekey(nvalid, 0, EK_UNDERRUN_NV));
            __syncthreads();
            const unsigned long long ek = S.errkey;
            if (ek != ~0ull) {
                // first failing entry in sequential order -> status + nibble position
                const uint32_t ent = (uint32_t)(ek >> 8);
                const int code = (int)(ek & 0xF);
                int st;
                int64_t pos;
                if (code == EK_UNDERRUN_NV) {
                    if ((sr.flags & CSV_SF_PARTIAL) && leaf && (sr.partial_op & 8u)) {
                        st = CSV_ST_LEAF_STOP;
                        pos = (int64_t)sr.fail_nibble - 1;
                    } else {
                        st = CSV_ST_UNDERRUN;
                        pos = (sr.flags & CSV_SF_FAILED) ? (int64_t)sr.fail_nibble : (int64_t)ent;
                    }
                } else {
                    // nibble index of entry `ent` = ent + #payload nibbles before it
                    uint64_t cnt = 0;
                    for (uint32_t g = threadIdx.x; g < (ent + 7) / 8; g += blockDim.x) {
                        uint64_t w = (8 * g + 8 <= ecap) ? __ldg(reinterpret_cast<const uint64_t*>(Eb) + g) : 0ull;
                        uint32_t lim = ent - 8 * g;
                        uint64_t m = op_eq(w, 5);
                        if (lim < 8) m &= (1ull << (8 * lim)) - 1ull;
                        cnt += __popcll(m);
                    }
                    pos = (int64_t)ent + (int64_t)block_sum64(cnt, 0, S);
                    st = code;
                    if (code == CSV_ST_DELTA_RANGE) pos += 1;   // reported at the payload nibble
                }
                write_result(P, r, st, leaf ? 1 : 0, pos, 0, 0);
                failed = true;
                break;
            }
            // (R) same-level chains (codec.py:422-423, nm < j): a child copies its -1
            // neighbour once that one is final.  Hops make coordinates odd, so a
            // chain is at most 3 deep and resolves within 3 rounds.
            for (int round = 0; round < 4; ++round) {
                int any = 0;
                for (uint32_t wdx = threadIdx.x; wdx < PW; wdx += blockDim.x) {
                    uint32_t bits = *(volatile uint32_t*)&pend[wdx];
                    while (bits) {
                        const int bit = __ffs(bits) - 1;
                        bits &= bits - 1;
                        const uint32_t j = 32 * wdx + bit;
                        const uint32_t q = j >> 3;
                        const int c = j & 7;
                        const uint32_t rk = wpre[q >> 5] + __popc(pmask[q >> 5] & ((1u << (q & 31)) - 1u));
                        const uint32_t e = __ldg(Eb + e0 + 8 * rk + c);
                        const int a = (int)(e & 7u) - 1;
                        const uint32_t M = axis_mask(a, cbits);
                        const uint32_t nm = (((j & M) - 1u) & M) | (j & ~M);
                        if ((*(volatile uint32_t*)&pend[nm >> 5] >> (nm & 31)) & 1u) { any = 1; continue; }
                        __threadfence_block();
                        uint32_t* dst = child_slot<MODE>(final_level, clev, out_m, R, P, j);
                        if (dst) {
                            const uint32_t* srcp = child_slot<MODE>(final_level, clev, out_m, R, P, nm);
                            *(volatile uint32_t*)dst = *(volatile const uint32_t*)srcp;
                        }
                        __threadfence_block();
                        atomicAnd(&pend[j >> 5], ~(1u << (j & 31)));
                    }
                }
                if (!__syncthreads_or(any)) break;
            }
            if (leaf) cur_d = e0 + 8 * nact; else cur_c = e0 + 8 * nact;
            ipbase += tot_pa;
            cur ^= 1;
        }
        if (!failed) {
            const int64_t pdc = (int64_t)block_sum64(pd_c, 0, S);
            const int64_t pdd = (int64_t)block_sum64(pd_d, 1, S);
            const int64_t ci = (int64_t)cur_c + pdc, di = (int64_t)cur_d + pdd;
            int st = 0, stream = 0;
            int64_t pos = 0;
            if (V.entropy) {   // full consumption must land on the initial state (codec.py:464-470)
                if (nc_raw > 0 && ci == (int64_t)nc_raw && (src.flags & CSV_SF_DESYNC)) { st = CSV_ST_DESYNC; stream = 0; pos = ci; }
                else if (t == 0 && nd_raw > 0 && di == (int64_t)nd_raw && (srd.flags & CSV_SF_DESYNC)) { st = CSV_ST_DESYNC; stream = 1; pos = di; }
            }
            write_result(P, r, st, stream, pos, ci, di);
        }
        __syncthreads();
    }
}

// Coarsest-LOD raster (t == N): one voxel per brick.
__global__ void k_root_raster(VolView V, Plan P) {
    uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (b >= V.nb) return;
    uint32_t plen = V.pal_len[b];
    if (P.res) {
        csv_result o{plen == 0 ? CSV_ST_EMPTY_PALETTE : 0, 0, 0, 0, 0};
        P.res[b] = o;
    }
    if (plen == 0) return;
    uint64_t gb = V.brick_begin + b;
    int64_t x = gb % V.gx, y = (gb / V.gx) % V.gy, z = gb / (V.gx * V.gy);
    if (x < P.cx && y < P.cy && z >= P.z_begin && z < P.z_end)
        P.out[((z - P.z_begin) * P.cy + y) * P.cx + x] = V.palette[V.pal_off[b]];
}

// ============================================================================ host launchers
template <bool E>
static void launch_k1(const VolView& V, const Plan& P, unsigned long long* counter, int nsm, cudaStream_t st) {
    uint64_t items = 2 * P.n;
    uint64_t want = (items + 31) / 32;                 // warps needed at one item per lane
    uint64_t blocks = (want + K1_THREADS / 32 - 1) / (K1_THREADS / 32);
    uint64_t cap = (uint64_t)nsm * 8;                  // 8 x 256 threads per SM resident (32 KB smem each)
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    k1_streams<E><<<(unsigned)blocks, K1_THREADS, 0, st>>>(V, P, counter);
}

}  // namespace csv

// ---------------------------------------------------------------------------- internal host API
namespace csv {

struct Runtime {
    int nsm = 148;
};

cudaError_t run_scan(const uint64_t* sizes, uint64_t* out, uint64_t n, uint64_t* tmp, cudaStream_t st) {
    // out has n+1 slots; tmp >= nblocks + 1 slots
    uint64_t nblocks = (n + SCAN_ITEMS - 1) / SCAN_ITEMS;
    if (nblocks == 0) nblocks = 1;
    if (nblocks > 4096) return cudaErrorInvalidValue;
    k_scan_blocks<<<(unsigned)nblocks, 256, 0, st>>>(sizes, out, n, tmp);
    k_scan_sums<<<1, 1024, 0, st>>>(tmp, (int)nblocks, out + n);
    k_scan_add<<<(unsigned)((n + 255) / 256 ? (n + 255) / 256 : 1), 256, 0, st>>>(out, n, tmp);
    return cudaGetLastError();
}

size_t k2_smem_bytes(int L) { return (size_t)make_layout(L, 2).words * 4; }
uint64_t k2_gws_words(int L) { return make_layout(L, 4).words; }

// Decode a plan: sizes -> scan -> K1 -> K2.  Workspace pointers are provided by the caller.
cudaError_t run_decode(const VolView& V, Plan P, int mode, uint64_t* sizes_tmp, uint64_t* scan_tmp,
                       unsigned long long* counter, uint32_t* gws, uint64_t gws_stride, int gws_ctas,
                       int nsm, int min_t, cudaStream_t st, cudaEvent_t* ev) {
    if (P.n == 0) return cudaSuccess;
    if (ev) cudaEventRecord(ev[0], st);
    unsigned nb = (unsigned)((2 * P.n + 255) / 256);
    k_region_sizes<<<nb, 256, 0, st>>>(V, P, sizes_tmp);
    cudaError_t e = run_scan(sizes_tmp, P.eoff, 2 * P.n, scan_tmp, st);
    if (e != cudaSuccess) return e;
    cudaMemsetAsync(counter, 0, sizeof(unsigned long long), st);
    if (ev) cudaEventRecord(ev[1], st);
    if (V.entropy) launch_k1<true>(V, P, counter, nsm, st);
    else launch_k1<false>(V, P, counter, nsm, st);
    if (ev) cudaEventRecord(ev[2], st);
    // K2 smem variant (N - t <= 5)
    int Ls = V.N - min_t;
    if (Ls > 5) Ls = 5;
    if (Ls < 1) Ls = 1;
    size_t smem = k2_smem_bytes(Ls);
    unsigned grid = (unsigned)(P.n < 0x7fffffffull ? P.n : 0x7fffffffull);
    if (mode == OUT_RASTER) {
        cudaFuncSetAttribute(k2_replay<OUT_RASTER, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k2_replay<OUT_RASTER, true><<<grid, K2_THREADS, smem, st>>>(V, P, Ls, nullptr, 0);
    } else {
        cudaFuncSetAttribute(k2_replay<OUT_MORTON, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k2_replay<OUT_MORTON, true><<<grid, K2_THREADS, smem, st>>>(V, P, Ls, nullptr, 0);
    }
    if (V.N - min_t > 5 && gws) {
        unsigned g = (unsigned)(P.n < (uint64_t)gws_ctas ? P.n : (uint64_t)gws_ctas);
        int Lg = V.N - min_t;
        if (mode == OUT_RASTER) k2_replay<OUT_RASTER, false><<<g, K2_THREADS, 0, st>>>(V, P, Lg, gws, gws_stride);
        else k2_replay<OUT_MORTON, false><<<g, K2_THREADS, 0, st>>>(V, P, Lg, gws, gws_stride);
    }
    if (ev) cudaEventRecord(ev[3], st);
    return cudaGetLastError();
}

cudaError_t run_root_raster(const VolView& V, Plan P, cudaStream_t st) {
    unsigned nb = (unsigned)((V.nb + 255) / 256);
    if (nb == 0) return cudaSuccess;
    k_root_raster<<<nb, 256, 0, st>>>(V, P);
    return cudaGetLastError();
}

cudaError_t run_streams_only(const VolView& V, Plan P, uint64_t* sizes_tmp, uint64_t* scan_tmp,
                             unsigned long long* counter, int nsm, cudaStream_t st) {
    if (P.n == 0) return cudaSuccess;
    unsigned nb = (unsigned)((2 * P.n + 255) / 256);
    k_region_sizes<<<nb, 256, 0, st>>>(V, P, sizes_tmp);
    cudaError_t e = run_scan(sizes_tmp, P.eoff, 2 * P.n, scan_tmp, st);
    if (e != cudaSuccess) return e;
    cudaMemsetAsync(counter, 0, sizeof(unsigned long long), st);
    if (V.entropy) launch_k1<true>(V, P, counter, nsm, st);
    else launch_k1<false>(V, P, counter, nsm, st);
    return cudaGetLastError();
}

}  // namespace csv
