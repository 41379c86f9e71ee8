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
//                     operation and stores them 16 at a time.  Lanes refill
//                     work dynamically from a global counter (warp-aggregated
//                     atomics), detail streams (long) first.
//  K2w k2_warp     -- replay stage (csv_replay_warp.cuh), the default: one
//                     WARP per brick, persistent warps, values as u8/u16
//                     palette indices, compacted active parents, chain rounds
//                     by popcount class, plane-sweep final level written to HBM
//                     as whole raster rows (K3, decompress_volume) or Morton
//                     sectors (K4, brick cache).
//  K2 k2_fast / k2_replay -- the earlier CTA-per-brick level-synchronous replay
//                     (csv_replay_fast.cuh, below): kept for palettes > 65535
//                     entries and for N - t = 6, 7 (global workspace).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include "csv_device.cuh"
#include "csv_eval8.cuh"

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
    sizes[i] = round32(lim);
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

// Small plans (2n <= SCAN_ITEMS streams): region sizes + exclusive scan + the K1/K2w
// work counters in ONE launch (per-brick calls are launch-latency bound).
__global__ void __launch_bounds__(256) k_plan_small(VolView V, Plan P, unsigned long long* counter) {
    __shared__ uint64_t sh[33];
    constexpr int PER = SCAN_ITEMS / 256;
    const uint64_t n2 = 2 * P.n;
    uint64_t loc[PER];
    uint64_t sum = 0;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const uint64_t i = threadIdx.x * PER + k;
        uint64_t v = 0;
        if (i < n2) {
            const uint64_t b = req_local(V, P, i >> 1);
            const int t = req_lod(P, i >> 1);
            v = round32((b < V.nb && t < V.N) ? stream_limit(V, b, t, (int)(i & 1)) : 0);
        }
        loc[k] = v;
        sum += v;
    }
    uint64_t tot;
    uint64_t pre = block_excl_scan(sum, sh, &tot);
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const uint64_t i = threadIdx.x * PER + k;
        if (i < n2) P.eoff[i] = pre;
        pre += loc[k];
    }
    if (threadIdx.x == 0) {
        P.eoff[n2] = tot;
        for (int i = 0; i < kCounterSlots; ++i) counter[i] = 0;
    }
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
// (renorm bytes are consumed in stream order, rans.py:9-11) fed from 16-byte
// aligned chunks with one chunk in flight (~25 symbols of prefetch distance).
struct Lane {
    const uint4* qp;        // next 16-byte chunk to prefetch
    uint4 cq;               // current chunk (words consumed from .x, rotated)
    uint4 nq;               // prefetched chunk
    uint64_t buf;           // upcoming stream bits, MSB first
    uint32_t alo, ahi;      // last <= 8 entry bytes, newest in the top byte of ahi
    uint32_t plo, phi;      // the previous complete 8-entry group (stored in 16-byte pairs)
    uint64_t* outp;         // entry region (32-byte aligned)
    uint64_t c03, c47;      // count mode: per-op counters, 4 x 16 bits each
    const uint8_t* rawp;    // raw mode: packed nibble bytes
    uint32_t x;             // rANS state (fits 32 bits: f*(x>>12) < 2^32)
    uint32_t pos, len;      // bytes consumed (incl. 4 state bytes) / stream bytes
    uint32_t i, lim, n;     // nibble index, nibble limit, stored count
    uint32_t ne;            // entries emitted
    uint32_t cur;           // current entry byte
    uint64_t item;
    int nb;                 // valid bits in buf
    int cw;                 // words left in cq
    uint32_t tbase;         // decode table offset in shared memory (0 interior, 4096 leaf)
    uint32_t since;         // count mode: ops since the last flush
    bool pend;              // next nibble is a P_delta payload
    bool slow;              // first step from a state < 2^23 (corrupt streams only)
};

__device__ __forceinline__ uint32_t bswap32(uint32_t v) { return __byte_perm(v, 0, 0x0123); }

__device__ __forceinline__ uint32_t lane_next_word(Lane& L) {
    if (L.cw == 0) {
        L.cq = L.nq;
        L.nq = __ldg(L.qp);
        ++L.qp;
        L.cw = 4;
    }
    const uint32_t w = L.cq.x;
    L.cq.x = L.cq.y; L.cq.y = L.cq.z; L.cq.z = L.cq.w;
    --L.cw;
    return w;
}

__device__ __forceinline__ void lane_refill(Lane& L) {
    L.buf |= (uint64_t)bswap32(lane_next_word(L)) << (32 - L.nb);
    L.nb += 32;
}

// count-mode flush of the packed per-op counters (stats(), container.py:485-495)
__device__ __forceinline__ void lane_flush_counts(Lane& L, unsigned long long* counts) {
#pragma unroll
    for (int op = 0; op < 8; ++op) {
        const uint64_t v = ((op < 4 ? L.c03 : L.c47) >> (16 * (op & 3))) & 0xFFFFull;
        if (v) atomicAdd(counts + op, (unsigned long long)v);
    }
    L.c03 = 0; L.c47 = 0; L.since = 0;
}

template <bool COUNT>
__device__ __forceinline__ void lane_emit(Lane& L, uint32_t s) {
    bool pay = L.pend;
    L.pend = !pay && ((s & 7u) == 5u);
    if (COUNT) {   // every op nibble counts, its payload does not (container.py:485-495)
        if (!pay) {
            const uint64_t inc = 1ull << (16 * (s & 3u));
            if (s & 4u) L.c47 += inc; else L.c03 += inc;
            ++L.since;
        }
        return;
    }
    L.cur = pay ? (L.cur | (s << 4)) : s;
    // shift the 8-byte window down one byte and append the entry on top (after 8
    // appends the first entry sits in the lowest byte, little-endian order); selects
    // instead of a branch on the payload flag, which diverges within a warp
    const bool em = !L.pend;
    const uint32_t nlo = __byte_perm(L.alo, L.ahi, 0x4321), nhi = __byte_perm(L.ahi, L.cur, 0x4321);
    L.alo = em ? nlo : L.alo;
    L.ahi = em ? nhi : L.ahi;
    L.ne += em ? 1u : 0u;
    if (em && (L.ne & 7u) == 0u) {
        if (L.ne & 8u) { L.plo = L.alo; L.phi = L.ahi; }   // first group of a pair: hold it
        else __stcs(reinterpret_cast<uint4*>(L.outp) + ((L.ne >> 4) - 1), make_uint4(L.plo, L.phi, L.alo, L.ahi));
    }
}

__device__ __forceinline__ void lane_finish(Lane& L, const Plan& P, bool failed, bool entropy) {
    if (P.op_counts) lane_flush_counts(L, P.op_counts);
    else if (L.ne & 8u) L.outp[(L.ne >> 3) - 1] = ((uint64_t)L.phi << 32) | L.plo;   // unpaired last group
    if (!P.op_counts && (L.ne & 7u)) {   // partial group: move its entries down to byte 0, zero above
        const uint64_t a = ((uint64_t)L.ahi << 32) | L.alo;
        L.outp[L.ne >> 3] = a >> (8 * (8 - (L.ne & 7u)));
    }
    csv_stream_result r;
    r.n_entries = L.ne;
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
template <bool ENTROPY, bool COUNT>
__device__ bool lane_init(Lane& L, const VolView& V, const Plan& P, uint64_t item) {
    uint64_t r = item < P.n ? item : item - P.n;
    int s = item < P.n ? 1 : 0;           // detail streams first (longest chains)
    uint64_t w = 2 * r + s;               // result / region index
    L.item = w;
    L.alo = 0; L.ahi = 0; L.ne = 0; L.pend = false; L.cur = 0; L.i = 0; L.slow = false;
    L.x = 0; L.pos = 0; L.len = 0; L.nb = 0; L.buf = 0;
    uint64_t b = req_local(V, P, r);
    int t = req_lod(P, r);
    L.c03 = 0; L.c47 = 0; L.since = 0;
    L.outp = COUNT ? nullptr : reinterpret_cast<uint64_t*>(P.entries + P.eoff[w]);
    bool ok = b < V.nb && t < V.N && !(s == 1 && t != 0);
    L.n = ok ? eff_nibbles(V, b, s) : 0;
    L.lim = ok ? (COUNT ? L.n : stream_limit(V, b, t, s)) : 0;
    L.tbase = (uint32_t)s << 12;
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
    const uint4* aq = reinterpret_cast<const uint4*>(q & ~uintptr_t(15));
    L.cq = __ldg(aq);
    L.nq = __ldg(aq + 1);
    L.qp = aq + 2;
    L.cw = 4;
    for (int skip = (int)((q & 15) >> 2); skip > 0; --skip) (void)lane_next_word(L);
    const int sh = (int)(q & 3);
    L.buf = (uint64_t)bswap32(lane_next_word(L)) << (32 + 8 * sh);
    L.nb = 32 - 8 * sh;
    L.slow = L.x < kStateLower;
    return true;
}

// One symbol; returns false when the lane's item is finished.  With REFILL =
// false the caller guarantees >= 16 buffered bits (pairs of steps after one
// `nb < 32` refill: the refill block then runs on every other step of the warp
// instead of nearly every step, since some lane always needs bytes).
// SLOWCHK = false: the caller has already taken the (rare) first step of a
// stream whose initial state is below 2^23, so no per-step check is needed.
template <bool ENTROPY, bool COUNT, bool REFILL = true, bool SLOWCHK = true>
__device__ __forceinline__ bool lane_step(Lane& L, const Plan& P, const uint32_t* tab) {
    uint32_t s;
    if (ENTROPY) {
        if (REFILL && L.nb < 16) lane_refill(L);
        uint32_t e = tab[L.tbase + (L.x & (kTotalFreq - 1))];
        s = e & 15u;
        uint32_t xn = (e >> 16) * (L.x >> kPrecision) + ((e >> 4) & 0xFFFu);
        if (!SLOWCHK || !L.slow) {
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
            if (!REFILL && L.nb < 16) lane_refill(L);   // the pair's next step reads without a check
        }
    } else {
        s = (L.rawp[L.i >> 1] >> (4 * (L.i & 1))) & 15u;
    }
    lane_emit<COUNT>(L, s);
    if (++L.i == L.lim) {
        lane_finish(L, P, false, ENTROPY);
        return false;
    }
    return true;
}

// Two register budgets: MINB 5 (48 registers, 40 warps/SM) for plans that fill
// several waves (throughput), MINB 3 (55 registers) for smaller plans whose time is the
// longest lane's chain (latency): 9.5 vs 10.6 ms on config 3, 1.12 vs 1.17 ms on config 2.
constexpr int K1_MINB_THROUGHPUT = 5;
constexpr int K1_MINB_LATENCY = 3;
// K1f (the rANS lanes of csv_k1fast.cuh) reverses that: at 48 registers its step schedules
// worse than at the ~62 it takes when allowed 64, so multi-wave plans run 4 blocks/SM of the
// 64-register build (config 3: K1 6.05 -> 5.72 ms; config-4 batch K1 3.3 -> 2.4 ms)
constexpr int K1F_MINB_MULTI = 4;
constexpr uint64_t kK1TinyBlocks = 8;   // plans of <= 8 K1 blocks (<= 1024 requests) use the latency-optimised steps
template <bool ENTROPY, bool COUNT, int MINB>
__global__ void __launch_bounds__(K1_THREADS, MINB) k1_streams(VolView V, Plan P, unsigned long long* counter) {
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
                if (my < total) has = lane_init<ENTROPY, COUNT>(L, V, P, my);
                else done = true;
            }
        }
        if (__all_sync(FULL, done)) break;
        if (has) {
            if (ENTROPY) {
                if (L.slow && !lane_step<ENTROPY, COUNT, true, true>(L, P, tab)) has = false;
                if (has) {
#pragma unroll 8
                    for (int u = 0; u < 32; ++u) {
                        if (L.nb < 32) lane_refill(L);
                        if (!lane_step<ENTROPY, COUNT, false, false>(L, P, tab)) { has = false; break; }
                        if (!lane_step<ENTROPY, COUNT, false, false>(L, P, tab)) { has = false; break; }
                    }
                }
            } else {
#pragma unroll 4
                for (int u = 0; u < 32; ++u) {
                    if (!lane_step<ENTROPY, COUNT>(L, P, tab)) { has = false; break; }
                }
            }
            if (COUNT && has && L.since > 16000u) lane_flush_counts(L, P.op_counts);
        }
    }
}

#include "csv_k1fast.cuh"

// ============================================================================ K2: replay
// Per-brick working set, sized for LMAX = N - t levels (compile-time):
//   lev  : values of levels t+1..N in Morton order; level N-j at levoffA(j)
//          (16-byte aligned for j >= 1)
//   mask : 2 x W words, active-parent bitmask ping-pong
//   wpre : W+1 words, exclusive popcount prefix of the parent mask
//   ipb  : per active parent (by rank) palette-advance prefix, level-relative
//   list : per active parent (by rank) its Morton index
//   pend : one bit per child of the level (or final tile): "chain, value pending"
//   pax  : two bits per child: the chain's axis
//   buf  : final-level tile of 4096 children (16^3 voxels) staged before the HBM write
// LMAX <= 5 lives in shared memory with 16-bit ipb/list (<= 4096 parents and
// <= 32768 entries per level); LMAX 6, 7 (b = 64, 128 at fine LODs) use a
// per-CTA global workspace with 32-bit indices.
__host__ __device__ constexpr uint32_t levoffA(int j) {
    return j == 0 ? 0u : 4u + ((1u << (3 * j)) - 8u) / 7u;
}
struct Layout {
    uint32_t lev, mask, wpre, ipb, list, pend, pax, buf, words, W;   // offsets in u32 units
};
__host__ __device__ constexpr Layout make_layout(int L, int idx_bytes) {
    Layout Y{};
    uint32_t nlev = levoffA(L);
    uint32_t maxP = 1u << (3 * (L - 1));              // parents at level t+1 (= children of level t+2)
    uint32_t ts = L >= 4 ? 4096u : (1u << (3 * L));   // final-level tile (children), k2_replay only
    uint32_t pbits = 8u * maxP;                       // children of the final level
    Y.W = (maxP + 31) / 32;
    Y.lev = 0;
    Y.mask = (nlev + 3) & ~3u;
    Y.wpre = Y.mask + 2 * Y.W;
    Y.ipb = (Y.wpre + Y.W + 1 + 3) & ~3u;
    uint32_t idx_words = (maxP * idx_bytes + 15) / 16 * 4;
    Y.list = Y.ipb + idx_words;
    Y.pend = Y.list + idx_words;
    Y.pax = Y.pend + (pbits + 31) / 32;
    Y.buf = (Y.pax + (maxP > ts ? maxP : ts) / 16 + 3) & ~3u;
    Y.words = idx_bytes == 2 ? Y.buf : Y.buf + ts;    // k2_fast (16-bit) has no tile buffer
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
    uint32_t scan2[K2_WARPS + 1];
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

// Raster placement of one brick at LOD t (replaces morton_to_grid + slice
// assignment, container.py:465-468).  Fast bricks (fully inside crop and slab,
// even row pitch, 15-bit Morton indices) address voxels through the per-CTA
// LUT with 32-bit offsets from `base`; edge bricks take the general path.
struct Raster {
    uint32_t* base;     // voxel (ox, oy, oz) of the slab
    int64_t ox, oy, oz; // brick origin in LOD-t voxels
    bool fast;
};

__device__ __forceinline__ void write_result(const Plan& P, uint64_t r, int st, int stream, int64_t pos,
                                             int64_t ci, int64_t di) {
    if (P.res && threadIdx.x == 0) {
        csv_result o;
        o.status = st; o.stream = stream; o.pos = pos; o.ci = ci; o.di = di;
        P.res[r] = o;
    }
}

// Evaluation of one child (lane-per-child; 8 consecutive lanes = one parent).
// Returns the value for every op whose source is already final; sets *chain
// for an even-coordinate reuse whose -1 neighbour has an active parent (its
// value is produced at this level, codec.py:422-423) and reports that
// neighbour in *nm_out.  Op-specific errors go to *st.
struct ChildCtx {
    const uint32_t* plev;
    const uint32_t* pmask;
    const uint32_t* pal;
    uint32_t plen;
    int32_t ipbase;
    uint32_t Mx, My, Mz;
};

__device__ __forceinline__ uint32_t eval_child(const ChildCtx& C, uint32_t q, uint32_t c, uint32_t e, int32_t ipq,
                                               uint32_t pam, int lane, int* st, bool* chain, uint32_t* nm_out,
                                               uint32_t* axis) {
    const uint32_t op = e & 7u;
    const uint32_t j = (q << 3) | c;
    *st = 0;
    *chain = false;
    if (op - 1u < 3u) {
        const uint32_t a = op - 1u;
        const uint32_t M = a == 0 ? C.Mx : (a == 1 ? C.My : C.Mz);
        const uint32_t part = j & M;
        *axis = a;
        if ((c >> a) & 1u) {   // odd: the +1 neighbour is decoded later -> its parent's value
            *st = part == M ? CSV_ST_BAD_NEIGHBOR : 0;
            return C.plev[((((part | ~M) + 1u) & M) | (j & ~M)) >> 3];
        }
        *st = part == 0 ? CSV_ST_BAD_NEIGHBOR : 0;    // even: the -1 neighbour, same level
        const uint32_t nm = ((part - 1u) & M) | (j & ~M);
        const uint32_t qn = nm >> 3;
        *nm_out = nm;
        *chain = *st == 0 && ((C.pmask[qn >> 5] >> (qn & 31)) & 1u);
        return C.plev[qn];                                  // final when that parent is inactive
    }
    if (op - 4u < 3u) {
        const int32_t ip = ipq + __popc(pam & (0xFFu << (lane & 24)) & ((1u << lane) - 1u));
        int32_t idx = op == 4u ? ip : (op == 5u ? ip - (int32_t)(e >> 4) - 1 : ip + 1);
        *st = idx < 0 ? CSV_ST_DELTA_RANGE : (idx >= (int32_t)C.plen ? CSV_ST_PALETTE_RANGE : 0);
        idx = min(max(idx, 0), (int32_t)C.plen - 1);
        return __ldg(C.pal + idx);
    }
    return C.plev[q];
}

__device__ __forceinline__ void record_error(K2Shared& S, uint32_t ent, uint32_t nvalid, uint32_t e, bool leaf, int st) {
    const uint32_t op = e & 7u;
    if (ent < nvalid && (op == 7u || (leaf && (e & 8u)) || st)) {
        const unsigned long long kk = op == 7u ? ekey(ent, 0, CSV_ST_BAD_OP)
                                               : (leaf && (e & 8u)) ? ekey(ent, 1, CSV_ST_LEAF_STOP) : ekey(ent, 2, st);
        atomicMin(&S.errkey, kk);
    }
}

// Raster address of final-level child j (brick-local Morton at LOD t); nullptr if cropped.
__device__ __forceinline__ uint32_t* raster_of(const Raster& R, const Plan& P, uint32_t j) {
    const uint32_t x = compact3(j), y = compact3(j >> 1), z = compact3(j >> 2);
    if (R.fast) return R.base + ((uint32_t)z * (uint32_t)(P.cx * P.cy) + (uint32_t)y * (uint32_t)P.cx + x);
    const int64_t gx = R.ox + x, gy = R.oy + y, gz = R.oz + z;
    if (gz < P.z_begin || gz >= P.z_end || gy >= P.cy || gx >= P.cx) return nullptr;
    return P.out + ((gz - P.z_begin) * P.cy + gy) * P.cx + gx;
}

template <int MODE, int LMAX>
#ifndef K2_MINB
#define K2_MINB 4
#endif
__global__ void __launch_bounds__(K2_THREADS, LMAX <= 5 ? K2_MINB : 1)
k2_replay(VolView V, Plan P, uint32_t* gws, uint64_t ws_stride) {
    constexpr bool SMEM = LMAX <= 5;
    using IdxT = typename std::conditional<SMEM, uint16_t, uint32_t>::type;
    constexpr Layout Y = make_layout(LMAX, sizeof(IdxT));
    extern __shared__ __align__(16) uint32_t dsm[];
    __shared__ K2Shared S;
    uint32_t* ws;
    if constexpr (SMEM) ws = dsm;
    else ws = gws + blockIdx.x * ws_stride;
    uint32_t* const lev = ws + Y.lev;
    uint32_t* const mask0 = ws + Y.mask;
    uint32_t* const wpre = ws + Y.wpre;
    IdxT* const ipb = reinterpret_cast<IdxT*>(ws + Y.ipb);
    IdxT* const list = reinterpret_cast<IdxT*>(ws + Y.list);
    uint32_t* const pend = ws + Y.pend;
    uint32_t* const pax = ws + Y.pax;
    uint32_t* const buf = ws + Y.buf;
    const int N = V.N;
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    for (uint64_t r = blockIdx.x; r < P.n; r += gridDim.x) {
        const uint64_t b = req_local(V, P, r);
        const int t = req_lod(P, r);
        if (b >= V.nb || t > N) { write_result(P, r, -1, 0, 0, 0, 0); continue; }
        if (t < N && N - t > LMAX) continue;            // served by a larger instantiation
        if (!SMEM && N - t <= 5) continue;
        uint32_t* out_m = MODE == OUT_MORTON ? P.out + P.dst[r] : nullptr;
        const uint32_t plen = V.pal_len[b];
        const uint32_t* pal = V.palette + V.pal_off[b];
        Raster R{};
        if (MODE == OUT_RASTER) {
            const uint64_t gb = V.brick_begin + b;
            const int64_t side = 1ll << (N - t);
            R.ox = (int64_t)(gb % V.gx) * side;
            R.oy = (int64_t)((gb / V.gx) % V.gy) * side;
            R.oz = (int64_t)(gb / (V.gx * V.gy)) * side;
            R.base = P.out + ((R.oz - P.z_begin) * P.cy + R.oy) * P.cx + R.ox;
            R.fast = R.ox + side <= P.cx && R.oy + side <= P.cy && R.oz >= P.z_begin && R.oz + side <= P.z_end &&
                     (uint64_t)P.cx * P.cy * side < (1ull << 32);
        }
        if (LMAX == 6 && P.k2w6 && plen <= e8::kMarkPal) continue;   // decoded by K2w<6>
        if (plen == 0) { write_result(P, r, CSV_ST_EMPTY_PALETTE, 0, 0, 0, 0); continue; }
        if (t == N) {   // coarsest LOD: palette[0] (codec.py:514-516, container.py:178-182)
            if (threadIdx.x == 0) {
                uint32_t* p = MODE == OUT_MORTON ? out_m : raster_of(R, P, 0);
                if (p) *p = __ldg(pal);
            }
            write_result(P, r, 0, 0, 0, 0, 0);
            continue;
        }
        const uint32_t nc_raw = V.c_nib[b], nd_raw = t == 0 ? V.d_nib[b] : 0;
        const uint32_t nc = eff_nibbles(V, b, 0), nd = t == 0 ? eff_nibbles(V, b, 1) : 0;
        if (V.entropy) {   // state-word checks come first (codec.py:331-351)
            if (nc_raw > 0 && V.c_bytes[b] < 4) { write_result(P, r, CSV_ST_UNDERRUN, 0, 0, 0, 0); continue; }
            if (t == 0 && nd_raw > 0 && V.d_bytes[b] < 4) { write_result(P, r, CSV_ST_UNDERRUN, 1, 0, 0, 0); continue; }
        }
        const csv_stream_result src = P.sres[2 * r], srd = P.sres[2 * r + 1];
        const uint64_t eo0 = P.eoff[2 * r], eo1 = P.eoff[2 * r + 1], eo2 = P.eoff[2 * r + 2];
        const bool trivial = (uint64_t)nc + nd == 0;     // relevant == 0: fill palette[0] (codec.py:353-358)
        if (threadIdx.x == 0) {
            lev[0] = __ldg(pal);      // root (codec.py:353)
            mask0[0] = trivial ? 0u : 1u;
            S.errkey = ~0ull;
        }
        __syncthreads();
        uint32_t cur_c = 0, cur_d = 0;
        uint64_t pd_c = 0, pd_d = 0;
        int32_t ipbase = 0;
        int cur = 0;
        bool failed = false;
        for (int l = N; l > t; --l) {
            const bool leaf = l == 1;
            const bool final_level = (l - 1 == t);
            const uint32_t Pn = 1u << (3 * (N - l));
            const uint32_t W = (Pn + 31) >> 5;
            uint32_t* const pmask = mask0 + cur * Y.W;
            uint8_t* const cmask = reinterpret_cast<uint8_t*>(mask0 + (cur ^ 1) * Y.W);
            const csv_stream_result sr = leaf ? srd : src;
            const uint32_t e0 = leaf ? cur_d : cur_c;
            const uint8_t* const Eb = P.entries + (leaf ? eo1 : eo0);   // this stream's entry bytes
            const uint32_t ecap = (uint32_t)((leaf ? eo2 : eo1) - (leaf ? eo1 : eo0));
            uint32_t* const clev = lev + levoffA(N - l + 1);
            const int cbits = N - l + 1;
            ChildCtx C;
            C.plev = lev + levoffA(N - l);
            C.pmask = pmask;
            C.pal = pal;
            C.plen = plen;
            C.ipbase = ipbase;
            C.Mx = axis_mask(0, cbits); C.My = axis_mask(1, cbits); C.Mz = axis_mask(2, cbits);
            // (A) rank prefix of active parents
            for (uint32_t i = threadIdx.x; i < W; i += blockDim.x) {
                uint32_t mw = pmask[i];
                if (Pn < 32) mw &= (1u << Pn) - 1u;
                pmask[i] = mw;
                wpre[i] = __popc(mw);
            }
            __syncthreads();
            const uint32_t nact = block_scan_inplace(wpre, W, S);
            // (B) active list + palette-advance counts per active parent
            for (uint32_t i = threadIdx.x; i < W; i += blockDim.x) {
                uint32_t mw = pmask[i], rk = wpre[i];
                while (mw) {
                    const int bit = __ffs(mw) - 1;
                    mw &= mw - 1;
                    list[rk++] = (IdxT)(32 * i + bit);
                }
            }
            uint64_t pdl = 0;
            for (uint32_t i = threadIdx.x; i < nact; i += blockDim.x) {
                const uint32_t off = e0 + 8 * i;
                const uint64_t w = off + 8 <= ecap ? __ldg(reinterpret_cast<const uint64_t*>(Eb + off)) : 0ull;
                ipb[i] = (IdxT)__popcll(op_eq(w, 6));
                pdl += __popcll(op_eq(w, 5));
            }
            if (leaf) pd_d += pdl; else pd_c += pdl;
            __syncthreads();
            const uint32_t tot_pa = block_scan_inplace(ipb, nact, S);
            const uint32_t nvalid = sr.n_entries;
            if (threadIdx.x == 0 && (uint64_t)e0 + 8ull * nact > nvalid)
                atomicMin(&S.errkey, ekey(nvalid, 0, EK_UNDERRUN_NV));
            // tiles: the whole child level for intermediate levels (shared level
            // array), 4096-child Morton tiles staged in `buf` for the final level
            const uint32_t Cn = 8 * Pn;
            const uint32_t TS = final_level ? (Cn < 4096u ? Cn : 4096u) : Cn;
            const uint32_t NT = Cn / TS;
            const uint32_t PT = TS / 8;                   // parents per tile
            for (uint32_t o = 0; o < NT; ++o) {
                uint32_t* const dst = final_level ? buf : clev;
                const uint32_t q0 = o * PT, q1 = q0 + PT;
                const uint32_t j0 = 8 * q0;
                const uint32_t r0 = wpre[q0 >> 5] + __popc(pmask[q0 >> 5] & ((1u << (q0 & 31)) - 1u));
                const uint32_t r1 = q1 >= Pn ? nact : wpre[q1 >> 5] + __popc(pmask[q1 >> 5] & ((1u << (q1 & 31)) - 1u));
                for (uint32_t i = threadIdx.x; i < TS / 32; i += blockDim.x) pend[i] = 0;
                for (uint32_t i = threadIdx.x; i < TS / 16; i += blockDim.x) pax[i] = 0;
                __syncthreads();
                // (C1) children of active parents in this tile, one lane each
                for (uint32_t kb = 8 * r0 + (threadIdx.x - lane); kb < 8 * r1; kb += blockDim.x) {
                    const uint32_t k = kb + lane;
                    const bool valid = k < 8 * r1;
                    const uint32_t rk = k >> 3;
                    const uint32_t c = k & 7;
                    const uint32_t q = valid ? (uint32_t)list[rk] : q0;
                    const uint32_t ent = e0 + k;
                    const uint32_t e = (valid && ent < ecap) ? (uint32_t)__ldg(Eb + ent) : 0u;
                    const uint32_t pam = __ballot_sync(FULL, valid && (e & 7u) == 6u);
                    if (!final_level) {
                        const uint32_t nstop = __ballot_sync(FULL, valid && !(e & 8u));
                        if (valid && c == 0) cmask[q] = (uint8_t)(nstop >> (lane & 24));
                    }
                    if (!valid) continue;
                    int st;
                    bool chain;
                    uint32_t nm = 0, a = 0;
                    uint32_t val = eval_child(C, q, c, e, ipbase + (int32_t)ipb[rk], pam, lane, &st, &chain, &nm, &a);
                    record_error(S, ent, nvalid, e, leaf, st);
                    const uint32_t jl = ((q << 3) | c) - j0;
                    if (chain && nm < j0) {       // neighbour in an earlier (already stored) tile
                        chain = false;
                        const uint32_t* p = MODE == OUT_MORTON ? out_m + nm : raster_of(R, P, nm);
                        val = p ? *p : 0u;
                    }
                    if (chain) {
                        atomicOr(&pend[jl >> 5], 1u << (jl & 31));
                        atomicOr(&pax[jl >> 4], a << (2 * (jl & 15)));
                    } else {
                        dst[jl] = val;
                    }
                }
                // (C2) inactive parents of this tile: children repeat the parent value
                for (uint32_t q = q0 + threadIdx.x; q < q1; q += blockDim.x) {
                    if ((pmask[q >> 5] >> (q & 31)) & 1u) continue;
                    const uint32_t pv = C.plev[q];
                    reinterpret_cast<uint4*>(dst + 8 * (q - q0))[0] = make_uint4(pv, pv, pv, pv);
                    reinterpret_cast<uint4*>(dst + 8 * (q - q0))[1] = make_uint4(pv, pv, pv, pv);
                    if (!final_level) cmask[q] = 0;
                }
                __syncthreads();
                // (W) same-level chains: walk -1 neighbours (<= 3 hops: each hop makes
                // one more coordinate odd) to the first child whose value is final
                for (uint32_t w = threadIdx.x; w < TS / 32; w += blockDim.x) {
                    uint32_t bits = pend[w];
                    while (bits) {
                        const uint32_t jl = 32 * w + (__ffs(bits) - 1);
                        bits &= bits - 1;
                        uint32_t cl = jl;
                        for (int hop = 0; hop < 4; ++hop) {
                            const uint32_t a = (pax[cl >> 4] >> (2 * (cl & 15))) & 3u;
                            const uint32_t M = a == 0 ? C.Mx : (a == 1 ? C.My : C.Mz);
                            const uint32_t jg = cl + j0;
                            cl = ((((jg & M) - 1u) & M) | (jg & ~M)) - j0;
                            if (!((pend[cl >> 5] >> (cl & 31)) & 1u)) break;
                        }
                        dst[jl] = dst[cl];
                    }
                }
                __syncthreads();
                if (!final_level) continue;
                // (T) stream the tile to HBM: Morton pool (linear) or raster rows
                if (MODE == OUT_MORTON) {
                    uint32_t* d = out_m + (size_t)TS * o;
                    const bool al = (reinterpret_cast<uintptr_t>(d) & 15) == 0;
                    for (uint32_t i = threadIdx.x; i < TS / 4; i += blockDim.x) {
                        const uint4 v = reinterpret_cast<const uint4*>(buf)[i];
                        if (al) reinterpret_cast<uint4*>(d)[i] = v;
                        else { d[4 * i] = v.x; d[4 * i + 1] = v.y; d[4 * i + 2] = v.z; d[4 * i + 3] = v.w; }
                    }
                } else {
                    const int tb = (31 - __clz(TS)) / 3;          // log2 of the tile side
                    const uint32_t ts = 1u << tb;
                    const uint32_t tx = compact3(o) << tb, ty = compact3(o >> 1) << tb, tz = compact3(o >> 2) << tb;
                    const uint32_t xs = ts >= 4 ? 4u : ts;         // voxels per item along x
                    const uint32_t ipr = ts / xs;                   // items per row
                    for (uint32_t i = threadIdx.x; i < TS / xs; i += blockDim.x) {
                        const uint32_t x = (i % ipr) * xs, y = (i / ipr) % ts, z = i / (ipr * ts);
                        const uint32_t myz = (spread3_u32(y) << 1) | (spread3_u32(z) << 2);
                        uint32_t v[4];
#pragma unroll
                        for (int k = 0; k < 4; ++k) v[k] = k < (int)xs ? buf[myz | spread3_u32(x + k)] : 0u;
                        if (R.fast) {
                            uint32_t* p = R.base + ((tz + z) * (uint32_t)(P.cx * P.cy) + (ty + y) * (uint32_t)P.cx + tx + x);
                            if (xs == 4 && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
                                *reinterpret_cast<uint4*>(p) = make_uint4(v[0], v[1], v[2], v[3]);
                            } else {
                                for (uint32_t k = 0; k < xs; ++k) p[k] = v[k];
                            }
                        } else {
                            const int64_t gz = R.oz + tz + z, gy = R.oy + ty + y;
                            if (gz < P.z_begin || gz >= P.z_end || gy >= P.cy) continue;
                            uint32_t* row = P.out + ((gz - P.z_begin) * P.cy + gy) * P.cx;
                            for (uint32_t k = 0; k < xs; ++k) {
                                const int64_t gx = R.ox + tx + x + k;
                                if (gx < P.cx) row[gx] = v[k];
                            }
                        }
                    }
                }
                __syncthreads();
            }
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
            if (leaf) cur_d = e0 + 8 * nact; else cur_c = e0 + 8 * nact;
            ipbase += (int32_t)tot_pa;
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

#include "csv_replay_fast.cuh"
#include "csv_replay_warp.cuh"

// Coarsest-LOD raster (t == N): one voxel per brick.
__global__ void k_root_raster(VolView V, Plan P) {
    uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (r >= P.n) return;
    uint64_t b = P.first + r;
    if (b >= V.nb) return;
    uint32_t plen = V.pal_len[b];
    if (P.res) {
        csv_result o{plen == 0 ? CSV_ST_EMPTY_PALETTE : 0, 0, 0, 0, 0};
        P.res[r] = o;
    }
    if (plen == 0) return;
    uint64_t gb = V.brick_begin + b;
    int64_t x = gb % V.gx, y = (gb / V.gx) % V.gy, z = gb / (V.gx * V.gy);
    if (x < P.cx && y < P.cy && z >= P.z_begin && z < P.z_end)
        P.out[((z - P.z_begin) * P.cy + y) * P.cx + x] = V.palette[V.pal_off[b]];
}

// ============================================================================ host launchers
template <bool E, bool COUNT, int MINB>
static void launch_k1_variant(const VolView& V, const Plan& P, unsigned long long* counter, int nsm, uint64_t blocks,
                              cudaStream_t st) {
    static int per_sm = 0;                              // resident blocks per SM (registers / 32 KB tables)
    if (per_sm == 0) {
        int b = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k1_streams<E, COUNT, MINB>, K1_THREADS, 0) != cudaSuccess ||
            b < 1)
            b = MINB;
        per_sm = b;
    }
    const uint64_t cap = (uint64_t)nsm * per_sm;        // persistent blocks: one resident wave
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    k1_streams<E, COUNT, MINB><<<(unsigned)blocks, K1_THREADS, 0, st>>>(V, P, counter);
}

template <int MINB, bool LAT = false>
static unsigned launch_k1f_variant(const VolView& V, const Plan& P, unsigned long long* counter, int nsm, uint64_t blocks,
                                   cudaStream_t st) {
    static int per_sm = 0;
    if (per_sm == 0) {
        int b = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k1_fast<MINB, LAT>, K1_THREADS, 0) != cudaSuccess || b < 1)
            b = MINB;
        per_sm = b;
    }
    const uint64_t cap = (uint64_t)nsm * per_sm;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    k1_fast<MINB, LAT><<<(unsigned)blocks, K1_THREADS, 0, st>>>(V, P, counter);
    return (unsigned)blocks;
}

static bool k1_old() {
    static int v = -1;
    if (v < 0) { const char* e = getenv("CSVGPU_K1"); v = (e && strcmp(e, "old") == 0) ? 1 : 0; }
    return v == 1;
}

// returns K1f's grid (0 for k1_streams)
template <bool E, bool COUNT = false>
static unsigned launch_k1(const VolView& V, const Plan& P, unsigned long long* counter, int nsm, cudaStream_t st) {
    const uint64_t items = 2 * P.n;
    const uint64_t want = (items + 31) / 32;           // warps needed at one item per lane
    const uint64_t blocks = (want + K1_THREADS / 32 - 1) / (K1_THREADS / 32);
    if (E && !COUNT && V.fast_tab && !k1_old()) {
        if (blocks > (uint64_t)nsm * K1_MINB_LATENCY) return launch_k1f_variant<K1F_MINB_MULTI>(V, P, counter, nsm, blocks, st);
        if (blocks > kK1TinyBlocks) return launch_k1f_variant<K1_MINB_LATENCY>(V, P, counter, nsm, blocks, st);
        return launch_k1f_variant<K1_MINB_LATENCY, true>(V, P, counter, nsm, blocks, st);   // per-brick calls
    }
    if (blocks > (uint64_t)nsm * K1_MINB_LATENCY)      // more than one wave of the latency variant
        launch_k1_variant<E, COUNT, K1_MINB_THROUGHPUT>(V, P, counter, nsm, blocks, st);
    else
        launch_k1_variant<E, COUNT, K1_MINB_LATENCY>(V, P, counter, nsm, blocks, st);
    return 0;
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
template <int MODE, int L>
static void k2_launch_one(unsigned grid, size_t smem, const VolView& V, const Plan& P, cudaStream_t st) {
    cudaFuncSetAttribute(k2_fast<MODE, L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k2_fast<MODE, L><<<grid, K2_THREADS, smem, st>>>(V, P);
}
template <int MODE>
static void k2_launch_mode(int L, unsigned grid, size_t smem, const VolView& V, const Plan& P, cudaStream_t st) {
    switch (L) {
        case 1: k2_launch_one<MODE, 1>(grid, smem, V, P, st); break;
        case 2: k2_launch_one<MODE, 2>(grid, smem, V, P, st); break;
        case 3: k2_launch_one<MODE, 3>(grid, smem, V, P, st); break;
        case 4: k2_launch_one<MODE, 4>(grid, smem, V, P, st); break;
        default: k2_launch_one<MODE, 5>(grid, smem, V, P, st); break;
    }
}
// K2w: persistent warps (K2W_WARPS per CTA), as many CTAs as fit per SM
// per_sm > 0: the overlap launch (warps per SM beside K1), 0: as many warps as fit, < 0: only
// the one-time set-up (function attributes, occupancy query -- which also loads the kernel).
template <int MODE, int L, typename IT, bool Q = false>
static void k2w_launch_one(const VolView& V, const Plan& P, unsigned long long* counter, int nsm, cudaStream_t st,
                           int per_sm = 0) {
    const size_t smem = (size_t)K2W_WARPS * wk::make_wlayout(L, sizeof(IT)).bytes;
    static int occ = 0;
    if (!occ) {
        cudaFuncSetAttribute(k2_warp<MODE, L, IT, Q>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k2_warp<MODE, L, IT, Q>, 32 * K2W_WARPS, smem);
        if (occ < 1) occ = 1;
        if (occ * K2W_WARPS > 32) occ = 32 / K2W_WARPS;   // wscratch: 64 warp slots per SM, the upper half for the overlap launch
        if (L >= 6 && occ * K2W_WARPS > kK2W6MaxWarpsPerSM) occ = kK2W6MaxWarpsPerSM / K2W_WARPS;   // wscratch6 slots
    }
    if (per_sm < 0) return;   // prepare only: attributes set and the kernel loaded before K1 runs
    uint64_t want = (P.n + K2W_WARPS - 1) / K2W_WARPS;
    uint64_t grid = (uint64_t)nsm * (per_sm > 0 ? (uint64_t)per_sm / K2W_WARPS : (uint64_t)occ);
    if (grid > want) grid = want;
    if (grid < 1) grid = 1;
    k2_warp<MODE, L, IT, Q><<<(unsigned)grid, 32 * K2W_WARPS, smem, st>>>(V, P, counter);
}
template <int MODE, typename IT, bool Q = false>
static void k2w_launch_mode(int L, const VolView& V, const Plan& P, unsigned long long* counter, int nsm, cudaStream_t st,
                            int per_sm = 0) {
    switch (L) {
        case 1: k2w_launch_one<MODE, 1, IT, Q>(V, P, counter, nsm, st, per_sm); break;
        case 2: k2w_launch_one<MODE, 2, IT, Q>(V, P, counter, nsm, st, per_sm); break;
        case 3: k2w_launch_one<MODE, 3, IT, Q>(V, P, counter, nsm, st, per_sm); break;
        case 4: k2w_launch_one<MODE, 4, IT, Q>(V, P, counter, nsm, st, per_sm); break;
        default: k2w_launch_one<MODE, 5, IT, Q>(V, P, counter, nsm, st, per_sm); break;
    }
}
// K1 -> K2w overlap: CSVGPU_OVERLAP=0 disables it; CSVGPU_OVL_WARPS overrides the overlap
// launch's warps per SM.  Default 32 (the whole upper half of the wscratch slots): the CTAs
// that do not fit beside K1 queue and take the SMs K1's finished blocks leave, so the
// overlap launch becomes the full-occupancy replay as K1 drains (config-4 batch and the
// config-3 shares measured at 4 / 8 / 12 / 16 / 24 / 32 warps).
static int ovl_warps(uint64_t k1_blocks, int nsm) {
    static int v = -2;
    if (v == -2) {
        const char* e = getenv("CSVGPU_OVERLAP");
        const char* w = getenv("CSVGPU_OVL_WARPS");
        v = (e && strcmp(e, "0") == 0) ? 0 : (w ? atoi(w) : -1);
        if (v < -1) v = 0;
        if (v > 32) v = 32;
    }
    if (v >= 0) return v;
    (void)k1_blocks; (void)nsm;
    return 32;
}
static bool k2w6_disabled() {
    static int v = -1;
    if (v < 0) { const char* e = getenv("CSVGPU_K2W6"); v = (e && strcmp(e, "0") == 0) ? 1 : 0; }
    return v == 1;
}
static bool k2w_disabled() {
    static int v = -1;
    if (v < 0) { const char* e = getenv("CSVGPU_K2"); v = (e && strcmp(e, "cta") == 0) ? 1 : 0; }
    return v == 1;
}

static void launch_k2_smem(int mode, int L, unsigned grid, size_t smem, const VolView& V, const Plan& P, cudaStream_t st) {
    if (mode == OUT_RASTER) k2_launch_mode<OUT_RASTER>(L, grid, smem, V, P, st);
    else k2_launch_mode<OUT_MORTON>(L, grid, smem, V, P, st);
}

cudaError_t run_decode(const VolView& V, Plan P, int mode, uint64_t* sizes_tmp, uint64_t* scan_tmp,
                       unsigned long long* counter, uint32_t* gws, uint64_t gws_stride, int gws_ctas,
                       int nsm, int min_t, cudaStream_t st, cudaEvent_t* ev, const Overlap* ov) {
    if (P.n == 0) return cudaSuccess;
    // K2: shared-memory instantiation for N - t <= 5, global workspace above
    int Ls = V.N - min_t;
    if (Ls > 5) Ls = 5;
    if (Ls < 1) Ls = 1;
    const bool small = 2 * P.n <= (uint64_t)SCAN_ITEMS;
    const bool k2w = V.max_pal <= 65535u && !k2w_disabled();
    // K1 -> K2w overlap for plans K1 runs in one wave (strong-scaling shares, cache fills): K1's
    // long chains leave the SMs idle at the end, so the u8 K2w pass starts on the bricks whose
    // streams are done.  Needs K1f (it publishes the ready queue).  Not for multi-wave plans
    // (the full volume): K1 then fills every SM to the end and the overlap costs 0.3 ms.
    const uint64_t k1_blocks = (2 * P.n + K1_THREADS - 1) / K1_THREADS;
    const int ow = ovl_warps(k1_blocks, nsm);
    const bool ovl = ov && ov->side && ow > 0 && !small && k2w && V.entropy && V.fast_tab && !k1_old() &&
                     k1_blocks > (uint64_t)kK1TinyBlocks && k1_blocks <= (uint64_t)nsm * K1_MINB_THROUGHPUT;
    if (ev) cudaEventRecord(ev[0], st);
    if (small) {
        k_plan_small<<<1, 256, 0, st>>>(V, P, counter);
    } else {
        unsigned nb = (unsigned)((2 * P.n + 255) / 256);
        k_region_sizes<<<nb, 256, 0, st>>>(V, P, sizes_tmp);
        cudaError_t e = run_scan(sizes_tmp, P.eoff, 2 * P.n, scan_tmp, st);
        if (e != cudaSuccess) return e;
        // K1 items, K2w u8 / u16 / 64^3 bricks, ready-queue tail
        cudaMemsetAsync(counter, 0, kCounterSlots * sizeof(unsigned long long), st);
        if (ovl) {   // the region sizes are dead after the scan: per-request counts + ready queue
            P.rcnt = reinterpret_cast<uint32_t*>(sizes_tmp);
            P.rq = P.rcnt + P.n;
            P.rq_tail = counter + 4;
            cudaMemsetAsync(sizes_tmp, 0, 2 * P.n * sizeof(uint32_t), st);
        }
    }
    if (ev) cudaEventRecord(ev[1], st);
    if (ovl) {
        // The overlap launch spins on slots K1 publishes, so K1 must be launched FIRST and
        // no host call may wait for the device in between: with lazy module loading, the
        // first load of a kernel can wait for the running ones, which would wait for K1.
        if (mode == OUT_RASTER) k2w_launch_mode<OUT_RASTER, uint8_t, true>(Ls, V, P, counter + 1, nsm, st, -1);
        else k2w_launch_mode<OUT_MORTON, uint8_t, true>(Ls, V, P, counter + 1, nsm, st, -1);
        cudaEventRecord(ov->fork, st);
    }
    unsigned k1_grid = 0;
    if (ovl) P.k1_started = counter + 5;
    if (V.entropy) k1_grid = launch_k1<true>(V, P, counter, nsm, st);
    else launch_k1<false>(V, P, counter, nsm, st);
    P.k1_started = nullptr;
    if (ovl) {   // overlap launch on the side stream, ordered after the plan, running beside K1
        Plan Po = P;
        Po.wslot0 = (uint32_t)nsm * 32u;
        Po.k1_started = counter + 5;
        Po.k1_grid = k1_grid;
        cudaStreamWaitEvent(ov->side, ov->fork, 0);
        if (mode == OUT_RASTER) k2w_launch_mode<OUT_RASTER, uint8_t, true>(Ls, V, Po, counter + 1, nsm, ov->side, ow);
        else k2w_launch_mode<OUT_MORTON, uint8_t, true>(Ls, V, Po, counter + 1, nsm, ov->side, ow);
        cudaEventRecord(ov->join, ov->side);
    }
    if (ev) cudaEventRecord(ev[2], st);
    if (k2w) {   // palette-index space: u8 pass, then u16 for long palettes
        if (ovl) {   // the rest of the ready queue, at full occupancy once K1 is done
            if (mode == OUT_RASTER) k2w_launch_mode<OUT_RASTER, uint8_t, true>(Ls, V, P, counter + 1, nsm, st);
            else k2w_launch_mode<OUT_MORTON, uint8_t, true>(Ls, V, P, counter + 1, nsm, st);
            cudaStreamWaitEvent(st, ov->join, 0);
        } else if (mode == OUT_RASTER) k2w_launch_mode<OUT_RASTER, uint8_t>(Ls, V, P, counter + 1, nsm, st);
        else k2w_launch_mode<OUT_MORTON, uint8_t>(Ls, V, P, counter + 1, nsm, st);
        if (V.max_pal > e8::kMarkPal) {   // the u8 pass takes palettes of <= 253 labels (markers 253-255)
            if (mode == OUT_RASTER) k2w_launch_mode<OUT_RASTER, uint16_t>(Ls, V, P, counter + 2, nsm, st);
            else k2w_launch_mode<OUT_MORTON, uint16_t>(Ls, V, P, counter + 2, nsm, st);
        }
    } else {
        size_t smem = k2_smem_bytes(Ls);
        unsigned grid = (unsigned)(P.n < 0x7fffffffull ? P.n : 0x7fffffffull);
        launch_k2_smem(mode, Ls, grid, smem, V, P, st);
    }
    if (V.N - min_t >= 6 && P.wscratch6 && !k2w6_disabled()) {   // 64^3 replays with <= 253 labels: K2w<6>
        P.k2w6 = 1;
        if (mode == OUT_RASTER) k2w_launch_one<OUT_RASTER, 6, uint8_t>(V, P, counter + 3, nsm, st);
        else k2w_launch_one<OUT_MORTON, 6, uint8_t>(V, P, counter + 3, nsm, st);
    }
    if (V.N - min_t > 5 && gws) {
        unsigned g = (unsigned)(P.n < (uint64_t)gws_ctas ? P.n : (uint64_t)gws_ctas);
        if (V.N - min_t == 6) {
            if (mode == OUT_RASTER) k2_replay<OUT_RASTER, 6><<<g, K2_THREADS, 0, st>>>(V, P, gws, gws_stride);
            else k2_replay<OUT_MORTON, 6><<<g, K2_THREADS, 0, st>>>(V, P, gws, gws_stride);
        } else {
            if (mode == OUT_RASTER) k2_replay<OUT_RASTER, 7><<<g, K2_THREADS, 0, st>>>(V, P, gws, gws_stride);
            else k2_replay<OUT_MORTON, 7><<<g, K2_THREADS, 0, st>>>(V, P, gws, gws_stride);
        }
    }
    if (ev) cudaEventRecord(ev[3], st);
    return cudaGetLastError();
}

cudaError_t run_root_raster(const VolView& V, Plan P, cudaStream_t st) {
    unsigned nb = (unsigned)((P.n + 255) / 256);
    if (nb == 0) return cudaSuccess;
    k_root_raster<<<nb, 256, 0, st>>>(V, P);
    return cudaGetLastError();
}

// stats(): K1 in count mode over every brick of the volume (no entry stores)
cudaError_t run_op_counts(const VolView& V, Plan P, unsigned long long* counter, int nsm, cudaStream_t st) {
    if (P.n == 0) return cudaSuccess;
    cudaMemsetAsync(counter, 0, sizeof(unsigned long long), st);
    if (V.entropy) launch_k1<true, true>(V, P, counter, nsm, st);
    else launch_k1<false, true>(V, P, counter, nsm, st);
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
