// csv_encode.cu -- B200 (sm_100a) encoder for the CSV1 format
// and the synthetic Voronoi volume generator used for the large benchmark configs.
//
// Byte-identical to the reference compress_volume (container.py:374-453):
//  E1  pyramid      : per-brick mode-of-8 with first-occurrence ties + constant
//                     flags (pyramid.py:43-78), levels 1..N in shared memory,
//                     level 0 read straight from the raster volume (edge clamp =
//                     np.pad mode="edge", container.py:352-366).
//  E2  operations   : every child's reuse op (R_p, R_x, R_y, R_z) is decided in
//                     parallel (codec.py:150-181); only children needing a palette
//                     op go to an ordered list, which ONE warp replays serially
//                     with a 32-lane register ring of the palette tail (P_0 /
//                     P_delta lookback of 16 via ballot, P_a append, codec.py:182-198).
//  E3  rANS lanes   : one lane per stream encodes in reverse (rans.py:120-137).
//  E4  assembly     : sizes scanned, blobs and 44-byte directory rows written in
//                     brick order (container.py:424-445).
#include <cstdio>
#include <cstring>
#include <cmath>
#include <string>
#include <vector>
#include <algorithm>
#include <mutex>
#include <chrono>
#include <cstdlib>
#include "csv_device.cuh"

namespace csv {

constexpr int E_THREADS = 256;

struct EncView {
    const void* vol;
    int width;                 // 16 or 32 (element size of vol)
    int64_t X, Y, Z;
    int N;
    int64_t gx, gy, gz;
    const uint32_t* list;      // chunk brick list (global indices) or nullptr
    uint64_t b0, nb;           // chunk = b0 + [0, nb) when list == nullptr
    uint8_t* ent;              // entries slots
    uint64_t ent_stride;       // bytes per brick
    uint32_t ent_doff;         // detail entries offset inside a slot
    uint32_t* need;            // need list slots (pairs), reused for encoded bytes
    uint64_t need_stride;      // u32 per brick
    uint32_t* pal;
    uint64_t pal_stride;       // u32 per brick
    uint32_t* cnt;             // 8 u32 per brick
    unsigned long long* hist;  // [2][16] or nullptr
    uint32_t* ws;              // global workspace (N == 7)
    uint64_t ws_stride;
};

__device__ __forceinline__ uint64_t enc_brick(const EncView& E, uint64_t i) {
    return E.list ? (uint64_t)E.list[i] : E.b0 + i;
}


__device__ __forceinline__ uint32_t voxel(const EncView& E, int64_t x, int64_t y, int64_t z) {
    x = x < E.X ? x : E.X - 1;
    y = y < E.Y ? y : E.Y - 1;
    z = z < E.Z ? z : E.Z - 1;
    uint64_t idx = ((uint64_t)z * E.Y + y) * E.X + x;
    return E.width == 16 ? (uint32_t)reinterpret_cast<const uint16_t*>(E.vol)[idx]
                         : reinterpret_cast<const uint32_t*>(E.vol)[idx];
}

// mode of 8 with first-occurrence ties (pyramid.py:43-55); also "all equal"
__device__ __forceinline__ uint32_t mode_first8(const uint32_t* v, bool* uniform) {
    int c0 = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) c0 += v[j] == v[0];
    *uniform = c0 == 8;
    if (c0 >= 4) return v[0];   // no other label can exceed it, and ties go to the first occurrence
    int best = 0, bestc = c0;
#pragma unroll
    for (int k = 1; k < 8; ++k) {
        int cnt = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) cnt += v[j] == v[k];
        if (cnt > bestc) { bestc = cnt; best = k; }
    }
    return v[best];
}

struct EncLayout { uint32_t lev, cst, mask, wpre, nmask, words; };
__host__ __device__ inline EncLayout enc_layout(int N) {
    EncLayout Y;
    uint32_t nlev = 0;
    for (int j = 0; j < N; ++j) nlev += 1u << (3 * j);        // levels N..1
    uint32_t maxP = 1u << (3 * (N - 1));                       // parents at level 1
    uint32_t W = (maxP + 31) / 32;
    Y.lev = 0;
    Y.cst = nlev;                                              // bytes: nlev, in words (nlev+3)/4
    Y.mask = Y.cst + (nlev + 3) / 4;
    Y.wpre = Y.mask + W;
    Y.nmask = Y.wpre + W + 1;                                  // bytes: per parent, its palette-needing children
    Y.words = Y.nmask + (maxP + 3) / 4;
    return Y;
}

struct EncShared {
    uint32_t scan[E_THREADS / 32 + 1];
    uint32_t hist[32];
    uint32_t misc[8];
};

__device__ uint32_t eblock_scan_inplace(uint32_t* arr, uint32_t n, EncShared& S) {
    // exclusive in-place scan (single warp walks warp totals)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, NW = E_THREADS / 32;
    uint32_t per = (n + NW - 1) / NW;
    uint32_t lo = wid * per, hi = min(n, lo + per);
    uint32_t sum = 0;
    for (uint32_t i = lo + lane; i < hi; i += 32) sum += arr[i];
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) S.scan[wid] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (int w = 0; w < NW; ++w) { uint32_t v = S.scan[w]; S.scan[w] = run; run += v; }
        S.scan[NW] = run;
    }
    __syncthreads();
    uint32_t carry = S.scan[wid];
    for (uint32_t c0 = lo; c0 < hi; c0 += 32) {
        uint32_t i = c0 + lane;
        uint32_t v = i < hi ? arr[i] : 0, inc = v;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += u;
        }
        if (i < hi) arr[i] = carry + inc - v;
        carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    uint32_t tot = S.scan[NW];
    __syncthreads();
    return tot;
}

// E1 + E2: one CTA per brick.
template <bool SMEM>
__global__ void __launch_bounds__(E_THREADS) e12_bricks(EncView E) {
    extern __shared__ __align__(16) uint32_t dsm[];
    __shared__ EncShared S;
    const int N = E.N;
    const EncLayout Y = enc_layout(N);
    uint32_t* ws = SMEM ? dsm : E.ws + blockIdx.x * E.ws_stride;
    const uint64_t i = blockIdx.x;
    if (i >= E.nb) return;
    const uint64_t gb = enc_brick(E, i);
    const int64_t bx = gb % E.gx, by = (gb / E.gx) % E.gy, bz = gb / (E.gx * E.gy);
    const int64_t side = 1ll << N;
    const int64_t ox = bx * side, oy = by * side, oz = bz * side;
    uint32_t* lev = ws + Y.lev;
    uint8_t* cst = reinterpret_cast<uint8_t*>(ws + Y.cst);
    uint32_t* pmask = ws + Y.mask;
    uint32_t* wpre = ws + Y.wpre;
    // ---- E1: level 1 from the raster volume, then levels 2..N
    {
        const uint32_t P1 = 1u << (3 * (N - 1));
        uint32_t* l1 = lev + levoff(N - 1);
        uint8_t* c1 = cst + levoff(N - 1);
        for (uint32_t m = threadIdx.x; m < P1; m += blockDim.x) {
            int64_t x1 = compact3(m), y1 = compact3(m >> 1), z1 = compact3(m >> 2);
            uint32_t v[8];
#pragma unroll
            for (int c = 0; c < 8; ++c)
                v[c] = voxel(E, ox + 2 * x1 + (c & 1), oy + 2 * y1 + ((c >> 1) & 1), oz + 2 * z1 + (c >> 2));
            bool u;
            l1[m] = mode_first8(v, &u);
            c1[m] = u;
        }
        __syncthreads();
        for (int k = 2; k <= N; ++k) {
            const uint32_t Pk = 1u << (3 * (N - k));
            uint32_t* lk = lev + levoff(N - k);
            uint8_t* ck = cst + levoff(N - k);
            const uint32_t* lc = lev + levoff(N - k + 1);
            const uint8_t* cc = cst + levoff(N - k + 1);
            for (uint32_t m = threadIdx.x; m < Pk; m += blockDim.x) {
                uint32_t v[8];
                bool allc = true;
#pragma unroll
                for (int c = 0; c < 8; ++c) { v[c] = lc[8 * m + c]; allc &= cc[8 * m + c] != 0; }
                bool u;
                lk[m] = mode_first8(v, &u);
                ck[m] = u && allc;
            }
            __syncthreads();
        }
    }
    // ---- E2: reuse ops in parallel, palette-needing children to an ordered list
    uint8_t* ent = E.ent + i * E.ent_stride;
    uint32_t* need = E.need + i * E.need_stride;
    uint32_t cursor[2] = {0, 0};
    uint32_t nneed = 0;
    for (int l = N; l >= 1; --l) {
        const int s = l == 1 ? 1 : 0;
        const uint32_t P = 1u << (3 * (N - l));
        const uint32_t W = (P + 31) >> 5;
        const uint32_t* lp = lev + levoff(N - l);
        const uint8_t* cp = cst + levoff(N - l);
        const uint32_t* lc = l > 1 ? lev + levoff(N - l + 1) : nullptr;
        const uint8_t* cc = l > 1 ? cst + levoff(N - l + 1) : nullptr;
        for (uint32_t w = threadIdx.x; w < W; w += blockDim.x) {
            uint32_t mw = 0;
            for (int b = 0; b < 32; ++b) {
                uint32_t m = 32 * w + b;
                if (m < P && !cp[m]) mw |= 1u << b;
            }
            pmask[w] = mw;
            wpre[w] = __popc(mw);
        }
        __syncthreads();
        const uint32_t nact = eblock_scan_inplace(wpre, W, S);
        (void)nact;
        uint8_t* es = ent + (s ? E.ent_doff : 0);
        const uint32_t e0 = cursor[s];
        const int cbits = N - l + 1;
        const int64_t child_side = 1ll << cbits;
        // pass 1: every active parent's 8 reuse ops (codec.py:150-181); the children that need a
        // palette op are flagged per parent (nmask), their entries completed by the replay
        uint8_t* const nmask = reinterpret_cast<uint8_t*>(ws + Y.nmask);
        for (uint32_t m = threadIdx.x; m < P; m += blockDim.x) {
            uint32_t needmask = 0;
            if ((pmask[m >> 5] >> (m & 31)) & 1u) {
                const uint32_t rk = wpre[m >> 5] + __popc(pmask[m >> 5] & ((1u << (m & 31)) - 1u));
                const uint32_t par = lp[m];
                uint64_t bytes = 0;
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const uint32_t j = (m << 3) | c;
                    uint32_t jx = compact3(j), jy = compact3(j >> 1), jz = compact3(j >> 2);
                    uint32_t lab = l > 1 ? lc[j] : voxel(E, ox + jx, oy + jy, oz + jz);
                    uint32_t stop = (l > 1 && cc[j]) ? 1u : 0u;
                    uint32_t op = 7;
                    if (lab == par) {
                        op = 0;
                    } else {
                        for (int a = 0; a < 3; ++a) {
                            int64_t ccrd = a == 0 ? jx : (a == 1 ? jy : jz);
                            int64_t nc = (ccrd & 1) == 0 ? ccrd - 1 : ccrd + 1;
                            if (nc < 0 || nc >= child_side) continue;
                            uint32_t nx = a == 0 ? (uint32_t)nc : jx, ny = a == 1 ? (uint32_t)nc : jy,
                                     nz = a == 2 ? (uint32_t)nc : jz;
                            uint32_t nm = spread3_u32(nx) | (spread3_u32(ny) << 1) | (spread3_u32(nz) << 2);
                            uint32_t obs;
                            if (nm < j) obs = l > 1 ? lc[nm] : voxel(E, ox + nx, oy + ny, oz + nz);
                            else obs = lp[nm >> 3];
                            if (obs == lab) { op = 1 + a; break; }
                        }
                    }
                    if (op == 7) needmask |= 1u << c;
                    bytes |= (uint64_t)(op | (stop << 3)) << (8 * c);
                }
                *reinterpret_cast<uint64_t*>(es + e0 + 8 * rk) = bytes;
            }
            nmask[m] = (uint8_t)needmask;
        }
        __syncthreads();
        // pass 2: ordered compaction (rank order == Morton order): each thread owns a contiguous
        // run of parents, one block scan of the run totals, then the run's needs in order
        {
            const uint32_t per = (P + blockDim.x - 1) / blockDim.x;
            const uint32_t m0 = min(P, threadIdx.x * per), m1 = min(P, m0 + per);
            uint32_t cnt = 0;
            for (uint32_t m = m0; m < m1; ++m) cnt += __popc((uint32_t)nmask[m]);
            const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
            uint32_t inc = cnt;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += u;
            }
            if (lane == 31) S.scan[wid] = inc;
            __syncthreads();
            if (threadIdx.x < 32) {
                const uint32_t v = threadIdx.x < E_THREADS / 32 ? S.scan[threadIdx.x] : 0u;
                uint32_t x = v;
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t u = __shfl_up_sync(0xffffffffu, x, o);
                    if ((int)threadIdx.x >= o) x += u;
                }
                if (threadIdx.x < E_THREADS / 32) S.scan[threadIdx.x] = x - v;
                if (threadIdx.x == E_THREADS / 32 - 1) S.scan[E_THREADS / 32] = x;
            }
            __syncthreads();
            uint32_t pos = nneed + S.scan[wid] + inc - cnt;
            for (uint32_t m = m0; m < m1; ++m) {
                uint32_t nmk = nmask[m];
                if (!nmk) continue;
                const uint32_t rk = wpre[m >> 5] + __popc(pmask[m >> 5] & ((1u << (m & 31)) - 1u));
                while (nmk) {
                    const int c = __ffs(nmk) - 1;
                    nmk &= nmk - 1;
                    const uint32_t j = (m << 3) | (uint32_t)c;
                    const uint32_t lab = l > 1 ? lc[j] : voxel(E, ox + compact3(j), oy + compact3(j >> 1), oz + compact3(j >> 2));
                    const uint32_t stop = (l > 1 && cc[j]) ? 1u : 0u;
                    need[2 * pos] = (e0 + 8 * rk + (uint32_t)c) | ((uint32_t)s << 31) | (stop << 30);
                    need[2 * pos + 1] = lab;
                    ++pos;
                }
            }
            nneed += S.scan[E_THREADS / 32];
            __syncthreads();
        }
        cursor[s] = e0 + 8 * nact;
        __syncthreads();
    }
    // ---- E2b: serial palette replay by warp 0 (codec.py:182-198)
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        uint32_t* pal = E.pal + i * E.pal_stride;
        const uint32_t root = lev[0];
        uint32_t ring = root;                   // lane k: palette[p_len-1-k]
        uint32_t p_len = 1;
        uint32_t pd[2] = {0, 0};
        if (lane == 0) pal[0] = root;
        for (uint32_t b0 = 0; b0 < nneed; b0 += 32) {
            uint32_t key_l = 0, lab_l = 0;
            if (b0 + lane < nneed) { key_l = need[2 * (b0 + lane)]; lab_l = need[2 * (b0 + lane) + 1]; }
            uint32_t cntb = min(32u, nneed - b0);
            for (uint32_t q = 0; q < cntb; ++q) {
                uint32_t key = __shfl_sync(0xffffffffu, key_l, q);
                uint32_t lab = __shfl_sync(0xffffffffu, lab_l, q);
                bool valid = (uint32_t)lane < p_len && lane <= 16;
                uint32_t match = __ballot_sync(0xffffffffu, valid && ring == lab);
                uint32_t op, d = 0;
                if (match & 1u) op = 4;
                else if (match & 0x1FFFEu) { op = 5; d = __ffs(match & 0x1FFFEu) - 2; }
                else {
                    op = 6;
                    uint32_t up = __shfl_up_sync(0xffffffffu, ring, 1);
                    ring = lane == 0 ? lab : up;
                    if (lane == 0) pal[p_len] = lab;
                    ++p_len;
                }
                uint32_t s = key >> 31, stop = (key >> 30) & 1u, eidx = key & 0x3FFFFFFFu;
                if (lane == 0) (s ? ent + E.ent_doff : ent)[eidx] = (uint8_t)(op | (stop << 3) | (d << 4));
                if (op == 5) pd[s] += 1;
            }
        }
        if (lane == 0) {
            uint32_t* c = E.cnt + 8 * i;
            c[0] = cursor[0]; c[1] = cursor[1];
            c[2] = cursor[0] + pd[0]; c[3] = cursor[1] + pd[1];
            c[4] = p_len;
        }
    }
    // ---- prepass histograms of raw nibbles (rans.py:94-117)
    if (E.hist) {
        __syncthreads();
        if (threadIdx.x < 32) S.hist[threadIdx.x] = 0;
        __syncthreads();
        for (int s = 0; s < 2; ++s) {
            const uint8_t* es = ent + (s ? E.ent_doff : 0);
            for (uint32_t e = threadIdx.x; e < cursor[s]; e += blockDim.x) {
                uint32_t b = es[e];
                atomicAdd(&S.hist[16 * s + (b & 15u)], 1u);
                if ((b & 7u) == 5u) atomicAdd(&S.hist[16 * s + (b >> 4)], 1u);
            }
        }
        __syncthreads();
        if (threadIdx.x < 32 && S.hist[threadIdx.x]) atomicAdd(&E.hist[threadIdx.x], (unsigned long long)S.hist[threadIdx.x]);
    }
}

// E3: one lane per stream, reverse rANS (rans.py:120-137) or nibble packing (container.py:340-345).
// Per symbol: the reciprocal form of x -> (x / f) * 4096 + x % f + cum (rans.py:133): with
// q = umulhi(x, rcp) >> rsh = x / f (exact for 2^15 <= x < 2^31), the state update is
// x + bias + q * (4096 - f) -- no integer division in the lane's loop.  f = 1 uses
// rcp = ~0, rsh = 0, bias = cum + 4095 (q = x - 1).
struct EncTables {
    uint32_t freq[2][16]; uint32_t cum[2][17];
    uint32_t rcp[2][16], rsh[2][16], bias[2][16], cmpl[2][16];
};

__global__ void __launch_bounds__(256) e3_streams(EncView E, EncTables T, int entropy, uint32_t enc_doff) {
    uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (w >= 2 * E.nb) return;
    uint64_t i = w >> 1;
    int s = (int)(w & 1);
    const uint32_t* c = E.cnt + 8 * i;
    uint32_t n_ent = c[s];
    uint32_t n_nib = c[2 + s];
    const uint8_t* es = E.ent + i * E.ent_stride + (s ? E.ent_doff : 0);
    uint8_t* slot = reinterpret_cast<uint8_t*>(E.need + i * E.need_stride) + (s ? enc_doff : 0);
    uint32_t nbytes;
    if (n_nib == 0) {
        nbytes = 0;   // empty stream -> b"" (container.py:410-411)
    } else if (entropy) {
        uint32_t cap = 2 * n_nib + 8;
        uint32_t ptr = cap;
        uint32_t x = kStateLower;
        for (int64_t e = (int64_t)n_ent - 1; e >= 0; --e) {
            uint32_t b = es[e];
            uint32_t syms[2];
            int ns = 0;
            if ((b & 7u) == 5u) syms[ns++] = b >> 4;    // payload follows the op nibble
            syms[ns++] = b & 15u;
            for (int k = 0; k < ns; ++k) {
                uint32_t sy = syms[k];
                uint32_t f = T.freq[s][sy];
                uint32_t xmax = ((kStateLower >> kPrecision) << 8) * f;
                while (x >= xmax) { slot[--ptr] = (uint8_t)(x & 0xFF); x >>= 8; }
                const uint32_t q = __umulhi(x, T.rcp[s][sy]) >> T.rsh[s][sy];
                x = x + T.bias[s][sy] + q * T.cmpl[s][sy];
            }
        }
        slot[--ptr] = (uint8_t)(x >> 24);
        slot[--ptr] = (uint8_t)(x >> 16);
        slot[--ptr] = (uint8_t)(x >> 8);
        slot[--ptr] = (uint8_t)x;
        nbytes = cap - ptr;
        // move to the slot start so assembly copies from offset 0
        for (uint32_t k = 0; k < nbytes; ++k) slot[k] = slot[ptr + k];
    } else {
        uint32_t k = 0;
        uint32_t half = 0;
        bool hi = false;
        for (uint32_t e = 0; e < n_ent; ++e) {
            uint32_t b = es[e];
            uint32_t syms[2] = {b & 15u, b >> 4};
            int ns = ((b & 7u) == 5u) ? 2 : 1;
            for (int q = 0; q < ns; ++q) {
                if (!hi) { half = syms[q]; hi = true; }
                else { slot[k++] = (uint8_t)(half | (syms[q] << 4)); hi = false; }
            }
        }
        if (hi) slot[k++] = (uint8_t)half;
        nbytes = k;
    }
    E.cnt[8 * i + 5 + s] = nbytes;
}

// E4: gather sizes (palette entries, coarse bytes, detail bytes) per brick
__global__ void e4_sizes(EncView E, uint64_t* sizes) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= E.nb) return;
    const uint32_t* c = E.cnt + 8 * i;
    sizes[i] = c[4];
    sizes[E.nb + i] = c[5];
    sizes[2 * E.nb + i] = c[6];
}

__device__ __forceinline__ void put_u64(uint8_t* p, uint64_t v) { for (int k = 0; k < 8; ++k) p[k] = (uint8_t)(v >> (8 * k)); }
__device__ __forceinline__ void put_u32(uint8_t* p, uint32_t v) { for (int k = 0; k < 4; ++k) p[k] = (uint8_t)(v >> (8 * k)); }

// E4: copy a chunk's parts into the blobs; write 44-byte directory rows.
__global__ void e4_assemble(EncView E, const uint64_t* offs, uint64_t pbase, uint64_t cbase, uint64_t dbase,
                            uint8_t* dir44, uint32_t* opal, uint8_t* ocoarse, uint8_t* odetail, uint32_t enc_doff) {
    uint64_t i = blockIdx.x;
    if (i >= E.nb) return;
    const uint32_t* c = E.cnt + 8 * i;
    uint64_t po = pbase + offs[i], co = cbase + offs[E.nb + i], d_o = dbase + offs[2 * E.nb + i];
    const uint32_t* pal = E.pal + i * E.pal_stride;
    const uint8_t* slot = reinterpret_cast<const uint8_t*>(E.need + i * E.need_stride);
    for (uint32_t k = threadIdx.x; k < c[4]; k += blockDim.x) opal[po + k] = pal[k];
    for (uint32_t k = threadIdx.x; k < c[5]; k += blockDim.x) ocoarse[co + k] = slot[k];
    for (uint32_t k = threadIdx.x; k < c[6]; k += blockDim.x) odetail[d_o + k] = slot[enc_doff + k];
    if (threadIdx.x == 0) {
        uint8_t* row = dir44 + 44 * enc_brick(E, i);
        put_u64(row + 0, po); put_u32(row + 8, c[4]);
        put_u64(row + 12, co); put_u32(row + 20, c[5]); put_u32(row + 24, c[2]);
        put_u64(row + 28, d_o); put_u32(row + 36, c[6]); put_u32(row + 40, c[3]);
    }
}

// ---------------------------------------------------------------------------- synthetic volumes
// Jittered-grid Voronoi (configs 2-5): g^3 cells of side `cell`
// voxels, one seed per cell at a hashed fixed-point offset (1/256 voxel), label
// = nearest seed id + 1 (ties -> lower id).  With `membrane`, label 0 marks
// voxels whose nearest seed differs from that of the +x/+y/+z neighbour
// (1-voxel boundaries).  `drift` shifts all seeds by a per-seed hashed
// offset of at most `drift` voxels (time series, config 5).
__device__ __forceinline__ uint32_t hash32(uint32_t a) {
    a ^= a >> 16; a *= 0x7feb352du; a ^= a >> 15; a *= 0x846ca68bu; a ^= a >> 16;
    return a;
}
struct Synth { int64_t X, Y, Z; int g; int64_t cell256; uint32_t seed; int drift256; uint32_t dseed; };

__device__ __forceinline__ void seed_pos(const Synth& S, int cx, int cy, int cz, int64_t* p) {
    uint32_t id = ((uint32_t)cz * S.g + cy) * S.g + cx;
    int c3[3] = {cx, cy, cz};
    for (int a = 0; a < 3; ++a) {
        uint32_t h = hash32(id * 3u + a + S.seed * 0x9e3779b9u);
        int64_t off = (int64_t)(h % (uint32_t)S.cell256);
        int64_t base = c3[a] * S.cell256 + off;
        if (S.drift256) {
            uint32_t hd = hash32(id * 7u + a + S.dseed * 0x85ebca6bu);
            base += (int64_t)(hd % (uint32_t)(2 * S.drift256 + 1)) - S.drift256;
        }
        p[a] = base;
    }
}

__device__ uint32_t nearest_seed(const Synth& S, int64_t x, int64_t y, int64_t z) {
    int64_t v[3] = {x * 256 + 128, y * 256 + 128, z * 256 + 128};
    int c[3];
    for (int a = 0; a < 3; ++a) {
        int64_t q = v[a] / S.cell256;
        c[a] = (int)(q >= S.g ? S.g - 1 : q);
    }
    uint64_t best = ~0ull;
    uint32_t bid = 0;
    for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                int cx = c[0] + dx, cy = c[1] + dy, cz = c[2] + dz;
                if (cx < 0 || cy < 0 || cz < 0 || cx >= S.g || cy >= S.g || cz >= S.g) continue;
                int64_t p[3];
                seed_pos(S, cx, cy, cz, p);
                uint64_t d = 0;
                for (int a = 0; a < 3; ++a) { int64_t e = v[a] - p[a]; d += (uint64_t)(e * e); }
                uint32_t id = ((uint32_t)cz * S.g + cy) * S.g + cx;
                if (d < best || (d == best && id < bid)) { best = d; bid = id; }
            }
    return bid + 1;
}

__global__ void k_synth(Synth S, uint32_t* out, int membrane) {
    uint64_t n = (uint64_t)S.X * S.Y * S.Z;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        int64_t x = i % S.X, y = (i / S.X) % S.Y, z = i / (S.X * S.Y);
        uint32_t lab = nearest_seed(S, x, y, z);
        if (membrane) {
            if ((x + 1 < S.X && nearest_seed(S, x + 1, y, z) != lab) ||
                (y + 1 < S.Y && nearest_seed(S, x, y + 1, z) != lab) ||
                (z + 1 < S.Z && nearest_seed(S, x, y, z + 1) != lab))
                lab = 0;
        }
        out[i] = lab;
    }
}

}  // namespace csv

// ============================================================================ host driver + C-ABI
using namespace csv;

namespace csv {
cudaError_t run_scan(const uint64_t* sizes, uint64_t* out, uint64_t n, uint64_t* tmp, cudaStream_t st);
}


struct csv_encoded {
    int device = 0;
    uint8_t head[120]{};
    uint64_t n = 0;
    uint64_t sizes[3]{};          // palette entries, coarse bytes, detail bytes
    uint8_t* d_dir = nullptr;
    uint32_t* d_pal = nullptr;
    uint8_t* d_coarse = nullptr;
    uint8_t* d_detail = nullptr;
    uint64_t cap[3]{};
};

namespace {

int efail(int code, const char* msg) {
    csv::set_error(msg);
    return code;
}

// quantize_counts (rans.py:73-91): floor 1, largest remainder over 4080, ties to lower symbol
void quantize(const unsigned long long* hist, uint16_t* out) {
    long long raw[16], tot = 0;
    for (int s = 0; s < 16; ++s) { raw[s] = (long long)hist[s]; tot += raw[s]; }
    if (tot == 0) { for (int s = 0; s < 16; ++s) raw[s] = 1; tot = 16; }
    const long long spread = 4096 - 16;
    double rem[16];
    long long base[16], bs = 0;
    for (int s = 0; s < 16; ++s) {
        double share = (double)(raw[s] * spread) / (double)tot;
        base[s] = (long long)std::floor(share);
        rem[s] = share - (double)base[s];
        bs += base[s];
    }
    int order[16];
    for (int s = 0; s < 16; ++s) order[s] = s;
    std::stable_sort(order, order + 16, [&](int a, int b) { return rem[a] > rem[b]; });
    for (long long k = 0; k < spread - bs && k < 16; ++k) base[order[k]] += 1;
    for (int s = 0; s < 16; ++s) out[s] = (uint16_t)(base[s] + 1);
}

uint32_t max_ent_coarse(int N) { return max_entries(N, 0, 0); }
uint32_t max_ent_detail(int N) { return max_entries(N, 0, 1); }

// Per-device scratch arena, grow-only and reused by every encode on that device
// (the encode synchronises its stream before returning, and the mutex serialises
// encodes on one device).  Allocating the ~2 GB of chunk scratch per call made the
// encode time depend on the driver's page-mapping cost (30 ms .. 1.4 s per 1024^3).
struct Scratch {
    uint8_t* ent = nullptr; uint32_t* need = nullptr; uint32_t* pal = nullptr; uint32_t* cnt = nullptr;
    uint32_t* ws = nullptr; uint32_t* list = nullptr; uint64_t* sizes = nullptr; uint64_t* offs = nullptr;
    uint64_t* tmp = nullptr; unsigned long long* hist = nullptr;
    uint64_t cap[10] = {};
};
struct ScratchArena {
    std::mutex mu;
    Scratch s;
    uint64_t budget = 0;        // chunk scratch budget, fixed at the first encode on the device
    bool pool_ready = false;    // default memory pool kept (release threshold) for the output blobs
};
constexpr int kMaxDevices = 64;
ScratchArena g_arena[kMaxDevices];

template <typename T>
cudaError_t reserve(T** p, uint64_t* cap, uint64_t bytes) {
    if (bytes <= *cap && *p) return cudaSuccess;
    cudaFree(*p);
    *p = nullptr;
    *cap = 0;
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), bytes ? bytes : 16);
    if (e == cudaSuccess) *cap = bytes;
    return e;
}

}  // namespace

// Output blobs and the directory come from the device's default memory pool (stream-ordered,
// kept by a release threshold): per-timestep encodes reuse the same physical pages instead of
// paying cudaMalloc/cudaFree page mapping (which made a 1024^3 encode take 14-120 ms).
static cudaError_t grow(void** p, uint64_t* cap, uint64_t need, uint64_t used, cudaStream_t st) {
    if (need <= *cap) return cudaSuccess;
    uint64_t nc = std::max<uint64_t>(need + 64, *cap * 3 / 2 + 64);
    void* q = nullptr;
    cudaError_t e = cudaMallocAsync(&q, nc, st);
    if (e != cudaSuccess) return e;
    cudaMemsetAsync(q, 0, nc, st);
    if (*p && used) cudaMemcpyAsync(q, *p, used, cudaMemcpyDeviceToDevice, st);
    if (*p) cudaFreeAsync(*p, st);
    *p = q;
    *cap = nc;
    return cudaSuccess;
}

static void keep_default_pool(int device) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
}

extern "C" {

int csv_synth_voronoi(uint32_t* d_out, int64_t X, int64_t Y, int64_t Z, int cells_per_axis, uint32_t seed,
                      int membrane, double drift, uint32_t drift_seed, uintptr_t stream) {
    if (!d_out || X < 1 || Y < 1 || Z < 1 || cells_per_axis < 1) return efail(CSV_E_ARG, "bad synth arguments");
    Synth S;
    S.X = X; S.Y = Y; S.Z = Z; S.g = cells_per_axis; S.seed = seed;
    int64_t maxd = std::max(X, std::max(Y, Z));
    S.cell256 = std::max<int64_t>(1, (maxd * 256 + cells_per_axis - 1) / cells_per_axis);
    S.drift256 = (int)std::llround(drift * 256.0);
    S.dseed = drift_seed;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    k_synth<<<148 * 16, 256, 0, st>>>(S, d_out, membrane);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? CSV_OK : efail(CSV_E_CUDA, cudaGetErrorString(e));
}

// GPU compress_volume (container.py:374-453).  d_volume: (Z,Y,X) C-order u16 (width 16) or u32.
int csv_encode_volume(int device, const void* d_volume, int width, int64_t X, int64_t Y, int64_t Z,
                      int brick_log2, int64_t prepass_stride, int entropy, int label_width, uintptr_t stream,
                      csv_encoded** out) {
    if (!d_volume || !out || (width != 16 && width != 32)) return efail(CSV_E_ARG, "bad encode arguments");
    if (brick_log2 < 1 || brick_log2 > 7) return efail(CSV_E_ARG, "brick_log2 must be in [1, 7]");
    if (X < 1 || Y < 1 || Z < 1) return efail(CSV_E_ARG, "need a non-empty 3-D volume");
    cudaSetDevice(device);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int N = brick_log2;
    const int64_t b = 1ll << N;
    const int64_t gx = (X + b - 1) / b, gy = (Y + b - 1) / b, gz = (Z + b - 1) / b;
    const uint64_t n = (uint64_t)(gx * gy * gz);
    const uint32_t mec = max_ent_coarse(N), med = max_ent_detail(N);
    const uint64_t ent_stride = round16(mec) + round16(med);
    const uint32_t ent_doff = (uint32_t)round16(mec);
    const uint64_t need_stride = 2ull * (mec + med) + 64;            // u32
    const uint32_t enc_doff = (uint32_t)round16(2ull * 2 * mec + 16); // bytes inside the need slot
    const uint64_t pal_stride = 1ull + mec + med;
    const bool smem = N <= 6;
    const EncLayout Y_ = enc_layout(N);
    const size_t smem_bytes = (size_t)Y_.words * 4;
    uint64_t per_brick = ent_stride + need_stride * 4 + pal_stride * 4 + 32 + (smem ? 0 : (uint64_t)Y_.words * 4);
    // CSVGPU_ENC_TRACE=1: host-clock phase times on stderr (encode timing investigations)
    static const bool trace = std::getenv("CSVGPU_ENC_TRACE") != nullptr;
    const auto t_start = std::chrono::steady_clock::now();
    auto mark = [&](const char* what, long long k) {
        if (!trace) return;
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
        std::fprintf(stderr, "[enc] %8.2f ms  %s %lld\n", ms, what, k);
    };
    if (device < 0 || device >= kMaxDevices) return efail(CSV_E_ARG, "device index out of range");
    std::lock_guard<std::mutex> arena_lock(g_arena[device].mu);
    Scratch& Sc = g_arena[device].s;
    if (!g_arena[device].budget) {
        // chunk scratch budget, sized once per device (cudaMemGetInfo waits for the driver's
        // deferred frees: 15-90 ms inside a timed encode).  CSVGPU_ENC_BUDGET_GB overrides the
        // default (8 GB: a 1024^3 volume of 32^3 bricks encodes in 2 chunks; 2 GB: 8 chunks, +55 %)
        size_t freeb = 0, totb = 0;
        cudaMemGetInfo(&freeb, &totb);
        const char* bg = std::getenv("CSVGPU_ENC_BUDGET_GB");
        const double budget_gb = bg ? std::atof(bg) : 8.0;
        g_arena[device].budget = std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)(freeb * 0.35),
                                                                           (uint64_t)(budget_gb * (1ull << 30))));
    }
    if (!g_arena[device].pool_ready) {
        keep_default_pool(device);
        g_arena[device].pool_ready = true;
    }
    mark("budget", 0);
    uint64_t chunk = std::max<uint64_t>(1, std::min<uint64_t>(n, g_arena[device].budget / per_brick));
    chunk = std::min<uint64_t>(chunk, 65536);
    csv_encoded* enc = new csv_encoded();
    enc->device = device;
    enc->n = n;
    auto cleanup = [&](int rc, const char* msg) {
        if (rc != CSV_OK) {
            cudaFree(enc->d_dir); cudaFree(enc->d_pal); cudaFree(enc->d_coarse); cudaFree(enc->d_detail);
            delete enc;
            return efail(rc, msg);
        }
        return CSV_OK;
    };
#define ETRY(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) return cleanup(CSV_E_CUDA, cudaGetErrorString(e_)); } while (0)
    ETRY(reserve(&Sc.ent, &Sc.cap[0], chunk * ent_stride));
    ETRY(reserve(&Sc.need, &Sc.cap[1], chunk * need_stride * 4));
    ETRY(reserve(&Sc.pal, &Sc.cap[2], chunk * pal_stride * 4));
    ETRY(reserve(&Sc.cnt, &Sc.cap[3], chunk * 32));
    if (!smem) ETRY(reserve(&Sc.ws, &Sc.cap[4], chunk * (uint64_t)Y_.words * 4));
    ETRY(reserve(&Sc.sizes, &Sc.cap[5], 3 * chunk * 8));
    ETRY(reserve(&Sc.offs, &Sc.cap[6], (3 * chunk + 1) * 8));
    ETRY(reserve(&Sc.tmp, &Sc.cap[7], 4104 * 8));
    ETRY(reserve(&Sc.hist, &Sc.cap[8], 32 * 8));
    ETRY(cudaMallocAsync(reinterpret_cast<void**>(&enc->d_dir), n * 44 + 16, st));
    if (smem) ETRY(cudaFuncSetAttribute(e12_bricks<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes));
    mark("scratch reserved, chunk", (long long)chunk);

    EncView E{};
    E.vol = d_volume; E.width = width; E.X = X; E.Y = Y; E.Z = Z; E.N = N; E.gx = gx; E.gy = gy; E.gz = gz;
    E.ent = Sc.ent; E.ent_stride = ent_stride; E.ent_doff = ent_doff;
    E.need = Sc.need; E.need_stride = need_stride; E.pal = Sc.pal; E.pal_stride = pal_stride; E.cnt = Sc.cnt;
    E.ws = Sc.ws; E.ws_stride = Y_.words;
    auto launch_e12 = [&](const EncView& V) {
        if (smem) e12_bricks<true><<<(unsigned)V.nb, E_THREADS, smem_bytes, st>>>(V);
        else e12_bricks<false><<<(unsigned)V.nb, E_THREADS, 0, st>>>(V);
    };
    // ---- tables: prepass over range(0, n, stride) (container.py:399-403)
    uint16_t icnt[16], lcnt[16];
    if (entropy) {
        uint64_t stride = prepass_stride < 1 ? 1 : (uint64_t)prepass_stride;
        std::vector<uint32_t> ids;
        for (uint64_t k = 0; k < n; k += stride) ids.push_back((uint32_t)k);
        ETRY(reserve(&Sc.list, &Sc.cap[9], ids.size() * 4));
        ETRY(cudaMemcpyAsync(Sc.list, ids.data(), ids.size() * 4, cudaMemcpyHostToDevice, st));
        ETRY(cudaMemsetAsync(Sc.hist, 0, 32 * 8, st));
        for (uint64_t k0 = 0; k0 < ids.size(); k0 += chunk) {
            EncView V = E;
            V.list = Sc.list + k0;
            V.nb = std::min<uint64_t>(chunk, ids.size() - k0);
            V.hist = Sc.hist;
            launch_e12(V);
            ETRY(cudaGetLastError());
        }
        unsigned long long h[32];
        ETRY(cudaMemcpyAsync(h, Sc.hist, sizeof h, cudaMemcpyDeviceToHost, st));
        ETRY(cudaStreamSynchronize(st));
        mark("prepass", (long long)ids.size());
        for (int s = 0; s < 32; ++s) h[s] += 1;   // +1 smoothing (rans.py:115-116)
        quantize(h, icnt);
        quantize(h + 16, lcnt);
    } else {
        for (int s = 0; s < 16; ++s) icnt[s] = lcnt[s] = 256;
    }
    EncTables T;
    for (int tb = 0; tb < 2; ++tb) {
        const uint16_t* cn = tb ? lcnt : icnt;
        T.cum[tb][0] = 0;
        for (int s = 0; s < 16; ++s) { T.freq[tb][s] = cn[s]; T.cum[tb][s + 1] = T.cum[tb][s] + cn[s]; }
        for (int s = 0; s < 16; ++s) {
            const uint32_t f = T.freq[tb][s];
            T.cmpl[tb][s] = kTotalFreq - f;
            if (f < 2) {
                T.rcp[tb][s] = 0xFFFFFFFFu; T.rsh[tb][s] = 0; T.bias[tb][s] = T.cum[tb][s] + kTotalFreq - 1;
            } else {
                uint32_t sh = 0;
                while (f > (1u << sh)) ++sh;
                T.rcp[tb][s] = (uint32_t)(((1ull << (sh + 31)) + f - 1) / f);
                T.rsh[tb][s] = sh - 1;
                T.bias[tb][s] = T.cum[tb][s];
            }
        }
    }
    // ---- main pass, chunk by chunk
    uint64_t pos[3] = {0, 0, 0};
    for (uint64_t c0 = 0; c0 < n; c0 += chunk) {
        EncView V = E;
        V.list = nullptr;
        V.b0 = c0;
        V.nb = std::min<uint64_t>(chunk, n - c0);
        V.hist = nullptr;
        launch_e12(V);
        ETRY(cudaGetLastError());
        e3_streams<<<(unsigned)((2 * V.nb + 255) / 256), 256, 0, st>>>(V, T, entropy, enc_doff);
        ETRY(cudaGetLastError());
        e4_sizes<<<(unsigned)((V.nb + 255) / 256), 256, 0, st>>>(V, Sc.sizes);
        ETRY(run_scan(Sc.sizes, Sc.offs, 3 * V.nb, Sc.tmp, st));
        // per-part totals: offs[nb], offs[2nb] are prefix boundaries; read three values
        uint64_t h[4];
        ETRY(cudaMemcpyAsync(&h[0], Sc.offs + V.nb, 8, cudaMemcpyDeviceToHost, st));
        ETRY(cudaMemcpyAsync(&h[1], Sc.offs + 2 * V.nb, 8, cudaMemcpyDeviceToHost, st));
        ETRY(cudaMemcpyAsync(&h[2], Sc.offs + 3 * V.nb, 8, cudaMemcpyDeviceToHost, st));
        ETRY(cudaStreamSynchronize(st));
        mark("chunk sized", (long long)c0);
        uint64_t tp = h[0], tc = h[1] - h[0], td = h[2] - h[1];
        // offsets of parts 1 and 2 are relative to the start of the whole scan: subtract in the kernel via bases
        if (c0 == 0 && V.nb < n) {   // size the blobs once from the first chunk (+12.5 %), not by regrowth
            const double sc = (double)n / (double)V.nb * 1.125;
            ETRY(grow((void**)&enc->d_pal, &enc->cap[0], (uint64_t)(tp * 4 * sc) + kBlobPad, 0, st));
            ETRY(grow((void**)&enc->d_coarse, &enc->cap[1], (uint64_t)(tc * sc) + kBlobPad, 0, st));
            ETRY(grow((void**)&enc->d_detail, &enc->cap[2], (uint64_t)(td * sc) + kBlobPad, 0, st));
        }
        ETRY(grow((void**)&enc->d_pal, &enc->cap[0], (pos[0] + tp) * 4 + kBlobPad, pos[0] * 4, st));
        ETRY(grow((void**)&enc->d_coarse, &enc->cap[1], pos[1] + tc + kBlobPad, pos[1], st));
        ETRY(grow((void**)&enc->d_detail, &enc->cap[2], pos[2] + td + kBlobPad, pos[2], st));
        e4_assemble<<<(unsigned)V.nb, 128, 0, st>>>(V, Sc.offs, pos[0], pos[1] - h[0], pos[2] - h[1], enc->d_dir,
                                                      enc->d_pal, enc->d_coarse, enc->d_detail, enc_doff);
        ETRY(cudaGetLastError());
        pos[0] += tp; pos[1] += tc; pos[2] += td;
        mark("chunk assembled", (long long)c0);
    }
    ETRY(cudaStreamSynchronize(st));
    mark("done", 0);
    enc->sizes[0] = pos[0]; enc->sizes[1] = pos[1]; enc->sizes[2] = pos[2];
    // head (container.py:235-253)
    uint8_t* hd = enc->head;
    memcpy(hd, "CSV1", 4);
    uint16_t ver = 1; memcpy(hd + 4, &ver, 2);
    hd[6] = entropy ? 1 : 0; hd[7] = 0;
    uint16_t lw = (uint16_t)label_width; memcpy(hd + 8, &lw, 2);
    uint16_t bl = (uint16_t)N; memcpy(hd + 10, &bl, 2);
    uint32_t d3[3] = {(uint32_t)X, (uint32_t)Y, (uint32_t)Z}; memcpy(hd + 12, d3, 12);
    uint32_t ps = (uint32_t)prepass_stride; memcpy(hd + 24, &ps, 4);
    uint32_t z0 = 0; memcpy(hd + 28, &z0, 4);
    memcpy(hd + 32, icnt, 32); memcpy(hd + 64, lcnt, 32);
    uint64_t bs[3] = {pos[0] * 4, pos[1], pos[2]}; memcpy(hd + 96, bs, 24);
    // guarantee non-null, padded blobs even when empty
    if (!enc->d_pal) ETRY(grow((void**)&enc->d_pal, &enc->cap[0], kBlobPad, 0, st));
    if (!enc->d_coarse) ETRY(grow((void**)&enc->d_coarse, &enc->cap[1], kBlobPad, 0, st));
    if (!enc->d_detail) ETRY(grow((void**)&enc->d_detail, &enc->cap[2], kBlobPad, 0, st));
    *out = enc;
    return cleanup(CSV_OK, "");
#undef ETRY
}

int csv_encoded_info(csv_encoded* enc, uint8_t* head120, uint64_t* n_bricks, uint64_t* sizes3) {
    if (!enc) return efail(CSV_E_ARG, "null encoded");
    if (head120) memcpy(head120, enc->head, 120);
    if (n_bricks) *n_bricks = enc->n;
    if (sizes3) memcpy(sizes3, enc->sizes, 24);
    return CSV_OK;
}

int csv_encoded_device_ptrs(csv_encoded* enc, const uint8_t** d_dir44, const uint32_t** d_palette,
                            const uint8_t** d_coarse, const uint8_t** d_detail) {
    if (!enc) return efail(CSV_E_ARG, "null encoded");
    if (d_dir44) *d_dir44 = enc->d_dir;
    if (d_palette) *d_palette = enc->d_pal;
    if (d_coarse) *d_coarse = enc->d_coarse;
    if (d_detail) *d_detail = enc->d_detail;
    return CSV_OK;
}

int csv_encoded_copy_to_host(csv_encoded* enc, uint8_t* dir44, uint32_t* palette, uint8_t* coarse, uint8_t* detail,
                             uintptr_t stream) {
    if (!enc) return efail(CSV_E_ARG, "null encoded");
    cudaSetDevice(enc->device);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (dir44 && enc->n) cudaMemcpyAsync(dir44, enc->d_dir, enc->n * 44, cudaMemcpyDeviceToHost, st);
    if (palette && enc->sizes[0]) cudaMemcpyAsync(palette, enc->d_pal, enc->sizes[0] * 4, cudaMemcpyDeviceToHost, st);
    if (coarse && enc->sizes[1]) cudaMemcpyAsync(coarse, enc->d_coarse, enc->sizes[1], cudaMemcpyDeviceToHost, st);
    if (detail && enc->sizes[2]) cudaMemcpyAsync(detail, enc->d_detail, enc->sizes[2], cudaMemcpyDeviceToHost, st);
    cudaError_t e = cudaStreamSynchronize(st);
    return e == cudaSuccess ? CSV_OK : efail(CSV_E_CUDA, cudaGetErrorString(e));
}

int csv_encoded_free(csv_encoded* enc) {
    if (!enc) return CSV_OK;
    cudaSetDevice(enc->device);
    cudaFree(enc->d_dir); cudaFree(enc->d_pal); cudaFree(enc->d_coarse); cudaFree(enc->d_detail);
    delete enc;
    return CSV_OK;
}

}  // extern "C"
