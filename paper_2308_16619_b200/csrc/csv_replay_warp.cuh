// csv_replay_warp.cuh -- K2w: one WARP per brick, persistent warps pulling
// requests from a global counter.  Included by csv_decode.cu after the shared
// K2 helpers (Raster, ekey, raster_of, op_eq, ...).
//
// Reference: _decode_kernel (codec.py:303-471) replays levels N..t+1, parents
// in Morton order, 8 children each.  The GPU restatement keeps a brick inside
// one warp (no CTA barriers, a dozen or more bricks in flight per SM) and
// works in palette-index space (u8 when the palette has <= 256 entries, else
// u16 in a second pass), so a warp's whole working set is 9 KB (17 KB) of
// shared memory.  Per level:
//
//  * fill: every parent's 8 children get the parent's value (stop fill /
//    occupancy skip, codec.py:367-370, :458-463); active parents (those the
//    reference visits) are ranked by a popcount prefix of the level's mask,
//    which is also the index of their 8 entries (K1's entry groups).
//  * active pass: one lane per ACTIVE parent (compacted, so no lane idles on
//    the 70 % of parents that are constant) evaluates its 8 children
//    (codec.py:400-457); the palette base i_p is a warp scan of the P_a
//    counts of the preceding parents in entry order.
//  * chain rounds: an even-coordinate neighbour op reuses the already decoded
//    child of the -1 neighbour parent (codec.py:422-423), whose local index is
//    c | (1 << axis) -- one more odd coordinate.  Resolving children by
//    decreasing popcount of the local index (7 | 3,5,6 | 1,2,4 | 0) therefore
//    takes exactly three rounds and never a loop.
//
// Coarse levels keep their children in the shared level array.  The final
// level is swept plane by plane (parent z): the children of the current
// parent plane and the odd-z voxel plane below live in a 3-plane ring, the
// inactive parents are written to HBM straight from the fill, the active ones
// after their rounds.

#include "csv_eval8.cuh"

#ifndef K2W_RUNROLL
#define K2W_RUNROLL 1   // u8 final level: unroll of the per-plane row loop
#endif
constexpr int kRUnroll = K2W_RUNROLL;

#ifndef K2W_SPAL
#define K2W_SPAL 1      // u8 mode: copy the brick's palette into the warp's shared slice
#endif

namespace wk {

// Entry words.  CG (the overlap launch, which reads regions while K1 is still running):
// L2-coherent loads (ld.global.cg); otherwise the read-only path.  Each word is read once,
// so L1 holds nothing useful either way; .cg costs ~1 % in the full-volume kernel.
template <bool CG>
__device__ __forceinline__ uint64_t ldent(const uint64_t* p) {
    if constexpr (CG) return __ldcg(p);
    else return __ldg(p);
}

__host__ __device__ constexpr uint32_t wofs(int j) {   // u16 offset of level N-j (root j = 0), 8-aligned
    return j == 0 ? 0u : 8u + ((1u << (3 * j)) - 8u) / 7u;
}
__host__ __device__ constexpr uint32_t al16(uint32_t v) { return (v + 15u) & ~15u; }
__host__ __device__ constexpr uint32_t umax(uint32_t a, uint32_t b) { return a > b ? a : b; }

// Per-warp shared-memory slice for LMAX = N - t levels, values of `isz` bytes
// (u8 palette indices when the palette has <= 256 entries, else u16):
//   lev   : level values t+1..N, root first (wofs)
//   pm/cm : active-parent bitmask of the level / of its children
//   wpre  : popcount prefix of pm per word (rank of an active parent)
//   ring  : final level: voxel planes 2pz-1, 2pz, 2pz+1 (3 x (2R)^2 values)
//   plist : final level: per-plane active parents (u8 index in the plane)
//   pdesc : final level: their pending-chain descriptors (u16); aliases cm
//   amask : final level: active parents of the plane (bit per parent, raster
//           order) + exclusive popcount per word (list index of a parent)
//   clist/cdesc : coarse levels: active list / descriptors (u16); alias the ring
struct WLayout {
    uint32_t lev, pm, cm, wpre, ring, plist, pdesc, clist, cdesc, spal, amask, bytes;   // byte offsets in one warp's slice
};
__host__ __device__ constexpr WLayout make_wlayout(int L, uint32_t isz) {
    WLayout Y{};
    const uint32_t maxP = 1u << (3 * (L - 1));            // final-level parents (= coarse children max)
    const uint32_t W = (maxP + 31) / 32;
    const uint32_t R = 1u << (L - 1);
    const uint32_t ringb = 3u * (2u * R) * (2u * R) * isz;
    const uint32_t cpar = L >= 2 ? (1u << (3 * (L - 2))) : 1u;   // coarse-level parents (max)
    const bool gfin = L >= 6;                             // final parent level in global scratch (64^3 replays)
    Y.lev = 0;
    Y.pm = al16((gfin ? wofs(L - 1) : wofs(L)) * isz);
    Y.cm = al16(Y.pm + 4 * W);
    Y.wpre = al16(Y.cm + 4 * W);
    Y.ring = al16(Y.wpre + 2 * W);
    Y.plist = al16(Y.ring + ringb);
    uint32_t end = al16(Y.plist + R * R * (R > 16 ? 2u : 1u));   // u16 plane indices above 16 x 16 parents
    if (2 * R * R <= 4 * W) {
        Y.pdesc = Y.cm;                                   // cm is dead during the final sweep
    } else {
        Y.pdesc = end;
        end = al16(end + 2 * R * R);
    }
    Y.clist = Y.ring;                                     // coarse levels: ring and plist are free
    if (!gfin) end = umax(end, al16(Y.ring + 4 * cpar));  // (64^3 replays: the largest coarse level's
    Y.cdesc = Y.clist + 2 * cpar;                         //  list lives in the warp's global slot)
    Y.spal = end;                                         // u8 mode: the brick's palette (<= 256 labels)
    if (isz == 1 && K2W_SPAL) end = al16(end + 1024);
    Y.amask = end;                                        // final level: per-plane active mask + word prefix (chain hops)
    end = al16(end + 6 * ((R * R + 31) / 32));
    Y.bytes = end;
    return Y;
}

// value storage: u8 or u16 palette indices; P2 holds two x-adjacent children
template <typename IT> struct IX;
template <> struct IX<uint8_t> { using P2 = uint16_t; static constexpr uint32_t B = 8; };
template <> struct IX<uint16_t> { using P2 = uint32_t; static constexpr uint32_t B = 16; };
template <typename IT>
__device__ __forceinline__ typename IX<IT>::P2 pack2(uint32_t a, uint32_t b) { return (typename IX<IT>::P2)(a | (b << IX<IT>::B)); }
template <typename IT>
__device__ __forceinline__ uint32_t lo2(uint32_t p) { return p & ((1u << IX<IT>::B) - 1u); }
template <typename IT>
__device__ __forceinline__ uint32_t hi2(uint32_t p) { return p >> IX<IT>::B; }
// the 8 children of one parent, contiguous (Morton order), 8 or 16 bytes
template <typename IT>
__device__ __forceinline__ void store8(IT* p, const uint32_t (&v)[8]) {
    if (sizeof(IT) == 1) {
        *reinterpret_cast<uint2*>(p) = make_uint2(v[0] | (v[1] << 8) | (v[2] << 16) | (v[3] << 24),
                                                  v[4] | (v[5] << 8) | (v[6] << 16) | (v[7] << 24));
    } else {
        *reinterpret_cast<uint4*>(p) = make_uint4(v[0] | (v[1] << 16), v[2] | (v[3] << 16), v[4] | (v[5] << 16),
                                                  v[6] | (v[7] << 16));
    }
}
template <typename IT>
__device__ __forceinline__ void store8_same(IT* p, uint32_t v) {
    if (sizeof(IT) == 1) {
        const uint32_t x = v * 0x01010101u;
        *reinterpret_cast<uint2*>(p) = make_uint2(x, x);
    } else {
        const uint32_t x = v | (v << 16);
        *reinterpret_cast<uint4*>(p) = make_uint4(x, x, x, x);
    }
}

constexpr unsigned FULL = 0xffffffffu;
constexpr uint64_t ONES = 0x0101010101010101ull;

__device__ __forceinline__ void put_result(const Plan& P, uint64_t r, int st, int stream, int64_t pos, int64_t ci,
                                           int64_t di) {
    if (P.res) {
        csv_result o;
        o.status = st; o.stream = stream; o.pos = pos; o.ci = ci; o.di = di;
        P.res[r] = o;
    }
}

__device__ __forceinline__ unsigned long long umin64(unsigned long long a, unsigned long long b) { return a < b ? a : b; }
__device__ __forceinline__ unsigned long long warp_min64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = umin64(v, __shfl_xor_sync(FULL, v, o));
    return v;
}
__device__ __forceinline__ uint32_t warp_sum(uint32_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}
__device__ __forceinline__ uint32_t lanemask_lt(int lane) { return (1u << lane) - 1u; }

// Exclusive popcount prefix of mask words [0, W) into wpre; returns the total (warp-uniform).
__device__ __forceinline__ uint32_t rank_prefix(const uint32_t* pm, uint32_t W, uint16_t* wpre, int lane) {
    uint32_t run = 0;
    for (uint32_t w0 = 0; w0 < W; w0 += 32) {
        const uint32_t i = w0 + lane;
        const uint32_t v = i < W ? __popc(pm[i]) : 0u;
        uint32_t inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(FULL, inc, o);
            if (lane >= o) inc += u;
        }
        if (i < W) wpre[i] = (uint16_t)(run + inc - v);
        run += __shfl_sync(FULL, inc, 31);
    }
    __syncwarp();
    return run;
}

// SWAR byte masks (0x01 per child byte) over the 8 entries of a group
__device__ __forceinline__ uint64_t m_op7(uint64_t w) { return w & (w >> 1) & (w >> 2) & ONES; }
__device__ __forceinline__ uint64_t m_op5(uint64_t w) { return w & ~(w >> 1) & (w >> 2) & ONES; }
__device__ __forceinline__ uint64_t m_pal(uint64_t w) { return (w >> 2) & ONES & ~m_op7(w); }   // ops 4, 5, 6
__device__ __forceinline__ uint64_t m_op6(uint64_t w) { return ~w & (w >> 1) & (w >> 2) & ONES; }
__device__ __forceinline__ uint32_t first_byte(uint64_t m) { return (uint32_t)(__ffsll((long long)m) - 1) >> 3; }
__device__ __forceinline__ uint64_t valid_mask(uint32_t nvalid, uint32_t ent0) {
    const uint32_t nv = nvalid > ent0 ? min(nvalid - ent0, 8u) : 0u;
    return nv == 8 ? ~0ull : ((1ull << (8 * nv)) - 1ull);
}

// Inclusive warp scan (u32).
__device__ __forceinline__ uint32_t warp_incl(uint32_t v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(FULL, v, o);
        if (lane >= o) v += u;
    }
    return v;
}

// Values of the 8 children of one active parent (codec.py:400-425): R_p and
// odd-coordinate neighbour ops resolved here, even-coordinate neighbour ops
// marked pending (axis + 1, 2 bits per child), boundary violations flagged.
// bf: bit 2a = parent at coordinate 0 on axis a, bit 2a+1 = at the maximum.
struct Group {
    uint32_t v[8];
    uint32_t pend;   // 2 bits per child: 0 none, 1 x, 2 y, 3 z
    uint32_t bn;     // BAD_NEIGHBOR children (bit c)
};
__device__ __forceinline__ void eval_group(uint64_t w, uint32_t pv, uint32_t pxp, uint32_t pyp, uint32_t pzp,
                                           uint32_t bf, Group& g) {
    const uint32_t lo = (uint32_t)w, hi = (uint32_t)(w >> 32);
    g.pend = 0;
    g.bn = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const uint32_t op = ((c < 4 ? lo : hi) >> (8 * (c & 3))) & 7u;
        const bool ox = c & 1, oy = c & 2, oz = c & 4;
        uint32_t val = pv;
        if (ox) val = op == 1u ? pxp : val;
        if (oy) val = op == 2u ? pyp : val;
        if (oz) val = op == 3u ? pzp : val;
        g.v[c] = val;
        // even coordinate at 0 or odd coordinate at the maximum: no neighbour (codec.py:416-417)
        const uint32_t bx = (bf >> (ox ? 1 : 0)) & 1u, by = (bf >> (oy ? 3 : 2)) & 1u, bz = (bf >> (oz ? 5 : 4)) & 1u;
        const bool bad = (op == 1u && bx) || (op == 2u && by) || (op == 3u && bz);
        uint32_t pa = 0;
        if (!ox && op == 1u) pa = 1u;
        if (!oy && op == 2u) pa = 2u;
        if (!oz && op == 3u) pa = 3u;
        if (bad) { pa = 0; g.bn |= 1u << c; }
        g.pend |= pa << (2 * c);
    }
}

// Error key of one group (codec.py:396-457 order per entry: BAD_OP, LEAF_STOP, op-specific).
__device__ __noinline__ unsigned long long group_errkey(uint32_t ent0, uint64_t w, uint64_t vmask, bool leaf,
                                                          uint32_t bn8) {
    unsigned long long k = ~0ull;
    const uint64_t bad = m_op7(w) & vmask;
    if (bad) k = umin64(k, ekey(ent0 + first_byte(bad), 0, CSV_ST_BAD_OP));
    if (leaf) {
        const uint64_t ls = (w >> 3) & ONES & vmask & ~bad;
        if (ls) k = umin64(k, ekey(ent0 + first_byte(ls), 1, CSV_ST_LEAF_STOP));
    }
    uint64_t bn = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) bn |= (uint64_t)((bn8 >> c) & 1u) << (8 * c);
    bn &= vmask;
    if (bn) k = umin64(k, ekey(ent0 + first_byte(bn), 2, CSV_ST_BAD_NEIGHBOR));
    return k;
}

// Palette ops of a group (P_last / P_delta / P_advance, codec.py:426-457):
// calls put(c, idx) for each; returns the first range-error key.
template <typename Put>
__device__ __forceinline__ unsigned long long palette_children(uint64_t w, uint64_t pmask, int32_t ipq, uint32_t plen,
                                                              uint32_t ent0, uint64_t vmask, Put put) {
    unsigned long long key = ~0ull;
    const uint64_t m6 = m_op6(w);
    while (pmask) {
        const uint32_t c = first_byte(pmask);
        pmask &= pmask - 1;
        const uint32_t e = (uint32_t)(w >> (8 * c)) & 0xFFu, op = e & 7u;
        const int32_t ip = ipq + (int32_t)prefix_bytes(m6, (int)c);
        int32_t idx = op == 4u ? ip : (op == 5u ? ip - (int32_t)(e >> 4) - 1 : ip + 1);
        const int st = idx < 0 ? CSV_ST_DELTA_RANGE : (idx >= (int32_t)plen ? CSV_ST_PALETTE_RANGE : 0);
        if (st && ((vmask >> (8 * c)) & 1u)) key = umin64(key, ekey(ent0 + c, 2, st));
        idx = min(max(idx, 0), (int32_t)plen - 1);
        put(c, (uint32_t)idx);
    }
    return key;
}

// Exact first-error key of a failing group (the per-child restatement; only
// runs when the SWAR evaluation flagged an error).
__device__ __noinline__ unsigned long long exact_key(uint64_t w, uint32_t bf, int32_t ipq, uint32_t plen, uint32_t ent0,
                                                     uint64_t vmask, bool leaf) {
    Group g;
    eval_group(w, 0u, 0u, 0u, 0u, bf, g);
    const uint64_t pmk = m_pal(w);
    unsigned long long pk = ~0ull;
    if (pmk) pk = palette_children(w, pmk, ipq, plen, ent0, vmask, [](uint32_t, uint32_t) {});
    return umin64(pk, group_errkey(ent0, w, vmask, leaf, g.bn));
}

struct Brick {
    uint64_t r;
    int N, t, n;
    uint32_t plen;
    const uint32_t* pal;
    Raster R;
    uint32_t pitch, plane;
    uint32_t* out_m;
    bool al8, al16;
    const uint32_t* spal;                // palette labels in shared memory (u8 mode)
    bool al16r;                          // raster rows may be written as 16-byte vectors
    const uint8_t* Ec;  uint32_t capc;   // coarse entries, entry capacity (bytes)
    const uint8_t* Ed;  uint32_t capd;
    uint16_t* ipb;                       // per-warp scratch: palette base per final-level active parent
    csv_stream_result src, srd;
};

// label of a palette index (shared copy in u8 mode)
template <typename IT>
__device__ __forceinline__ uint32_t label_of(const Brick& B, uint32_t idx) {
    return sizeof(IT) == 1 && K2W_SPAL ? B.spal[idx] : __ldg(B.pal + idx);
}

// raster voxel (x, y, z) of the brick at LOD t, nullptr if cropped (container.py:465-468)
__device__ __forceinline__ uint32_t* raster_xyz(const Raster& R, const Plan& P, uint32_t x, uint32_t y, uint32_t z) {
    const int64_t gx = R.ox + x, gy = R.oy + y, gz = R.oz + z;
    if (gz < P.z_begin || gz >= P.z_end || gy >= P.cy || gx >= P.cx) return nullptr;
    return P.out + ((gz - P.z_begin) * P.cy + gy) * P.cx + gx;
}

// one voxel plane of the final level to HBM, per voxel with cropping (edge bricks)
template <typename IT>
__device__ __noinline__ void plane_rows_slow(Raster R, const Plan& P, const uint32_t* spal, const uint32_t* pal,
                                             const IT* pl, uint32_t S2, uint32_t zz, int lane) {
    for (uint32_t e = lane; e < S2 * S2; e += 32) {
        uint32_t* const pp = raster_xyz(R, P, e % S2, e / S2, zz);
        if (pp) *pp = sizeof(IT) == 1 && K2W_SPAL ? spal[pl[e]] : __ldg(pal + pl[e]);
    }
}

// Store the 8 children (palette labels) of final-level parent q = (px, py, pz).
template <int MODE>
__device__ __forceinline__ void store_children(const Brick& B, const Plan& P, uint32_t q, uint32_t px, uint32_t py,
                                               uint32_t pz, const uint32_t (&lab)[8]) {
    if (MODE == OUT_MORTON) {
        uint32_t* g = B.out_m + 8ull * q;
        if (B.al16) {
            __stcs(reinterpret_cast<uint4*>(g), make_uint4(lab[0], lab[1], lab[2], lab[3]));   // streaming: keep
            __stcs(reinterpret_cast<uint4*>(g) + 1, make_uint4(lab[4], lab[5], lab[6], lab[7]));   // entries in L2
        } else {
#pragma unroll
            for (int c = 0; c < 8; ++c) g[c] = lab[c];
        }
    } else if (B.al8) {
        uint32_t* g = B.R.base + ((2 * pz) * B.plane + (2 * py) * B.pitch + 2 * px);
        *reinterpret_cast<uint2*>(g) = make_uint2(lab[0], lab[1]);
        *reinterpret_cast<uint2*>(g + B.pitch) = make_uint2(lab[2], lab[3]);
        *reinterpret_cast<uint2*>(g + B.plane) = make_uint2(lab[4], lab[5]);
        *reinterpret_cast<uint2*>(g + B.plane + B.pitch) = make_uint2(lab[6], lab[7]);
    } else {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            uint32_t* pp = raster_of(B.R, P, 8 * q + c);
            if (pp) *pp = lab[c];
        }
    }
}

// Error epilogue (warp): status/stream/nibble position of the winning key.
template <bool CG = false>
__device__ __noinline__ void report_error(const Plan& P, uint64_t r, const uint8_t* Eb, uint32_t ecap,
                                          csv_stream_result sr, unsigned long long ek, bool leaf, int lane) {
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
        uint32_t cnt = 0;      // nibble index of entry `ent` = ent + #payload nibbles before it
        for (uint32_t g = lane; g < (ent + 7) / 8; g += 32) {
            uint64_t w = (8 * g + 8 <= ecap) ? ldent<CG>(reinterpret_cast<const uint64_t*>(Eb) + g) : 0ull;
            uint32_t lim = ent - 8 * g;
            uint64_t m = m_op5(w);
            if (lim < 8) m &= (1ull << (8 * lim)) - 1ull;
            cnt += __popcll(m);
        }
        pos = (int64_t)ent + (int64_t)warp_sum(cnt);
        st = code;
        if (code == CSV_ST_DELTA_RANGE) pos += 1;   // reported at the payload nibble
    }
    if (lane == 0) put_result(P, r, st, leaf ? 1 : 0, pos, 0, 0);
}

// pending-descriptor masks (2 bits per child) of the three chain rounds:
// children 3,5,6 (targets: child 7), 1,2,4 (targets 3,5,6), 0 (targets 1,2,4)
constexpr uint32_t kClass1 = (3u << 6) | (3u << 10) | (3u << 12);
constexpr uint32_t kClass2 = (3u << 2) | (3u << 4) | (3u << 8);
constexpr uint32_t kClass3 = 3u;

// -1 / +1 neighbour along an axis of Morton index j (the axis' bits selected by M)
__device__ __forceinline__ uint32_t morton_dec(uint32_t j, uint32_t M) { return (((j & M) - 1u) & M) | (j & ~M); }
__device__ __forceinline__ uint32_t morton_inc(uint32_t j, uint32_t M) { return ((((j & M) | ~M) + 1u) & M) | (j & ~M); }

// ---------------------------------------------------------------- coarse level (Morton, smem)
// Parents at level N - j (j bits per axis), children kept in the level array.
// Returns the warp-uniform error key; adds the level's payload nibbles to pdl.
template <typename IT, bool CG = false>
__device__ __forceinline__ unsigned long long coarse_level(const Brick& B, int j, IT* lev, const uint32_t* pm,
                                                          uint32_t* cm, uint16_t* wpre, uint16_t* list,
                                                          uint16_t* pdesc, uint32_t& cur_c, uint32_t& ip_run,
                                                          uint32_t& pdl, int lane, IT* fin = nullptr) {
    const uint32_t Pn = 1u << (3 * j);
    const uint32_t W = (Pn + 31) >> 5;
    const IT* plev = lev + wofs(j);
    IT* clev = fin ? fin : lev + wofs(j + 1);   // fin: the final parent level lives in global scratch
    const uint32_t Mx = axis_mask(0, j), My = axis_mask(1, j), Mz = axis_mask(2, j);        // parent level
    const uint32_t Cx = axis_mask(0, j + 1), Cy = axis_mask(1, j + 1), Cz = axis_mask(2, j + 1);   // child level
    const uint32_t nact = rank_prefix(pm, W, wpre, lane);
    const uint32_t e0 = cur_c, nvalid = B.src.n_entries;
    unsigned long long ek = ~0ull;
    if ((uint64_t)e0 + 8ull * nact > nvalid) ek = ekey(nvalid, 0, EK_UNDERRUN_NV);
    const uint32_t CW = (8 * Pn + 31) >> 5;
    for (uint32_t i = lane; i < CW; i += 32) cm[i] = 0u;
    // fill: children repeat the parent (codec.py:458-463); active list by rank
    for (uint32_t q0 = 0; q0 < Pn; q0 += 32) {
        const uint32_t q = q0 + lane;
        if (q < Pn) {
            store8_same<IT>(clev + 8 * q, plev[q]);
            const uint32_t mw = pm[q >> 5];
            if ((mw >> (q & 31)) & 1u) list[wpre[q >> 5] + __popc(mw & ((1u << (q & 31)) - 1u))] = (uint16_t)q;
        }
    }
    __syncwarp();
    uint8_t* const cmb = reinterpret_cast<uint8_t*>(cm);
    uint32_t anyp = 0;
    for (uint32_t k0 = 0; k0 < nact; k0 += 32) {
        const uint32_t k = k0 + lane;
        const uint32_t ent0 = e0 + 8 * k;
        const uint64_t w = (k < nact && ent0 + 8 <= B.capc) ? ldent<CG>(reinterpret_cast<const uint64_t*>(B.Ec + ent0)) : 0ull;
        // palette base: i_p advances (P_a) of the preceding parents, in entry order (codec.py:453-457)
        const uint32_t c6 = __popcll(m_op6(w)), inc6 = warp_incl(c6, lane);
        const int32_t ipq = (int32_t)(ip_run + inc6 - c6);
        ip_run += __shfl_sync(FULL, inc6, 31);
        if (k < nact) {
            const uint32_t q = list[k];
            const uint64_t vmask = valid_mask(nvalid, ent0);
            pdl += __popcll(m_op5(w) & vmask);
            const uint32_t pv = plev[q];
            const uint32_t qx = q & Mx, qy = q & My, qz = q & Mz;
            const uint32_t bf = (qx == 0) | ((qx == Mx) << 1) | ((qy == 0) << 2) | ((qy == My) << 3) |
                                ((qz == 0) << 4) | ((qz == Mz) << 5);
            const uint32_t pxp = qx != Mx ? plev[morton_inc(q, Mx)] : 0u;
            const uint32_t pyp = qy != My ? plev[morton_inc(q, My)] : 0u;
            const uint32_t pzp = qz != Mz ? plev[morton_inc(q, Mz)] : 0u;
            cmb[q] = (uint8_t)(((~(w >> 3) & ONES) * 0x0102040810204080ull) >> 56);   // no stop: visited next level
            if constexpr (sizeof(IT) == 1) {
                e8::Out g;
                e8::eval8<true>(w, pv, pxp, pyp, pzp, bf, ipq, B.plen, vmask, false, g);   // pending: markers
                *reinterpret_cast<uint2*>(clev + 8 * q) = make_uint2(g.vlo, g.vhi);
                pdesc[k] = (uint16_t)g.pend;
                anyp |= g.pend;
                if (g.err) ek = umin64(ek, exact_key(w, bf, ipq, B.plen, ent0, vmask, false));
            } else {
                Group g;
                eval_group(w, pv, pxp, pyp, pzp, bf, g);
                store8<IT>(clev + 8 * q, g.v);
                pdesc[k] = (uint16_t)g.pend;
                anyp |= g.pend;
                const uint64_t pmk = m_pal(w);
                unsigned long long pk = ~0ull;
                if (pmk) {
                    pk = palette_children(w, pmk, ipq, B.plen, ent0, vmask,
                                          [&](uint32_t c, uint32_t idx) { clev[8 * q + c] = (IT)idx; });
                }
                if (((m_op7(w) & vmask) != 0) | (g.bn != 0) | (pk != ~0ull))
                    ek = umin64(ek, umin64(pk, group_errkey(ent0, w, vmask, false, g.bn)));
            }
        }
    }
    __syncwarp();
    if (sizeof(IT) == 1 && __any_sync(FULL, anyp != 0u)) {
        // u8: one pass.  A pending child holds the marker 252 + axis; it copies the -1
        // neighbour on that axis (codec.py:422-423), following markers (at most three hops,
        // each adds an odd coordinate) until a final value.  The warp reads first and the
        // parents' 8-child words are rewritten after a __syncwarp.
#pragma unroll 1
        for (uint32_t k0 = 0; k0 < nact; k0 += 32) {
            const uint32_t k = k0 + lane;
            uint32_t m = k < nact ? (uint32_t)pdesc[k] : 0u;
            const uint32_t q = m ? list[k] : 0u;
            uint32_t nlo = 0, nhi = 0, mlo = 0, mhi = 0;
            while (m) {
                const uint32_t c = (uint32_t)(__ffs(m) - 1) >> 1;
                uint32_t a = (m >> (2 * c)) & 3u;
                m &= ~(3u << (2 * c));
                uint32_t src = (q << 3) | c, v;
#pragma unroll 1
                do {
                    src = morton_dec(src, a == 1u ? Cx : (a == 2u ? Cy : Cz));
                    v = clev[src];
                    a = v - 252u;
                } while (v >= 253u);
                if (c < 4) { nlo |= v << (8 * c); mlo |= 0xFFu << (8 * c); }
                else { nhi |= v << (8 * (c - 4)); mhi |= 0xFFu << (8 * (c - 4)); }
            }
            __syncwarp();
            if (mlo | mhi) {
                uint2* const p = reinterpret_cast<uint2*>(clev + 8 * q);
                const uint2 o = *p;
                *p = make_uint2((o.x & ~mlo) | nlo, (o.y & ~mhi) | nhi);
            }
            __syncwarp();
        }
    } else if (__any_sync(FULL, anyp != 0u)) {
        // rounds by decreasing popcount of the child index: targets are final
#pragma unroll 1
        for (int rd = 0; rd < 3; ++rd) {
            const uint32_t cls = rd == 0 ? kClass1 : (rd == 1 ? kClass2 : kClass3);
#pragma unroll 1
            for (uint32_t k0 = 0; k0 < nact; k0 += 32) {
                const uint32_t k = k0 + lane;
                uint32_t m = k < nact ? (uint32_t)pdesc[k] & cls : 0u;
                const uint32_t q = m ? list[k] : 0u;
                while (m) {
                    const uint32_t c = (uint32_t)(__ffs(m) - 1) >> 1;
                    const uint32_t a1 = (m >> (2 * c)) & 3u;
                    m &= ~(3u << (2 * c));
                    const uint32_t M = a1 == 1 ? Cx : (a1 == 2 ? Cy : Cz);
                    const uint32_t jj = (q << 3) | c;
                    clev[jj] = clev[morton_dec(jj, M)];
                }
            }
            __syncwarp();
        }
    }
    cur_c = e0 + 8 * nact;
    return warp_min64(ek);
}

__host__ __device__ __forceinline__ constexpr uint32_t spread3_c(uint32_t v) {   // spread3 of a (compile-time) coordinate < 32
    return (v & 1u) | ((v & 2u) << 2) | ((v & 4u) << 4) | ((v & 8u) << 6) | ((v & 16u) << 8);
}
// ---------------------------------------------------------------- final level (plane sweep)
// offset of child c (x, y bits) of plane parent i = px + RR * py inside a ring voxel plane
template <int RR>
__device__ __forceinline__ uint32_t child_off(uint32_t i, uint32_t c) {
    return (2 * (i / RR) + ((c >> 1) & 1u)) * (2 * RR) + 2 * (i % RR) + (c & 1u);
}

// Ring voxel plane z (u16, (2R)^2) at ring + (z % 3) * (2R)^2; child (cx, cy) at cy * 2R + cx.
template <int MODE, int RR, typename IT, bool CG = false>
__device__ __forceinline__ unsigned long long final_sweep(const Brick& B, const Plan& P, const IT* plev,
                                                         const uint32_t* pm, uint16_t* wpre, IT* ring,
                                                         uint8_t* plist, uint16_t* pdesc, uint32_t* amask,
                                                         uint32_t& cur, uint32_t& ip_run, uint32_t& pdl, int lane) {
    constexpr uint32_t Pn = RR * RR * RR, W = (Pn + 31) / 32;
    constexpr uint32_t PP = RR * RR;                    // parents per plane
    constexpr uint32_t S2 = 2 * RR;                     // children per row
    constexpr uint32_t PL = S2 * S2;                    // u16 per voxel plane
    constexpr uint32_t AW = (PP + 31) / 32;             // active-mask words per plane
    uint16_t* const apre = reinterpret_cast<uint16_t*>(amask + AW);
    const bool leaf = B.t == 0;
    const uint32_t nact = rank_prefix(pm, W, wpre, lane);
    const uint8_t* const E = leaf ? B.Ed : B.Ec;
    const uint32_t cap = leaf ? B.capd : B.capc;
    const uint32_t nvalid = leaf ? B.srd.n_entries : B.src.n_entries;
    const uint32_t e0 = cur;
    unsigned long long ek = ~0ull;
    if ((uint64_t)e0 + 8ull * nact > nvalid) ek = ekey(nvalid, 0, EK_UNDERRUN_NV);
    // palette base per active parent, in entry (rank) order (codec.py:453-457) -> per-warp scratch
    {
        auto ld = [&](uint32_t k) -> uint64_t {
            const uint32_t ent0 = e0 + 8 * k;
            return (k < nact && ent0 + 8 <= cap) ? ldent<CG>(reinterpret_cast<const uint64_t*>(E + ent0)) : 0ull;
        };
        uint64_t wn = ld(lane), wnn = ld(32 + lane);   // two chunks in flight
        for (uint32_t k0 = 0; k0 < nact; k0 += 32) {
            const uint32_t k = k0 + lane;
            const uint64_t w = wn;
            wn = wnn;
            wnn = ld(k0 + 64 + lane);
            const uint32_t c6 = __popcll(m_op6(w)), inc6 = warp_incl(c6, lane);
            if (k < nact) B.ipb[k] = (uint16_t)(ip_run + inc6 - c6);
            ip_run += __shfl_sync(FULL, inc6, 31);
        }
    }
    __syncwarp();
    using P2 = typename IX<IT>::P2;
    P2* const ring2 = reinterpret_cast<P2*>(ring);
    for (uint32_t pz = 0; pz < RR; ++pz) {
        const uint32_t sz = spread3_u32(pz) << 2;
        P2* const r0 = ring2 + ((2 * pz) % 3) * (PL / 2);       // voxel plane 2pz   (2 children in x per P2)
        P2* const r1 = ring2 + ((2 * pz + 1) % 3) * (PL / 2);   // voxel plane 2pz+1
        // ---- fill: ring <- parent values; inactive parents straight to HBM; active list
        uint32_t nl = 0;
        for (uint32_t i0 = 0; i0 < PP; i0 += 32) {
            const uint32_t i = i0 + lane;
            const bool ok = i < PP;
            const uint32_t px = i % RR, py = i / RR;
            const uint32_t q = spread3_u32(px) | (spread3_u32(py) << 1) | sz;
            uint32_t mw = 0, pv = 0;
            if (ok) {
                pv = plev[q];
                mw = pm[q >> 5];
            }
            const bool act = ok && ((mw >> (q & 31)) & 1u);
            if (ok && !act) {   // active parents' children are all written by the active pass
                const P2 pp = pack2<IT>(pv, pv);
                r0[(2 * py) * RR + px] = pp;
                r0[(2 * py + 1) * RR + px] = pp;
                r1[(2 * py) * RR + px] = pp;
                r1[(2 * py + 1) * RR + px] = pp;
            }
            const uint32_t bal = __ballot_sync(FULL, act);
            if (lane == 0 && i0 < PP) {
                amask[i0 >> 5] = bal;
                apre[i0 >> 5] = (uint16_t)nl;
            }
            if (act) {
                plist[nl + __popc(bal & lanemask_lt(lane))] = (uint8_t)i;
            } else if (MODE == OUT_MORTON && ok) {
                const uint32_t l = label_of<IT>(B, pv);
                const uint32_t lab[8] = {l, l, l, l, l, l, l, l};
                store_children<MODE>(B, P, q, px, py, pz, lab);
            }
            nl += __popc(bal);
        }
        __syncwarp();
        // ---- active parents of this plane: one lane each
        uint32_t anyp = 0;
        for (uint32_t k0 = 0; k0 < nl; k0 += 32) {
            const uint32_t k = k0 + lane;
            if (k < nl) {
                const uint32_t i = plist[k];
                const uint32_t px = i % RR, py = i / RR;
                const uint32_t sx = spread3_u32(px), sy = spread3_u32(py) << 1;
                const uint32_t q = sx | sy | sz;
                const uint32_t rank = wpre[q >> 5] + __popc(pm[q >> 5] & ((1u << (q & 31)) - 1u));
                const uint32_t ent0 = e0 + 8 * rank;
                const uint64_t w = ent0 + 8 <= cap ? ldent<CG>(reinterpret_cast<const uint64_t*>(E + ent0)) : 0ull;
                const uint64_t vmask = valid_mask(nvalid, ent0);
                const uint32_t pv = plev[q];
                const uint32_t bf = (px == 0) | ((px == RR - 1) << 1) | ((py == 0) << 2) | ((py == RR - 1) << 3) |
                                    ((pz == 0) << 4) | ((pz == RR - 1) << 5);
                const uint32_t pxp = px + 1 < RR ? plev[spread3_u32(px + 1) | sy | sz] : 0u;
                const uint32_t pyp = py + 1 < RR ? plev[sx | (spread3_u32(py + 1) << 1) | sz] : 0u;
                const uint32_t pzp = pz + 1 < RR ? plev[sx | sy | (spread3_u32(pz + 1) << 2)] : 0u;
                if constexpr (sizeof(IT) == 1) {
                    // palette base only when the group has palette ops (op bit 2)
                    const int32_t ipq = (w & 0x0404040404040404ull) ? (int32_t)B.ipb[rank] : 0;
                    e8::Out g;
                    e8::eval8(w, pv, pxp, pyp, pzp, bf, ipq, B.plen, vmask, leaf, g);
                    pdl += g.n5;
                    r0[(2 * py) * RR + px] = (P2)(g.vlo & 0xFFFFu);
                    r0[(2 * py + 1) * RR + px] = (P2)(g.vlo >> 16);
                    r1[(2 * py) * RR + px] = (P2)(g.vhi & 0xFFFFu);
                    r1[(2 * py + 1) * RR + px] = (P2)(g.vhi >> 16);
                    pdesc[k] = (uint16_t)g.pend;
                    anyp |= g.pend;
                    if (g.err) ek = umin64(ek, exact_key(w, bf, ipq, B.plen, ent0, vmask, leaf));
                    continue;
                }
                pdl += __popcll(m_op5(w) & vmask);
                Group g;
                eval_group(w, pv, pxp, pyp, pzp, bf, g);
                r0[(2 * py) * RR + px] = pack2<IT>(g.v[0], g.v[1]);
                r0[(2 * py + 1) * RR + px] = pack2<IT>(g.v[2], g.v[3]);
                r1[(2 * py) * RR + px] = pack2<IT>(g.v[4], g.v[5]);
                r1[(2 * py + 1) * RR + px] = pack2<IT>(g.v[6], g.v[7]);
                pdesc[k] = (uint16_t)g.pend;
                anyp |= g.pend;
                const uint64_t pmk = m_pal(w);
                unsigned long long pk = ~0ull;
                if (pmk) {
                    const int32_t ipq = B.ipb[rank];
                    IT* const p0 = reinterpret_cast<IT*>(r0);
                    IT* const p1 = reinterpret_cast<IT*>(r1);
                    pk = palette_children(w, pmk, ipq, B.plen, ent0, vmask, [&](uint32_t c, uint32_t idx) {
                        IT* pl = (c & 4) ? p1 : p0;
                        pl[(2 * py + ((c >> 1) & 1)) * S2 + 2 * px + (c & 1)] = (IT)idx;
                    });
                }
                const uint64_t errs = m_op7(w) | (leaf ? (w >> 3) & ONES : 0ull);
                if (((errs & vmask) != 0) | (g.bn != 0) | (pk != ~0ull))
                    ek = umin64(ek, umin64(pk, group_errkey(ent0, w, vmask, leaf, g.bn)));
            }
        }
        __syncwarp();
        const IT* const pr = ring + ((2 * pz + 2) % 3) * PL;   // voxel plane 2pz-1
        IT* const p0 = ring + ((2 * pz) % 3) * PL;
        IT* const p1 = ring + ((2 * pz + 1) % 3) * PL;
        // ---- pending chains: child c of an active parent copies child c | (1 << axis) of
        // the -1 neighbour parent (codec.py:422-423); that child is final unless it is
        // itself pending (one more odd coordinate, so at most three hops), or lies in the
        // previous voxel plane (z), which is final.  One pass, no rounds.
        if (__any_sync(FULL, anyp != 0u)) {
#pragma unroll 1
            for (uint32_t k0 = 0; k0 < nl; k0 += 32) {
                const uint32_t k = k0 + lane;
                uint32_t d = k < nl ? (uint32_t)pdesc[k] : 0u;
                if (!__any_sync(FULL, d != 0u)) continue;
                const uint32_t i = d ? plist[k] : 0u;
                while (d) {
                    const uint32_t c = (uint32_t)(__ffs(d) - 1) >> 1;
                    uint32_t a = (d >> (2 * c)) & 3u;
                    d &= ~(3u << (2 * c));
                    uint32_t ii = i, cc = c;
                    const IT* src;
#pragma unroll 1
                    for (;;) {
                        cc |= 1u << (a - 1u);
                        if (a == 3u) { src = pr + child_off<RR>(ii, cc); break; }
                        ii -= a == 1u ? 1u : RR;
                        const uint32_t wd = amask[ii >> 5], bit = 1u << (ii & 31);
                        uint32_t a2 = 0;
                        if (wd & bit) a2 = ((uint32_t)pdesc[apre[ii >> 5] + __popc(wd & (bit - 1u))] >> (2 * cc)) & 3u;
                        if (a2 == 0u) { src = ((cc & 4) ? p1 : p0) + child_off<RR>(ii, cc); break; }
                        a = a2;
                    }
                    (((c & 4) ? p1 : p0) + child_off<RR>(i, c))[0] = *src;
                }
            }
            __syncwarp();
        }
        if (MODE == OUT_RASTER) {
            // ---- the plane pair to HBM as whole rows (each sector written once)
#pragma unroll 1
            for (int dz = 0; dz < 2; ++dz) {
                const IT* const pl = dz ? p1 : p0;
                const uint32_t zz = 2 * pz + dz;
                if (S2 >= 4 && B.al16r) {
                    uint32_t* const zb = B.R.base + zz * B.plane;
                    for (uint32_t e = 4 * lane; e < PL; e += 128) {
                        uint32_t v0, v1, v2, v3;
                        if (sizeof(IT) == 1) {
                            const uint32_t x = *reinterpret_cast<const uint32_t*>(pl + e);
                            v0 = x & 0xFFu; v1 = (x >> 8) & 0xFFu; v2 = (x >> 16) & 0xFFu; v3 = x >> 24;
                        } else {
                            const uint2 x = *reinterpret_cast<const uint2*>(pl + e);
                            v0 = x.x & 0xFFFFu; v1 = x.x >> 16; v2 = x.y & 0xFFFFu; v3 = x.y >> 16;
                        }
                        const uint4 lab = make_uint4(label_of<IT>(B, v0), label_of<IT>(B, v1), label_of<IT>(B, v2),
                                                     label_of<IT>(B, v3));
                        __stcs(reinterpret_cast<uint4*>(zb + (e / S2) * B.pitch + (e % S2)), lab);   // evict-first
                    }
                } else {
                    plane_rows_slow<IT>(B.R, P, B.spal, B.pal, pl, S2, zz, lane);
                }
            }
        } else {
        // ---- active parents to HBM (Morton: 8 children = one 32-byte sector)
        for (uint32_t k0 = 0; k0 < nl; k0 += 32) {
            const uint32_t k = k0 + lane;
            if (k < nl) {
                const uint32_t i = plist[k];
                const uint32_t px = i % RR, py = i / RR;
                const uint32_t q = spread3_u32(px) | (spread3_u32(py) << 1) | sz;
                const P2* const q0 = reinterpret_cast<const P2*>(p0);
                const P2* const q1 = reinterpret_cast<const P2*>(p1);
                const uint32_t a = q0[(2 * py) * RR + px], b = q0[(2 * py + 1) * RR + px];
                const uint32_t c = q1[(2 * py) * RR + px], d = q1[(2 * py + 1) * RR + px];
                const uint32_t vv[8] = {lo2<IT>(a), hi2<IT>(a), lo2<IT>(b), hi2<IT>(b), lo2<IT>(c), hi2<IT>(c), lo2<IT>(d), hi2<IT>(d)};
                uint32_t lab[8];
#pragma unroll
                for (int cc = 0; cc < 8; ++cc) lab[cc] = label_of<IT>(B, vv[cc]);
                store_children<MODE>(B, P, q, px, py, pz, lab);
            }
        }
        }
        __syncwarp();
    }
    cur = e0 + 8 * nact;
    return warp_min64(ek);
}

// One voxel plane's rows of one parity: resolve the chain markers word by word
// (4 children per lane), write the words back where later phases / the next
// plane read them, and (fast raster) store the labels as whole 16-byte rows.
//   DZ = 0: even voxel plane 2pz (z markers from the previous plane `pr`),
//   PH = 0: odd rows (no y markers), PH = 1: even rows (y from the odd row above).
__device__ __forceinline__ uint32_t marker_bytes(uint32_t x) {   // bit 7 of every byte >= 253
    return ((x & 0x7F7F7F7Fu) + 0x03030303u) & x & 0x80808080u;
}
// z / y step of one word: markers of axis (a0, a1 at bit 7) take the source word's byte
__device__ __forceinline__ uint32_t take_bytes(uint32_t y, uint32_t m7, uint32_t src) {
    const uint32_t M = (m7 >> 7) * 0xFFu;
    return (y & ~M) | (src & M);
}

template <int RR, int DZ, int PH>
__device__ __forceinline__ void resolve_rows(const Brick& B, uint8_t* pl, const uint8_t* pr, bool fast, uint32_t* zb,
                                             int lane) {
    static_assert(K2W_SPAL, "the u8 pass reads labels from the shared palette copy");
    // one lane = 8 children (two words) of a row; RPI row pairs per warp iteration
    constexpr uint32_t S2 = 2 * RR, WPR = S2 / 8, HW = RR * RR / 4, RPI = 32 / WPR;
    const uint32_t rp0 = lane / WPR, cw = lane % WPR;
    const uint32_t row0 = 2 * rp0 + (PH ? 0u : 1u);
    uint2* wp = reinterpret_cast<uint2*>(pl + row0 * S2) + cw;
    const uint2* pw = reinterpret_cast<const uint2*>(pr + row0 * S2) + cw;
    uint32_t* op = fast ? zb + row0 * B.pitch + 8 * cw : nullptr;
    const uint8_t* const lab = reinterpret_cast<const uint8_t*>(B.spal);
    // write-back needed unless nothing reads these words again (even rows of the even plane, fast raster)
    const bool keep = !(DZ == 0 && PH == 1) || !fast;
#pragma unroll kRUnroll
    for (uint32_t w0 = 0; w0 < HW; w0 += 32) {
        const bool okw = HW >= 32 || lane < (int)HW;
        const uint2 x = okw ? *wp : make_uint2(0u, 0u);
        const uint32_t f0 = marker_bytes(x.x), f1 = marker_bytes(x.y);
        const uint32_t a00 = x.x << 7, a01 = x.x << 6, a10 = x.y << 7, a11 = x.y << 6;   // axis bits at bit 7
        uint32_t y0 = x.x, y1 = x.y;
        if (DZ == 0) {   // z: the previous voxel plane (final)
            const uint2 z = okw ? *pw : make_uint2(0u, 0u);
            y0 = take_bytes(y0, f0 & a00 & a01, z.x);
            y1 = take_bytes(y1, f1 & a10 & a11, z.y);
        }
        if (PH == 1) {   // y: the odd row above (resolved in phase 0)
            const uint2 u = okw ? *(wp - WPR) : make_uint2(0u, 0u);
            y0 = take_bytes(y0, f0 & ~a00 & a01, u.x);
            y1 = take_bytes(y1, f1 & ~a10 & a11, u.y);
        }
        // x: the byte to the left (word 0's byte 0 from the left lane's word 1; odd-x sources are final)
        const uint32_t left = __shfl_up_sync(FULL, y1, 1);
        y0 = take_bytes(y0, f0 & a00 & ~a01, __byte_perm(y0, left, 0x2107));
        y1 = take_bytes(y1, f1 & a10 & ~a11, __byte_perm(y1, y0, 0x2107));
        if (keep && (f0 | f1)) *wp = make_uint2(y0, y1);
        if (fast && okw) {
            const uint4 v0 = make_uint4(*reinterpret_cast<const uint32_t*>(lab + 4 * __byte_perm(y0, 0, 0x4440)),
                                        *reinterpret_cast<const uint32_t*>(lab + 4 * __byte_perm(y0, 0, 0x4441)),
                                        *reinterpret_cast<const uint32_t*>(lab + 4 * __byte_perm(y0, 0, 0x4442)),
                                        *reinterpret_cast<const uint32_t*>(lab + 4 * __byte_perm(y0, 0, 0x4443)));
            const uint4 v1 = make_uint4(*reinterpret_cast<const uint32_t*>(lab + 4 * __byte_perm(y1, 0, 0x4440)),
                                        *reinterpret_cast<const uint32_t*>(lab + 4 * __byte_perm(y1, 0, 0x4441)),
                                        *reinterpret_cast<const uint32_t*>(lab + 4 * __byte_perm(y1, 0, 0x4442)),
                                        *reinterpret_cast<const uint32_t*>(lab + 4 * __byte_perm(y1, 0, 0x4443)));
            __stcs(reinterpret_cast<uint4*>(op), v0);   // evict-first
            __stcs(reinterpret_cast<uint4*>(op) + 1, v1);
            op += 2 * RPI * B.pitch;
        }
        wp += 2 * RPI * WPR;
        pw += 2 * RPI * WPR;
    }
    __syncwarp();
}

// ---------------------------------------------------------------- final level, u8 (marker chains)
// The u8 pass (palettes of <= 253 labels, indices <= 252) leaves every pending
// child as the marker byte 252 + axis (e8::eval8<true>) and resolves the chains
// word by word over the ring rows instead of per child:
//   * a pending child copies the -1 neighbour on its axis (codec.py:422-423);
//     x-pending children sit at even x, y at even y, z at even z;
//   * odd rows have no y markers, and their x markers' sources (odd x) are
//     final once the z markers are: phase 0 resolves odd rows (z from the
//     previous voxel plane, then x from the byte to the left, a byte_perm with
//     the left lane's word);
//   * phase 1 resolves even rows: z, y from the already resolved odd row
//     above, then x.
// Resolution is fused with the whole-row raster write (each 16-byte row chunk
// is resolved, written back for later readers and stored as labels).
template <int MODE, int RR, bool CG = false>
__device__ __forceinline__ unsigned long long final_sweep8(const Brick& B, const Plan& P, const uint8_t* plev,
                                                          const uint32_t* pm, uint16_t* wpre, uint8_t* ring,
                                                          uint8_t* plist_raw, uint32_t& cur, uint32_t& ip_run,
                                                          uint32_t& pdl, int lane) {
    static_assert(RR >= 4, "word-wise rows need >= 8 children per row");
    using PLT = typename std::conditional<(RR > 16), uint16_t, uint8_t>::type;   // plane index of an active parent
    PLT* const plist = reinterpret_cast<PLT*>(plist_raw);
    constexpr int kFillUnroll = RR <= 16 ? 8 : 1;   // RR <= 16: Morton parts of the fill are compile-time
    constexpr uint32_t Pn = RR * RR * RR, W = (Pn + 31) / 32;
    constexpr uint32_t PP = RR * RR;           // parents per plane
    constexpr uint32_t S2 = 2 * RR;            // children (bytes) per row
    constexpr uint32_t PL = S2 * S2;           // bytes per voxel plane
    constexpr uint32_t LG = RR == 4 ? 2 : (RR == 8 ? 3 : (RR == 16 ? 4 : 5));
    constexpr uint32_t MX = 0x49249u & ((1u << (3 * LG)) - 1u), MY = MX << 1, MZ = MX << 2;
    const bool leaf = B.t == 0;
    const uint32_t nact = rank_prefix(pm, W, wpre, lane);
    const uint8_t* const E = leaf ? B.Ed : B.Ec;
    const uint32_t cap = leaf ? B.capd : B.capc;
    const uint32_t nvalid = leaf ? B.srd.n_entries : B.src.n_entries;
    const uint32_t e0 = cur;
    unsigned long long ek = ~0ull;
    if ((uint64_t)e0 + 8ull * nact > nvalid) ek = ekey(nvalid, 0, EK_UNDERRUN_NV);
    {   // palette base per active parent, in entry (rank) order (codec.py:453-457) -> per-warp scratch
        auto ld = [&](uint32_t k) -> uint64_t {
            const uint32_t ent0 = e0 + 8 * k;
            return (k < nact && ent0 + 8 <= cap) ? ldent<CG>(reinterpret_cast<const uint64_t*>(E + ent0)) : 0ull;
        };
        uint64_t wn = ld(lane), wnn = ld(32 + lane);
        for (uint32_t k0 = 0; k0 < nact; k0 += 32) {
            const uint32_t k = k0 + lane;
            const uint64_t w = wn;
            wn = wnn;
            wnn = ld(k0 + 64 + lane);
            const uint32_t c6 = __popcll(m_op6(w)), inc6 = warp_incl(c6, lane);
            if (k < nact) B.ipb[k] = (uint16_t)(ip_run + inc6 - c6);
            ip_run += __shfl_sync(FULL, inc6, 31);
        }
    }
    __syncwarp();
    const bool fast = MODE == OUT_RASTER && B.al16r;
    const uint32_t qlane = spread3_u32(2 * (lane % (RR / 2))) | (spread3_u32((lane / (RR / 2)) % RR) << 1);
#pragma unroll 1
    for (uint32_t pz = 0; pz < RR; ++pz) {
        const uint32_t sz = spread3_u32(pz) << 2;
        uint8_t* const r0 = ring + ((2 * pz) % 3) * PL;         // voxel plane 2pz
        uint8_t* const r1 = ring + ((2 * pz + 1) % 3) * PL;     // voxel plane 2pz+1
        const uint8_t* const pr = ring + ((2 * pz + 2) % 3) * PL;   // voxel plane 2pz-1 (final)
        uint16_t* const h0 = reinterpret_cast<uint16_t*>(r0);
        uint16_t* const h1 = reinterpret_cast<uint16_t*>(r1);
        // ---- fill: every parent's children = the parent value (ring; Morton: inactive ones to HBM),
        // two x-adjacent parents per lane (Morton codes q, q | 1: one u16 load, one u32 store per row);
        // active parents are listed (and overwritten by the active pass)
        uint32_t nl = 0;
#pragma unroll kFillUnroll
        for (uint32_t i0 = 0; i0 < PP / 2; i0 += 32) {
            const uint32_t j = i0 + lane;
            const bool ok = j < PP / 2;
            const uint32_t px = 2 * (j % (RR / 2)), py = j / (RR / 2);
            // i0 / (RR/2) and lane / (RR/2) have disjoint bits: the Morton code splits into a
            // per-lane part and a (compile-time when unrolled) part of this iteration
            const uint32_t q = qlane | (spread3_c(i0 / (RR / 2)) << 1) | sz;
            uint32_t mw = 0, pv2 = 0;
            if (ok) {
                pv2 = *reinterpret_cast<const uint16_t*>(plev + q);   // parents q and q | 1
                mw = pm[q >> 5] >> (q & 31);
            }
            const bool act0 = ok && (mw & 1u), act1 = ok && (mw & 2u);
            if (ok) {
                const uint32_t pp = (pv2 & 0xFFu) * 0x0101u | (pv2 >> 8) * 0x01010000u;
                uint32_t* const w0 = reinterpret_cast<uint32_t*>(r0 + (2 * py) * S2 + 2 * px);
                uint32_t* const w1 = reinterpret_cast<uint32_t*>(r1 + (2 * py) * S2 + 2 * px);
                w0[0] = pp;
                w0[S2 / 4] = pp;
                w1[0] = pp;
                w1[S2 / 4] = pp;
                if (MODE == OUT_MORTON) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        if (h ? act1 : act0) continue;
                        const uint32_t l = label_of<uint8_t>(B, h ? pv2 >> 8 : pv2 & 0xFFu);
                        const uint32_t lab[8] = {l, l, l, l, l, l, l, l};
                        store_children<MODE>(B, P, q | (uint32_t)h, px + h, py, pz, lab);
                    }
                }
            }
            const uint32_t bal0 = __ballot_sync(FULL, act0), bal1 = __ballot_sync(FULL, act1);
            const uint32_t lt = lanemask_lt(lane);
            const uint32_t i = py * RR + px;
            if (act0) plist[nl + __popc(bal0 & lt)] = (PLT)i;
            if (act1) plist[nl + __popc(bal0) + __popc(bal1 & lt)] = (PLT)(i + 1);
            nl += __popc(bal0) + __popc(bal1);
        }
        __syncwarp();
        // ---- active parents: one lane each, SWAR evaluation, pending children as markers
        for (uint32_t k0 = 0; k0 < nl; k0 += 32) {
            const uint32_t k = k0 + lane;
            if (k < nl) {
                const uint32_t i = plist[k];
                const uint32_t px = i % RR, py = i / RR;
                const uint32_t q = spread3_u32(px) | (spread3_u32(py) << 1) | sz;
                const uint32_t rank = wpre[q >> 5] + __popc(pm[q >> 5] & ((1u << (q & 31)) - 1u));
                const uint32_t ent0 = e0 + 8 * rank;
                const uint64_t w = ent0 + 8 <= cap ? ldent<CG>(reinterpret_cast<const uint64_t*>(E + ent0)) : 0ull;
                const uint64_t vmask = valid_mask(nvalid, ent0);
                const uint32_t pv = plev[q];
                const uint32_t bf = (px == 0) | ((px == RR - 1) << 1) | ((py == 0) << 2) | ((py == RR - 1) << 3) |
                                    ((pz == 0) << 4) | ((pz == RR - 1) << 5);
                // +1 neighbours (wrap around at the maximum: value unused, BAD_NEIGHBOR)
                const uint32_t pxp = plev[morton_inc(q, MX)];
                const uint32_t pyp = plev[morton_inc(q, MY)];
                const uint32_t pzp = plev[morton_inc(q, MZ)];
                const int32_t ipq = B.ipb[rank];   // (issued with the entry load, not after it)
                e8::Out g;
                e8::eval8<true>(w, pv, pxp, pyp, pzp, bf, ipq, B.plen, vmask, leaf, g);
                pdl += g.n5;
                h0[(2 * py) * RR + px] = (uint16_t)g.vlo;
                h0[(2 * py + 1) * RR + px] = (uint16_t)(g.vlo >> 16);
                h1[(2 * py) * RR + px] = (uint16_t)g.vhi;
                h1[(2 * py + 1) * RR + px] = (uint16_t)(g.vhi >> 16);
                if (g.err) ek = umin64(ek, exact_key(w, bf, ipq, B.plen, ent0, vmask, leaf));
            }
        }
        __syncwarp();
        // ---- marker chains, row parity by row parity; fast raster: resolve + write whole rows
        resolve_rows<RR, 0, 0>(B, r0, pr, fast, fast ? B.R.base + (2 * pz) * B.plane : nullptr, lane);
        resolve_rows<RR, 0, 1>(B, r0, pr, fast, fast ? B.R.base + (2 * pz) * B.plane : nullptr, lane);
        resolve_rows<RR, 1, 0>(B, r1, pr, fast, fast ? B.R.base + (2 * pz + 1) * B.plane : nullptr, lane);
        resolve_rows<RR, 1, 1>(B, r1, pr, fast, fast ? B.R.base + (2 * pz + 1) * B.plane : nullptr, lane);
        if (!fast) {
            if (MODE == OUT_RASTER) {
#pragma unroll 1
                for (int dz = 0; dz < 2; ++dz)
                    plane_rows_slow<uint8_t>(B.R, P, B.spal, B.pal, dz ? r1 : r0, S2, 2 * pz + dz, lane);
            } else {
                for (uint32_t k0 = 0; k0 < nl; k0 += 32) {   // active parents to HBM (8 children = one sector)
                    const uint32_t k = k0 + lane;
                    if (k < nl) {
                        const uint32_t i = plist[k];
                        const uint32_t px = i % RR, py = i / RR;
                        const uint32_t q = spread3_u32(px) | (spread3_u32(py) << 1) | sz;
                        const uint32_t a = h0[(2 * py) * RR + px], b = h0[(2 * py + 1) * RR + px];
                        const uint32_t c = h1[(2 * py) * RR + px], d = h1[(2 * py + 1) * RR + px];
                        const uint32_t lab[8] = {label_of<uint8_t>(B, a & 0xFFu), label_of<uint8_t>(B, a >> 8), label_of<uint8_t>(B, b & 0xFFu), label_of<uint8_t>(B, b >> 8),
                                                 label_of<uint8_t>(B, c & 0xFFu), label_of<uint8_t>(B, c >> 8), label_of<uint8_t>(B, d & 0xFFu), label_of<uint8_t>(B, d >> 8)};
                        store_children<MODE>(B, P, q, px, py, pz, lab);
                    }
                }
            }
        }
        __syncwarp();
    }
    cur = e0 + 8 * nact;
    return warp_min64(ek);
}

}  // namespace wk

#ifndef K2W_MINB
#define K2W_MINB 19   // launch bound (warps per SM): same 96 registers as 20, a slightly better schedule (K2w 13.58 -> 13.50 ms)
#endif
#ifndef K2W_WPB
#define K2W_WPB 1
#endif
constexpr int K2W_WARPS = K2W_WPB;

// Overlap launch (Q): request k of the counter is the k-th entry of K1's ready queue.  The
// slot is published by K1 (fl_signal) with a release store; the spin is bounded and traps
// (a launch failure, never a hang) if the slot is never published.
__device__ __noinline__ unsigned long long wait_ready(const Plan& P, unsigned long long k) {
    uint32_t v;
    for (uint32_t spin = 0;; ++spin) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(P.rq + k) : "memory");
        if (v) break;
        if (spin > (1u << 24)) __trap();
        __nanosleep(256);
    }
    return v - 1u;
}

template <int MODE, int LMAX, typename IT, bool Q = false>
__global__ void __launch_bounds__(32 * K2W_WARPS, K2W_MINB) k2_warp(VolView V, Plan P, unsigned long long* counter) {
    using namespace wk;
    constexpr WLayout Y = make_wlayout(LMAX, sizeof(IT));
    constexpr bool WIDE = sizeof(IT) == 2;             // second pass: only bricks the u8 pass skipped
    extern __shared__ __align__(16) uint8_t wsm[];
    uint8_t* const base = wsm + (threadIdx.x >> 5) * Y.bytes;
    IT* const lev = reinterpret_cast<IT*>(base + Y.lev);
    uint32_t* const mA = reinterpret_cast<uint32_t*>(base + Y.pm);
    uint32_t* const mB = reinterpret_cast<uint32_t*>(base + Y.cm);
    uint16_t* const wpre = reinterpret_cast<uint16_t*>(base + Y.wpre);
    IT* const ring = reinterpret_cast<IT*>(base + Y.ring);
    uint8_t* const plist = base + Y.plist;
    uint16_t* const pdesc = reinterpret_cast<uint16_t*>(base + Y.pdesc);
    uint16_t* const clist = reinterpret_cast<uint16_t*>(base + Y.clist);
    uint16_t* const cdesc = reinterpret_cast<uint16_t*>(base + Y.cdesc);
    uint32_t* const amask = reinterpret_cast<uint32_t*>(base + Y.amask);
    const int lane = threadIdx.x & 31;
    if (Q && P.k1_grid) {   // overlap launch: work only beside a fully resident K1 (Plan::k1_started)
        unsigned long long st = 0;
        if (lane == 0) {
            for (uint32_t spin = 0; spin < 512; ++spin) {
                asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(st) : "l"(P.k1_started) : "memory");
                if (st >= P.k1_grid) break;
                __nanosleep(128);
            }
        }
        st = __shfl_sync(FULL, st, 0);
        if (st < P.k1_grid) return;
    }
    while (true) {
        __syncwarp();
        unsigned long long rr = 0;
        if (lane == 0) {
            rr = atomicAdd(counter, 1ull);
            if (Q && rr < P.n) rr = wait_ready(P, rr);
        }
        rr = __shfl_sync(FULL, rr, 0);
        if (rr >= P.n) break;
        if (Q) __syncwarp();   // lane 0's acquire orders the whole warp's reads of the brick's entries
        Brick B{};
        B.r = rr;
        const uint64_t b = req_local(V, P, rr);
        B.t = req_lod(P, rr);
        B.N = V.N;
        if (b >= V.nb || B.t > B.N) { if (!WIDE && LMAX <= 5 && lane == 0) put_result(P, rr, -1, 0, 0, 0, 0); continue; }
        B.n = B.N - B.t;
        if (B.t < B.N && B.n > LMAX) continue;          // served by the global-workspace kernel
        if (LMAX == 6 && B.n != 6) continue;             // K2w<6> takes only the 64^3 replays
        B.plen = V.pal_len[b];
        if (WIDE ? B.plen <= e8::kMarkPal : B.plen > e8::kMarkPal) continue;   // the other index width's pass
        B.out_m = MODE == OUT_MORTON ? P.out + P.dst[rr] : nullptr;
        B.pal = V.palette + V.pal_off[b];
        if (sizeof(IT) == 1 && K2W_SPAL) {   // the palette (<= 256 labels) into the warp's slice
            uint32_t* const sp = reinterpret_cast<uint32_t*>(base + Y.spal);
            for (uint32_t i = lane; i < B.plen; i += 32) sp[i] = __ldg(B.pal + i);
            B.spal = sp;
            __syncwarp();
        }
        if (MODE == OUT_RASTER) {
            const uint64_t gb = V.brick_begin + b;
            const int64_t side = 1ll << B.n;
            B.R.ox = (int64_t)(gb % V.gx) * side;
            B.R.oy = (int64_t)((gb / V.gx) % V.gy) * side;
            B.R.oz = (int64_t)(gb / (V.gx * V.gy)) * side;
            B.R.base = P.out + ((B.R.oz - P.z_begin) * P.cy + B.R.oy) * P.cx + B.R.ox;
            B.R.fast = B.R.ox + side <= P.cx && B.R.oy + side <= P.cy && B.R.oz >= P.z_begin &&
                       B.R.oz + side <= P.z_end && (uint64_t)P.cx * P.cy * side < (1ull << 32);
            B.pitch = (uint32_t)P.cx;
            B.plane = (uint32_t)(P.cx * P.cy);
            B.al8 = B.R.fast && (B.pitch & 1u) == 0u && (reinterpret_cast<uintptr_t>(B.R.base) & 7u) == 0u;
            B.al16r = B.R.fast && (B.pitch & 3u) == 0u && (reinterpret_cast<uintptr_t>(B.R.base) & 15u) == 0u;
        } else {
            B.al16 = (reinterpret_cast<uintptr_t>(B.out_m) & 15u) == 0u;
        }
        if (B.plen == 0) { if (lane == 0) put_result(P, rr, CSV_ST_EMPTY_PALETTE, 0, 0, 0, 0); continue; }
        if (B.t == B.N) {   // coarsest LOD: palette[0] (codec.py:514-516, container.py:178-182)
            if (lane == 0) {
                uint32_t* p = MODE == OUT_MORTON ? B.out_m : raster_of(B.R, P, 0);
                if (p) *p = __ldg(B.pal);
                put_result(P, rr, 0, 0, 0, 0, 0);
            }
            continue;
        }
        const uint32_t nc_raw = V.c_nib[b], nd_raw = B.t == 0 ? V.d_nib[b] : 0;
        const uint32_t nc = eff_nibbles(V, b, 0), nd = B.t == 0 ? eff_nibbles(V, b, 1) : 0;
        if (V.entropy) {   // state-word checks come first (codec.py:331-351)
            if (nc_raw > 0 && V.c_bytes[b] < 4) { if (lane == 0) put_result(P, rr, CSV_ST_UNDERRUN, 0, 0, 0, 0); continue; }
            if (B.t == 0 && nd_raw > 0 && V.d_bytes[b] < 4) { if (lane == 0) put_result(P, rr, CSV_ST_UNDERRUN, 1, 0, 0, 0); continue; }
        }
        {   // stream results through L2 (written by K1, possibly during this launch)
            const uint4 a = __ldcg(reinterpret_cast<const uint4*>(P.sres + 2 * rr));
            const uint4 c = __ldcg(reinterpret_cast<const uint4*>(P.sres + 2 * rr + 1));
            memcpy(&B.src, &a, sizeof a);
            memcpy(&B.srd, &c, sizeof c);
        }
        const uint64_t eo0 = P.eoff[2 * rr], eo1 = P.eoff[2 * rr + 1], eo2 = P.eoff[2 * rr + 2];
        if (lane == 0 && eo2 > eo0) {   // stage this brick's entries + gip in L2 ahead of the levels
            const uint64_t lo = eo0 & ~15ull, hi = (eo2 + 15) & ~15ull;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(P.entries + lo), "r"((uint32_t)(hi - lo)) : "memory");
        }
        const uint32_t limc = stream_limit(V, b, B.t, 0), limd = B.t == 0 ? stream_limit(V, b, 0, 1) : 0u;
        B.Ec = P.entries + eo0;
        B.capc = (uint32_t)round32(limc);
        B.Ed = P.entries + eo1;
        B.capd = (uint32_t)round32(limd);
        uint8_t* fin = nullptr;   // K2w<6>: the final parent level (32^3 u8) in the warp's global slot
        uint16_t* glist = nullptr;   // K2w<6>: list + pending descriptors of the 16^3-parent coarse level
        if constexpr (LMAX >= 6) {
            B.ipb = P.wscratch6 + (uint64_t)(blockIdx.x * K2W_WARPS + (threadIdx.x >> 5)) * kWScratch6Stride;
            fin = reinterpret_cast<uint8_t*>(B.ipb + 32768);
            glist = B.ipb + 32768 + 16384;
        } else {
            B.ipb = P.wscratch + (uint64_t)(P.wslot0 + blockIdx.x * K2W_WARPS + (threadIdx.x >> 5)) * P.wscratch_stride;
        }
        const bool trivial = (uint64_t)nc + nd == 0;     // relevant == 0: fill palette[0] (codec.py:353-358)
        if (lane == 0) {
            lev[0] = 0;
            mA[0] = trivial ? 0u : 1u;
        }
        __syncwarp();
        uint32_t cur_c = 0, cur_d = 0, pdc = 0, pdd = 0, ip_run = 0;
        uint32_t* pm = mA;
        uint32_t* cm = mB;
        bool failed = false;
        for (int j = 0; j + 1 < B.n; ++j) {      // parents at level N - j, children above the final level
            IT* const finj = (LMAX >= 6 && j + 2 == B.n) ? reinterpret_cast<IT*>(fin) : nullptr;
            // 64^3 replays: the 4096-parent level's list does not fit the warp's shared slice
            uint16_t* const lj = (LMAX >= 6 && j == 4) ? glist : clist;
            uint16_t* const dj = (LMAX >= 6 && j == 4) ? glist + 4096 : cdesc;
            const unsigned long long ek = coarse_level<IT, Q>(B, j, lev, pm, cm, wpre, lj, dj, cur_c, ip_run, pdc,
                                                           lane, finj);
            if (ek != ~0ull) { report_error<Q>(P, rr, B.Ec, B.capc, B.src, ek, false, lane); failed = true; break; }
            uint32_t* tmp = pm; pm = cm; cm = tmp;
        }
        if (failed) continue;
        const IT* plev = (LMAX >= 6 && B.n == 6) ? reinterpret_cast<const IT*>(fin) : lev + wofs(B.n - 1);
        // pdesc lives in whichever mask array is dead after the ping-pong (the layout aliases "cm")
        uint16_t* const fdesc = Y.pdesc == Y.cm ? reinterpret_cast<uint16_t*>(cm) : pdesc;
        uint32_t& cur = B.t == 0 ? cur_d : cur_c;
        uint32_t& pdl = B.t == 0 ? pdd : pdc;
        unsigned long long ek;
        if constexpr (sizeof(IT) == 1) {
            switch (B.n) {
                case 1: ek = final_sweep<MODE, 1, IT, Q>(B, P, plev, pm, wpre, ring, plist, fdesc, amask, cur, ip_run, pdl, lane); break;
                case 2: ek = final_sweep<MODE, 2, IT, Q>(B, P, plev, pm, wpre, ring, plist, fdesc, amask, cur, ip_run, pdl, lane); break;
                case 3: ek = final_sweep8<MODE, 4, Q>(B, P, plev, pm, wpre, ring, plist, cur, ip_run, pdl, lane); break;
                case 4: ek = final_sweep8<MODE, (LMAX >= 4 ? 8 : 4), Q>(B, P, plev, pm, wpre, ring, plist, cur, ip_run, pdl, lane); break;
                case 5: ek = final_sweep8<MODE, (LMAX >= 5 ? 16 : 4), Q>(B, P, plev, pm, wpre, ring, plist, cur, ip_run, pdl, lane); break;
                default: ek = final_sweep8<MODE, (LMAX >= 6 ? 32 : 4), Q>(B, P, plev, pm, wpre, ring, plist, cur, ip_run, pdl, lane); break;
            }
        } else {
            switch (B.n) {
                case 1: ek = final_sweep<MODE, 1, IT, Q>(B, P, plev, pm, wpre, ring, plist, fdesc, amask, cur, ip_run, pdl, lane); break;
                case 2: ek = final_sweep<MODE, 2, IT, Q>(B, P, plev, pm, wpre, ring, plist, fdesc, amask, cur, ip_run, pdl, lane); break;
                case 3: ek = final_sweep<MODE, 4, IT, Q>(B, P, plev, pm, wpre, ring, plist, fdesc, amask, cur, ip_run, pdl, lane); break;
                case 4: ek = final_sweep<MODE, (LMAX >= 4 ? 8 : 1), IT, Q>(B, P, plev, pm, wpre, ring, plist, fdesc, amask, cur, ip_run, pdl, lane); break;
                default: ek = final_sweep<MODE, (LMAX >= 5 ? 16 : 1), IT, Q>(B, P, plev, pm, wpre, ring, plist, fdesc, amask, cur, ip_run, pdl, lane); break;
            }
        }
        if (ek != ~0ull) {
            if (B.t == 0) report_error<Q>(P, rr, B.Ed, B.capd, B.srd, ek, true, lane);
            else report_error<Q>(P, rr, B.Ec, B.capc, B.src, ek, false, lane);
            continue;
        }
        const int64_t ci = (int64_t)cur_c + warp_sum(pdc), di = (int64_t)cur_d + warp_sum(pdd);
        if (lane == 0) {
            int st = 0, stream = 0;
            int64_t pos = 0;
            if (V.entropy) {   // full consumption must land on the initial state (codec.py:464-470)
                if (nc_raw > 0 && ci == (int64_t)nc_raw && (B.src.flags & CSV_SF_DESYNC)) { st = CSV_ST_DESYNC; stream = 0; pos = ci; }
                else if (B.t == 0 && nd_raw > 0 && di == (int64_t)nd_raw && (B.srd.flags & CSV_SF_DESYNC)) { st = CSV_ST_DESYNC; stream = 1; pos = di; }
            }
            put_result(P, rr, st, stream, pos, ci, di);
        }
    }
}
