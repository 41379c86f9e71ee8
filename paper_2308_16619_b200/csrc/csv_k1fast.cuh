// csv_k1fast.cuh -- K1f: the entropy lanes for rANS streams, issue-diet version.
// Included by csv_decode.cu after k1_streams (shared: Plan, VolView, bswap32, lane
// work distribution).
//
// Reference: _rans_pull (codec.py:290-300) over one single-state rANS chain per
// (brick, stream), nibbles parsed into one entry byte per operation
// (op | stop << 3 | delta << 4, codec.py:374-395).  Same output as k1_streams
// (entry regions + per-stream csv_stream_result), restructured so that the
// common step carries no checks at all:
//
//  * the warp runs blocks of K1F_BLOCK symbols; a block is "fast" when every
//    active lane has more than K1F_BLOCK symbols left before its limit and is
//    not in checked mode.  Fast steps have no limit, underrun or slow-state
//    test and no branch: table lookup, state update, byte renormalisation
//    from a 64-bit bit buffer, entry append, predicated 8-byte group store.
//  * underruns (corrupt streams only) are detected once per block from the
//    bytes consumed; the lane then restarts its stream in CHECKED mode, whose
//    steps replay the reference's order of checks exactly (underrun at the
//    failing symbol, the slow first renormalisation of a state below 2^23).
//    Lanes within K1F_BLOCK symbols of their limit also take checked steps.
//  * the bit buffer refills from a two-word lookahead queue (4-byte loads from
//    the stream, predicated, no divergent branch) once per pair of steps.
//  * entry bytes are appended as they are parsed: a P_delta op byte first,
//    its payload nibble patched into the byte's high half on the next symbol.
//    A group of 8 entries, once its last entry is complete, goes to the
//    lane's 32-byte ring in shared memory; every 8 steps a lane with 4
//    complete groups writes them to HBM as ONE 32-byte store (a full sector:
//    partial-sector writes cost DRAM read-modify-writes).
//  * decode table in shared memory, one word per slot:
//    f << 20 | (slot - cum[s]) << 8 | s   (f <= 4095; containers whose tables
//    have a count of 4096 use k1_streams).
// (included inside namespace csv)
#pragma once

#ifndef K1F_FMA_DECODE
#define K1F_FMA_DECODE 1
#endif
#ifndef K1F_EVICT_FIRST
#define K1F_EVICT_FIRST 1   // entry stores L2::evict_first (K1 DRAM reads 1.30x -> 1.18x of the stream bytes)
#endif
#ifndef K1F_OR_ADDR
#define K1F_OR_ADDR 1   // table base | slot offset (16 KB-aligned tables): one instruction less per symbol
#endif
#ifndef K1F_BLOCK
#define K1F_BLOCK 16
#endif

struct FLane {
    uint32_t hi, lo;        // upcoming stream bits, MSB first: nb valid bits from the top of hi:lo
    int nb;
    const uint32_t* wbase;  // 4-byte aligned word pointer of the stream (word 0 holds byte 4 - sh)
    uint32_t wo;            // index of the word to load next into nxt1
    uint32_t nxt0, nxt1;    // lookahead words (stream byte order)
    uint32_t sh;            // bytes of word 0 before the first renormalisation byte
    uint32_t x;             // rANS state
    uint32_t alo, ahi;      // last 8 entry bytes, newest in the top byte of ahi
    uint32_t ne;            // entries appended (a pending P_delta op included)
    uint32_t fl;            // entries written to HBM (multiple of 32 until the finish)
    uint32_t ring;          // shared-memory byte address of the lane's 4-group ring (group g in slot (g+1) & 3)
    uint64_t* outp;         // entry region (32-byte aligned)
    uint32_t i, lim, n, len;
    uint32_t tb;            // shared-memory byte address of the stream's decode table
    uint64_t item;
    uint64_t pol;           // L2 evict-first cache policy of the entry stores (K1F_EVICT_FIRST)
    bool pend;              // the top entry is a P_delta op waiting for its payload
    bool checked;           // exact per-step checks (corrupt stream or restart after an underrun)
};

__device__ __forceinline__ uint32_t fl_pos(const FLane& L) {   // stream bytes consumed (state bytes included)
    return 4u + 4u * (L.wo - 2u) - L.sh - (uint32_t)(L.nb >> 3);
}

__device__ __forceinline__ void fl_refill(FLane& L) {   // requires nb < 32 (then lo == 0)
    const uint32_t w = bswap32(L.nxt0);
    L.hi |= w >> L.nb;
    L.lo = __funnelshift_r(0u, w, (uint32_t)L.nb);        // w << (32 - nb); 0 for nb == 0
    L.nb += 32;
    L.nxt0 = L.nxt1;
    L.nxt1 = __ldg(L.wbase + L.wo);
    ++L.wo;
}

// Consume s8 (0, 8, 16) bits into the state: x = xn << s8 | next s8 bits.
__device__ __forceinline__ void fl_shift_in(FLane& L, uint32_t xn, uint32_t s8) {
    L.x = __funnelshift_l(L.hi, xn, s8);
    L.hi = __funnelshift_l(L.lo, L.hi, s8);
    L.lo <<= s8;
    L.nb -= (int)s8;
}

// Append symbol e (table word, symbol in the low byte) to the entry window;
// store a completed group.  pay: this symbol is the payload of the top entry.
__device__ __forceinline__ void fl_emit(FLane& L, uint32_t e) {
    const bool pay = L.pend;
    L.pend = !pay && ((e & 7u) == 5u);
    const uint32_t nlo = __byte_perm(L.alo, L.ahi, 0x4321), nhi = __byte_perm(L.ahi, e, 0x4321);
    L.alo = pay ? L.alo : nlo;
    L.ahi = pay ? L.ahi + (e << 28) : nhi;
    L.ne += pay ? 0u : 1u;
    if (((L.ne & 7u) == 0u) & !L.pend)   // the group's last entry is complete: into the ring
        asm volatile("st.shared.v2.u32 [%0], {%1, %2};" :: "r"(L.ring | (L.ne & 24u)), "r"(L.alo), "r"(L.ahi) : "memory");
}

// Four complete groups in the ring (entries [fl, fl + 32)): one 32-byte store.
__device__ __forceinline__ void fl_flush(FLane& L) {
    if (L.ne - (L.pend ? 1u : 0u) >= L.fl + 32u) {
        uint32_t a0, a1, a2, a3, b0, b1, b2, b3;   // slots 0..3 = groups 3, 0, 1, 2 of the chunk
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3) : "r"(L.ring) : "memory");
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(b0), "=r"(b1), "=r"(b2), "=r"(b3) : "r"(L.ring + 16u) : "memory");
#if K1F_EVICT_FIRST
        // entries stream through L2 (3.5 GB on config 3): evict them first so the lanes'
        // stream bytes stay resident until consumed
        asm volatile("st.global.L2::cache_hint.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8}, %9;"
                     :: "l"(reinterpret_cast<uint8_t*>(L.outp) + L.fl), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "r"(b2),
                        "r"(b3), "r"(a0), "r"(a1), "l"(L.pol) : "memory");
#else
        asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
                     :: "l"(reinterpret_cast<uint8_t*>(L.outp) + L.fl), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "r"(b2),
                        "r"(b3), "r"(a0), "r"(a1) : "memory");
#endif
        L.fl += 32u;
    }
}

#if K1F_OR_ADDR
// The decode tables at file scope: their shared address is a link-time constant that folds
// into the LDS immediate, so a slot's address is one LOP3 (s << 12 | x & 4095) + the scale.
__shared__ uint32_t k1f_tab[2 * 4096];
#endif

// One symbol without checks (fast blocks).  L.tb: s << 12 (K1F_OR_ADDR), else the table's
// shared byte address.
__device__ __forceinline__ uint32_t fl_lookup(const FLane& L) {
#if K1F_OR_ADDR
    return k1f_tab[L.tb | (L.x & (kTotalFreq - 1u))];
#else
    uint32_t e;
    asm("ld.shared.u32 %0, [%1];" : "=r"(e) : "r"(L.tb + 4u * (L.x & (kTotalFreq - 1u))));
    return e;
#endif
}

// LAT (the single-wave variant, where the longest stream's chain sets the time): the
// renormalisation is taken from three candidates chosen by two compares instead of
// count-leading-zeros -> shift amount -> funnel shift, and the table address is one
// AND + one multiply-add; fewer cycles on the symbol-to-symbol dependency chain, a few
// more ALU instructions.
template <bool LAT = false>
__device__ __forceinline__ uint32_t fl_lookup_t(const FLane& L) {
    uint32_t e;
    if (LAT && !K1F_OR_ADDR) {
        uint32_t a;
        asm("mad.lo.u32 %0, %1, 4, %2;" : "=r"(a) : "r"(L.x & (kTotalFreq - 1u)), "r"(L.tb));
        asm("ld.shared.u32 %0, [%1];" : "=r"(e) : "r"(a));
    } else {
        e = fl_lookup(L);
    }
    return e;
}

template <bool LAT = false>
__device__ __forceinline__ void fl_step_fast(FLane& L) {
    const uint32_t e = fl_lookup_t<LAT>(L);
    if (LAT) {
        const uint32_t f = __umulhi(e, 1u << 12), g = __umulhi(e, 1u << 24);
        const uint32_t xn = f * (__umulhi(L.x, 1u << 20) - 4096u) + g;
        const bool r1 = xn < kStateLower, r2 = xn < (1u << 15);   // 1 / 2 renormalisation bytes
        const uint32_t x8 = __funnelshift_l(L.hi, xn, 8u), x16 = __funnelshift_l(L.hi, xn, 16u);
        const uint32_t s8 = r2 ? 16u : (r1 ? 8u : 0u);
        L.x = r2 ? x16 : (r1 ? x8 : xn);
        L.hi = __funnelshift_l(L.lo, L.hi, s8);
        L.lo <<= s8;
        L.nb -= (int)s8;
        fl_emit(L, e);
        return;
    }
#if K1F_FMA_DECODE
    // the same xn with the field extractions on the FMA pipe (the ALU pipe is the bottleneck):
    // e >> 8 = f << 12 | bias, so xn = f * ((x >> 12) - 4096) + (e >> 8) (mod 2^32)
    const uint32_t f = __umulhi(e, 1u << 12), g = __umulhi(e, 1u << 24);
    const uint32_t xn = f * (__umulhi(L.x, 1u << 20) - 4096u) + g;
#else
    const uint32_t f = e >> 20, bias = (e >> 8) & 0xFFFu;
    const uint32_t xn = f * (L.x >> kPrecision) + bias;
#endif
    const uint32_t s8 = ((uint32_t)__clz(xn) - 1u) & 0x18u;   // 8 * renormalisation bytes (xn >= 2^11)
    fl_shift_in(L, xn, s8);
    fl_emit(L, e);
}

// K1 -> K2w overlap (Plan::rcnt): stream w of request w >> 1 is final (its entries and
// csv_stream_result are written).  The second stream of a request to finish appends the
// request to the ready queue with a release store; K2w's acquire load of the slot then
// sees both streams' writes (each lane fences before its count increment).
__device__ __forceinline__ void fl_signal(const Plan& P, uint64_t w) {
    if (P.rcnt == nullptr) return;
    __threadfence();
    const uint64_t r = w >> 1;
    if (atomicAdd(P.rcnt + r, 1u) == 1u) {
        __threadfence();
        const unsigned long long pos = atomicAdd(P.rq_tail, 1ull);
        asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(P.rq + pos), "r"((uint32_t)r + 1u) : "memory");
    }
}

__device__ __forceinline__ void fl_finish(FLane& L, const Plan& P, bool failed) {
    const uint32_t ne = L.ne - (L.pend ? 1u : 0u);          // the pending P_delta op is not an entry
    for (; L.fl + 8u <= ne; L.fl += 8u) {                     // complete groups still in the ring
        uint32_t lo, hi;
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(L.ring | ((L.fl + 8u) & 24u)) : "memory");
        L.outp[L.fl >> 3] = ((uint64_t)hi << 32) | lo;
    }
    const uint32_t k = ne & 7u;
    if (k) {   // partial group: its entries down to byte 0, zero above
        uint64_t a = ((uint64_t)L.ahi << 32) | L.alo;
        if (L.pend) a <<= 8;
        a >>= 8 * (8 - k);
        L.outp[ne >> 3] = a;
    }
    csv_stream_result r;
    r.n_entries = ne;
    r.flags = 0;
    r.fail_nibble = 0xffffffffu;
    r.partial_op = 0;
    if (failed) {
        r.flags |= CSV_SF_FAILED;
        r.fail_nibble = L.i;
    } else if (L.i == L.n) {
        r.flags |= CSV_SF_FAILED | CSV_SF_COMPLETE;
        r.fail_nibble = L.n;
        if (L.n > 0 && (L.x != kStateLower || fl_pos(L) != L.len)) r.flags |= CSV_SF_DESYNC;
    }
    if (L.pend) {
        r.flags |= CSV_SF_PARTIAL;
        r.partial_op = L.ahi >> 24;
    }
    P.sres[L.item] = r;
    fl_signal(P, L.item);
}

// One symbol with the reference's checks; returns false when the lane's item is finished.
__device__ __forceinline__ bool fl_step_checked(FLane& L, const Plan& P) {
    if (L.nb < 32) fl_refill(L);
    const uint32_t e = fl_lookup(L);
    uint32_t xn = (e >> 20) * (L.x >> kPrecision) + ((e >> 8) & 0xFFFu);
    if (L.x >= kStateLower) {
        // after a step from x >= 2^23, xn >= 2^11: at most two renormalisation bytes
        const uint32_t s8 = ((uint32_t)__clz(xn) - 1u) & 0x18u;
        if (fl_pos(L) + (s8 >> 3) > L.len) {   // underrun (codec.py:295-297)
            fl_finish(L, P, true);
            return false;
        }
        fl_shift_in(L, xn, s8);
    } else {   // first step from a state below 2^23 (corrupt stream): byte by byte
        while (xn < kStateLower) {
            if (fl_pos(L) >= L.len) {
                fl_finish(L, P, true);
                return false;
            }
            if (L.nb < 8) fl_refill(L);
            fl_shift_in(L, xn, 8u);
            xn = L.x;
        }
        L.x = xn;
    }
    fl_emit(L, e);
    fl_flush(L);
    if (++L.i == L.lim) {
        fl_finish(L, P, false);
        return false;
    }
    return true;
}

// Initialise the lane for work item `item` (detail streams first); false if it finished at once.
__device__ bool fl_init(FLane& L, const VolView& V, const Plan& P, uint64_t item, bool checked, uint32_t tab_s) {
    const uint64_t r = item < P.n ? item : item - P.n;
    const int s = item < P.n ? 1 : 0;
    const uint64_t w = 2 * r + s;
    L.item = w;
    L.alo = 0; L.ahi = 0; L.ne = 0; L.fl = 0; L.pend = false; L.i = 0; L.checked = checked;
    L.x = 0; L.len = 0; L.nb = 0; L.hi = 0; L.lo = 0; L.sh = 0; L.wo = 2; L.nxt0 = 0; L.nxt1 = 0;
    const uint64_t b = req_local(V, P, r);
    const int t = req_lod(P, r);
    L.outp = reinterpret_cast<uint64_t*>(P.entries + P.eoff[w]);
    const bool ok = b < V.nb && t < V.N && !(s == 1 && t != 0);
    L.n = ok ? eff_nibbles(V, b, s) : 0;
    L.lim = ok ? stream_limit(V, b, t, s) : 0;
    L.tb = K1F_OR_ADDR ? ((uint32_t)s << 12) : tab_s + ((uint32_t)s << 14);
    if (!ok) {
        P.sres[w] = csv_stream_result{0, 0xffffffffu, 0, 0};
        fl_signal(P, w);
        return false;
    }
    const uint8_t* base = s ? V.detail + V.d_off[b] : V.coarse + V.c_off[b];
    L.len = s ? V.d_bytes[b] : V.c_bytes[b];
    if (L.lim == 0) {
        if (L.n == 0) P.sres[w] = csv_stream_result{0, 0, CSV_SF_FAILED | CSV_SF_COMPLETE, 0};
        else P.sres[w] = csv_stream_result{0, 0xffffffffu, 0, 0};
        fl_signal(P, w);
        return false;
    }
    if (L.len < 4) {   // entropy stream shorter than its state word (codec.py:333-334)
        P.sres[w] = csv_stream_result{0, 0, CSV_SF_FAILED, 0};
        fl_signal(P, w);
        return false;
    }
    L.x = (uint32_t)base[0] | ((uint32_t)base[1] << 8) | ((uint32_t)base[2] << 16) | ((uint32_t)base[3] << 24);
    const uintptr_t q = reinterpret_cast<uintptr_t>(base) + 4;
    L.wbase = reinterpret_cast<const uint32_t*>(q & ~uintptr_t(3));
    L.sh = (uint32_t)(q & 3);
    const uint32_t w0 = bswap32(__ldg(L.wbase));
    L.hi = w0 << (8 * L.sh);
    L.lo = 0;
    L.nb = 32 - 8 * (int)L.sh;
    L.nxt0 = __ldg(L.wbase + 1);
    L.nxt1 = __ldg(L.wbase + 2);
    L.wo = 3;
    if (L.x < kStateLower) L.checked = true;
    return true;
}

template <int MINB, bool LAT>
__global__ void __launch_bounds__(K1_THREADS, MINB) k1_fast(VolView V, Plan P, unsigned long long* counter) {
    // LAT: plans of a few blocks (per-brick calls), where one lane's chain is the whole time
#if K1F_OR_ADDR
    uint32_t* const tab = k1f_tab;
#else
    __shared__ uint32_t tab[2 * 4096];
#endif
    __shared__ __align__(32) uint2 ring[K1_THREADS][4];
    if (P.k1_started && threadIdx.x == 0) atomicAdd(P.k1_started, 1ull);   // resident (overlap launch)
    // {f:16 | (slot-cum):12 | s:4} -> {f:12 | (slot-cum):12 | 0:4 | s:4}
    if (MINB >= 5) {   // throughput variant (48 registers): the plain loop
        for (int i = threadIdx.x; i < 2 * 4096; i += blockDim.x) {
            const uint32_t o = V.dtab[i];
            tab[i] = ((o >> 16) << 20) | (((o >> 4) & 0xFFFu) << 8) | (o & 15u);
        }
    } else {   // single-wave / per-brick variants: all 8 vector loads of a thread in flight at once
        static_assert(2 * 4096 == 8 * 4 * K1_THREADS, "table fill: 8 uint4 per thread");
        const uint4* const src = reinterpret_cast<const uint4*>(V.dtab);
        uint4 w[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) w[k] = __ldg(src + k * K1_THREADS + threadIdx.x);
        auto cv = [](uint32_t o) { return ((o >> 16) << 20) | (((o >> 4) & 0xFFFu) << 8) | (o & 15u); };
#pragma unroll
        for (int k = 0; k < 8; ++k)
            reinterpret_cast<uint4*>(tab)[k * K1_THREADS + threadIdx.x] =
                make_uint4(cv(w[k].x), cv(w[k].y), cv(w[k].z), cv(w[k].w));
    }
    __syncthreads();
    const uint32_t tab_s = (uint32_t)__cvta_generic_to_shared(tab);
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const uint64_t total = 2 * P.n;
    FLane L;
    L.ring = (uint32_t)__cvta_generic_to_shared(&ring[threadIdx.x][0]);
#if K1F_EVICT_FIRST
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(L.pol));
#else
    L.pol = 0;
#endif
    bool has = false, done = false;
    while (true) {
        const bool need = !has && !done;
        const unsigned m = __ballot_sync(FULL, need);
        if (m) {
            const int leader = __ffs(m) - 1;
            unsigned long long base = 0;
            if (lane == leader) base = atomicAdd(counter, (unsigned long long)__popc(m));
            base = __shfl_sync(FULL, base, leader);
            if (need) {
                const uint64_t my = base + __popc(m & ((1u << lane) - 1u));
                if (my < total) has = fl_init(L, V, P, my, false, tab_s);
                else done = true;
            }
        }
        if (__all_sync(FULL, done)) break;
        const bool fast = !has || (!L.checked && L.lim - L.i > (uint32_t)K1F_BLOCK);
        if (__all_sync(FULL, fast)) {
            if (has) {
#pragma unroll
                for (int u = 0; u < K1F_BLOCK / 2; ++u) {
                    if (L.nb < 32) fl_refill(L);
                    fl_step_fast<LAT>(L);
                    fl_step_fast<LAT>(L);
                    if ((u & 3) == 3) fl_flush(L);   // <= 8 entries between flushes: the ring never overflows
                }
                L.i += K1F_BLOCK;
                // an underrun inside the block (corrupt stream): redo the stream with exact checks
                if (fl_pos(L) > L.len) has = fl_init(L, V, P, (L.item & 1) ? (L.item >> 1) : P.n + (L.item >> 1), true, tab_s);
            }
        } else if (has) {
#pragma unroll 1
            for (int u = 0; u < K1F_BLOCK; ++u) {
                if (!fl_step_checked(L, P)) { has = false; break; }
            }
        }
    }
}

