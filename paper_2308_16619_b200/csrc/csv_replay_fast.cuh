// csv_replay_fast.cuh -- K2 for N - t <= 5 (every LOD of b <= 32, coarse LODs of
// b = 64/128): the whole per-brick working set lives in shared memory and is
// addressed directly through `dsm[]`, so the hot loops compile to plain
// LDS/STS without generic-address materialisation.  Included by csv_decode.cu
// after the shared K2 helpers (Layout, K2Shared, scans, Raster, ekey).
//
// Per level l (parents at l, children at l-1), reference _decode_kernel
// (codec.py:361-463) restated level-synchronously:
//   A  rank prefix of the active-parent bitmask (occupancy skip, :367-370)
//   B  active list + palette-advance counts -> i_p base per parent (:453-457)
//   C1 one lane per child of an active parent: op -> value (:400-457)
//   C2 inactive parents: children repeat the parent (stop fill, :460-463)
//   W  same-level chains (even-coordinate reuse, :422-423) walked in smem
//   T  final level only: the 16^3 tile streamed to HBM (raster or Morton pool)

// position of the r-th (0-based) set bit of m (r < popc(m)); branch-free bisection
__device__ __forceinline__ uint32_t nth_set_bit(uint32_t m, uint32_t r) {
    uint32_t pos = 0;
#pragma unroll
    for (int width = 16; width > 0; width >>= 1) {
        const uint32_t lo = __popc(m & ((1u << width) - 1u));
        const bool up = r >= lo;
        r -= up ? lo : 0u;
        m = up ? (m >> width) : m;
        pos += up ? (uint32_t)width : 0u;
    }
    return pos;
}

#ifndef K2F_MINB
#define K2F_MINB 5
#endif
template <int MODE, int LMAX>
__global__ void __launch_bounds__(K2_THREADS, K2F_MINB) k2_fast(VolView V, Plan P) {
    static_assert(LMAX <= 5, "shared-memory replay covers N - t <= 5");
    constexpr Layout Y = make_layout(LMAX, 2);
    extern __shared__ __align__(16) uint32_t dsm[];
    __shared__ K2Shared S;
    uint16_t* const ipb = reinterpret_cast<uint16_t*>(dsm + Y.ipb);
    uint16_t* const list = reinterpret_cast<uint16_t*>(dsm + Y.list);
    const int lane = threadIdx.x & 31;
    const int N = V.N;
    const uint64_t r = blockIdx.x;
    if (r >= P.n) return;
    const uint64_t b = req_local(V, P, r);
    const int t = req_lod(P, r);
    if (b >= V.nb || t > N) { write_result(P, r, -1, 0, 0, 0, 0); return; }
    if (t < N && N - t > LMAX) return;            // served by the global-workspace kernel
    uint32_t* const out_m = MODE == OUT_MORTON ? P.out + P.dst[r] : nullptr;
    const uint32_t plen = V.pal_len[b];
    const uint32_t* const pal = V.palette + V.pal_off[b];
    Raster R{};
    uint32_t pitch = 0, plane = 0;
    if (MODE == OUT_RASTER) {
        const uint64_t gb = V.brick_begin + b;
        const int64_t side = 1ll << (N - t);
        R.ox = (int64_t)(gb % V.gx) * side;
        R.oy = (int64_t)((gb / V.gx) % V.gy) * side;
        R.oz = (int64_t)(gb / (V.gx * V.gy)) * side;
        R.base = P.out + ((R.oz - P.z_begin) * P.cy + R.oy) * P.cx + R.ox;
        asm volatile("" : "+l"(R.base));   // computed once: keep it in registers, not rematerialised
        R.fast = R.ox + side <= P.cx && R.oy + side <= P.cy && R.oz >= P.z_begin && R.oz + side <= P.z_end &&
                 (uint64_t)P.cx * P.cy * side < (1ull << 32);
        pitch = (uint32_t)P.cx;
        plane = (uint32_t)(P.cx * P.cy);
    }
    if (plen == 0) { write_result(P, r, CSV_ST_EMPTY_PALETTE, 0, 0, 0, 0); return; }
    if (t == N) {   // coarsest LOD: palette[0] (codec.py:514-516, container.py:178-182)
        if (threadIdx.x == 0) {
            uint32_t* p = MODE == OUT_MORTON ? out_m : raster_of(R, P, 0);
            if (p) *p = __ldg(pal);
        }
        write_result(P, r, 0, 0, 0, 0, 0);
        return;
    }
    const uint32_t nc_raw = V.c_nib[b], nd_raw = t == 0 ? V.d_nib[b] : 0;
    const uint32_t nc = eff_nibbles(V, b, 0), nd = t == 0 ? eff_nibbles(V, b, 1) : 0;
    if (V.entropy) {   // state-word checks come first (codec.py:331-351)
        if (nc_raw > 0 && V.c_bytes[b] < 4) { write_result(P, r, CSV_ST_UNDERRUN, 0, 0, 0, 0); return; }
        if (t == 0 && nd_raw > 0 && V.d_bytes[b] < 4) { write_result(P, r, CSV_ST_UNDERRUN, 1, 0, 0, 0); return; }
    }
    const csv_stream_result src = P.sres[2 * r], srd = P.sres[2 * r + 1];
    const uint64_t eo0 = P.eoff[2 * r], eo1 = P.eoff[2 * r + 1], eo2 = P.eoff[2 * r + 2];
    if (threadIdx.x == 0 && eo2 > eo0) {   // stage this brick's entries in L2 ahead of the level loop
        const uint64_t lo = eo0 & ~15ull, hi = (eo2 + 15) & ~15ull;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(P.entries + lo), "r"((uint32_t)(hi - lo)) : "memory");
    }
    const bool trivial = (uint64_t)nc + nd == 0;     // relevant == 0: fill palette[0] (codec.py:353-358)
    if (threadIdx.x == 0) {
        dsm[Y.lev] = __ldg(pal);      // root (codec.py:353)
        dsm[Y.mask] = trivial ? 0u : 1u;
        S.errkey = ~0ull;
    }
    __syncthreads();
    uint32_t cur_c = 0, cur_d = 0;
    uint32_t pd_c = 0, pd_d = 0;
    int32_t ipbase = 0;
    uint32_t cur = 0;
    for (int l = N; l > t; --l) {
        const bool leaf = l == 1;
        const bool final_level = (l - 1 == t);
        const uint32_t Pn = 1u << (3 * (N - l));
        const uint32_t W = (Pn + 31) >> 5;
        uint32_t* const pmask = dsm + Y.mask + cur * Y.W;
        uint8_t* const cmask = reinterpret_cast<uint8_t*>(dsm + Y.mask + (cur ^ 1u) * Y.W);
        const uint32_t* const plev = dsm + Y.lev + levoffA(N - l);
        uint32_t* const clev = dsm + Y.lev + levoffA(N - l + 1);
        const uint32_t e0 = leaf ? cur_d : cur_c;
        const uint8_t* const Eb = P.entries + (leaf ? eo1 : eo0);
        const uint32_t ecap = (uint32_t)((leaf ? eo2 : eo1) - (leaf ? eo1 : eo0));
        const uint32_t nvalid = leaf ? srd.n_entries : src.n_entries;
        const int cbits = N - l + 1;
        const uint32_t Mx = axis_mask(0, cbits), My = axis_mask(1, cbits), Mz = axis_mask(2, cbits);
        // (A) rank prefix of the active-parent bitmask: each warp scans its own
        // contiguous word range, one barrier, then adds the preceding warps' totals
        const uint32_t wid = threadIdx.x >> 5;
        if (Pn < 32 && threadIdx.x == 0) pmask[0] &= (1u << Pn) - 1u;
        if (Pn < 32) __syncwarp();
        const uint32_t cw = (W + K2_WARPS - 1) / K2_WARPS;
        const uint32_t wb = min(wid * cw, W), we = min(wb + cw, W);
        {
            uint32_t run = 0;
            for (uint32_t c0 = wb; c0 < we; c0 += 32) {
                const uint32_t i = c0 + lane;
                const uint32_t v = i < we ? __popc(pmask[i]) : 0u;
                uint32_t inc = v;
#pragma unroll
                for (int o2 = 1; o2 < 32; o2 <<= 1) {
                    const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o2);
                    if (lane >= o2) inc += u;
                }
                if (i < we) dsm[Y.wpre + i] = run + inc - v;
                run += __shfl_sync(0xffffffffu, inc, 31);
            }
            if (lane == 0) S.scan[wid] = run;
        }
        __syncthreads();
        uint32_t nact = 0, woff = 0;
#pragma unroll
        for (int k = 0; k < K2_WARPS; ++k) {
            const uint32_t v = S.scan[k];
            woff += (uint32_t)k < wid ? v : 0u;
            nact += v;
        }
        // (B) active list (rank -> parent) and palette-advance counts per active
        // parent, scanned the same way; F1 below reads only its own warp's ranks
        for (uint32_t i = wb + lane; i < we; i += 32) {
            uint32_t mw = pmask[i], rk = dsm[Y.wpre + i] + woff;
            dsm[Y.wpre + i] = rk;
            while (mw) {
                list[rk++] = (uint16_t)(32 * i + (__ffs(mw) - 1));
                mw &= mw - 1;
            }
        }
        const uint32_t cr = (nact + K2_WARPS - 1) / K2_WARPS;
        const uint32_t rb = min(wid * cr, nact), re = min(rb + cr, nact);
        {
            uint32_t run = 0, pdl = 0;
            for (uint32_t c0 = rb; c0 < re; c0 += 32) {
                const uint32_t i = c0 + lane;
                const uint32_t off = e0 + 8 * i;
                const uint64_t w = (i < re && off + 8 <= ecap) ? __ldg(reinterpret_cast<const uint64_t*>(Eb + off)) : 0ull;
                const uint32_t v = __popcll(op_eq(w, 6));
                pdl += __popcll(op_eq(w, 5));
                uint32_t inc = v;
#pragma unroll
                for (int o2 = 1; o2 < 32; o2 <<= 1) {
                    const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o2);
                    if (lane >= o2) inc += u;
                }
                if (i < re) ipb[i] = (uint16_t)(run + inc - v);
                run += __shfl_sync(0xffffffffu, inc, 31);
            }
            if (lane == 0) S.scan2[wid] = run;
            if (leaf) pd_d += pdl; else pd_c += pdl;
        }
        {
            const uint32_t Cn0 = 8 * Pn;
            for (uint32_t i = threadIdx.x; i < (Cn0 + 31) / 32; i += K2_THREADS) dsm[Y.pend + i] = 0;
            if (!final_level)
                for (uint32_t i = threadIdx.x; i < (Cn0 + 15) / 16; i += K2_THREADS) dsm[Y.pax + i] = 0;
        }
        if (threadIdx.x == 0 && (uint64_t)e0 + 8ull * nact > nvalid)
            atomicMin(&S.errkey, ekey(nvalid, 0, EK_UNDERRUN_NV));
        __syncthreads();
        uint32_t tot_pa = 0, ioff = 0;
#pragma unroll
        for (int k = 0; k < K2_WARPS; ++k) {
            const uint32_t v = S.scan2[k];
            ioff += (uint32_t)k < wid ? v : 0u;
            tot_pa += v;
        }
        for (uint32_t i = rb + lane; i < re; i += 32) ipb[i] = (uint16_t)(ipb[i] + ioff);
        __syncwarp();
        const uint32_t Cn = 8 * Pn;
        const int pb = N - l;                        // bits per axis at the parent level
        const uint32_t pm = (1u << pb) - 1u;
        const bool al8 = MODE == OUT_RASTER && R.fast && (pitch & 1u) == 0u &&
                         (reinterpret_cast<uintptr_t>(R.base) & 7u) == 0u;
        const bool al16 = MODE == OUT_MORTON && (reinterpret_cast<uintptr_t>(out_m) & 15u) == 0u;
        // storage of child j of this level: shared level array, Morton pool slot or raster voxel
        auto child_ptr = [&](uint32_t j) -> uint32_t* {
            if (!final_level) return clev + j;
            if (MODE == OUT_MORTON) return out_m + j;
            return raster_of(R, P, j);
        };
        // all 8 children of parent q take value v
        auto fill_group = [&](uint32_t q, uint32_t v) {
            if (!final_level) {
                reinterpret_cast<uint4*>(clev + 8 * q)[0] = make_uint4(v, v, v, v);
                reinterpret_cast<uint4*>(clev + 8 * q)[1] = make_uint4(v, v, v, v);
            } else if (MODE == OUT_MORTON) {
                uint32_t* g = out_m + 8ull * q;
                if (al16) {
                    reinterpret_cast<uint4*>(g)[0] = make_uint4(v, v, v, v);
                    reinterpret_cast<uint4*>(g)[1] = make_uint4(v, v, v, v);
                } else {
#pragma unroll
                    for (int c = 0; c < 8; ++c) g[c] = v;
                }
            } else if (al8) {
                uint32_t* g = R.base + ((2 * compact3(q >> 2)) * plane + (2 * compact3(q >> 1)) * pitch + 2 * compact3(q));
                const uint2 v2 = make_uint2(v, v);
                *reinterpret_cast<uint2*>(g) = v2;
                *reinterpret_cast<uint2*>(g + pitch) = v2;
                *reinterpret_cast<uint2*>(g + plane) = v2;
                *reinterpret_cast<uint2*>(g + plane + pitch) = v2;
            } else {
#pragma unroll
                for (uint32_t c = 0; c < 8; ++c) {
                    uint32_t* pp = raster_of(R, P, 8 * q + c);
                    if (pp) *pp = v;
                }
            }
        };
        // (F0) inactive parents: children repeat the parent value (stop fill, codec.py:460-463);
        // raster order of parents for raster output so warps write whole row segments
        if (final_level && MODE == OUT_RASTER && al8) {
            for (uint32_t i = threadIdx.x; i < Pn; i += K2_THREADS) {
                const uint32_t qx = i & pm, qy = (i >> pb) & pm, qz = i >> (2 * pb);
                const uint32_t q = spread3_u32(qx) | (spread3_u32(qy) << 1) | (spread3_u32(qz) << 2);
                if ((pmask[q >> 5] >> (q & 31)) & 1u) continue;
                const uint32_t v = plev[q];
                uint32_t* g = R.base + ((2 * qz) * plane + (2 * qy) * pitch + 2 * qx);
                const uint2 v2 = make_uint2(v, v);
                *reinterpret_cast<uint2*>(g) = v2;
                *reinterpret_cast<uint2*>(g + pitch) = v2;
                *reinterpret_cast<uint2*>(g + plane) = v2;
                *reinterpret_cast<uint2*>(g + plane + pitch) = v2;
            }
        } else {
            for (uint32_t i = threadIdx.x; i < Pn; i += K2_THREADS) {
                const uint32_t q = (final_level && MODE == OUT_RASTER)
                    ? (spread3_u32(i & pm) | (spread3_u32((i >> pb) & pm) << 1) | (spread3_u32(i >> (2 * pb)) << 2)) : i;
                if ((pmask[q >> 5] >> (q & 31)) & 1u) continue;
                fill_group(q, plev[q]);
                if (!final_level) cmask[q] = 0;
            }
        }
        // (F1) active parents in 32-parent chunks per warp: each lane sets its
        // parent's 8 children to the parent value (R_p, 2/3 of all entries), then
        // the chunk's other children are spread one per lane (warp scan +
        // shuffle search), evaluated (codec.py:400-457) and stored.
        {
            const uint32_t wb0 = rb, we0 = re;          // same rank partition as (B)
            const uint64_t ones = 0x0101010101010101ull;
            for (uint32_t cb = wb0; cb < we0; cb += 32) {
                const uint32_t rk = cb + lane;
                const bool valid = rk < we0;
                const uint32_t q = valid ? (uint32_t)list[rk] : 0u;
                const uint32_t ent0 = e0 + 8 * rk;
                const uint64_t w = (valid && ent0 + 8 <= ecap) ? __ldg(reinterpret_cast<const uint64_t*>(Eb + ent0)) : 0ull;
                const uint32_t nv = nvalid > ent0 ? (nvalid - ent0 < 8 ? nvalid - ent0 : 8) : 0;
                uint32_t todo = 0;
                int32_t ipq = 0;
                if (valid) {
                    fill_group(q, plev[q]);
                    const uint64_t stops = (w >> 3) & ones;
                    if (!final_level) cmask[q] = (uint8_t)~(uint32_t)((stops * 0x0102040810204080ull) >> 56);
                    const uint64_t vmask = nv == 8 ? ~0ull : ((1ull << (8 * nv)) - 1ull);
                    const uint64_t b7 = op_eq(w, 7) & vmask, ls = leaf ? (stops & vmask & ~b7) : 0ull;
                    if (b7 | ls) {   // BAD_OP / LEAF_STOP of the whole group (codec.py:396-399)
                        if (b7) atomicMin(&S.errkey, ekey(ent0 + (__ffsll((long long)b7) - 1) / 8, 0, CSV_ST_BAD_OP));
                        if (ls) atomicMin(&S.errkey, ekey(ent0 + (__ffsll((long long)ls) - 1) / 8, 1, CSV_ST_LEAF_STOP));
                    }
                    todo = (uint32_t)(((~op_eq(w, 0) & ones & ~op_eq(w, 7)) * 0x0102040810204080ull) >> 56);
                    ipq = ipbase + (int32_t)ipb[rk];
                }
                const uint32_t cnt = __popc(todo);
                uint32_t inc = cnt;
#pragma unroll
                for (int o2 = 1; o2 < 32; o2 <<= 1) {
                    const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o2);
                    if (lane >= o2) inc += u;
                }
                const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
                const uint32_t excl = inc - cnt;
                const uint32_t wlo = (uint32_t)w, whi = (uint32_t)(w >> 32);
                __syncwarp();
                for (uint32_t k0 = 0; k0 < total; k0 += 32) {
                    const uint32_t sidx = k0 + lane;
                    int src = 0;
#pragma unroll
                    for (int step = 16; step > 0; step >>= 1) {
                        const uint32_t ex = __shfl_sync(0xffffffffu, excl, src + step);
                        if (src + step < 32 && ex <= sidx) src += step;
                    }
                    const uint32_t sq = __shfl_sync(0xffffffffu, q, src);
                    const uint32_t stodo = __shfl_sync(0xffffffffu, todo, src);
                    const uint32_t sexcl = __shfl_sync(0xffffffffu, excl, src);
                    const uint32_t slo = __shfl_sync(0xffffffffu, wlo, src);
                    const uint32_t shi = __shfl_sync(0xffffffffu, whi, src);
                    const int32_t sip = __shfl_sync(0xffffffffu, ipq, src);
                    const uint32_t sent0 = __shfl_sync(0xffffffffu, ent0, src);
                    const uint32_t snv = __shfl_sync(0xffffffffu, nv, src);
                    if (sidx >= total) continue;
                    const uint32_t c = nth_set_bit(stodo, sidx - sexcl);
                    const uint64_t sw = ((uint64_t)shi << 32) | slo;
                    const uint32_t e = (uint32_t)(sw >> (8 * c)) & 0xFFu;
                    const uint32_t op = e & 7u;
                    const uint32_t j = (sq << 3) | c;
                    uint32_t val;
                    int st = 0;
                    bool chain = false;
                    const uint32_t a = op - 1u;
                    if (a < 3u) {
                        const uint32_t M = a == 0 ? Mx : (a == 1 ? My : Mz);
                        const uint32_t part = j & M, rest = j & ~M;
                        if ((c >> a) & 1u) {   // odd: the +1 neighbour is decoded later -> its parent's value
                            st = part == M ? CSV_ST_BAD_NEIGHBOR : 0;
                            val = plev[((((part | ~M) + 1u) & M) | rest) >> 3];
                        } else {               // even: the -1 neighbour at this level
                            st = part == 0 ? CSV_ST_BAD_NEIGHBOR : 0;
                            const uint32_t qn = (((part - 1u) & M) | rest) >> 3;
                            val = plev[qn];    // final when that parent is inactive
                            chain = st == 0 && ((pmask[qn >> 5] >> (qn & 31)) & 1u);
                        }
                    } else {
                        const int32_t ip = sip + (int32_t)prefix_bytes(op_eq(sw, 6), c);
                        int32_t idx = op == 4u ? ip : (op == 5u ? ip - (int32_t)(e >> 4) - 1 : ip + 1);
                        st = idx < 0 ? CSV_ST_DELTA_RANGE : (idx >= (int32_t)plen ? CSV_ST_PALETTE_RANGE : 0);
                        idx = min(max(idx, 0), (int32_t)plen - 1);
                        val = __ldg(pal + idx);
                    }
                    if (st && c < snv && !(leaf && (e & 8u))) atomicMin(&S.errkey, ekey(sent0 + c, 2, st));
                    if (chain) {
                        atomicOr(&dsm[Y.pend + (j >> 5)], 1u << (j & 31));
                        if (!final_level) atomicOr(&dsm[Y.pax + (j >> 4)], a << (2 * (j & 15)));
                    } else {
                        uint32_t* pp = child_ptr(j);
                        if (pp) *pp = val;
                    }
                }
            }
        }
        __syncthreads();
        // (W) chains (codec.py:422-423, nm < j): walk -1 neighbours (<= 3 hops, each
        // makes one more coordinate odd) to the first child whose value is final
        if (S.errkey == ~0ull) {
            const uint32_t NWd = (Cn + 31) / 32;
            const uint32_t wpw = (NWd + K2_WARPS - 1) / K2_WARPS;
            const uint32_t wbeg = (threadIdx.x >> 5) * wpw, wend = min(wbeg + wpw, NWd);
            for (uint32_t wb = wbeg; wb < wend; wb += 32) {
                const uint32_t wi = wb + lane;
                const uint32_t word = wi < wend ? dsm[Y.pend + wi] : 0u;
                const uint32_t cnt = __popc(word);
                uint32_t inc = cnt;
#pragma unroll
                for (int o2 = 1; o2 < 32; o2 <<= 1) {
                    const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o2);
                    if (lane >= o2) inc += u;
                }
                const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
                const uint32_t excl = inc - cnt;
                for (uint32_t k0 = 0; k0 < total; k0 += 32) {
                    const uint32_t sidx = k0 + lane;
                    int src = 0;
#pragma unroll
                    for (int step = 16; step > 0; step >>= 1) {
                        const uint32_t ex = __shfl_sync(0xffffffffu, excl, src + step);
                        if (src + step < 32 && ex <= sidx) src += step;
                    }
                    const uint32_t wsrc = __shfl_sync(0xffffffffu, word, src);
                    const uint32_t esrc = __shfl_sync(0xffffffffu, excl, src);
                    if (sidx >= total) continue;
                    const uint32_t j = 32 * (wb + src) + nth_set_bit(wsrc, sidx - esrc);
                    uint32_t cl = j;
#pragma unroll 1
                    for (int hop = 0; hop < 4; ++hop) {
                        uint32_t aa;
                        if (!final_level) {
                            aa = (dsm[Y.pax + (cl >> 4)] >> (2 * (cl & 15))) & 3u;
                        } else {
                            const uint32_t qc = cl >> 3;
                            const uint32_t rkc = dsm[Y.wpre + (qc >> 5)] + __popc(pmask[qc >> 5] & ((1u << (qc & 31)) - 1u));
                            aa = (__ldg(Eb + e0 + 8 * rkc + (cl & 7)) & 7u) - 1u;
                        }
                        const uint32_t MM = aa == 0 ? Mx : (aa == 1 ? My : Mz);
                        cl = (((cl & MM) - 1u) & MM) | (cl & ~MM);
                        if (!((dsm[Y.pend + (cl >> 5)] >> (cl & 31)) & 1u)) break;
                    }
                    uint32_t* d = child_ptr(j);
                    if (!d) continue;
                    if (!final_level) { *d = clev[cl]; continue; }
                    // final level: evaluate the chain's end child cl from shared state
                    // instead of reading back the output it was stored to
                    const uint32_t qc = cl >> 3, cc = cl & 7u;
                    const uint32_t mwc = pmask[qc >> 5];
                    uint32_t val = plev[qc];
                    if ((mwc >> (qc & 31)) & 1u) {
                        const uint32_t rkc = dsm[Y.wpre + (qc >> 5)] + __popc(mwc & ((1u << (qc & 31)) - 1u));
                        const uint32_t ec0 = e0 + 8 * rkc;
                        const uint64_t wc = ec0 + 8 <= ecap ? __ldg(reinterpret_cast<const uint64_t*>(Eb + ec0)) : 0ull;
                        const uint32_t e = (uint32_t)(wc >> (8 * cc)) & 0xFFu;
                        const uint32_t op = e & 7u;
                        const uint32_t a = op - 1u;
                        if (a < 3u) {   // not pending: odd -> +1 parent, even -> inactive -1 parent
                            const uint32_t M = a == 0 ? Mx : (a == 1 ? My : Mz);
                            const uint32_t part = cl & M, rest = cl & ~M;
                            const uint32_t nb = (cc >> a) & 1u ? ((((part | ~M) + 1u) & M) | rest)
                                                                : (((part - 1u) & M) | rest);
                            val = plev[nb >> 3];
                        } else if (op >= 4u && op <= 6u) {
                            const int32_t ip = ipbase + (int32_t)ipb[rkc] + (int32_t)prefix_bytes(op_eq(wc, 6), cc);
                            int32_t idx = op == 4u ? ip : (op == 5u ? ip - (int32_t)(e >> 4) - 1 : ip + 1);
                            idx = min(max(idx, 0), (int32_t)plen - 1);
                            val = __ldg(pal + idx);
                        }
                    }
                    *d = val;
                }
            }
        }
        __syncthreads();
        const unsigned long long ek = S.errkey;
        if (ek != ~0ull) {
            const csv_stream_result& sr = leaf ? srd : src;
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
                uint64_t cnt = 0;      // nibble index of entry `ent` = ent + #payload nibbles before it
                for (uint32_t g = threadIdx.x; g < (ent + 7) / 8; g += K2_THREADS) {
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
            return;
        }
        if (leaf) cur_d = e0 + 8 * nact; else cur_c = e0 + 8 * nact;
        ipbase += (int32_t)tot_pa;
        cur ^= 1u;
    }
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
