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

template <int MODE, int LMAX>
__global__ void __launch_bounds__(K2_THREADS, 4) k2_fast(VolView V, Plan P) {
    static_assert(LMAX <= 5, "shared-memory replay covers N - t <= 5");
    constexpr Layout Y = make_layout(LMAX, 2);
    constexpr uint32_t TSMAX = LMAX >= 4 ? 4096u : (1u << (3 * LMAX));
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
        // (A) rank prefix of active parents
        for (uint32_t i = threadIdx.x; i < W; i += K2_THREADS) {
            uint32_t mw = pmask[i];
            if (Pn < 32) mw &= (1u << Pn) - 1u;
            pmask[i] = mw;
            dsm[Y.wpre + i] = __popc(mw);
        }
        __syncthreads();
        const uint32_t nact = block_scan_inplace(dsm + Y.wpre, W, S);
        // (B) active list + palette-advance counts per active parent
        for (uint32_t i = threadIdx.x; i < W; i += K2_THREADS) {
            uint32_t mw = pmask[i], rk = dsm[Y.wpre + i];
            while (mw) {
                list[rk++] = (uint16_t)(32 * i + (__ffs(mw) - 1));
                mw &= mw - 1;
            }
        }
        uint32_t pdl = 0;
        for (uint32_t i = threadIdx.x; i < nact; i += K2_THREADS) {
            const uint32_t off = e0 + 8 * i;
            const uint64_t w = off + 8 <= ecap ? __ldg(reinterpret_cast<const uint64_t*>(Eb + off)) : 0ull;
            ipb[i] = (uint16_t)__popcll(op_eq(w, 6));
            pdl += __popcll(op_eq(w, 5));
        }
        if (leaf) pd_d += pdl; else pd_c += pdl;
        __syncthreads();
        const uint32_t tot_pa = block_scan_inplace(ipb, nact, S);
        if (threadIdx.x == 0 && (uint64_t)e0 + 8ull * nact > nvalid)
            atomicMin(&S.errkey, ekey(nvalid, 0, EK_UNDERRUN_NV));
        const uint32_t Cn = 8 * Pn;
        const uint32_t TS = final_level ? (Cn < TSMAX ? Cn : TSMAX) : Cn;
        const uint32_t NT = Cn / TS;
        const uint32_t PT = TS / 8;
        const uint32_t dst_off = final_level ? Y.buf : Y.lev + levoffA(N - l + 1);
        for (uint32_t o = 0; o < NT; ++o) {
            const uint32_t q0 = o * PT, q1 = q0 + PT;
            const uint32_t j0 = 8 * q0;
            const uint32_t r0 = dsm[Y.wpre + (q0 >> 5)] + __popc(pmask[q0 >> 5] & ((1u << (q0 & 31)) - 1u));
            const uint32_t r1 = q1 >= Pn ? nact
                                         : dsm[Y.wpre + (q1 >> 5)] + __popc(pmask[q1 >> 5] & ((1u << (q1 & 31)) - 1u));
            for (uint32_t i = threadIdx.x; i < TS / 32; i += K2_THREADS) dsm[Y.pend + i] = 0;
            for (uint32_t i = threadIdx.x; i < TS / 16; i += K2_THREADS) dsm[Y.pax + i] = 0;
            __syncthreads();
            // (C1) active parents of this tile, one lane per parent: the 8 entry
            // bytes are read at once, all children start as the parent value
            // (R_p, 2/3 of all entries), and only the other ops are evaluated.
            for (uint32_t rk = r0 + threadIdx.x; rk < r1; rk += K2_THREADS) {
                const uint32_t q = list[rk];
                const uint32_t ent0 = e0 + 8 * rk;
                const uint64_t w = ent0 + 8 <= ecap ? __ldg(reinterpret_cast<const uint64_t*>(Eb + ent0)) : 0ull;
                const uint32_t pv = plev[q];
                uint32_t* const d = dsm + dst_off + 8 * (q - q0);
                reinterpret_cast<uint4*>(d)[0] = make_uint4(pv, pv, pv, pv);
                reinterpret_cast<uint4*>(d)[1] = make_uint4(pv, pv, pv, pv);
                const uint64_t ones = 0x0101010101010101ull;
                const uint64_t stops = (w >> 3) & ones;
                if (!final_level) cmask[q] = (uint8_t)~(uint32_t)((stops * 0x0102040810204080ull) >> 56);
                // flag errors of the whole group first (BAD_OP, LEAF_STOP; codec.py:396-399)
                const uint32_t nv = nvalid > ent0 ? (nvalid - ent0 < 8 ? nvalid - ent0 : 8) : 0;
                const uint64_t vmask = nv == 8 ? ~0ull : ((1ull << (8 * nv)) - 1ull);
                const uint64_t b7 = op_eq(w, 7) & vmask, ls = leaf ? (stops & vmask & ~b7) : 0ull;
                if (b7 | ls) {
                    if (b7) atomicMin(&S.errkey, ekey(ent0 + (__ffsll((long long)b7) - 1) / 8, 0, CSV_ST_BAD_OP));
                    if (ls) atomicMin(&S.errkey, ekey(ent0 + (__ffsll((long long)ls) - 1) / 8, 1, CSV_ST_LEAF_STOP));
                }
                const uint64_t pa = op_eq(w, 6);
                const int32_t ipq = ipbase + (int32_t)ipb[rk];
                // non-R_p children: bytes whose op is not 0 (op 7 keeps pv; flagged above)
                uint32_t todo = (uint32_t)(((~op_eq(w, 0) & ones & ~op_eq(w, 7)) * 0x0102040810204080ull) >> 56);
                while (todo) {
                    const uint32_t c = __ffs(todo) - 1;
                    todo &= todo - 1;
                    const uint32_t e = (uint32_t)(w >> (8 * c)) & 0xFFu;
                    const uint32_t op = e & 7u;
                    const uint32_t j = (q << 3) | c;
                    uint32_t val;
                    int st = 0;
                    bool chain = false;
                    uint32_t a = op - 1u;
                    if (a < 3u) {
                        const uint32_t M = a == 0 ? Mx : (a == 1 ? My : Mz);
                        const uint32_t part = j & M, rest = j & ~M;
                        if ((c >> a) & 1u) {   // odd: the +1 neighbour is decoded later -> its parent's value
                            st = part == M ? CSV_ST_BAD_NEIGHBOR : 0;
                            val = plev[((((part | ~M) + 1u) & M) | rest) >> 3];
                        } else {               // even: the -1 neighbour at this level
                            st = part == 0 ? CSV_ST_BAD_NEIGHBOR : 0;
                            const uint32_t nb = ((part - 1u) & M) | rest;
                            const uint32_t qn = nb >> 3;
                            val = plev[qn];    // final when that parent is inactive
                            chain = st == 0 && ((pmask[qn >> 5] >> (qn & 31)) & 1u);
                            if (chain && nb < j0) {          // earlier tile: already in HBM
                                chain = false;
                                const uint32_t* p = MODE == OUT_MORTON ? out_m + nb : raster_of(R, P, nb);
                                val = p ? *p : 0u;
                            }
                        }
                    } else {
                        const int32_t ip = ipq + (int32_t)prefix_bytes(pa, c);
                        int32_t idx = op == 4u ? ip : (op == 5u ? ip - (int32_t)(e >> 4) - 1 : ip + 1);
                        st = idx < 0 ? CSV_ST_DELTA_RANGE : (idx >= (int32_t)plen ? CSV_ST_PALETTE_RANGE : 0);
                        idx = min(max(idx, 0), (int32_t)plen - 1);
                        val = __ldg(pal + idx);
                    }
                    if (st && c < nv && !(leaf && (e & 8u))) atomicMin(&S.errkey, ekey(ent0 + c, 2, st));
                    const uint32_t jl = j - j0;
                    if (chain) {
                        atomicOr(&dsm[Y.pend + (jl >> 5)], 1u << (jl & 31));
                        atomicOr(&dsm[Y.pax + (jl >> 4)], a << (2 * (jl & 15)));
                    } else {
                        d[c] = val;
                    }
                }
            }
            // (C2) inactive parents of this tile
            for (uint32_t q = q0 + threadIdx.x; q < q1; q += K2_THREADS) {
                if ((pmask[q >> 5] >> (q & 31)) & 1u) continue;
                const uint32_t pv = plev[q];
                uint4* d = reinterpret_cast<uint4*>(dsm + dst_off + 8 * (q - q0));
                d[0] = make_uint4(pv, pv, pv, pv);
                d[1] = make_uint4(pv, pv, pv, pv);
                if (!final_level) cmask[q] = 0;
            }
            __syncthreads();
            // (W) chains: walk -1 neighbours to the first final value (<= 3 hops).
            // Each warp compacts the pending bits of its words (ballot-free scan
            // over lanes) so that every lane walks one chain.
            {
                const uint32_t NWd = TS / 32;
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
                        const uint32_t jl = 32 * (wb + src) + __fns(wsrc, 0, (int)(sidx - esrc) + 1);
                        uint32_t cl = jl;
#pragma unroll 1
                        for (int hop = 0; hop < 4; ++hop) {
                            const uint32_t aa = (dsm[Y.pax + (cl >> 4)] >> (2 * (cl & 15))) & 3u;
                            const uint32_t MM = aa == 0 ? Mx : (aa == 1 ? My : Mz);
                            const uint32_t jg = cl + j0;
                            cl = ((((jg & MM) - 1u) & MM) | (jg & ~MM)) - j0;
                            if (!((dsm[Y.pend + (cl >> 5)] >> (cl & 31)) & 1u)) break;
                        }
                        dsm[dst_off + jl] = dsm[dst_off + cl];
                    }
                }
            }
            __syncthreads();
            if (!final_level) continue;
            // (T) stream the tile to HBM
            if (MODE == OUT_MORTON) {
                uint32_t* d = out_m + (size_t)TS * o;
                const bool al = (reinterpret_cast<uintptr_t>(d) & 15) == 0;
                for (uint32_t i = threadIdx.x; i < TS / 4; i += K2_THREADS) {
                    const uint4 v = reinterpret_cast<const uint4*>(dsm + Y.buf)[i];
                    if (al) reinterpret_cast<uint4*>(d)[i] = v;
                    else { d[4 * i] = v.x; d[4 * i + 1] = v.y; d[4 * i + 2] = v.z; d[4 * i + 3] = v.w; }
                }
            } else if (TS == 4096 && R.fast) {
                // 16^3 tile: lane = (x-group 4, y0y1 4, z0 2); each lane reads its 4
                // x-consecutive voxels rotated by its x-group so every LDS hits 32
                // distinct banks, then writes them as one 16-byte row segment
                const uint32_t xg = lane & 3, y01 = (lane >> 2) & 3, z0 = (lane >> 4) & 1;
                const uint32_t ox = (compact3(o) << 4) + 4 * xg;
                const uint32_t oy = compact3(o >> 1) << 4, oz = compact3(o >> 2) << 4;
                const uint32_t mx = spread3_u32(4 * xg);
                const uint32_t s0 = spread3_u32(xg & 3), s1 = spread3_u32((xg + 1) & 3),
                               s2 = spread3_u32((xg + 2) & 3), s3 = spread3_u32((xg + 3) & 3);
                const bool al = ((pitch & 3u) == 0u) && ((reinterpret_cast<uintptr_t>(R.base) & 15u) == 0u);
                auto tile_rows = [&](auto vec) {
#pragma unroll
                    for (int it = 0; it < 4; ++it) {
                        const uint32_t combo = (threadIdx.x >> 5) * 4 + it;      // 0..31
                        const uint32_t y = y01 | ((combo & 3) << 2), z = z0 | ((combo >> 2) << 1);
                        const uint32_t mb = (spread3_u32(y) << 1) | (spread3_u32(z) << 2) | mx;
                        const uint32_t u0 = dsm[Y.buf + (mb | s0)], u1 = dsm[Y.buf + (mb | s1)],
                                       u2 = dsm[Y.buf + (mb | s2)], u3 = dsm[Y.buf + (mb | s3)];
                        // un-rotate: v[x] = u[(x - xg) & 3]
                        uint32_t v0 = u0, v1 = u1, v2 = u2, v3 = u3;
                        if (xg & 1) { uint32_t tt = v3; v3 = v2; v2 = v1; v1 = v0; v0 = tt; }
                        if (xg & 2) { uint32_t t0 = v0, t1 = v1; v0 = v2; v1 = v3; v2 = t0; v3 = t1; }
                        uint32_t* p = R.base + ((oz + z) * plane + (oy + y) * pitch + ox);
                        if (decltype(vec)::value) {
                            *reinterpret_cast<uint4*>(p) = make_uint4(v0, v1, v2, v3);
                        } else {
                            asm volatile("st.global.v2.u32 [%0], {%1, %2};" :: "l"(p), "r"(v0), "r"(v1) : "memory");
                            asm volatile("st.global.v2.u32 [%0], {%1, %2};" :: "l"(p + 2), "r"(v2), "r"(v3) : "memory");
                        }
                    }
                };
                if (al) tile_rows(std::true_type{});
                else if ((pitch & 1u) == 0u && (reinterpret_cast<uintptr_t>(R.base) & 7u) == 0u) tile_rows(std::false_type{});
                else {
                    for (int it = 0; it < 4; ++it) {
                        const uint32_t combo = (threadIdx.x >> 5) * 4 + it;
                        const uint32_t y = y01 | ((combo & 3) << 2), z = z0 | ((combo >> 2) << 1);
                        const uint32_t mb = (spread3_u32(y) << 1) | (spread3_u32(z) << 2) | mx;
                        uint32_t* p = R.base + ((oz + z) * plane + (oy + y) * pitch + ox);
#pragma unroll
                        for (uint32_t k = 0; k < 4; ++k) {
                            const uint32_t v = dsm[Y.buf + (mb | spread3_u32(k))];
                            asm volatile("st.global.u32 [%0], %1;" :: "l"(p + k), "r"(v) : "memory");
                        }
                    }
                }
            } else {
                const int tb = (31 - __clz(TS)) / 3;          // log2 of the tile side
                const uint32_t ts = 1u << tb;
                const uint32_t tx = compact3(o) << tb, ty = compact3(o >> 1) << tb, tz = compact3(o >> 2) << tb;
                for (uint32_t i = threadIdx.x; i < TS; i += K2_THREADS) {
                    const uint32_t x = i & (ts - 1), y = (i >> tb) & (ts - 1), z = i >> (2 * tb);
                    const uint32_t v = dsm[Y.buf + (spread3_u32(x) | (spread3_u32(y) << 1) | (spread3_u32(z) << 2))];
                    if (R.fast) {
                        R.base[(tz + z) * plane + (ty + y) * pitch + tx + x] = v;
                    } else {
                        const int64_t gx = R.ox + tx + x, gy = R.oy + ty + y, gz = R.oz + tz + z;
                        if (gz >= P.z_begin && gz < P.z_end && gy < P.cy && gx < P.cx)
                            P.out[((gz - P.z_begin) * P.cy + gy) * P.cx + gx] = v;
                    }
                }
            }
            __syncthreads();
        }
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
