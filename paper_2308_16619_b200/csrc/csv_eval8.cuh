// csv_eval8.cuh -- SWAR evaluation of the 8 children of one active parent in
// u8 palette-index space (K2w's u8 pass).  Host + device so that
// tools/eval8_check.cu can compare it exhaustively with the per-child
// restatement (wk::eval_group + wk::palette_children).
//
// Reference: the per-child op rules of _decode_kernel, codec.py:400-457.
// One 8-byte entry group w (byte c = child c: op | stop << 3 | delta << 4)
// is evaluated with bit-sliced byte masks over two 32-bit halves (children
// 0-3 / 4-7) instead of eight select chains:
//
//   * R_p / odd-coordinate neighbour ops (codec.py:400-425): the value is the
//     parent's or the +1 neighbour parent's index -- a byte blend of
//     broadcast candidates, the masks built on the FMA pipe (x * 0xFF);
//   * even-coordinate neighbour ops are left "pending" (2 bits per child, the
//     axis) for the chain pass, which copies child c | (1 << axis) of the -1
//     neighbour parent;
//   * palette ops (codec.py:426-457): i_p at child c is ipq + #P_a before c
//     (a byte prefix by one multiply), P_l -> i_p, P_d -> i_p - delta - 1,
//     P_a -> i_p + 1, all as biased bytes (16 + offset in [0, 24]) so the
//     range checks are byte compares against a broadcast threshold;
//   * errors (BAD_OP, LEAF_STOP, BAD_NEIGHBOR, DELTA_RANGE, PALETTE_RANGE)
//     only raise a flag here: the exact first-error key is recomputed by the
//     per-child path, which only runs for failing groups.
#pragma once
#include <cstdint>

namespace e8 {

#if defined(__CUDA_ARCH__)
__device__ __forceinline__ uint32_t popc32(uint32_t v) { return (uint32_t)__popc(v); }
#else
inline uint32_t popc32(uint32_t v) { return (uint32_t)__builtin_popcount(v); }
#endif

constexpr uint32_t O = 0x01010101u;
constexpr uint32_t MXO = 0x01000100u;   // children with an odd x coordinate (bytes 1, 3 of a half)
constexpr uint32_t MYO = 0x01010000u;   // odd y (bytes 2, 3)
constexpr uint32_t MXE = 0x00010001u;   // even x
constexpr uint32_t MYE = 0x00000101u;   // even y

struct Out {
    uint32_t vlo, vhi;   // child values (u8 indices), byte c of (vhi:vlo) = child c
    uint32_t pend;       // 2 bits per child: pending neighbour axis (1 x, 2 y, 3 z), 0 none
    uint32_t err;        // nonzero: some valid entry of the group is an error
    uint32_t n5;         // P_d payload nibbles among the valid entries
};

// bf: bit 2a = parent at coordinate 0 on axis a, bit 2a+1 = at the maximum.
// vmask: 0xFF per valid entry byte.  ipq: i_p before this group.  The +1
// neighbour values at a maximum coordinate are never used (BAD_NEIGHBOR).
// MARK: pending children hold the marker byte 252 + axis (253 x, 254 y, 255 z)
// instead of the parent's value; needs palettes of at most kMarkPal entries
// (indices <= 252).
constexpr uint32_t kMarkPal = 253;
template <bool MARK = false>
__host__ __device__ __forceinline__ void eval8(uint64_t w, uint32_t pv, uint32_t pxp, uint32_t pyp, uint32_t pzp,
                                               uint32_t bf, int32_t ipq, uint32_t plen, uint64_t vmask, bool leaf,
                                               Out& g) {
    const uint32_t PV = pv * O;
    const uint32_t DX = (pv ^ pxp) * O, DY = (pv ^ pyp) * O, DZ = (pv ^ pzp) * O;
    // boundary masks: children whose neighbour on that axis lies outside the level
    const uint32_t fx = bf & 3u, fy = (bf >> 2) & 3u;
    const uint32_t vx = fx * MXE, vy = fy * MYE;
    const uint32_t BX = (vx & MXE) | ((vx & (MXE << 1)) << 7);
    const uint32_t BY = (vy & MYE) | ((vy & (MYE << 1)) << 15);
    const uint32_t BZ0 = ((bf >> 4) & 1u) * O, BZ1 = ((bf >> 5) & 1u) * O;
    // palette index bytes: idx = ipq - 16 + B, added bytewise without carries (B <= 24)
    const uint32_t kb = ((uint32_t)(ipq - 16) & 0xFFu) * O;
    const uint32_t K7 = kb & 0x7F7F7F7Fu, K8 = kb & 0x80808080u;
    const int32_t room = (int32_t)plen - ipq;
    const bool chk_lo = ipq < 16, chk_hi = room <= 8;
    const uint32_t TL = (128u - (uint32_t)(16 - ipq)) * O;                       // B < 16 - ipq  <=>  idx < 0
    const uint32_t TH = (128u - (uint32_t)(room + 16 > 0 ? room + 16 : 0)) * O;   // B >= room + 16 <=> idx >= plen
    uint32_t carry6 = 0, err = 0, n5 = 0, pend = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const uint32_t x = h ? (uint32_t)(w >> 32) : (uint32_t)w;
        const uint32_t vm = h ? (uint32_t)(vmask >> 32) : (uint32_t)vmask;
        const uint32_t a = x & O, b = (x >> 1) & O, c = (x >> 2) & O;
        const uint32_t is1 = a & ~b & ~c, is2 = b & ~a & ~c, is3 = a & b & ~c;
        const uint32_t is5 = a & c & ~b, is6 = b & c & ~a, is7 = a & b & c;
        const uint32_t isP = c & ~(a & b);
        // neighbour ops
        const uint32_t BZ = h ? BZ1 : BZ0;
        const uint32_t bad = (is1 & BX) | (is2 & BY) | (is3 & BZ);
        uint32_t v = PV ^ (DX & ((is1 & MXO) * 0xFFu)) ^ (DY & ((is2 & MYO) * 0xFFu));
        if (h) v ^= DZ & (is3 * 0xFFu);
        const uint32_t pb = ((is1 & MXE) | ((is2 & MYE) << 1) | (h ? 0u : is3 * 3u)) & ~(bad * 3u);
        pend |= ((pb * 0x01041040u) >> 24) << (8 * h);
        if (MARK) {   // pending children hold the marker 252 + axis until the chain pass
            const uint32_t PM = ((pb | (pb >> 1)) & O) * 0xFFu;
            v = (v & ~PM) | ((pb | 0xFCFCFCFCu) & PM);
        }
        // palette ops
        const uint32_t pre = is6 * 0x01010100u + carry6 * O;
        carry6 += popc32(is6);
        const uint32_t d1 = (((x >> 4) & 0x0F0F0F0Fu) + O) & (is5 * 0xFFu);
        const uint32_t B = 0x10101010u + pre + is6 - d1;
        const uint32_t idx = (B + K7) ^ K8;
        const uint32_t FP = isP * 0xFFu;
        v = (v & ~FP) | (idx & FP);
        uint32_t rng = 0;
        if (chk_lo) rng |= ~(B + TL) & (is5 << 7);
        if (chk_hi) rng |= (B + TH) & (is6 << 7);
        uint32_t e = is7 | bad | (rng >> 7);
        if (leaf) e |= (x >> 3) & O;
        err |= e & vm;
        n5 += popc32(is5 & vm);
        if (h) g.vhi = v; else g.vlo = v;
    }
    g.pend = pend;
    g.err = err;
    g.n5 = n5;
}

}  // namespace e8
