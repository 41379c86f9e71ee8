// csv_device.cuh -- shared device-side types and helpers for the B200 CSV decoder.
//
// Data layout in HBM: the container's directory is unpacked
// once into SoA columns (local brick index), the three blobs stay exactly as
// in the CSV1 file (palette u32, coarse bytes, detail bytes) plus 16 B of
// tail padding so the entropy lanes may prefetch one word past a stream.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/csvgpu.h"

namespace csv {

// thread-local last-error text shared by every C-ABI entry point (csv_last_error)
void set_error(const char* msg);

constexpr uint32_t kStateLower = 1u << 23;   // rans.py:27
constexpr int kPrecision = 12;               // rans.py:25
constexpr uint32_t kTotalFreq = 1u << 12;    // rans.py:26

// Read-only view of one uploaded volume (bricks [brick_begin, brick_begin + nb)).
struct VolView {
    const uint64_t* pal_off;   // rebased to the uploaded palette slice (entries)
    const uint32_t* pal_len;   // clamped like numpy slicing
    const uint64_t* c_off;
    const uint32_t* c_bytes;
    const uint32_t* c_nib;
    const uint64_t* d_off;
    const uint32_t* d_bytes;
    const uint32_t* d_nib;
    const uint32_t* palette;
    const uint8_t* coarse;
    const uint8_t* detail;
    const uint32_t* dtab;      // 2 x 4096 packed decode tables (interior, leaf)
    int N;                     // brick_log2
    int entropy;               // header flag bit 0 (container.py:7)
    int64_t X, Y, Z;           // original dims
    int64_t gx, gy, gz;        // brick grid
    uint64_t brick_begin;
    uint64_t nb;
    uint32_t max_pal;          // longest palette (K2w works in u16 palette-index space)
    int fast_tab;              // every table count <= 4095: K1f's packed table applies
};

constexpr uint32_t kWScratch6Stride = 57344;   // K2w<6> scratch per warp slot (u16): palette bases 32768,
                                               // final parent level 16384 (32 KB), coarse list + descriptors 8192
constexpr int kK2W6MaxWarpsPerSM = 8;          // K2w<6> warp slots per SM
constexpr uint32_t kWScratchStride = 4096;   // K2w scratch per warp slot (final-level parents, LMAX <= 5)
constexpr int kScanTmpSlots = 4104;           // u64 scan workspace (4096 block sums + total + pad)
constexpr int kCounterSlots = 8;              // work counters of one decode (K1 items, K2w passes, ready-queue tail)

// Side stream + fork/join events of a volume's K1 -> K2w overlap launch (run_decode).
struct Overlap {
    cudaStream_t side = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};

// One decode call: n requests; request r decodes brick `brick[r]` at LOD lod[r].
struct Plan {
    uint64_t n;
    uint64_t first;            // implicit requests: local brick first + r
    const uint32_t* brick;     // global brick index, or nullptr => brick_begin + first + r
    const uint8_t* lod;        // per-request LOD, or nullptr => t_uniform
    int t_uniform;
    const uint64_t* dst;       // Morton mode: pool element offset per request
    uint32_t* out;             // raster slab base or pool base
    int64_t z_begin, z_end;    // raster slab (LOD-t voxel rows)
    int64_t cx, cy;            // cropped LOD-t x/y extent
    uint64_t* eoff;            // [2n+1] entry-region offsets (bytes)
    csv_stream_result* sres;   // [2n]
    uint8_t* entries;
    csv_result* res;           // [n] or nullptr
    unsigned long long* op_counts;   // K1 count mode (stats): 8 per-op totals, else nullptr
    uint16_t* wscratch;        // K2w: per resident warp, palette base per final-level active parent
    uint32_t wscratch_stride;  // u16 per warp slot
    uint16_t* wscratch6;       // K2w<6> (64^3 replays): per warp slot kWScratch6Stride u16 =
                               //   palette bases (32768 u16) + the final parent level (32768 u8)
    int k2w6;                  // K2w<6> serves the u8 bricks with N - t = 6 (k2_replay<6> skips them)
    // K1 -> K2w overlap (single-wave plans): K1 counts finished streams per request in
    // rcnt and appends a request to the ready queue rq (r + 1, 0 = not yet) once both of
    // its streams are done; the u8 K2w pass takes queue slots instead of request indices.
    uint32_t* rcnt;            // [n] or nullptr (no overlap)
    uint32_t* rq;              // [n]
    unsigned long long* rq_tail;
    uint32_t wslot0;           // first wscratch warp slot of this K2w launch (the overlap launch runs beside another)
    // overlap launch only: K1's grid and its count of started blocks.  Its warps replay bricks
    // only once every K1 block is resident (else they could hold the SM resources a K1 block
    // waits for while spinning on that block's bricks); otherwise they exit and the launch
    // after K1 takes the whole queue.
    unsigned long long* k1_started;
    uint32_t k1_grid;
};

__device__ __forceinline__ uint64_t req_local(const VolView& V, const Plan& P, uint64_t r) {
    return P.brick ? (uint64_t)P.brick[r] - V.brick_begin : P.first + r;
}
__device__ __forceinline__ int req_lod(const Plan& P, uint64_t r) {
    return P.lod ? (int)P.lod[r] : P.t_uniform;
}

// Max entries the replay can consume from a stream (coarse: levels N..max(t+1,2);
// detail: level 1 when t == 0).  Entries are at most 2 nibbles (codec.py:203-211),
// so K1 never needs more than 2x this many nibbles (prefix decode, codec.py:330).
__host__ __device__ __forceinline__ uint32_t max_entries(int N, int t, int s) {
    if (s == 1) return t == 0 ? (1u << (3 * N)) : 0u;
    uint32_t tot = 0;
    int lo = t + 1 > 2 ? t + 1 : 2;
    for (int l = N; l >= lo; --l) tot += 1u << (3 * (N - l + 1));
    return tot;
}

// Effective nibble count: raw containers unpack 2 nibbles/byte and slice to the
// stored count (container.py:333-337), so the count saturates at 2*bytes.
__device__ __forceinline__ uint32_t eff_nibbles(const VolView& V, uint64_t b, int s) {
    uint32_t n = s ? V.d_nib[b] : V.c_nib[b];
    if (!V.entropy) {
        uint64_t cap = 2ull * (s ? V.d_bytes[b] : V.c_bytes[b]);
        if (n > cap) n = (uint32_t)cap;
    }
    return n;
}

__device__ __forceinline__ uint32_t stream_limit(const VolView& V, uint64_t b, int t, int s) {
    if (s == 1 && t != 0) return 0;
    uint32_t n = eff_nibbles(V, b, s);
    uint32_t cap = 2u * max_entries(V.N, t, s);
    return n < cap ? n : cap;
}

__host__ __device__ __forceinline__ uint64_t round16(uint64_t v) { return (v + 15) & ~15ull; }
__host__ __device__ __forceinline__ uint64_t round32(uint64_t v) { return (v + 31) & ~31ull; }
constexpr uint64_t kBlobPad = 64;   // readable bytes past every blob (chunk prefetch)

// ---- Morton (x lowest bit, morton.py:3-6) on brick-local indices (<= 21 bits)
__device__ __forceinline__ uint32_t axis_mask(int a, int bits_per_axis) {
    uint32_t m = 0x49249u << a;                   // bits a, a+3, ..., a+18
    return m & ((1u << (3 * bits_per_axis)) - 1u);
}
__device__ __forceinline__ uint32_t spread3_u32(uint32_t v) {   // 7-bit coordinate -> bits 0,3,..,18
    v = (v | (v << 8)) & 0x0000F00Fu;
    v = (v | (v << 4)) & 0x000C30C3u;
    v = (v | (v << 2)) & 0x00249249u;
    return v;
}

// offset of level (N - j) inside a coarse-to-fine level array (root first)
__host__ __device__ __forceinline__ uint32_t levoff(int j) {
    return ((1u << (3 * j)) - 1u) / 7u;
}

__device__ __forceinline__ uint32_t compact3(uint32_t v) {   // bits 0,3,6.. -> 0,1,2..
    v &= 0x00249249u;
    v = (v ^ (v >> 2)) & 0x000C30C3u;
    v = (v ^ (v >> 4)) & 0x0000F00Fu;
    v = (v ^ (v >> 8)) & 0x000000FFu;
    return v;
}

// ---- SWAR helpers over 8 entry bytes (entry = op | stop<<3 | delta<<4)
__device__ __forceinline__ uint64_t op_eq(uint64_t w, uint32_t op) {
    const uint64_t ones = 0x0101010101010101ull;
    uint64_t d = (w & 0x0707070707070707ull) ^ (ones * op);
    uint64_t nz = (d | (d >> 1) | (d >> 2)) & ones;
    return nz ^ ones;   // 0x01 in every byte whose op == `op`
}
__device__ __forceinline__ uint32_t prefix_bytes(uint64_t m, int c) {   // # flagged bytes before byte c
    return (uint32_t)__popcll(m & ((1ull << (8 * c)) - 1ull));
}

}  // namespace csv
