// csv_rans.cu -- stand-alone entry points of the drop-in surface that are not
// the fused decode: the raw-nibble rANS coder (rans_decode / rans_encode,
// csvol/rans.py:120-198) and the per-brick resolution pyramid
// (build_pyramid / downsample_level, csvol/pyramid.py:43-104).
//
//  * k_rans_decode: one thread per stream.  The 4096-slot table is packed
//    into shared memory as {freq:16 | slot - cum:12 | sym:4} (the K1
//    layout), so a step is one LDS + one IMAD; renormalisation reads bytes
//    until the state is back in [2^23, 2^31).  Truncation and desync are
//    reported as (status, symbol position) exactly as _decode_core does
//    (rans.py:140-165).
//  * k_rans_encode: one thread per stream, reverse encode into the back of a
//    2n + 8 byte slot (rans.py:120-137, byte-exact).
//  * k_pyramid_level: one thread per parent node, mode of the 8 Morton
//    children with first-occurrence ties + subtree-constant flag
//    (pyramid.py:43-63); one launch per level over all bricks.
//  * k_downsample: the same rule on a (z, y, x) grid (pyramid.py:81-96).
#include <cuda_runtime.h>
#include <cstdint>
#include "../../include/csvgpu.h"

namespace csv { void set_error(const char* msg); }

namespace {

constexpr uint32_t kLower = 1u << 23;
constexpr uint32_t kPrec = 12;

struct RansTable { uint32_t freq[16]; uint32_t cum[17]; };

__device__ __forceinline__ uint32_t mode8(const uint32_t (&v)[8], bool* uniform) {
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

__global__ void __launch_bounds__(256) k_rans_decode(const uint8_t* data, const uint64_t* off, const uint32_t* nbytes,
                                                     const uint32_t* nsym, uint64_t n, RansTable T, uint8_t* out,
                                                     const uint64_t* out_off, int32_t* status) {
    __shared__ uint32_t tab[4096];
    for (uint32_t s = 0; s < 16; ++s)
        for (uint32_t k = T.cum[s] + threadIdx.x; k < T.cum[s + 1]; k += blockDim.x)
            tab[k] = (T.freq[s] << 16) | ((k - T.cum[s]) << 4) | s;
    __syncthreads();
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint8_t* d = data + off[i];
    const uint32_t nb = nbytes[i], ns = nsym[i];
    uint8_t* o = out + out_off[i];
    int32_t st = 0, pos = 0;
    if (nb < 4) {
        st = 1;
    } else {
        uint32_t x = d[0] | (d[1] << 8) | (d[2] << 16) | ((uint32_t)d[3] << 24);
        uint32_t p = 4;
        uint32_t k = 0;
        for (; k < ns; ++k) {
            const uint32_t e = tab[x & 4095u];
            x = (e >> 16) * (x >> kPrec) + ((e >> 4) & 4095u);
            bool trunc = false;
            while (x < kLower) {
                if (p >= nb) { trunc = true; break; }
                x = (x << 8) | d[p++];
            }
            if (trunc) break;
            o[k] = (uint8_t)(e & 15u);
        }
        if (k < ns) { st = 1; pos = (int32_t)k; }
        else if (x != kLower || p != nb) { st = 2; pos = (int32_t)ns; }
        else pos = (int32_t)ns;
    }
    status[2 * i] = st;
    status[2 * i + 1] = pos;
}

__global__ void __launch_bounds__(256) k_rans_encode(const uint8_t* nib, const uint64_t* off, const uint32_t* nsym,
                                                     uint64_t n, RansTable T, uint8_t* buf, const uint64_t* buf_off,
                                                     uint32_t* start) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint8_t* s = nib + off[i];
    const uint32_t ns = nsym[i];
    uint8_t* b = buf + buf_off[i];
    uint32_t ptr = 2 * ns + 8;
    uint32_t x = kLower;
    for (int64_t k = (int64_t)ns - 1; k >= 0; --k) {
        const uint32_t sy = s[k], f = T.freq[sy];
        const uint32_t xmax = ((kLower >> kPrec) << 8) * f;
        while (x >= xmax) { b[--ptr] = (uint8_t)(x & 0xFF); x >>= 8; }
        x = ((x / f) << kPrec) + (x % f) + T.cum[sy];
    }
    b[--ptr] = (uint8_t)(x >> 24);
    b[--ptr] = (uint8_t)(x >> 16);
    b[--ptr] = (uint8_t)(x >> 8);
    b[--ptr] = (uint8_t)x;
    start[i] = ptr;
}

// level l+1 of every brick from level l (Morton: node j's children are 8j .. 8j+7)
__global__ void __launch_bounds__(256) k_pyramid_level(const uint32_t* child, const uint8_t* cconst, uint64_t child_stride,
                                                       uint32_t* parent, uint8_t* pconst, uint64_t parent_stride,
                                                       uint64_t n_parent, uint64_t n_bricks) {
    const uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (g >= n_parent * n_bricks) return;
    const uint64_t br = g / n_parent, j = g % n_parent;
    const uint32_t* c = child + br * child_stride + 8 * j;
    const uint8_t* cc = cconst + br * child_stride + 8 * j;
    uint32_t v[8];
    bool all_const = true;
#pragma unroll
    for (int k = 0; k < 8; ++k) { v[k] = c[k]; all_const &= cc[k] != 0; }
    bool uniform;
    const uint32_t m = mode8(v, &uniform);
    parent[br * parent_stride + j] = m;
    pconst[br * parent_stride + j] = (uint8_t)(uniform && all_const);
}

// (nz, ny, nx) -> (nz/2, ny/2, nx/2); children of a cell in (z, y, x) C order
__global__ void __launch_bounds__(256) k_downsample(const uint32_t* in, uint32_t* out, int64_t nz, int64_t ny, int64_t nx) {
    const int64_t oz = nz / 2, oy = ny / 2, ox = nx / 2;
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= oz * oy * ox) return;
    const int64_t x = g % ox, y = (g / ox) % oy, z = g / (ox * oy);
    uint32_t v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int64_t dz = k >> 2, dy = (k >> 1) & 1, dx = k & 1;
        v[k] = in[((2 * z + dz) * ny + (2 * y + dy)) * nx + (2 * x + dx)];
    }
    bool u;
    out[g] = mode8(v, &u);
}

bool make_table(const uint16_t* counts, RansTable* T) {
    uint32_t c = 0;
    for (int s = 0; s < 16; ++s) {
        T->freq[s] = counts[s];
        T->cum[s] = c;
        c += counts[s];
    }
    T->cum[16] = c;
    return c == 4096u;
}

int launch_status(const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        csv::set_error(what);
        return CSV_E_CUDA;
    }
    return CSV_OK;
}

}  // namespace

extern "C" {

int csv_rans_decode(const uint8_t* d_data, const uint64_t* d_off, const uint32_t* d_nbytes, const uint32_t* d_nsym,
                    uint64_t n_streams, const uint16_t* counts16, uint8_t* d_out, const uint64_t* d_out_off,
                    int32_t* d_status, uintptr_t stream) {
    RansTable T;
    if (!counts16 || !make_table(counts16, &T)) { csv::set_error("rANS counts must sum to 4096"); return CSV_E_ARG; }
    if (n_streams == 0) return CSV_OK;
    const unsigned grid = (unsigned)((n_streams + 255) / 256);
    k_rans_decode<<<grid, 256, 0, (cudaStream_t)stream>>>(d_data, d_off, d_nbytes, d_nsym, n_streams, T, d_out,
                                                          d_out_off, d_status);
    return launch_status("k_rans_decode launch failed");
}

int csv_rans_encode(const uint8_t* d_nibbles, const uint64_t* d_off, const uint32_t* d_nsym, uint64_t n_streams,
                    const uint16_t* counts16, uint8_t* d_buf, const uint64_t* d_buf_off, uint32_t* d_start,
                    uintptr_t stream) {
    RansTable T;
    if (!counts16 || !make_table(counts16, &T)) { csv::set_error("rANS counts must sum to 4096"); return CSV_E_ARG; }
    if (n_streams == 0) return CSV_OK;
    const unsigned grid = (unsigned)((n_streams + 255) / 256);
    k_rans_encode<<<grid, 256, 0, (cudaStream_t)stream>>>(d_nibbles, d_off, d_nsym, n_streams, T, d_buf, d_buf_off,
                                                          d_start);
    return launch_status("k_rans_encode launch failed");
}

int csv_build_pyramid(const uint32_t* d_labels, uint64_t n_bricks, int brick_log2, uint32_t* d_levels,
                      uint8_t* d_const, uintptr_t stream) {
    if (brick_log2 < 0 || brick_log2 > 7) { csv::set_error("brick_log2 outside [0, 7]"); return CSV_E_ARG; }
    if (n_bricks == 0) return CSV_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const uint64_t total = ((1ull << (3 * (brick_log2 + 1))) - 1) / 7;   // sum of 8^l, l = 0..N
    // level 0: the labels, all constant
    if (cudaMemcpy2DAsync(d_levels, total * 4, d_labels, (1ull << (3 * brick_log2)) * 4, (1ull << (3 * brick_log2)) * 4,
                          n_bricks, cudaMemcpyDeviceToDevice, st) != cudaSuccess ||
        cudaMemset2DAsync(d_const, total, 1, 1ull << (3 * brick_log2), n_bricks, st) != cudaSuccess) {
        csv::set_error("pyramid level-0 copy failed");
        return CSV_E_CUDA;
    }
    uint64_t off = 0;
    for (int l = 0; l < brick_log2; ++l) {
        const uint64_t nc = 1ull << (3 * (brick_log2 - l)), np = nc / 8;
        const uint64_t work = np * n_bricks;
        k_pyramid_level<<<(unsigned)((work + 255) / 256), 256, 0, st>>>(d_levels + off, d_const + off, total,
                                                                        d_levels + off + nc, d_const + off + nc,
                                                                        total, np, n_bricks);
        off += nc;
    }
    return launch_status("k_pyramid_level launch failed");
}

int csv_downsample(const uint32_t* d_in, int64_t nz, int64_t ny, int64_t nx, uint32_t* d_out, uintptr_t stream) {
    if (nz % 2 || ny % 2 || nx % 2 || nz < 0 || ny < 0 || nx < 0) { csv::set_error("grid sides must be even"); return CSV_E_ARG; }
    const int64_t n = (nz / 2) * (ny / 2) * (nx / 2);
    if (n == 0) return CSV_OK;
    k_downsample<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(d_in, d_out, nz, ny, nx);
    return launch_status("k_downsample launch failed");
}

}  // extern "C"
