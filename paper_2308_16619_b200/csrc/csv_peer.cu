// csv_peer.cu -- peer-memory output buffers for the fused decode + gather
// (SURVEY.md §8e).  The receiving rank allocates the (Z, Y, X) volume with
// csv_peer_alloc and publishes its 64-byte IPC handle; every other rank maps
// it with csv_peer_open and runs csv_decode_volume with d_out pointing at its
// own z-rows INSIDE the receiver's volume.  On a multi-GPU node the mapping is
// NVLink peer memory (cudaIpcMemLazyEnablePeerAccess), so K2w's whole-row
// label stores travel straight to the receiver while later bricks are still
// being decoded: the decode IS the gather, no NCCL data-path collective and no
// staging copy.  Two processes on one device share the allocation the same way
// (that is how the single-GPU test exercises it).
#include <cuda_runtime.h>
#include <cstdint>
#include <cstring>
#include "../../include/csvgpu.h"

namespace csv { void set_error(const char* msg); }

extern "C" {

int csv_peer_alloc(int device, uint64_t bytes, void** d_ptr, uint8_t* handle64) {
    if (!d_ptr || !handle64) { csv::set_error("null argument"); return CSV_E_ARG; }
    if (cudaSetDevice(device) != cudaSuccess) { csv::set_error("cudaSetDevice failed"); return CSV_E_CUDA; }
    void* p = nullptr;
    if (cudaMalloc(&p, bytes ? bytes : 16) != cudaSuccess) { csv::set_error("cudaMalloc of the peer buffer failed"); return CSV_E_NOMEM; }
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, p) != cudaSuccess) {
        cudaFree(p);
        csv::set_error("cudaIpcGetMemHandle failed");
        return CSV_E_CUDA;
    }
    static_assert(sizeof(h) == 64, "IPC handle size");
    memcpy(handle64, &h, 64);
    *d_ptr = p;
    return CSV_OK;
}

int csv_peer_free(int device, void* d_ptr) {
    cudaSetDevice(device);
    return cudaFree(d_ptr) == cudaSuccess ? CSV_OK : CSV_E_CUDA;
}

int csv_peer_open(int device, const uint8_t* handle64, void** d_ptr) {
    if (!d_ptr || !handle64) { csv::set_error("null argument"); return CSV_E_ARG; }
    if (cudaSetDevice(device) != cudaSuccess) { csv::set_error("cudaSetDevice failed"); return CSV_E_CUDA; }
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, 64);
    const cudaError_t e = cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) { csv::set_error(cudaGetErrorString(e)); return CSV_E_CUDA; }
    return CSV_OK;
}

int csv_peer_close(int device, void* d_ptr) {
    cudaSetDevice(device);
    return cudaIpcCloseMemHandle(d_ptr) == cudaSuccess ? CSV_OK : CSV_E_CUDA;
}

}  // extern "C"
