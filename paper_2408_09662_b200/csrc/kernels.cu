// Static sm_100a kernels compiled by nvcc into libvsb200.so.
//
// Layout conversion between the reference's env-major workspace layout
// ([B, nnz] row-major, batchrt.py:78-169) and the structure-of-arrays
// [nnz, ld] layout the SoA entry point consumes.  Tiled through shared
// memory so both the read and the write side are coalesced.
#include <cuda_runtime.h>
#include <stdint.h>

#include "vsb200.h"

namespace {

constexpr int TILE = 32;
constexpr int ROWS = 8;

// src: [rows, cols] row-major with leading dim lds; dst: [cols, rows] with leading dim ldd
template <typename T>
__global__ void __launch_bounds__(TILE * ROWS) transpose_kernel(const T* __restrict__ src, T* __restrict__ dst,
                                                                 int64_t rows, int64_t cols, int64_t lds, int64_t ldd) {
    __shared__ T tile[TILE][TILE + 1];
    const int64_t c0 = static_cast<int64_t>(blockIdx.x) * TILE, r0 = static_cast<int64_t>(blockIdx.y) * TILE;
    for (int k = threadIdx.y; k < TILE; k += ROWS) {
        const int64_t r = r0 + k, c = c0 + threadIdx.x;
        if (r < rows && c < cols) tile[k][threadIdx.x] = src[r * lds + c];
    }
    __syncthreads();
    for (int k = threadIdx.y; k < TILE; k += ROWS) {
        const int64_t c = c0 + k, r = r0 + threadIdx.x;
        if (r < rows && c < cols) dst[c * ldd + r] = tile[threadIdx.x][k];
    }
}

template <typename T>
int launch_transpose(const void* src, void* dst, int64_t rows, int64_t cols, int64_t lds, int64_t ldd, cudaStream_t s) {
    if (rows <= 0 || cols <= 0) return VSB_OK;
    const int64_t gx = (cols + TILE - 1) / TILE, gy = (rows + TILE - 1) / TILE;
    if (gy > 65535) {
        // long batches: sweep the row dimension in slabs of 65535 tiles
        const int64_t slab = 65535LL * TILE;
        for (int64_t r = 0; r < rows; r += slab) {
            const int64_t m = rows - r < slab ? rows - r : slab;
            int rc = launch_transpose<T>(static_cast<const T*>(src) + r * lds, static_cast<T*>(dst) + r, m, cols, lds,
                                         ldd, s);
            if (rc != VSB_OK) return rc;
        }
        return VSB_OK;
    }
    transpose_kernel<T><<<dim3(static_cast<unsigned>(gx), static_cast<unsigned>(gy)), dim3(TILE, ROWS), 0, s>>>(
        static_cast<const T*>(src), static_cast<T*>(dst), rows, cols, lds, ldd);
    return cudaGetLastError() == cudaSuccess ? VSB_OK : VSB_ERR_CUDA;
}

}  // namespace

extern "C" int vsb_transpose(const void* src, void* dst, int64_t rows, int64_t cols, int64_t lds, int64_t ldd,
                             int32_t dtype, void* stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    return dtype == VSB_F32 ? launch_transpose<float>(src, dst, rows, cols, lds, ldd, s)
                            : launch_transpose<double>(src, dst, rows, cols, lds, ldd, s);
}
