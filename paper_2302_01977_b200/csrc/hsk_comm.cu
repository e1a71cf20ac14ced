// hsk_comm.cu -- peer-memory plumbing for the row-sharded S' = A^T R^T of
// BASELINE.json C5 (one process per GPU, NVLink/NVSwitch peers).
//
// The reference sums the per-shard partials of A^T R^T with a collective
// (SURVEY.md §8(e)); here every rank's S' kernel stores each destination
// block straight into the owning rank's receive slot through a CUDA-IPC
// mapping of that rank's buffer (the kernel's epilogue writes over NVLink,
// tile by tile, while other tiles are still being computed), and the owner
// sums its slots in rank order -- deterministic, no reduction collective.
//   hsk_ipc_alloc / hsk_ipc_free   receive buffer + its IPC handle
//   hsk_ipc_open / hsk_ipc_close   map / unmap a peer's buffer
//   hsk_sum_slices                 rank-ordered sum of the received slots
#include <string.h>

#include <algorithm>

#include "hsk_common.cuh"

namespace hsk {
namespace comm {

// out(r, c) = sum_{g = 0..nslices-1} base[g*stride + c*ld + r], in g order
__global__ void sum_slices_kernel(const double *__restrict__ base, int nslices, int64_t stride,
                                  int64_t rows, int64_t cols, int64_t ld, double *__restrict__ out,
                                  int64_t ldo) {
    const int64_t total = rows * cols;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = q / rows, r = q - c * rows;
        const double *src = base + c * ld + r;
        double acc = src[0];
        for (int g = 1; g < nslices; ++g) acc += src[g * stride];
        out[c * ldo + r] = acc;
    }
}

}  // namespace comm
}  // namespace hsk

using namespace hsk;

extern "C" int hsk_ipc_alloc(int64_t bytes, void **ptr, void *handle) {
    HSK_REQUIRE(bytes > 0 && ptr && handle, HSK_EINVAL, "ipc alloc: bad arguments");
    cudaError_t e = cudaMalloc(ptr, (size_t)bytes);
    if (e != cudaSuccess) return cuda_status(e, "ipc alloc: cudaMalloc");
    cudaIpcMemHandle_t h;
    e = cudaIpcGetMemHandle(&h, *ptr);
    if (e != cudaSuccess) {
        cudaFree(*ptr);
        *ptr = nullptr;
        return cuda_status(e, "ipc alloc: cudaIpcGetMemHandle");
    }
    static_assert(sizeof(h) == HSK_IPC_HANDLE_BYTES, "IPC handle size");
    memcpy(handle, &h, sizeof(h));
    return HSK_OK;
}

extern "C" int hsk_ipc_free(void *ptr) {
    if (!ptr) return HSK_OK;
    cudaError_t e = cudaFree(ptr);
    return e == cudaSuccess ? HSK_OK : cuda_status(e, "ipc free");
}

extern "C" int hsk_ipc_open(const void *handle, void **ptr) {
    HSK_REQUIRE(handle && ptr, HSK_EINVAL, "ipc open: bad arguments");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
    return e == cudaSuccess ? HSK_OK : cuda_status(e, "ipc open: cudaIpcOpenMemHandle");
}

extern "C" int hsk_ipc_close(void *ptr) {
    if (!ptr) return HSK_OK;
    cudaError_t e = cudaIpcCloseMemHandle(ptr);
    return e == cudaSuccess ? HSK_OK : cuda_status(e, "ipc close");
}

extern "C" int hsk_sum_slices(const double *base, int32_t nslices, int64_t stride, int64_t rows,
                              int64_t cols, int64_t ld, double *out, int64_t ldo, void *stream) {
    HSK_REQUIRE(nslices >= 1 && rows >= 0 && cols >= 0 && ld >= rows && ldo >= rows &&
                    stride >= ld * cols,
                HSK_EINVAL, "sum slices: bad shape");
    if (rows == 0 || cols == 0) return HSK_OK;
    HSK_REQUIRE(base && out, HSK_EINVAL, "sum slices: null pointer");
    const int64_t total = rows * cols;
    const unsigned blocks = (unsigned)std::min<int64_t>((total + 255) / 256, sm_count() * 8);
    comm::sum_slices_kernel<<<std::max(1u, blocks), 256, 0, as_stream(stream)>>>(
        base, nslices, stride, rows, cols, ld, out, ldo);
    HSK_CHECK_LAUNCH("sum_slices_kernel");
    return HSK_OK;
}

// Strided 2-D copy (host <-> device, async on `stream`): `height` rows of
// `width` bytes, pitches in bytes -- row slabs of column-major matrices for
// the pipelined host path (sketching.apply_right on pinned host arrays).
// kind: 1 = host to device, 2 = device to host.
extern "C" int hsk_memcpy2d(void *dst, int64_t dpitch, const void *src, int64_t spitch,
                            int64_t width, int64_t height, int32_t kind, void *stream) {
    HSK_REQUIRE(kind == 1 || kind == 2, HSK_EINVAL, "memcpy2d: kind must be 1 or 2");
    HSK_REQUIRE(width >= 0 && height >= 0 && dpitch >= width && spitch >= width, HSK_EINVAL,
                "memcpy2d: bad shape");
    if (width == 0 || height == 0) return HSK_OK;
    cudaError_t e = cudaMemcpy2DAsync(dst, (size_t)dpitch, src, (size_t)spitch, (size_t)width,
                                      (size_t)height,
                                      kind == 1 ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost,
                                      as_stream(stream));
    return e == cudaSuccess ? HSK_OK : cuda_status(e, "memcpy2d");
}
