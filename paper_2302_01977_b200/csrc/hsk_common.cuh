// hsk_common.cuh -- shared helpers for the sm_100a sketch kernels:
// error plumbing for the C ABI and inline-PTX wrappers for mbarrier,
// cp.async.bulk (TMA bulk copy engine) and cp.async.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/hsk.h"

namespace hsk {

// ---------------------------------------------------------------- errors
int set_error(int code, const char *fmt, ...);
int cuda_status(cudaError_t e, const char *what);

#define HSK_CHECK_LAUNCH(what)                                             \
    do {                                                                   \
        cudaError_t _e = cudaGetLastError();                               \
        if (_e != cudaSuccess) return ::hsk::cuda_status(_e, what);        \
    } while (0)

#define HSK_REQUIRE(cond, code, ...)                                       \
    do {                                                                   \
        if (!(cond)) return ::hsk::set_error(code, __VA_ARGS__);           \
    } while (0)

int sm_count();

// Run-time tuning knobs (HSK_* environment variables), read once and cached:
// a launch costs no getenv() scans.  hsk_tuning_reload() re-reads them (tests
// and A/B tools that change the environment in-process).  -1 = unset.
struct Tuning {
    int sjlt_w32, sjlt_tk, sjlt_tk_t, sjlt_rpt, sjlt_rpt_t, sjlt_prod, sjlt_streamk, sjlt_mc,
        sjlt_stages, sjlt_wait_ns, sjlt_dbg, sjlt_pf, sjlt_fused, sjlt_xp, sjlt_xp_gb, gauss_splits;
    char gauss_cfg[32];
};
const Tuning &tuning();

// Scratch for cross-CTA partial sums: a zero-initialised flag array plus a
// data area, one per (device, stream) so launches on different streams never
// share it; launches on one stream are ordered, and every kernel that uses
// the flags leaves them zero.  Grows on demand (never shrinks).
int stream_workspace(cudaStream_t st, size_t data_bytes, int nflags, void **data, int **flags);

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// 2-D float64 TMA descriptor over a column-major matrix: inner dimension =
// rows (contiguous), outer = columns, row stride lda*8 bytes (multiple of 16).
// Out-of-bounds box elements are zero-filled by the TMA unit.
// swizzle128: 128-byte TMA swizzle (16-byte chunk c of each 128-byte row r of
// the box lands at chunk c ^ (r % 8); needs a 1024-byte aligned destination).
int make_tmap_f64_2d(CUtensorMap *map, const void *base, uint64_t rows, uint64_t cols,
                     uint64_t lda, uint32_t box_rows, uint32_t box_cols, bool swizzle128 = false);

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// Non-blocking probe of the phase with the given parity.
__device__ __forceinline__ bool mbar_test_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// The wait loops are PTX loops inside one asm block (labels are local to its
// braces): a C++ loop around
// try_wait is a potentially divergent branch to ptxas, and any such branch on
// a path into the SJLT walker makes it bracket every walker branch with
// BSSY/BSYNC (see hsk_sjlt.cu).
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "HSK_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra HSK_WAIT;\n\t}"
        ::"r"(smem_u32(bar)), "r"(parity)
        : "memory");
}

// try_wait with an explicit suspend-time hint (ns): a waiting warp sleeps
// until the phase completes or the hint elapses instead of re-polling
__device__ __forceinline__ void mbar_wait_hint(uint64_t *bar, uint32_t parity, uint32_t ns) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "HSK_WAITH:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra HSK_WAITH;\n\t}"
        ::"r"(smem_u32(bar)), "r"(parity), "r"(ns)
        : "memory");
}

// TMA bulk copy global -> shared, completion counted on an mbarrier
// (SASS: UBLKCP).  dst/src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// TMA 2-D tile load (SASS: UTMALDG) into shared memory, completion counted
// on an mbarrier.  x = inner (row) coordinate, y = outer (column) coordinate.
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int x, int y,
                                            uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

// TMA 2-D tile load multicast to the CTAs of `mask` in this cluster: the box
// lands at the same shared offset in every destination CTA and completes
// bytes on the mbarrier at the same offset in each of them.
__device__ __forceinline__ void tma_load_2d_mc(void *dst, const CUtensorMap *map, int x, int y,
                                               uint64_t *bar, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
        "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar)), "h"(mask)
        : "memory");
}

// Arrive on the mbarrier at this shared offset in CTA `rank` of the cluster.
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t *bar, uint32_t rank) {
    asm volatile(
        "{\n\t.reg .b32 ra;\n\t"
        "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
        "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar)),
        "r"(rank)
        : "memory");
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// Pull a TMA box into L2 ahead of its shared-memory load (no completion).
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap *map, int x, int y) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(x), "r"(y)
                 : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// 8-byte cp.async with zero fill when !valid (src-size 0).
__device__ __forceinline__ void cp_async8(void *dst, const void *src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(valid ? 8 : 0)
                 : "memory");
}

__device__ __forceinline__ void cp_async16(void *dst, const void *src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(valid ? 16 : 0)
                 : "memory");
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }

template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Arrive on `bar` when all prior cp.async of this thread complete; the
// barrier's expected count must include this arrival (.noinc).
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t *bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

// Cluster-wide barrier (all threads of all CTAs in the cluster), with
// release/acquire so shared-memory writes before it are visible after it.
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
                 ::: "memory");
}

// Load a double from the same shared-memory offset in CTA `rank` of the
// cluster (distributed shared memory).
__device__ __forceinline__ double ld_dsmem_f64(const double *local, uint32_t rank) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(local)), "r"(rank));
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(remote) : "memory");
    return v;
}

// Named barrier over the first `nthreads` threads (id 1; id 0 = __syncthreads).
__device__ __forceinline__ void bar_named(int nthreads) {
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

__device__ __forceinline__ int ld_acquire_gpu(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_gpu(int *p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

}  // namespace hsk
