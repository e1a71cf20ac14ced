// hsk_misc.cu -- C-ABI plumbing (errors, device info), synthetic matrix
// generators for the BASELINE.json configs, and the L2 flush used between
// timed launches.
#include <math.h>
#include <stdarg.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <atomic>
#include <mutex>
#include <utility>

#include <cudaTypedefs.h>

#include "hsk_common.cuh"

namespace hsk {

static thread_local char g_err[512] = "";

int set_error(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

int cuda_status(cudaError_t e, const char *what) {
    return set_error(e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver ? HSK_ENODEV
                                                                                 : HSK_ECUDA,
                     "%s: %s", what, cudaGetErrorString(e));
}

int make_tmap_f64_2d(CUtensorMap *map, const void *base, uint64_t rows, uint64_t cols,
                     uint64_t lda, uint32_t box_rows, uint32_t box_cols, bool swizzle128) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
        if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn)
            return set_error(HSK_ECUDA, "cuTensorMapEncodeTiled unavailable");
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    cuuint64_t dims[2] = {rows, cols};
    cuuint64_t strides[1] = {lda * 8};
    cuuint32_t box[2] = {box_rows, box_cols};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void *>(base), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_error(HSK_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return HSK_OK;
}

int sm_count() {
    static int cached = 0;
    if (!cached) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
        if (cached <= 0) cached = 148;
    }
    return cached;
}

namespace {
Tuning g_tuning;
std::atomic<int> g_tuning_ready{0};
std::atomic<int> g_tuning_gen{0};
std::mutex g_tuning_mu;

int env_int(const char *name) {
    const char *v = getenv(name);
    return (v && *v) ? atoi(v) : -1;
}

void tuning_load() {
    Tuning t;
    t.sjlt_w32 = env_int("HSK_SJLT_W32");
    t.sjlt_tk = env_int("HSK_SJLT_TK");
    t.sjlt_tk_t = env_int("HSK_SJLT_TK_T");
    t.sjlt_rpt = env_int("HSK_SJLT_RPT");
    t.sjlt_rpt_t = env_int("HSK_SJLT_RPT_T");
    t.sjlt_prod = env_int("HSK_SJLT_PROD");
    t.sjlt_streamk = env_int("HSK_SJLT_STREAMK");
    t.sjlt_mc = env_int("HSK_SJLT_MC");
    t.sjlt_stages = env_int("HSK_SJLT_STAGES");
    t.sjlt_wait_ns = env_int("HSK_SJLT_WAIT_NS");
    t.sjlt_dbg = env_int("HSK_SJLT_DBG");
    t.sjlt_pf = env_int("HSK_SJLT_PF");
    t.sjlt_fused = env_int("HSK_SJLT_FUSED");
    t.sjlt_xp = env_int("HSK_SJLT_XP");
    t.sjlt_xp_gb = env_int("HSK_SJLT_XP_GB");
    t.gauss_splits = env_int("HSK_GAUSS_SPLITS");
    const char *g = getenv("HSK_GAUSS_CFG");
    snprintf(t.gauss_cfg, sizeof(t.gauss_cfg), "%s", g ? g : "");
    g_tuning = t;
}
}  // namespace

const Tuning &tuning() {
    if (!g_tuning_ready.load(std::memory_order_acquire)) {
        std::lock_guard<std::mutex> lk(g_tuning_mu);
        if (!g_tuning_ready.load(std::memory_order_relaxed)) {
            tuning_load();
            g_tuning_ready.store(1, std::memory_order_release);
        }
    }
    return g_tuning;
}

namespace {
struct Workspace {
    void *data = nullptr;
    size_t data_bytes = 0;
    int *flags = nullptr;
    int nflags = 0;
};
std::mutex g_ws_mu;
std::map<std::pair<int, cudaStream_t>, Workspace> g_ws;
}  // namespace

int stream_workspace(cudaStream_t st, size_t data_bytes, int nflags, void **data, int **flags) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_status(e, "workspace: device");
    std::lock_guard<std::mutex> lk(g_ws_mu);
    Workspace &w = g_ws[std::make_pair(dev, st)];
    if (w.data_bytes < data_bytes) {
        if (w.data) {
            cudaStreamSynchronize(st);
            cudaFree(w.data);
        }
        w.data = nullptr;
        w.data_bytes = 0;
        e = cudaMalloc(&w.data, data_bytes);
        if (e != cudaSuccess) return cuda_status(e, "workspace: allocate");
        w.data_bytes = data_bytes;
    }
    if (w.nflags < nflags) {
        if (w.flags) {
            cudaStreamSynchronize(st);
            cudaFree(w.flags);
        }
        w.flags = nullptr;
        w.nflags = 0;
        e = cudaMalloc(reinterpret_cast<void **>(&w.flags), (size_t)nflags * sizeof(int));
        if (e != cudaSuccess) return cuda_status(e, "workspace: allocate flags");
        e = cudaMemsetAsync(w.flags, 0, (size_t)nflags * sizeof(int), st);
        if (e != cudaSuccess) return cuda_status(e, "workspace: clear flags");
        w.nflags = nflags;
    }
    *data = w.data;
    *flags = w.flags;
    return HSK_OK;
}

// A_ij = exp(-|x_i - x_j|^2 / (2 h^2)) + diag*(i==j); thread per element,
// consecutive threads along the column (contiguous) dimension.
__global__ void gen_gauss_kernel(const double *__restrict__ pts, int64_t n, int dim,
                                 double inv2h2, double diag, int64_t row0, int64_t nrows,
                                 int64_t col0, int64_t ncols, double *__restrict__ A,
                                 int64_t lda) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t c = blockIdx.y;
    if (r >= nrows) return;
    for (int64_t cc = c; cc < ncols; cc += gridDim.y) {
        const int64_t i = row0 + r, j = col0 + cc;
        const double *xi = pts + i * dim, *xj = pts + j * dim;
        double s = 0.0;
        for (int q = 0; q < dim; ++q) {
            const double t = xi[q] - xj[q];
            s += t * t;
        }
        double v = exp(-s * inv2h2);
        if (i == j) v += diag;
        A[cc * lda + r] = v;
    }
}

// A_ij = 1/(1+|i-j|) + 0.1 sin(i+2j)/n
__global__ void gen_toeplitz_sin_kernel(int64_t n, int64_t row0, int64_t nrows, int64_t col0,
                                        int64_t ncols, double *__restrict__ A, int64_t lda) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= nrows) return;
    for (int64_t cc = blockIdx.y; cc < ncols; cc += gridDim.y) {
        const int64_t i = row0 + r, j = col0 + cc;
        const int64_t dd = i > j ? i - j : j - i;
        A[cc * lda + r] = 1.0 / (1.0 + (double)dd) + 0.1 * sin((double)(i + 2 * j)) / (double)n;
    }
}

__global__ void l2_flush_kernel(double4 *p, int64_t n4, double v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = make_double4(v, v, v, v);
}

}  // namespace hsk

using namespace hsk;

extern "C" int hsk_abi_version(void) { return HSK_ABI_VERSION; }

extern "C" int hsk_tuning_reload(void) {
    std::lock_guard<std::mutex> lk(g_tuning_mu);
    tuning_load();
    g_tuning_ready.store(1, std::memory_order_release);
    g_tuning_gen.fetch_add(1, std::memory_order_relaxed);
    return HSK_OK;
}

extern "C" int hsk_tuning_generation(void) { return g_tuning_gen.load(std::memory_order_relaxed); }

extern "C" int hsk_last_error(char *buf, size_t len) {
    const int n = (int)strlen(g_err);
    if (buf && len) {
        strncpy(buf, g_err, len - 1);
        buf[len - 1] = '\0';
    }
    return n;
}

extern "C" int hsk_device_info(int *sms, int *major, int *minor, int64_t *l2) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_status(e, "cudaGetDevice");
    int v = 0;
    if (sms) {
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        *sms = v;
    }
    if (major) {
        cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMajor, dev);
        *major = v;
    }
    if (minor) {
        cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMinor, dev);
        *minor = v;
    }
    if (l2) {
        cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, dev);
        *l2 = v;
    }
    return HSK_OK;
}

static int gen_grid(int64_t nrows, int64_t ncols, dim3 &grid) {
    const int64_t bx = (nrows + 255) / 256;
    HSK_REQUIRE(bx < (1ll << 31), HSK_EINVAL, "generator: too many rows");
    grid = dim3((unsigned)bx, (unsigned)std::min<int64_t>(std::max<int64_t>(ncols, 1), 65535), 1);
    return HSK_OK;
}

extern "C" int hsk_gen_gauss_kernel(const double *pts, int64_t n, int32_t dim, double h,
                                    double diag, int64_t row0, int64_t nrows, int64_t col0,
                                    int64_t ncols, double *A, int64_t lda, void *stream) {
    HSK_REQUIRE(n >= 0 && dim >= 1 && h > 0, HSK_EINVAL, "gen_gauss_kernel: bad n/dim/h");
    HSK_REQUIRE(row0 >= 0 && nrows >= 0 && row0 + nrows <= n && col0 >= 0 && ncols >= 0 &&
                    col0 + ncols <= n && lda >= std::max<int64_t>(nrows, 1),
                HSK_EINVAL, "gen_gauss_kernel: bad block");
    if (nrows == 0 || ncols == 0) return HSK_OK;
    dim3 grid;
    int rc = gen_grid(nrows, ncols, grid);
    if (rc) return rc;
    gen_gauss_kernel<<<grid, 256, 0, as_stream(stream)>>>(pts, n, dim, 1.0 / (2.0 * h * h), diag,
                                                          row0, nrows, col0, ncols, A, lda);
    HSK_CHECK_LAUNCH("gen_gauss_kernel");
    return HSK_OK;
}

extern "C" int hsk_gen_toeplitz_sin(int64_t n, int64_t row0, int64_t nrows, int64_t col0,
                                    int64_t ncols, double *A, int64_t lda, void *stream) {
    HSK_REQUIRE(n >= 0 && row0 >= 0 && nrows >= 0 && row0 + nrows <= n && col0 >= 0 &&
                    ncols >= 0 && col0 + ncols <= n && lda >= std::max<int64_t>(nrows, 1),
                HSK_EINVAL, "gen_toeplitz_sin: bad block");
    if (nrows == 0 || ncols == 0) return HSK_OK;
    dim3 grid;
    int rc = gen_grid(nrows, ncols, grid);
    if (rc) return rc;
    gen_toeplitz_sin_kernel<<<grid, 256, 0, as_stream(stream)>>>(n, row0, nrows, col0, ncols, A,
                                                                 lda);
    HSK_CHECK_LAUNCH("gen_toeplitz_sin_kernel");
    return HSK_OK;
}

// B = A^T through 64 x 64 shared tiles s[r][c] = A(r0 + r, c0 + c) with a
// 65-double pitch.  Both directions move whole 128-byte lines: eight lanes
// cover one 16-row run of a column as 16-byte pairs, a warp four such runs
// (partial sectors would make every HBM write a read-modify-write); eight
// pairs per thread in flight.  The shared stores and loads of a half-warp
// (two columns / rows x eight pairs) hit 16 distinct bank pairs.  Partial
// tiles and 8-byte-aligned operands take the scalar path.
__global__ void __launch_bounds__(256) transpose_kernel(const double *__restrict__ A, int64_t rows,
                                                        int64_t cols, int64_t lda,
                                                        double *__restrict__ B, int64_t ldb, int vec) {
    __shared__ double s[64 * 65];
    const int l8 = threadIdx.x & 7, gi = threadIdx.x >> 3;  // 16-byte chunk of a run, run group
    const int64_t r0 = (int64_t)blockIdx.x * 64;
    for (int64_t c0 = (int64_t)blockIdx.y * 64; c0 < cols; c0 += (int64_t)gridDim.y * 64) {
        const bool full = vec && r0 + 64 <= rows && c0 + 64 <= cols;
        if (full) {
            double2 v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {  // run p: column p % 64, rows 16 (p / 64) + 2 l8
                const int pr = gi + 32 * k, c = pr & 63, rb = pr >> 6;
                v[k] = __ldcs(reinterpret_cast<const double2 *>(A + (c0 + c) * lda + r0 + 16 * rb + 2 * l8));
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int pr = gi + 32 * k, c = pr & 63, rb = pr >> 6;
                s[(16 * rb + 2 * l8) * 65 + c] = v[k].x;
                s[(16 * rb + 2 * l8 + 1) * 65 + c] = v[k].y;
            }
        } else {
            for (int e = threadIdx.x; e < 64 * 64; e += 256) {
                const int c = e >> 6, r = e & 63;
                const int64_t gr = r0 + r, gc = c0 + c;
                s[r * 65 + c] = (gr < rows && gc < cols) ? A[gc * lda + gr] : 0.0;
            }
        }
        __syncthreads();
        if (full) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {  // run p: B column r0 + p % 64, entries 16 (p / 64) + 2 l8
                const int pr = gi + 32 * k, r = pr & 63, cb = pr >> 6;
                const int cc = 16 * cb + 2 * l8;
                __stcs(reinterpret_cast<double2 *>(B + (r0 + r) * ldb + c0 + cc),
                       make_double2(s[r * 65 + cc], s[r * 65 + cc + 1]));
            }
        } else {
            for (int e = threadIdx.x; e < 64 * 64; e += 256) {
                const int r = e >> 6, c = e & 63;
                const int64_t gr = r0 + r, gc = c0 + c;
                if (gr < rows && gc < cols) B[gr * ldb + gc] = s[r * 65 + c];
            }
        }
        __syncthreads();
    }
}

extern "C" int hsk_transpose(const double *A, int64_t rows, int64_t cols, int64_t lda, double *B,
                             int64_t ldb, void *stream) {
    HSK_REQUIRE(rows >= 0 && cols >= 0 && lda >= std::max<int64_t>(rows, 1) &&
                    ldb >= std::max<int64_t>(cols, 1),
                HSK_EINVAL, "transpose: bad shape rows=%lld cols=%lld lda=%lld ldb=%lld",
                (long long)rows, (long long)cols, (long long)lda, (long long)ldb);
    if (rows == 0 || cols == 0) return HSK_OK;
    HSK_REQUIRE(A && B, HSK_EINVAL, "transpose: null pointer");
    const int64_t gx = (rows + 63) / 64;
    HSK_REQUIRE(gx < (1ll << 31), HSK_EINVAL, "transpose: too many rows");
    const int vec = (lda % 2 == 0) && (ldb % 2 == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0) &&
                    ((reinterpret_cast<uintptr_t>(B) & 15) == 0);
    // ~8 column tiles per CTA: short CTAs balance the tail, enough of them
    // amortise the start-up
    const unsigned gy = (unsigned)std::min<int64_t>(std::max<int64_t>(1, (cols + 511) / 512), 65535);
    transpose_kernel<<<dim3((unsigned)gx, gy, 1), 256, 0, as_stream(stream)>>>(A, rows, cols, lda, B,
                                                                                 ldb, vec);
    HSK_CHECK_LAUNCH("transpose_kernel");
    return HSK_OK;
}

// Symmetry test of an n x n column-major A: CTA (bi, bj), bi <= bj, loads tile
// (bi, bj) into shared memory with the transpose kernel's whole-line pattern,
// then reads tile (bj, bi) the same way and compares each element bitwise with
// its mirror; any mismatch sets *flag.  CTAs start by polling the flag, so a
// nonsymmetric A costs about one wave.
__global__ void __launch_bounds__(256) symmetric_kernel(const double *__restrict__ A, int64_t n,
                                                        int64_t lda, int32_t *flag, int vec) {
    __shared__ unsigned long long s[64 * 65];
    __shared__ int bad;
    const int64_t bi = blockIdx.x, bj = blockIdx.y;
    if (bj < bi) return;
    if (threadIdx.x == 0) bad = *reinterpret_cast<volatile int32_t *>(flag);
    __syncthreads();
    if (bad) return;
    const unsigned long long *a = reinterpret_cast<const unsigned long long *>(A);
    const int l8 = threadIdx.x & 7, gi = threadIdx.x >> 3;
    const int64_t r0 = bi * 64, c0 = bj * 64;
    const bool full = vec && r0 + 64 <= n && c0 + 64 <= n;
    if (full) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {  // tile (bi, bj): s[r][c] = A(r0 + r, c0 + c)
            const int pr = gi + 32 * k, c = pr & 63, rb = pr >> 6;
            const ulonglong2 v =
                *reinterpret_cast<const ulonglong2 *>(a + (c0 + c) * lda + r0 + 16 * rb + 2 * l8);
            s[(16 * rb + 2 * l8) * 65 + c] = v.x;
            s[(16 * rb + 2 * l8 + 1) * 65 + c] = v.y;
        }
    } else {
        for (int e = threadIdx.x; e < 64 * 64; e += 256) {
            const int c = e >> 6, r = e & 63;
            const int64_t gr = r0 + r, gc = c0 + c;
            s[r * 65 + c] = (gr < n && gc < n) ? a[gc * lda + gr] : 0ull;
        }
    }
    __syncthreads();
    int mism = 0;
    if (full) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {  // tile (bj, bi): A(c0 + r', r0 + c') == s[c'][r']
            const int pr = gi + 32 * k, cc = pr & 63, rb = pr >> 6;
            const ulonglong2 v =
                *reinterpret_cast<const ulonglong2 *>(a + (r0 + cc) * lda + c0 + 16 * rb + 2 * l8);
            mism |= v.x != s[cc * 65 + 16 * rb + 2 * l8];
            mism |= v.y != s[cc * 65 + 16 * rb + 2 * l8 + 1];
        }
    } else {
        for (int e = threadIdx.x; e < 64 * 64; e += 256) {
            const int cc = e >> 6, rr = e & 63;  // A(c0 + rr, r0 + cc) vs A(r0 + cc, c0 + rr)
            const int64_t gr = c0 + rr, gc = r0 + cc;
            if (gr < n && gc < n) mism |= a[gc * lda + gr] != s[cc * 65 + rr];
        }
    }
    if (__syncthreads_or(mism) && threadIdx.x == 0) atomicExch(flag, 1);
}

extern "C" int hsk_is_symmetric(const double *A, int64_t n, int64_t lda, int32_t *flag, void *stream) {
    HSK_REQUIRE(n >= 0 && lda >= std::max<int64_t>(n, 1) && flag, HSK_EINVAL,
                "is_symmetric: bad arguments n=%lld lda=%lld", (long long)n, (long long)lda);
    cudaError_t e = cudaMemsetAsync(flag, 0, sizeof(int32_t), as_stream(stream));
    if (e != cudaSuccess) return cuda_status(e, "is_symmetric: memset");
    if (n == 0) return HSK_OK;
    HSK_REQUIRE(A, HSK_EINVAL, "is_symmetric: null matrix");
    const int64_t nb = (n + 63) / 64;
    HSK_REQUIRE(nb < 65536, HSK_EINVAL, "is_symmetric: n too large");
    const int vec = (lda % 2 == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
    symmetric_kernel<<<dim3((unsigned)nb, (unsigned)nb, 1), 256, 0, as_stream(stream)>>>(A, n, lda, flag,
                                                                                           vec);
    HSK_CHECK_LAUNCH("symmetric_kernel");
    return HSK_OK;
}

extern "C" int hsk_l2_flush(void *scratch, int64_t bytes, void *stream) {
    HSK_REQUIRE(scratch && bytes >= 32 && (reinterpret_cast<uintptr_t>(scratch) & 31) == 0,
                HSK_EINVAL, "l2_flush: need a 32-byte aligned scratch buffer");
    static double v = 0.0;
    v += 1.0;
    l2_flush_kernel<<<sm_count() * 4, 256, 0, as_stream(stream)>>>(
        static_cast<double4 *>(scratch), bytes / 32, v);
    HSK_CHECK_LAUNCH("l2_flush_kernel");
    return HSK_OK;
}
