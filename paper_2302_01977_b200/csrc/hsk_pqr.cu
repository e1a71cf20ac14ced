// hsk_pqr.cu -- column-pivoted Householder QR truncated at the numerical rank,
// the factorisation behind the interpolative decompositions of the HSS sweep.
//
// Replaces scipy.linalg.qr(S, mode="r", pivoting=True) (LAPACK dgeqp3) plus
// the rank count of interpolative_decomposition
// (/root/reference/pkg/src/hsskit/dense_kernels.py:54-82): the rank is the
// number of leading |R_jj| >= max(eps_abs, eps_rel * |R_00|), so the
// factorisation stops at the first step below that threshold (every later
// step is discarded by the reference).  Pivoting follows LAPACK's unblocked
// dgeqp2 / dlaqp2 exactly: at step j the pivot is the FIRST position >= j of
// maximal partial column norm (idamax), positions j and pivot are swapped,
// the reflector is dlarfg's (beta = -sign(alpha) * |x|, tau = (beta -
// alpha) / beta), and the partial norms are downdated with dlaqp2's formula,
// recomputed when the downdate has lost half the digits (tol3z = sqrt(eps)).
//
// One cooperative launch per factorisation: G CTAs own the physical columns
// cyclically (k mod G); every CTA computes the pivot and the reflector of
// the pivot column redundantly (identical inputs and reduction order, so
// identical results -- no broadcast needed), applies it to its own remaining
// columns (one warp per column) and downdates their norms; one grid barrier
// per step publishes the updated columns and norms.  Columns are never moved:
// the position -> column map (jpvt) is kept per CTA in shared memory and the
// R rows are gathered in pivot order at the end.
#include <math.h>

#include <algorithm>

#include "hsk_common.cuh"

namespace hsk {
namespace pqr {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

struct Ctl {
    unsigned count, gen;
    int rank, pad;
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// sense-counting grid barrier (the launch is cooperative: all CTAs resident)
__device__ __forceinline__ void grid_barrier(Ctl *c, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = ld_acquire_u32(&c->gen);
        __threadfence();
        if (atomicAdd(&c->count, 1u) == nblocks - 1) {
            c->count = 0;
            __threadfence();
            atomicAdd(&c->gen, 1u);
        } else {
            while (ld_acquire_u32(&c->gen) == g) __nanosleep(20);
        }
        __threadfence();
    }
    __syncthreads();
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// deterministic CTA sum (fixed shuffle tree, warps added in order)
__device__ double block_sum(double v, double *red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double s = red[0];
#pragma unroll
    for (int w = 1; w < kWarps; ++w) s += red[w];
    __syncthreads();
    return s;
}

// LAPACK dlapy2: sqrt(x^2 + y^2) without destructive underflow / overflow
__device__ __forceinline__ double dlapy2(double x, double y) {
    const double xa = fabs(x), ya = fabs(y);
    const double w = fmax(xa, ya), z = fmin(xa, ya);
    if (z == 0.0 || w == 0.0) return w;
    const double q = z / w;
    return w * sqrt(1.0 + q * q);
}

__global__ void __launch_bounds__(kThreads) pqr_kernel(double *__restrict__ M, int64_t m, int64_t n,
                                                       int64_t ldm, double eps_rel, double eps_abs,
                                                       int64_t *__restrict__ perm, double *__restrict__ R,
                                                       int64_t ldr, Ctl *ctl, double *__restrict__ vn1,
                                                       double *__restrict__ vn2, double *__restrict__ rdiag,
                                                       int v_in_smem) {
    extern __shared__ __align__(16) unsigned char smem[];
    double *red = reinterpret_cast<double *>(smem);                 // kWarps doubles (+pad)
    double *bestv = red + 16;                                       // kWarps
    int *bestp = reinterpret_cast<int *>(bestv + 16);               // kWarps
    int *jpvt = bestp + 16;                                         // n
    unsigned char *done = reinterpret_cast<unsigned char *>(jpvt + n);  // n
    double *vs = reinterpret_cast<double *>(smem + ((64 * 8 + 4 * n + n + 15) / 16) * 16);  // m
    const unsigned G = gridDim.x, b = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const double tol3z = sqrt(1.1102230246251565e-16);  // sqrt(dlamch('Epsilon')) = sqrt(2^-53)

    for (int64_t i = tid; i < n; i += kThreads) {
        jpvt[i] = (int)i;
        done[i] = 0;
    }
    // initial column norms of the owned columns (one warp per column)
    for (int64_t k = b + (int64_t)warp * G; k < n; k += (int64_t)G * kWarps) {
        const double *col = M + k * ldm;
        double s = 0.0;
        for (int64_t i = lane; i < m; i += 32) s = fma(col[i], col[i], s);
        s = sqrt(warp_sum(s));
        if (lane == 0) {
            vn1[k] = s;
            vn2[k] = s;
        }
    }
    grid_barrier(ctl, G);

    const int64_t kmax = m < n ? m : n;
    int64_t rank = kmax;
    double thresh = 0.0;
    for (int64_t j = 0; j < kmax; ++j) {
        // ---- pivot: first position >= j of maximal vn1 (LAPACK idamax)
        double bv = -1.0;
        int bp = 0x7fffffff;
        for (int64_t q = j + tid; q < n; q += kThreads) {
            const double v = vn1[jpvt[q]];
            if (v > bv) {  // positions visited in increasing order: keeps the first max
                bv = v;
                bp = (int)q;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int op = __shfl_xor_sync(0xffffffffu, bp, o);
            if (ov > bv || (ov == bv && op < bp)) {
                bv = ov;
                bp = op;
            }
        }
        if (lane == 0) {
            bestv[warp] = bv;
            bestp[warp] = bp;
        }
        __syncthreads();
        if (tid == 0) {
            double v = bestv[0];
            int pp = bestp[0];
            for (int w = 1; w < kWarps; ++w)
                if (bestv[w] > v || (bestv[w] == v && bestp[w] < pp)) {
                    v = bestv[w];
                    pp = bestp[w];
                }
            const int t = jpvt[j];
            jpvt[j] = jpvt[pp];
            jpvt[pp] = t;
            done[jpvt[j]] = 1;
            red[15] = v;
        }
        __syncthreads();
        const int64_t p = jpvt[j];
        if (j == 0 && red[15] == 0.0) {  // all-zero matrix: rank 0 (reference: `not np.any(S)`)
            rank = 0;
            break;
        }
        // ---- reflector of x = M[j:m, p] (dlarfg)
        double *xp = M + p * ldm;
        const double alpha = xp[j];
        double s = 0.0;
        for (int64_t i = j + 1 + tid; i < m; i += kThreads) s = fma(xp[i], xp[i], s);
        const double xnorm = sqrt(block_sum(s, red));
        double beta = alpha, tau = 0.0, scal = 0.0;
        if (m - j > 1 && xnorm != 0.0) {
            beta = -copysign(dlapy2(alpha, xnorm), alpha);
            tau = (beta - alpha) / beta;
            scal = 1.0 / (alpha - beta);
        }
        if (j == 0) thresh = fmax(eps_abs, eps_rel * fabs(beta));
        if (!(fabs(beta) >= thresh)) {  // the first diagonal below the threshold ends the rank
            rank = j;
            break;
        }
        const int64_t len = m - j;  // v[0] = 1, v[i] = x[j+i] * scal
        const double *v = v_in_smem ? vs : nullptr;
        if (v_in_smem) {
            for (int64_t i = tid; i < len; i += kThreads) vs[i] = i == 0 ? 1.0 : xp[j + i] * scal;
            __syncthreads();
        }
        // ---- apply H = I - tau v v^T to the owned remaining columns, downdate norms
        {
            for (int64_t k = b + (int64_t)warp * G; k < n; k += (int64_t)G * kWarps) {
                if (done[k]) continue;
                double *col = M + k * ldm + j;
                double dot = 0.0;
                for (int64_t i = lane; i < len; i += 32) {
                    const double vi = v ? v[i] : (i == 0 ? 1.0 : xp[j + i] * scal);
                    dot = fma(vi, col[i], dot);
                }
                dot = warp_sum(dot);
                const double t = -tau * dot;
                if (t != 0.0) {
                    for (int64_t i = lane; i < len; i += 32) {
                        const double vi = v ? v[i] : (i == 0 ? 1.0 : xp[j + i] * scal);
                        col[i] = fma(vi, t, col[i]);
                    }
                }
                __syncwarp();
                // dlaqp2 norm downdate with col[0] = R(j, k)
                double a1 = vn1[k];
                if (a1 != 0.0) {
                    double temp = fabs(col[0]) / a1;
                    temp = 1.0 - temp * temp;
                    temp = temp > 0.0 ? temp : 0.0;
                    const double r12 = a1 / vn2[k];
                    const double temp2 = temp * r12 * r12;
                    if (temp2 <= tol3z) {
                        double nrm = 0.0;
                        if (j < m - 1) {
                            double s2 = 0.0;
                            for (int64_t i = 1 + lane; i < len; i += 32) s2 = fma(col[i], col[i], s2);
                            nrm = sqrt(warp_sum(s2));
                        }
                        if (lane == 0) {
                            vn1[k] = nrm;
                            vn2[k] = nrm;
                        }
                    } else if (lane == 0) {
                        vn1[k] = a1 * sqrt(temp);
                    }
                }
                __syncwarp();
            }
        }
        // R(j, j) goes to its own array: column p's row j is still being read
        // as alpha by CTAs that have not reached this point
        if (b == 0 && tid == 0) rdiag[j] = beta;
        grid_barrier(ctl, G);
    }
    if (b == 0 && tid == 0) ctl->rank = (int)rank;
    // R rows 0..rank-1 in pivot order, and the permutation
    for (int64_t pos = b; pos < n; pos += G) {
        const int64_t k = jpvt[pos];
        if (tid == 0) perm[pos] = k;
        for (int64_t i = tid; i < rank; i += kThreads)
            R[pos * ldr + i] = pos > i ? M[k * ldm + i] : pos == i ? rdiag[i] : 0.0;
    }
}

}  // namespace pqr
}  // namespace hsk

using namespace hsk;

extern "C" int64_t hsk_pqr_work_bytes(int64_t m, int64_t n) {
    if (m < 0 || n < 0) return HSK_EINVAL;
    return (int64_t)sizeof(pqr::Ctl) + 16 + 8 * (2 * std::max<int64_t>(n, 1) + std::max<int64_t>(std::min(m, n), 1));
}

extern "C" int hsk_pqr(double *M, int64_t m, int64_t n, int64_t ldm, double eps_rel, double eps_abs,
                       int64_t *perm, double *R, int64_t ldr, int32_t *rank, void *work,
                       int64_t work_bytes, void *stream) {
    HSK_REQUIRE(m >= 0 && n >= 0 && ldm >= std::max<int64_t>(m, 1), HSK_EINVAL,
                "pqr: bad shape m=%lld n=%lld ldm=%lld", (long long)m, (long long)n, (long long)ldm);
    HSK_REQUIRE(eps_rel >= 0 && eps_abs >= 0, HSK_EINVAL, "tolerances must be nonnegative");
    HSK_REQUIRE(ldr >= std::max<int64_t>(std::min(m, n), 1), HSK_EINVAL, "pqr: ldr too small");
    HSK_REQUIRE(rank != nullptr && work != nullptr && work_bytes >= hsk_pqr_work_bytes(m, n),
                HSK_EINVAL, "pqr: workspace of %lld bytes, need %lld", (long long)work_bytes,
                (long long)hsk_pqr_work_bytes(m, n));
    HSK_REQUIRE(n <= (1 << 20), HSK_EINVAL, "pqr: n=%lld too large", (long long)n);
    cudaStream_t st = as_stream(stream);
    pqr::Ctl *ctl = static_cast<pqr::Ctl *>(work);
    cudaError_t e = cudaMemsetAsync(ctl, 0, sizeof(pqr::Ctl), st);
    if (e != cudaSuccess) return cuda_status(e, "pqr: memset");
    if (m == 0 || n == 0) {
        e = cudaMemcpyAsync(rank, &ctl->rank, sizeof(int), cudaMemcpyDeviceToDevice, st);
        return e == cudaSuccess ? HSK_OK : cuda_status(e, "pqr: rank");
    }
    HSK_REQUIRE(M && perm && R, HSK_EINVAL, "pqr: null pointer");
    double *vn1 = reinterpret_cast<double *>(static_cast<unsigned char *>(work) + sizeof(pqr::Ctl) + 16);
    vn1 = reinterpret_cast<double *>((reinterpret_cast<uintptr_t>(vn1) + 15) & ~uintptr_t(15));
    double *vn2 = vn1 + n;
    double *rdiag = vn2 + n;
    const size_t base = ((64 * 8 + 4 * n + n + 15) / 16) * 16;
    int v_in_smem = base + (size_t)m * 8 <= 200 * 1024;
    const size_t smem = base + (v_in_smem ? (size_t)m * 8 : 0);
    HSK_REQUIRE(smem <= 220 * 1024, HSK_EINVAL, "pqr: n=%lld too large for the pivot map", (long long)n);
    auto kern = pqr::pqr_kernel;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_status(e, "pqr: smem attribute");
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, pqr::kThreads, smem);
    if (e != cudaSuccess) return cuda_status(e, "pqr: occupancy");
    // one CTA per SM: two factorisations (a node's row and column IDs) can
    // then run concurrently on two streams, both grids co-resident
    per_sm = std::max(1, std::min(per_sm, 1));
    // a CTA per ~kWarps columns, at most what is co-resident
    const int64_t want = (n + pqr::kWarps - 1) / pqr::kWarps;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sm_count() * per_sm));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid, 1, 1);
    cfg.blockDim = dim3(pqr::kThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, M, m, n, ldm, eps_rel, eps_abs, perm, R, ldr, ctl, vn1, vn2,
                           rdiag, v_in_smem);
    if (e != cudaSuccess) return cuda_status(e, "pqr_kernel launch");
    HSK_CHECK_LAUNCH("pqr_kernel");
    e = cudaMemcpyAsync(rank, &ctl->rank, sizeof(int), cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return cuda_status(e, "pqr: rank");
    return HSK_OK;
}
