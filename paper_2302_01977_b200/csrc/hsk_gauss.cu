// hsk_gauss.cu -- Gaussian sketch S = A R^T / S' = A^T R^T as an FP64
// tensor-core contraction on sm_100a.
//
// Replaces GaussianBlock.apply_right (buf @ matrix.T) and
// apply_right_transposed ((matrix @ buf).T), sketching.py:134-138.
//
// tcgen05.mma has no f64 kind, so the FP64 tensor path on sm_100a is the
// warp-level mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4).  CTA tile BM x BN with
// BK = 32 k-steps staged by a STAGES-deep cp.async ring; 4 warps, each a
// (BM/2) x (BN/4) register tile of 8x8 DMMA fragments.  Shared-memory pitches
// are chosen so every fragment load is conflict-free
// (DESIGN.md §Gaussian).  R is the reference's d x n row-major `matrix`,
// i.e. R^T column-major with leading dimension n.
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include "hsk_common.cuh"

#ifndef HSK_TUNING
#define HSK_TUNING 0
#endif

namespace hsk {
namespace gauss {

// BK = 16, 2 stages, 2 x 2 warps: 38 KB of shared memory per CTA, so the
// register file (120 per thread) sets 4 resident CTAs = 16 warps per SM.  r02
// sweep on C2 (S / S' ms, cuBLAS 7.71): BK 32 2-st 8.16 / 8.20 (3 CTAs/SM);
// BK 16 2-st 7.95 / 7.89; 3-st 7.96 / 7.91; 4-st 7.98 / 8.01; BK 8 4-st
// 8.09 / 8.01; 2 x 4 warps 8.58 / 8.44; 5 CTAs (94 registers) 8.15 / 8.06.
#ifndef HSK_GAUSS_BK
#define HSK_GAUSS_BK 16
#endif
#ifndef HSK_GAUSS_STAGES
#define HSK_GAUSS_STAGES 2
#endif
#ifndef HSK_GAUSS_MINB
#define HSK_GAUSS_MINB 4  // <= 128 registers: 4 resident CTAs
#endif
#ifndef HSK_GAUSS_WGM
#define HSK_GAUSS_WGM 2
#endif
#ifndef HSK_GAUSS_WGN
#define HSK_GAUSS_WGN 2
#endif
constexpr int BK = HSK_GAUSS_BK;
constexpr int PKK = BK + 4;  // pitch of k-contiguous tiles (== 4 mod 16)

struct Args {
    const double *A;
    int64_t lda;
    const double *R;
    int64_t M, N, K;
    double *S;
    int64_t lds, col0;
    int a16, b16;  // 16-byte cp.async allowed
    int ntiles_n;
    // split-K: blockIdx.y = split; splits > 1 store partial tiles to ws
    // (split-major, column-major M x N each) for the ordered reduction
    int splits;
    double *ws;
};

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

// copy the two doubles src[0..1] (valid0/valid1) to dst, 16B if allowed
// (`safe` is any valid global address used when a half is out of range)
__device__ __forceinline__ void copy2(double *dst, const double *src, bool v0, bool v1,
                                      bool vec16, const double *safe) {
    if (vec16 && v0 && v1) {
        cp_async16(dst, src, true);
    } else {
        cp_async8(dst, v0 ? src : safe, v0);
        cp_async8(dst + 1, v1 ? src + 1 : safe, v1);
    }
}

template <int BM, int BN, int TRANS, int STAGES>
struct Smem {
    // 8-byte fragment loads are serviced per half-warp (4 k x 4 rows): a pitch
    // == 4 (mod 16) doubles puts the 4 k-rows on disjoint 8-bank groups.
    static constexpr int PA = TRANS ? PKK : BM + 4;  // trans0: [BK][BM+4]
    static constexpr int A_ELEMS = TRANS ? BM * PKK : BK * (BM + 4);
    static constexpr int B_ELEMS = BN * PKK;
    static constexpr int STAGE = A_ELEMS + B_ELEMS;
    static constexpr int BYTES = STAGES * STAGE * 8;
};

// WGM x WGN warps, each a (BM/WGM) x (BN/WGN) tile of 8x8 DMMA fragments.
template <int BM, int BN, int TRANS, int WGM, int WGN, int STAGES>
__global__ void __launch_bounds__(WGM * WGN * 32, HSK_GAUSS_MINB) gauss_kernel(const Args p) {
    using SM = Smem<BM, BN, TRANS, STAGES>;
    constexpr int NT = WGM * WGN * 32;
    constexpr int WM = BM / WGM, WN = BN / WGN;
    constexpr int MF = WM / 8, NF = WN / 8;
    extern __shared__ __align__(128) double sm[];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t nt = blockIdx.x % p.ntiles_n, mt = blockIdx.x / p.ntiles_n;
    const int64_t m0 = mt * BM, n0 = nt * BN;
    const int wm0 = (warp / WGN) * WM, wn0 = (warp % WGN) * WN;
    const int64_t ktiles_all = (p.K + BK - 1) / BK;
    const int64_t kper = (ktiles_all + p.splits - 1) / p.splits;
    const int64_t kt0 = std::min<int64_t>(ktiles_all, (int64_t)blockIdx.y * kper);
    const int64_t ktiles = std::min<int64_t>(ktiles_all, kt0 + kper) - kt0;

    // interior tiles (all rows/columns/k in range, 16-byte aligned operands)
    // take an unpredicated copy path.  Its addresses are per-thread constants
    // plus compile-time shared offsets and a runtime global pass stride, so a
    // 16-byte copy costs one 64-bit add and one LDGSTS (the generic per-copy
    // index arithmetic was ~10 integer instructions per copy: 190 per warp
    // and k-tile against 128 DMMAs, ncu r02; C2 8.30 -> 8.16 ms)
    const bool full_mn = (m0 + BM <= p.M) && (n0 + BN <= p.N) && p.a16 && p.b16;
    // A: !TRANS -- BK columns of BM rows, CA = BM/2 chunks per column;
    //     TRANS -- BM rows of BK k, CA = BK/2 chunks per row
    constexpr int CA = TRANS ? BK / 2 : BM / 2;
    constexpr int LA = NT / CA;                       // lines (columns / rows) per pass
    constexpr int PASS_A = (TRANS ? BM : BK) / LA;
    constexpr int CB = BK / 2, LB = NT / CB, PASS_B = BN / LB;
    static_assert(NT % CA == 0 && NT % CB == 0, "copy mapping");
    const int a_c = tid % CA, a_l = tid / CA, b_c = tid % CB, b_l = tid / CB;
    const uint32_t s_a0 = smem_u32(sm) + 8u * (uint32_t)(TRANS ? a_l * PKK + 2 * a_c : a_l * SM::PA + 2 * a_c);
    const uint32_t s_b0 = smem_u32(sm) + 8u * (uint32_t)(SM::A_ELEMS + b_l * PKK + 2 * b_c);
    const char *g_a0 = reinterpret_cast<const char *>(
        TRANS ? p.A + (m0 + a_l) * p.lda + 2 * a_c : p.A + (int64_t)a_l * p.lda + m0 + 2 * a_c);
    const char *g_b0 = reinterpret_cast<const char *>(p.R + (n0 + b_l) * p.K + 2 * b_c);
    const int64_t a_pass = (int64_t)LA * p.lda * 8, b_pass = (int64_t)LB * p.K * 8;
    auto load_stage = [&](int64_t kt, int s) {
        double *sA = sm + s * SM::STAGE;
        double *sB = sA + SM::A_ELEMS;
        const int64_t k0 = (kt0 + kt) * BK;
        if (full_mn && k0 + BK <= p.K) {
            const uint32_t so = (uint32_t)(s * SM::STAGE * 8);
            const char *ga = g_a0 + (TRANS ? k0 * 8 : k0 * p.lda * 8);
#pragma unroll
            for (int i = 0; i < PASS_A; ++i, ga += a_pass)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                                 s_a0 + so + 8u * (uint32_t)(i * LA * (TRANS ? PKK : SM::PA))),
                             "l"(ga)
                             : "memory");
            const char *gb = g_b0 + k0 * 8;
#pragma unroll
            for (int i = 0; i < PASS_B; ++i, gb += b_pass)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                                 s_b0 + so + 8u * (uint32_t)(i * LB * PKK)),
                             "l"(gb)
                             : "memory");
            return;
        }
        if (!TRANS) {
            // A(m,k) = A[k*lda + m]: BK columns of BM contiguous rows
            for (int q = tid; q < BK * (BM / 2); q += NT) {
                const int kk = q / (BM / 2), mm = (q % (BM / 2)) * 2;
                const int64_t gm = m0 + mm, gk = k0 + kk;
                const bool vk = gk < p.K;
                const double *src = p.A + gk * p.lda + gm;
                copy2(sA + kk * SM::PA + mm, src, vk && gm < p.M, vk && gm + 1 < p.M, p.a16, p.R);
            }
        } else {
            // A^T(m,k) = A[m*lda + k]: BM rows of BK contiguous k
            for (int q = tid; q < BM * (BK / 2); q += NT) {
                const int mm = q / (BK / 2), kk = (q % (BK / 2)) * 2;
                const int64_t gm = m0 + mm, gk = k0 + kk;
                const bool vm = gm < p.M;
                const double *src = p.A + gm * p.lda + gk;
                copy2(sA + mm * PKK + kk, src, vm && gk < p.K, vm && gk + 1 < p.K, p.a16, p.R);
            }
        }
        // B(k,j) = R[j*K + k]
        for (int q = tid; q < BN * (BK / 2); q += NT) {
            const int jj = q / (BK / 2), kk = (q % (BK / 2)) * 2;
            const int64_t gj = n0 + jj, gk = k0 + kk;
            const bool vj = gj < p.N;
            const double *src = p.R + gj * p.K + gk;
            copy2(sB + jj * PKK + kk, src, vj && gk < p.K, vj && gk + 1 < p.K, p.b16, p.R);
        }
    };

    double acc[MF][NF][2];
#pragma unroll
    for (int i = 0; i < MF; ++i)
#pragma unroll
        for (int j = 0; j < NF; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < ktiles) load_stage(s, s);
        cp_async_commit();
    }
    int rs = 0, ws = STAGES - 1;  // read / write stage (incremental, no division)
    for (int64_t kt = 0; kt < ktiles; ++kt) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        {
            const int64_t nk = kt + STAGES - 1;
            if (nk < ktiles) load_stage(nk, ws);
            cp_async_commit();
            if (++ws == STAGES) ws = 0;
        }
        const double *sA = sm + rs * SM::STAGE;
        if (++rs == STAGES) rs = 0;
        const double *sB = sA + SM::A_ELEMS;
        const int fr = lane >> 2, fc = lane & 3;
        // fragments double-buffered in registers: step k4 + 4's loads are in
        // flight while step k4's DMMAs issue
        double a[2][MF], b[2][NF];
        auto load_frags = [&](int k4, int buf) {
#pragma unroll
            for (int i = 0; i < MF; ++i) {
                const int m = wm0 + i * 8 + fr;
                a[buf][i] = TRANS ? sA[m * PKK + k4 + fc] : sA[(k4 + fc) * SM::PA + m];
            }
#pragma unroll
            for (int j = 0; j < NF; ++j) b[buf][j] = sB[(wn0 + j * 8 + fr) * PKK + k4 + fc];
        };
        load_frags(0, 0);
#pragma unroll
        for (int k4 = 0; k4 < BK; k4 += 4) {
            const int cur = (k4 / 4) & 1;
            if (k4 + 4 < BK) load_frags(k4 + 4, cur ^ 1);
#pragma unroll
            for (int i = 0; i < MF; ++i)
#pragma unroll
                for (int j = 0; j < NF; ++j) dmma(acc[i][j], a[cur][i], b[cur][j]);
        }
    }
    cp_async_wait<0>();

    const int fr = lane >> 2, fc = lane & 3;
    double *out = p.splits > 1 ? p.ws + (int64_t)blockIdx.y * p.M * p.N : p.S + p.col0 * p.lds;
    const int64_t ldo = p.splits > 1 ? p.M : p.lds;
#pragma unroll
    for (int i = 0; i < MF; ++i) {
        const int64_t m = m0 + wm0 + i * 8 + fr;
        if (m >= p.M) continue;
#pragma unroll
        for (int j = 0; j < NF; ++j) {
            const int64_t c = n0 + wn0 + j * 8 + 2 * fc;
            if (c < p.N) out[c * ldo + m] = acc[i][j][0];
            if (c + 1 < p.N) out[(c + 1) * ldo + m] = acc[i][j][1];
        }
    }
}

// S[:, col0 + c] = sum over splits s (in order) of ws[s] -- deterministic
__global__ void splitk_reduce_kernel(const double *__restrict__ ws, int splits, int64_t M, int64_t N,
                                     double *__restrict__ S, int64_t lds, int64_t col0) {
    const int64_t total = M * N, stride = M * N;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = q / M, m = q - c * M;
        double acc = ws[q];
        for (int s = 1; s < splits; ++s) acc += ws[s * stride + q];
        S[(col0 + c) * lds + m] = acc;
    }
}

template <int BM, int BN, int TRANS, int WGM, int WGN, int STAGES>
static int launch(Args a, cudaStream_t st) {
    using SM = Smem<BM, BN, TRANS, STAGES>;
    auto kern = gauss_kernel<BM, BN, TRANS, WGM, WGN, STAGES>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SM::BYTES);
    if (e != cudaSuccess) return cuda_status(e, "gauss: set smem attribute");
    a.ntiles_n = (int)((a.N + BN - 1) / BN);
    const int64_t grid = ((a.M + BM - 1) / BM) * a.ntiles_n;
    HSK_REQUIRE(grid < (1ll << 31), HSK_EINVAL, "gauss: grid too large");
    if (a.splits < 1) a.splits = 1;
    if (a.splits > 1) {
        void *ws = nullptr;
        int *flags = nullptr;
        int rc = stream_workspace(st, (size_t)a.splits * a.M * a.N * sizeof(double), 1, &ws, &flags);
        if (rc) return rc;
        a.ws = static_cast<double *>(ws);
    }
    kern<<<dim3((unsigned)grid, (unsigned)a.splits, 1), WGM * WGN * 32, SM::BYTES, st>>>(a);
    HSK_CHECK_LAUNCH("gauss_kernel");
    if (a.splits > 1) {
        splitk_reduce_kernel<<<sm_count() * 4, 256, 0, st>>>(a.ws, a.splits, a.M, a.N, a.S, a.lds,
                                                            a.col0);
        HSK_CHECK_LAUNCH("splitk_reduce_kernel");
    }
    return HSK_OK;
}

// FP64 tensor-pipe peak probe: independent DMMA.8x8x4 chains only (8 per
// warp), for the roofline denominator of the Gaussian product (bench.py)
__global__ void dmma_probe_kernel(double *out, int64_t iters) {
    double c[8][2];
    const double a = threadIdx.x * 1e-9, b = 1.0 + blockIdx.x * 1e-9;
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
    for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) dmma(c[i], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 1234.5) out[0] = s;  // keeps the chains live
}

}  // namespace gauss
}  // namespace hsk

using namespace hsk;

extern "C" int hsk_gauss_apply(const double *A, int64_t rows, int64_t cols, int64_t lda,
                               int32_t trans, const double *R, int64_t n, int32_t d, double *S,
                               int64_t lds, int64_t col0, void *stream) {
    HSK_REQUIRE(trans == 0 || trans == 1, HSK_EINVAL, "gauss apply: trans must be 0 or 1");
    HSK_REQUIRE(rows >= 0 && cols >= 0 && lda >= std::max<int64_t>(rows, 1), HSK_EINVAL,
                "gauss apply: bad A shape");
    HSK_REQUIRE(d >= 1, HSK_EINVAL, "gauss apply: d must be >= 1");
    const int64_t kdim = trans ? rows : cols;
    const int64_t m_out = trans ? cols : rows;
    if (kdim != n) {
        return set_error(HSK_EINVAL, "operator is over dimension %lld, matrix has %lld %s",
                         (long long)n, (long long)kdim, trans ? "rows" : "columns");
    }
    HSK_REQUIRE(lds >= std::max<int64_t>(m_out, 1) && col0 >= 0, HSK_EINVAL,
                "gauss apply: bad output lds/col0");
    if (m_out == 0) return HSK_OK;
    HSK_REQUIRE(S && R && (A || n == 0), HSK_EINVAL, "gauss apply: null pointer");
    gauss::Args a{};
    a.A = A;
    a.lda = lda;
    a.R = R;
    a.M = m_out;
    a.N = d;
    a.K = n;
    a.S = S;
    a.lds = lds;
    a.col0 = col0;
    a.a16 = ((reinterpret_cast<uintptr_t>(A) & 15) == 0) && (lda % 2 == 0);
    a.b16 = ((reinterpret_cast<uintptr_t>(R) & 15) == 0) && (n % 2 == 0);
    a.splits = tuning().gauss_splits > 0 ? tuning().gauss_splits : 1;
    cudaStream_t st = as_stream(stream);
    // 64 x 64 tiles, 2 x 2 warps (32 x 32 DMMA tiles each), BK 32, 2 stages: many
    // resident CTAs keep the FP64 tensor pipe fed (measured best among warp
    // tiles 32x32 / 32x64 / 64x32 / 64x64 and 2-6 stages).  HSK_GAUSS_CFG overrides: "128" (128x128, 2x4 warps),
    // "64x128" (2x4 warps).
#if HSK_TUNING  // A/B variants of DESIGN.md §7 (HSK_GAUSS_CFG); the 128-wide tiles spill
    const char *cfg = tuning().gauss_cfg;
    if (!strcmp(cfg, "64x128w"))
        return trans ? gauss::launch<64, 128, 1, 2, 2, 4>(a, st)
                     : gauss::launch<64, 128, 0, 2, 2, 4>(a, st);
    if (!strcmp(cfg, "128x64w"))
        return trans ? gauss::launch<128, 64, 1, 2, 2, 4>(a, st)
                     : gauss::launch<128, 64, 0, 2, 2, 4>(a, st);
    if (!strcmp(cfg, "128x128w"))
        return trans ? gauss::launch<128, 128, 1, 2, 2, 3>(a, st)
                     : gauss::launch<128, 128, 0, 2, 2, 3>(a, st);
    if (!strcmp(cfg, "64x64s3"))
        return trans ? gauss::launch<64, 64, 1, 2, 2, 3>(a, st)
                     : gauss::launch<64, 64, 0, 2, 2, 3>(a, st);
    if (!strcmp(cfg, "64x64s6"))
        return trans ? gauss::launch<64, 64, 1, 2, 2, 6>(a, st)
                     : gauss::launch<64, 64, 0, 2, 2, 6>(a, st);
    if (!strcmp(cfg, "128"))
        return trans ? gauss::launch<128, 128, 1, 2, 4, 3>(a, st)
                     : gauss::launch<128, 128, 0, 2, 4, 3>(a, st);
    if (!strcmp(cfg, "64x128"))
        return trans ? gauss::launch<64, 128, 1, 2, 4, 3>(a, st)
                     : gauss::launch<64, 128, 0, 2, 4, 3>(a, st);
    if (!strcmp(cfg, "64x64x8"))
        return trans ? gauss::launch<64, 64, 1, 2, 4, 4>(a, st)
                     : gauss::launch<64, 64, 0, 2, 4, 4>(a, st);
#endif
    return trans ? gauss::launch<64, 64, 1, HSK_GAUSS_WGM, HSK_GAUSS_WGN, HSK_GAUSS_STAGES>(a, st)
                 : gauss::launch<64, 64, 0, HSK_GAUSS_WGM, HSK_GAUSS_WGN, HSK_GAUSS_STAGES>(a, st);
}

extern "C" int64_t hsk_dmma_probe_flops(int64_t iters) {
    return (int64_t)sm_count() * 2 * 8 * iters * 8 * (2 * 8 * 8 * 4);
}

extern "C" int hsk_dmma_probe(int64_t iters, double *scratch, void *stream) {
    HSK_REQUIRE(iters >= 1 && scratch, HSK_EINVAL, "dmma probe: bad arguments");
    gauss::dmma_probe_kernel<<<sm_count() * 2, 8 * 32, 0, as_stream(stream)>>>(scratch, iters);
    HSK_CHECK_LAUNCH("dmma_probe_kernel");
    return HSK_OK;
}
