// hsk_srht.cu -- SRHT sketch S[r, t] = scale * FWHT(pad(x_r) .* signs)[sample[t]]
// and the standalone FWHT, on sm_100a.
//
// Replaces SrhtBlock._transform (sketching.py:162-176) and fwht
// (sketching.py:100-112).
//
// Two-level Walsh-Hadamard factorisation.  With
// k = g*B + k_lo and s = s_hi*B + s_lo (B = 256):
//     y[s] = sum_g (-1)^popcount(g & s_hi) * z_g[s_lo],
//     z_g  = FWHT_B(x'[g*B : (g+1)*B]).
// A CTA owns 32 vectors (lane = vector) and a slab of sampled outputs; it
// streams the n_pad/B segments of its vectors through a double-buffered
// shared tile X[k][r] (A read once from HBM), transforms each segment in
// registers (two passes of 16-value butterflies, 16 warps), and folds the
// segment into register accumulators of the d sampled outputs with a +-1
// DFMA.  Only the d sampled columns of the last log2(n_pad/B) stages are
// ever formed (pruned FWHT).  Sample indices may repeat (the reference
// draws with replacement, sketching.py:159).
#include <algorithm>

#include "hsk_common.cuh"

namespace hsk {
namespace srht {

constexpr int NW = 16;        // warps per CTA
constexpr int TM = 32;        // vectors per CTA (lane = vector)
constexpr int SEG = 256;      // segment length B

struct Args {
    const double *A;
    int64_t lda;
    int trans;
    int vec16;
    int64_t m_out;   // number of vectors
    int64_t n;       // vector length (before padding)
    int64_t n_pad;
    int seg;         // min(SEG, n_pad)
    const double *signs;
    const int64_t *sample;
    int d;
    double scale;
    double *S;
    int64_t lds, col0;
    int nslabs;
    int pitch;
};

// Load segment g of the 32 vectors into X[k][r] (pitch doubles per k).
__device__ __forceinline__ void load_segment(const Args &p, double *X, int64_t r0, int64_t g) {
    const int tid = threadIdx.x;
    const int64_t k0 = g * p.seg;
    if (!p.trans) {
        // vector r = row r0+r of A; element k at A[k*lda + r0 + r]; 16 B = 2 rows
        for (int q = tid; q < p.seg * (TM / 2); q += NW * 32) {
            const int kk = q / (TM / 2), rr = (q % (TM / 2)) * 2;
            const int64_t gk = k0 + kk, gr = r0 + rr;
            const bool vk = gk < p.n;
            const bool v0 = vk && gr < p.m_out, v1 = vk && gr + 1 < p.m_out;
            const double *src = p.A + gk * p.lda + gr;
            double *dst = X + kk * p.pitch + rr;
            if (p.vec16 && v0 && v1) {
                cp_async16(dst, src, true);
            } else {
                cp_async8(dst, v0 ? src : p.A, v0);
                cp_async8(dst + 1, v1 ? src + 1 : p.A, v1);
            }
        }
    } else {
        // vector r = column r0+r of A; element k at A[(r0+r)*lda + k].
        // 16 consecutive k per half-warp: coalesced reads; pitch 33 makes the
        // transposing shared stores conflict-free.
        const int lane = tid & 31, warp = tid >> 5;
        const int kl = lane & 15, rl = lane >> 4;
        for (int rb = warp * 2; rb < TM; rb += NW * 2) {
            const int rr = rb + rl;
            const int64_t gr = r0 + rr;
            const bool vr = gr < p.m_out;
            const double *col = p.A + gr * p.lda + k0;
            for (int kk = kl; kk < p.seg; kk += 16) {
                const bool v = vr && (k0 + kk < p.n);
                cp_async8(X + kk * p.pitch + rr, v ? col + kk : p.A, v);
            }
        }
    }
}

template <int TPW>
__global__ void __launch_bounds__(NW * 32, 1) srht_kernel(const Args p) {
    extern __shared__ __align__(128) double sm[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int slab = (int)(blockIdx.x % p.nslabs);
    const int64_t r0 = (blockIdx.x / p.nslabs) * TM;
    const int t0 = slab * NW * TPW;
    const int tile_elems = p.seg * p.pitch;
    double *X0 = sm;
    double *X1 = sm + tile_elems;
    int *s_samp = reinterpret_cast<int *>(sm + 2 * tile_elems);

    for (int i = tid; i < NW * TPW; i += NW * 32) {
        const int t = t0 + i;
        s_samp[i] = t < p.d ? (int)p.sample[t] : 0;
    }
    const int64_t G = p.n_pad / p.seg;
    const int lb = 31 - __clz(p.seg);  // log2(seg)

    double acc[TPW];
#pragma unroll
    for (int i = 0; i < TPW; ++i) acc[i] = 0.0;

    load_segment(p, X0, r0, 0);
    cp_async_commit();
    for (int64_t g = 0; g < G; ++g) {
        double *X = (g & 1) ? X1 : X0;
        if (g + 1 < G) load_segment(p, (g & 1) ? X0 : X1, r0, g + 1);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        const int64_t kb = g * p.seg;
        if (p.seg == SEG) {
            // pass A: k = w + 16 q, butterflies over k bits 4..7 (q bits)
            double x[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const int k = warp + 16 * q;
                const int64_t gk = kb + k;
                x[q] = X[k * p.pitch + lane] * (gk < p.n ? p.signs[gk] : 0.0);
            }
#pragma unroll
            for (int h = 1; h < 16; h <<= 1)
#pragma unroll
                for (int q = 0; q < 16; ++q)
                    if (!(q & h)) {
                        const double a = x[q], b = x[q + h];
                        x[q] = a + b;
                        x[q + h] = a - b;
                    }
#pragma unroll
            for (int q = 0; q < 16; ++q) X[(warp + 16 * q) * p.pitch + lane] = x[q];
            __syncthreads();
            // pass B: k = 16 w + q, butterflies over k bits 0..3
#pragma unroll
            for (int q = 0; q < 16; ++q) x[q] = X[(16 * warp + q) * p.pitch + lane];
#pragma unroll
            for (int h = 1; h < 16; h <<= 1)
#pragma unroll
                for (int q = 0; q < 16; ++q)
                    if (!(q & h)) {
                        const double a = x[q], b = x[q + h];
                        x[q] = a + b;
                        x[q + h] = a - b;
                    }
#pragma unroll
            for (int q = 0; q < 16; ++q) X[(16 * warp + q) * p.pitch + lane] = x[q];
        } else {
            // small n_pad (< 256): signs, then in-smem radix-2 stages
            for (int k = warp; k < p.seg; k += NW) {
                const int64_t gk = kb + k;
                X[k * p.pitch + lane] *= (gk < p.n ? p.signs[gk] : 0.0);
            }
            __syncthreads();
            for (int h = 1; h < p.seg; h <<= 1) {
                for (int pr = warp; pr < p.seg / 2; pr += NW) {
                    const int a_i = (pr / h) * 2 * h + (pr % h);
                    const double a = X[a_i * p.pitch + lane], b = X[(a_i + h) * p.pitch + lane];
                    X[a_i * p.pitch + lane] = a + b;
                    X[(a_i + h) * p.pitch + lane] = a - b;
                }
                __syncthreads();
            }
        }
        __syncthreads();
        // fold segment g into the sampled outputs owned by this warp
#pragma unroll
        for (int i = 0; i < TPW; ++i) {
            const int s = s_samp[warp * TPW + i];
            const int s_lo = s & (p.seg - 1);
            const int s_hi = s >> lb;
            const double sg = (__popcll((long long)(g & s_hi)) & 1) ? -1.0 : 1.0;
            acc[i] = fma(X[s_lo * p.pitch + lane], sg, acc[i]);
        }
        __syncthreads();  // X is overwritten by the load issued next iteration
    }
    cp_async_wait<0>();

    const int64_t row = r0 + lane;
    if (row < p.m_out) {
#pragma unroll
        for (int i = 0; i < TPW; ++i) {
            const int t = t0 + warp * TPW + i;
            if (t < p.d) p.S[(p.col0 + t) * p.lds + row] = acc[i] * p.scale;
        }
    }
}

template <int TPW>
static int launch(Args a, cudaStream_t st) {
    a.pitch = a.trans ? TM + 1 : TM;
    const int smem = 2 * a.seg * a.pitch * 8 + NW * TPW * 4 + 16;
    auto kern = srht_kernel<TPW>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return cuda_status(e, "srht: set smem attribute");
    a.nslabs = (a.d + NW * TPW - 1) / (NW * TPW);
    const int64_t grid = ((a.m_out + TM - 1) / TM) * a.nslabs;
    HSK_REQUIRE(grid < (1ll << 31), HSK_EINVAL, "srht: grid too large");
    kern<<<(unsigned)grid, NW * 32, smem, st>>>(a);
    HSK_CHECK_LAUNCH("srht_kernel");
    return HSK_OK;
}

// one radix-2 stage of the standalone FWHT over rows x n (row-major)
__global__ void fwht_stage_kernel(double *X, int64_t rows, int64_t n, int64_t h, double post) {
    const int64_t pairs = rows * (n / 2);
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < pairs;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = q / (n / 2), pr = q % (n / 2);
        const int64_t i = (pr / h) * 2 * h + (pr % h);
        double *y = X + r * n;
        const double a = y[i], b = y[i + h];
        double u = a + b, v = a - b;
        if (post != 1.0) {
            u /= post;
            v /= post;
        }
        y[i] = u;
        y[i + h] = v;
    }
}

__global__ void scale_kernel(double *X, int64_t cnt, double div) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < cnt;
         q += (int64_t)gridDim.x * blockDim.x)
        X[q] /= div;
}

}  // namespace srht
}  // namespace hsk

using namespace hsk;

extern "C" int hsk_srht_apply(const double *A, int64_t rows, int64_t cols, int64_t lda,
                              int32_t trans, const double *signs, int64_t n, int64_t n_pad,
                              const int64_t *sample, int32_t d, double scale, double *S,
                              int64_t lds, int64_t col0, void *stream) {
    HSK_REQUIRE(trans == 0 || trans == 1, HSK_EINVAL, "srht apply: trans must be 0 or 1");
    HSK_REQUIRE(rows >= 0 && cols >= 0 && lda >= std::max<int64_t>(rows, 1), HSK_EINVAL,
                "srht apply: bad A shape");
    HSK_REQUIRE(d >= 1 && n >= 1 && n_pad >= n && (n_pad & (n_pad - 1)) == 0, HSK_EINVAL,
                "srht apply: bad d/n/n_pad");
    HSK_REQUIRE(n_pad < (1ll << 31), HSK_EINVAL, "srht apply: n_pad too large");
    const int64_t kdim = trans ? rows : cols;
    const int64_t m_out = trans ? cols : rows;
    if (kdim != n) {
        return set_error(HSK_EINVAL, "operator is over dimension %lld, matrix has %lld %s",
                         (long long)n, (long long)kdim, trans ? "rows" : "columns");
    }
    HSK_REQUIRE(lds >= std::max<int64_t>(m_out, 1) && col0 >= 0, HSK_EINVAL,
                "srht apply: bad output lds/col0");
    if (m_out == 0) return HSK_OK;
    HSK_REQUIRE(A && S && signs && sample, HSK_EINVAL, "srht apply: null pointer");
    srht::Args a{};
    a.A = A;
    a.lda = lda;
    a.trans = trans;
    a.vec16 = ((reinterpret_cast<uintptr_t>(A) & 15) == 0) && (lda % 2 == 0);
    a.m_out = m_out;
    a.n = n;
    a.n_pad = n_pad;
    a.seg = (int)std::min<int64_t>(srht::SEG, n_pad);
    a.signs = signs;
    a.sample = sample;
    a.d = d;
    a.scale = scale;
    a.S = S;
    a.lds = lds;
    a.col0 = col0;
    cudaStream_t st = as_stream(stream);
    if (d <= srht::NW * 8) return srht::launch<8>(a, st);
    if (d <= srht::NW * 16) return srht::launch<16>(a, st);
    return srht::launch<32>(a, st);
}

extern "C" int hsk_fwht(double *X, int64_t rows, int64_t n, int32_t normalize, void *stream) {
    HSK_REQUIRE(n >= 1 && (n & (n - 1)) == 0, HSK_EINVAL, "fwht length must be a power of two");
    HSK_REQUIRE(rows >= 0, HSK_EINVAL, "fwht: rows must be >= 0");
    if (rows == 0) return HSK_OK;
    HSK_REQUIRE(X, HSK_EINVAL, "fwht: null pointer");
    cudaStream_t st = as_stream(stream);
    const int64_t pairs = rows * (n / 2);
    const unsigned blocks = (unsigned)std::min<int64_t>((pairs + 255) / 256, sm_count() * 8);
    for (int64_t h = 1; h < n; h <<= 1) {
        srht::fwht_stage_kernel<<<std::max(1u, blocks), 256, 0, st>>>(X, rows, n, h, 1.0);
        HSK_CHECK_LAUNCH("fwht_stage_kernel");
    }
    if (normalize && n > 1) {
        const int64_t cnt = rows * n;
        const unsigned b2 = (unsigned)std::min<int64_t>((cnt + 255) / 256, sm_count() * 8);
        srht::scale_kernel<<<std::max(1u, b2), 256, 0, st>>>(X, cnt, sqrt((double)n));
        HSK_CHECK_LAUNCH("scale_kernel");
    }
    return HSK_OK;
}
