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
#include <string.h>

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
    int use_tma;
    int use_tma_t;  // S' of aligned A: swizzled TMA staging read by pass A
    int64_t m_out;   // number of vectors
    int64_t n;       // vector length (before padding)
    int64_t n_pad;
    int seg;         // min(SEG, n_pad)
    const double *signs;
    const uint16_t *masks;  // seg == 256: per (segment, warp) sign bits of k = w + 16 u
    const int64_t *sample;
    int d;
    double scale;
    double *S;
    int64_t lds, col0;
    int nslabs;
    int pitch;
    int stages;
    int64_t nseg;    // n_pad / seg
};

constexpr int kMaxStages = 4;
// smem map: [full barriers 64 B][signs: kMaxStages x SEG doubles (n_pad < 256) or
// kMaxStages x 16 u16 sign masks][sorted samples, their columns]
// [tiles from kTileOff: 1024-byte aligned for the TMA destination]
constexpr int kSampOff = 64 + kMaxStages * SEG * 8;
constexpr int kTileOff = ((kSampOff + 2 * 32 * 32 * 4) + 1023) / 1024 * 1024;

// Sign masks for 256-element segments: bit u of masks[g*16 + w] is the sign
// of element g*256 + w + 16u -- what warp w of the kernel's pass A needs, in
// one 2-byte broadcast instead of 16 double loads.
__global__ void srht_mask_kernel(const double *__restrict__ signs, int64_t nseg,
                                 uint16_t *__restrict__ masks) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nseg * 16;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = q >> 4;
        const int w = (int)(q & 15);
        uint32_t m = 0;
        for (int u = 0; u < 16; ++u) m |= (signs[g * SEG + w + 16 * u] < 0.0 ? 1u : 0u) << u;
        masks[q] = (uint16_t)m;
    }
}

// Segment g of the 32 vectors into X[k][r] (pitch doubles per k) with 8/16-byte
// cp.async; used when TMA cannot be (S' tiles, unaligned A, n_pad < 256).
__device__ __forceinline__ void load_segment_async(const Args &p, double *X, int64_t r0,
                                                   int64_t g) {
    const int tid = threadIdx.x;
    const int64_t k0 = g * p.seg;
    if (!p.trans) {
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
        // vector r = column r0+r of A; thread keeps kk fixed and walks rows
        // (lanes along kk: coalesced reads; pitch 33: conflict-free stores)
        for (int kk = tid % p.seg; kk < p.seg; kk += NW * 32) {
            const int64_t gk = k0 + kk;
            const bool vk = gk < p.n;
            for (int rr = tid / p.seg; rr < TM; rr += (NW * 32 + p.seg - 1) / p.seg) {
                const bool v = vk && (r0 + rr < p.m_out);
                cp_async8(X + kk * p.pitch + rr, v ? p.A + (r0 + rr) * p.lda + gk : p.A, v);
            }
        }
    }
}

// In-register Walsh-Hadamard butterflies over the index bits of x[0..15].
__device__ __forceinline__ void wht16(double (&x)[16]) {
#pragma unroll
    for (int h = 1; h < 16; h <<= 1)
#pragma unroll
        for (int q = 0; q < 16; ++q)
            if (!(q & h)) {
                const double a = x[q], b = x[q + h];
                x[q] = a + b;
                x[q + h] = a - b;
            }
}

// PATH 0: cp.async segments (unaligned A, n_pad < 256); 1: TMA S tiles;
// 2: TMA S' staging (separate instantiations: code generation)
template <int TPW, int PATH>
__global__ void __launch_bounds__(NW * 32, 1)
    srht_kernel(const Args p, const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);
    double *sgn_all = reinterpret_cast<double *>(smem + 64);            // stages x seg doubles
    uint16_t *sgm_all = reinterpret_cast<uint16_t *>(smem + 64);        // stages x 16 masks
    int *s_samp = reinterpret_cast<int *>(smem + kSampOff);             // NW*TPW, sorted per warp
    int *s_col = s_samp + NW * 32;                                      // their output columns
    uint32_t *s_pk = reinterpret_cast<uint32_t *>(s_col + NW * 32);     // NW x 8 packed positions
    double *X0 = reinterpret_cast<double *>(smem + kTileOff);  // 1024-B aligned (TMA)
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // the TMA paths always run 256-input segments at pitch TM: compile-time
    // constants there (shared-memory addresses become immediate offsets)
    const int pitch = PATH == 0 ? p.pitch : TM;
    const int seg = PATH == 0 ? p.seg : SEG;
    const int slab = (int)(blockIdx.x % p.nslabs);
    const int64_t r0 = (blockIdx.x / p.nslabs) * TM;
    const int t0 = slab * NW * TPW;
    const int tile_elems = seg * pitch;
    const int stages = p.stages;
    constexpr bool tma = PATH == 1;  // == p.use_tma
    // S' (vectors = columns of A, contiguous): TMA lands each 32-vector x
    // 256 segment in A's natural layout -- 16 boxes of 16 inputs x 32
    // vectors, 128-byte swizzle -- in a staging buffer, and pass A reads it
    // from there (lane pairs share a 16-byte chunk: conflict-free) and
    // writes X[k][vector]; the next segment's TMA is issued
    // once pass A's barrier shows the staging buffer consumed.  Two X slots:
    // pass A of segment g+1 may run while slow warps still fold segment g
    // (slot g+1 was last read before the pass-A barrier of segment g), so
    // the fold needs no trailing barrier.
    constexpr bool tmat = PATH == 2;  // == p.use_tma_t
    uint64_t *stg_full = full + (kMaxStages - 1);
    const double *stg = X0 + (size_t)stages * tile_elems;

    // each warp sorts its TPW samples by position within a segment (s mod
    // seg) so repeated positions reuse one tile load in the fold
    {
        const int t = t0 + warp * TPW + lane;
        const bool valid = lane < TPW && t < p.d;
        const int sv = valid ? (int)p.sample[t] : 0;
        // key: (position, lane) -- invalid samples sort last
        uint64_t key = ((uint64_t)(valid ? (uint32_t)(sv & (seg - 1)) : 0xFFFFFFu) << 32) |
                       (uint32_t)lane;
#pragma unroll
        for (int kk = 2; kk <= 32; kk <<= 1)
#pragma unroll
            for (int jj = kk >> 1; jj > 0; jj >>= 1) {
                const uint64_t o = __shfl_xor_sync(0xffffffffu, key, jj);
                const bool up = ((lane & kk) == 0);
                const bool lower = (lane & jj) == 0;
                key = (lower == up) ? (o < key ? o : key) : (o > key ? o : key);
            }
        const int src = (int)(key & 31u);
        const int s_sorted = __shfl_sync(0xffffffffu, sv, src);
        const int valid_sorted = __shfl_sync(0xffffffffu, (int)valid, src);
        if (lane < TPW) {
            s_samp[warp * TPW + lane] = s_sorted;
            s_col[warp * TPW + lane] = valid_sorted ? t0 + warp * TPW + src : -1;
        }
        // the same positions within a segment, one byte each: the fold reads
        // them as two broadcast 16-byte loads per segment instead of TPW
        // 4-byte ones (registers are full: TPW = 32 sits at 127)
        const uint32_t byte = (uint32_t)(s_sorted & (seg - 1));
        uint32_t w = byte << (8 * (lane & 3));
        w |= __shfl_down_sync(0xffffffffu, w, 1);
        w |= __shfl_down_sync(0xffffffffu, w, 2);
        if ((lane & 3) == 0 && lane < TPW) s_pk[warp * 8 + (lane >> 2)] = w;
    }
    if (tid == 0) {
        for (int q = 0; q < stages; ++q) mbar_init(&full[q], 1);
        if (tmat) mbar_init(stg_full, 1);
        fence_mbar_init();
        if (tma || tmat) prefetch_tmap(&tmap);
    }
    __syncthreads();
    const int64_t G = p.nseg;
    const int lb = 31 - __clz(seg);  // log2(seg)

    // issue segment g into slot q == g % stages (TMA path: one thread; else all)
    auto issue = [&](int64_t g, int q) {
        double *X = X0 + (size_t)q * tile_elems;
        double *sg = sgn_all + q * SEG;
        if (tma) {  // (TMA implies seg == 256: sign masks)
            if (tid == 0) {
                mbar_arrive_expect_tx(&full[q], (uint32_t)(seg * TM * 8 + 32));
                tma_load_2d(X, &tmap, (int)r0, (int)(g * seg), &full[q]);
                bulk_g2s(sgm_all + q * 16, p.masks + g * 16, 32, &full[q]);
            }
        } else {
            load_segment_async(p, X, r0, g);
            if (seg == SEG) {
                if (tid < 2) cp_async16(sgm_all + q * 16 + 8 * tid, p.masks + g * 16 + 8 * tid, true);
            } else {
                for (int k = tid; k < seg; k += NW * 32) cp_async8(sg + k, p.signs + g * seg + k, true);
            }
        }
    };

    // S' staging issue (thread 0): segment g and its sign masks (mask slot g & 1)
    auto issue_t = [&](int64_t g) {
        mbar_arrive_expect_tx(stg_full, (uint32_t)(SEG * TM * 8 + 32));
        for (int u = 0; u < SEG / 16; ++u)  // box u: inputs 16u.. of the 32 vectors (4 KB)
            tma_load_2d(const_cast<double *>(stg) + u * 16 * TM, &tmap, (int)(g * SEG + 16 * u), (int)r0,
                        stg_full);
        bulk_g2s(sgm_all + (g & 1) * 16, p.masks + g * 16, 32, stg_full);
    };

    double acc[TPW];
#pragma unroll
    for (int i = 0; i < TPW; ++i) acc[i] = 0.0;

    if (tmat) {
        if (tid == 0 && G > 0) issue_t(0);
    } else {
        for (int64_t g = 0; g < stages - 1 && g < G; ++g) {
            issue(g, (int)g);
            if (!tma) cp_async_commit();
        }
    }
    // slot q = g % stages and its full-barrier parity (g / stages) & 1, kept
    // incrementally (no 64-bit division per segment); qi = slot of g - 1
    int q = 0, qi = stages - 1;
    uint32_t fph = 0;
    for (int64_t g = 0; g < G; ++g) {
        double *X = X0 + (size_t)q * tile_elems;
        const double *sg = sgn_all + q * SEG;
        if (tmat) {
            mbar_wait(stg_full, (uint32_t)(g & 1));
        } else {
        // the slot of segment g-1 is free: every thread passed its last sync
        // (TMA path: issued after pass A's barrier below instead)
        if (!tma && g + stages - 1 < G) issue(g + stages - 1, qi);
        if (tma) {
            mbar_wait(&full[q], fph);
        } else {
            cp_async_commit();
            if (stages == 2) cp_async_wait<1>(); else cp_async_wait<2>();
            __syncthreads();
        }
        }
        if (seg == SEG) {
            // pass A: k = w + 16 q, butterflies over k bits 4..7 (signs applied
            // by flipping sign bits: exact, as the reference's multiply by +-1)
            double x[16];
            if (tmat) {
                // lane -> (vector v = 16 (w/8) + l/2, input kl = 2 (w%8) + l%2): the
                // two lanes of a vector read the two 8-byte halves of one 16-byte
                // chunk, so each half-warp's 16 loads (64-bit loads are serviced
                // per half-warp) hit 16 distinct bank pairs -- one wavefront each
                // (one input of 16 vectors would share 8 bank pairs: ncu showed 4
                // wavefronts per load).  Input kl + 16u of vector v: box u,
                // 128-byte row v, 16-byte chunk (kl/2) ^ (v%8).  X columns of odd
                // inputs are XOR 8 permuted (vector v of input k at column
                // v ^ 8(k%2)), so the two lanes of a vector store to different
                // bank pairs as well; pass B undoes it when it reads.
                const int v = 16 * (warp >> 3) + (lane >> 1), kl = 2 * (warp & 7) + (lane & 1);
                const uint32_t msk = sgm_all[(int)(g & 1) * 16 + kl];
                const double *sb = stg + v * 16 + (((kl * 8) ^ ((v & 7) << 4)) >> 3);
#pragma unroll
                for (int u = 0; u < 16; ++u)
                    x[u] = __longlong_as_double(__double_as_longlong(sb[u * 16 * TM]) ^
                                                ((long long)((msk >> u) & 1u) << 63));
                wht16(x);
#pragma unroll
                for (int u = 0; u < 16; ++u) X[(kl + 16 * u) * pitch + (v ^ ((kl & 1) << 3))] = x[u];
            } else {
            const uint32_t msk = sgm_all[q * 16 + warp];
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    const int k = warp + 16 * u;
                    x[u] = __longlong_as_double(__double_as_longlong(X[k * pitch + lane]) ^
                                                ((long long)((msk >> u) & 1u) << 63));
                }
            wht16(x);
#pragma unroll
            for (int u = 0; u < 16; ++u) X[(warp + 16 * u) * pitch + lane] = x[u];
            }
            __syncthreads();
            // TMA path: every thread is past the fold of segment g-1 here, so
            // its slot is refilled now and the fold needs no trailing barrier
            if (tma && g + stages - 1 < G) issue(g + stages - 1, qi);
            // S': every warp is past pass A, the staging buffer is free
            if (tmat && tid == 0 && g + 1 < G) issue_t(g + 1);
            // pass B: k = 16 w + q, butterflies over k bits 0..3 (S': odd inputs
            // of vector `lane` at column lane ^ 8, see pass A)
#pragma unroll
            for (int u = 0; u < 16; ++u) x[u] = X[(16 * warp + u) * pitch + (tmat ? lane ^ ((u & 1) << 3) : lane)];
            wht16(x);
#pragma unroll
            for (int u = 0; u < 16; ++u) X[(16 * warp + u) * pitch + lane] = x[u];
        } else {
            // small n_pad (< 256): signs, then in-smem radix-2 stages
            for (int k = warp; k < seg; k += NW) X[k * pitch + lane] *= sg[k];
            __syncthreads();
            for (int h = 1; h < seg; h <<= 1) {
                for (int pr = warp; pr < seg / 2; pr += NW) {
                    const int a_i = (pr / h) * 2 * h + (pr % h);
                    const double a = X[a_i * pitch + lane], b = X[(a_i + h) * pitch + lane];
                    X[a_i * pitch + lane] = a + b;
                    X[(a_i + h) * pitch + lane] = a - b;
                }
                __syncthreads();
            }
        }
        __syncthreads();
        // fold segment g into the warp's sampled outputs.  Lane i computes the
        // Walsh sign of sample i for this segment; a ballot shares the mask.
        {
            const int sw = lane < TPW ? s_samp[warp * TPW + lane] : 0;
            const uint32_t neg = __ballot_sync(0xffffffffu,
                                               __popc((unsigned)(g & (sw >> lb))) & 1);
            uint32_t pk[(TPW + 3) / 4];
#pragma unroll
            for (int v = 0; v < (TPW + 3) / 4; v += 4) {
                const uint4 q4 = *reinterpret_cast<const uint4 *>(s_pk + warp * 8 + v);
                pk[v] = q4.x;
                if (v + 1 < (TPW + 3) / 4) pk[v + 1] = q4.y;
                if (v + 2 < (TPW + 3) / 4) pk[v + 2] = q4.z;
                if (v + 3 < (TPW + 3) / 4) pk[v + 3] = q4.w;
            }
            if constexpr (PATH != 0) {
                // pitch 32: byte offset s_lo*256 + lane*8 assembled by one PRMT
                // (byte 0 = lane*8, byte 1 = s_lo); the Walsh sign goes onto the
                // value's sign bit (exact, as the +-1 product) and a DADD adds it
                const char *xb = reinterpret_cast<const char *>(X);
                const uint32_t lane8 = (uint32_t)lane * 8u;
#pragma unroll
                for (int i = 0; i < TPW; ++i) {
                    const uint32_t off = __byte_perm(pk[i >> 2], lane8, 0x5504u | ((uint32_t)(i & 3) << 4));
                    const double v = *reinterpret_cast<const double *>(xb + off);
                    const int hi = __double2hiint(v) ^ (int)((neg << (31 - i)) & 0x80000000u);
                    acc[i] += __hiloint2double(hi, __double2loint(v));
                }
            } else {
#pragma unroll
                for (int i = 0; i < TPW; ++i) {
                    const int s_lo = (int)__byte_perm(pk[i >> 2], 0u, 0x4440u | (uint32_t)(i & 3));
                    const double gsg = __hiloint2double((int)(((neg >> i) & 1u) << 31 | 0x3FF00000u), 0);
                    acc[i] = fma(X[s_lo * pitch + lane], gsg, acc[i]);
                }
            }
        }
        if (!tma && !tmat) __syncthreads();  // X (slot q) is refilled by the issue of segment g + 1
        qi = q;
        if (++q == stages) {
            q = 0;
            fph ^= 1u;
        }
    }
    if (!tma && !tmat) cp_async_wait<0>();

    const int64_t row = r0 + lane;
    if (row < p.m_out) {
#pragma unroll
        for (int i = 0; i < TPW; ++i) {
            const int t = s_col[warp * TPW + i];
            if (t >= 0) p.S[(p.col0 + t) * p.lds + row] = acc[i] * p.scale;
        }
    }
}

template <int TPW>
static int launch(Args a, cudaStream_t st) {
    // TMA for row tiles of aligned A with full 256-column segments
    a.use_tma = !a.trans && a.vec16 && a.seg == SEG;
    a.use_tma_t = a.trans && a.vec16 && a.seg == SEG;
    a.pitch = a.trans && !a.use_tma_t ? TM + 1 : TM;  // pitch 33: transposing cp.async stores
    a.nseg = a.n_pad / a.seg;
    CUtensorMap tmap;
    memset(&tmap, 0, sizeof(tmap));
    if (a.use_tma) {
        int rc = make_tmap_f64_2d(&tmap, a.A, (uint64_t)a.m_out, (uint64_t)a.n, (uint64_t)a.lda,
                                  TM, SEG);
        if (rc) return rc;
    } else if (a.use_tma_t) {  // A is n x m_out: boxes of 16 input indices x TM vectors, swizzled
        int rc = make_tmap_f64_2d(&tmap, a.A, (uint64_t)a.n, (uint64_t)a.m_out, (uint64_t)a.lda,
                                  16, TM, true);
        if (rc) return rc;
    }
    const int tile = a.seg * a.pitch * 8;
    static_assert(kSampOff + NW * 32 * 4 * 2 + NW * 8 * 4 <= kTileOff, "sample tables must fit below kTileOff");
    const int fixed = kTileOff;
    a.stages = (int)std::min<int64_t>(3, std::max<int64_t>(2, a.nseg));
    while (a.stages > 2 && fixed + a.stages * tile > 227 * 1024) --a.stages;
    if (a.use_tma_t) a.stages = 2;  // two X slots + the staging tile
    const int smem = fixed + a.stages * tile + (a.use_tma_t ? SEG * TM * 8 : 0);
    auto kern = a.use_tma_t ? srht_kernel<TPW, 2> : a.use_tma ? srht_kernel<TPW, 1> : srht_kernel<TPW, 0>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return cuda_status(e, "srht: set smem attribute");
    a.nslabs = (a.d + NW * TPW - 1) / (NW * TPW);
    const int64_t grid = ((a.m_out + TM - 1) / TM) * a.nslabs;
    HSK_REQUIRE(grid < (1ll << 31), HSK_EINVAL, "srht: grid too large");
    kern<<<(unsigned)grid, NW * 32, smem, st>>>(a, tmap);
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
    cudaStream_t st0 = as_stream(stream);
    if (a.seg == srht::SEG) {  // per-(segment, warp) sign masks in the stream's workspace
        const int64_t nseg = n_pad / srht::SEG;
        void *ws = nullptr;
        int *flags = nullptr;
        int rc = stream_workspace(st0, (size_t)nseg * 16 * sizeof(uint16_t), 0, &ws, &flags);
        if (rc) return rc;
        a.masks = static_cast<const uint16_t *>(ws);
        const unsigned blocks = (unsigned)std::min<int64_t>((nseg * 16 + 255) / 256, sm_count() * 4);
        srht::srht_mask_kernel<<<std::max(1u, blocks), 256, 0, st0>>>(
            signs, nseg, static_cast<uint16_t *>(ws));
        HSK_CHECK_LAUNCH("srht_mask_kernel");
    }
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
