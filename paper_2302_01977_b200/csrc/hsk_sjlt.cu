// hsk_sjlt.cu -- SJLT sketch S = A R^T and S' = A^T R^T on sm_100a.
//
// Replaces SjltBlock._build_storage / apply_right / apply_right_transposed
// (/root/reference/pkg/src/hsskit/sketching.py:292-351; §6).
//
// Design:
//  * Plan.  The reference keeps R^T = s (B+ - B-) as index-only CSR/CSC.  The
//    GPU plan re-blocks the same pattern by k-chunks of TK input indices: per
//    chunk, its TK*alpha entries sorted by bucket (stable in (k, t)), plus
//    per-chunk bucket offsets.  An entry is 16 bytes, pre-decoded for the
//    consumer: {byte offset of row kk in the staged tile, 0, (double)+-1}, so
//    the inner loop spends no instructions on decoding.  Two entry arrays
//    are kept, one per tile pitch (S: TMA-dense, S': padded transpose).
//    Built on device by a per-chunk bitonic sort.
//  * Apply.  A CTA owns TM = 32*RPT output rows and a slab of NW*DB buckets.
//    Consumer warp w owns buckets [j0 + w*DB, +DB); lane l owns rows
//    l*RPT .. l*RPT+RPT-1, so each warp holds an RPT x DB register
//    accumulator block: owner-computes, no atomics, a fixed summation order
//    (deterministic).  Per entry: one broadcast LDS of the entry word, one
//    LDS.128 (RPT = 2) of the staged A tile, RPT DFMAs with +-1 (exactly the
//    reference's add/subtract, one rounding each; no data multiplies).
//  * Streaming.  A producer warp moves TK x TM tiles of A (every element
//    read once from HBM) plus the chunk's plan slice into a STAGES-deep
//    shared-memory ring: one TMA 2-D tile load (UTMALDG, OOB zero-filled)
//    per chunk when A's columns are 16-byte aligned, otherwise 8-byte
//    cp.async (which also transposes the tile for S' = A^T R^T).  mbarrier
//    full/empty pairs decouple producer and consumer warps, so per-chunk
//    load imbalance between warps is absorbed across stages.
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include "hsk_common.cuh"

namespace hsk {
namespace sjlt {

constexpr int kHeaderBytes = 128;
constexpr int kMaxChunkEntries = 4096;  // TK * alpha bound (12-bit local index)
constexpr int kPlanSlab = 512;          // bucket-offset rows padded for slabs | 512
constexpr int64_t kMaxD = (1 << 19);    // bucket index fits 19 bits of the sort key

struct Geom {
    int rpt;           // rows per lane: 4 for d <= 64, else 2
    int tm;            // rows per CTA = 32 * rpt
    int pitch;         // tile pitch (doubles) = tm: TMA writes densely; the S'
                       // producer orders its transposing stores conflict-free
    int tk;
    int64_t nchunks;
    int64_t bstride;   // uint16 per bucket-offset row
    int64_t estride;   // entries per chunk row (tk*alpha)
    int64_t bptr_off;  // bytes
    int64_t ent_off;   // bytes
    int64_t bytes;
};

static inline int64_t roundup(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// TK: as long as a stage (TK x TM x 8 B tile + TK*alpha 16-byte entries)
// leaves room for >= 3 stages in shared memory, capped at 128.
static inline int tk_for(int alpha, int tm) {
    int tk = 128;
    while (tk > 1 && (tk * alpha > kMaxChunkEntries || tk * (tm * 8 + 16 * alpha) > 74 * 1024))
        tk >>= 1;
    return tk;
}

static Geom geom(int64_t n, int d, int alpha) {
    Geom g;
    g.rpt = d <= 64 ? 4 : 2;
    g.tm = 32 * g.rpt;
    g.pitch = g.tm;
    g.tk = tk_for(alpha, g.tm);
    g.nchunks = (n + g.tk - 1) / g.tk;
    g.bstride = roundup(d, kPlanSlab) + 8;
    g.estride = (int64_t)g.tk * alpha;
    g.bptr_off = kHeaderBytes;
    g.ent_off = roundup(g.bptr_off + (g.nchunks + 1) * g.bstride * 2, 128);
    g.bytes = g.ent_off + roundup((g.nchunks + 1) * g.estride * 16, 128);
    return g;
}

// ------------------------------------------------------------ plan build
// One CTA per chunk: sort the chunk's (bucket, local index) keys, emit
// entry words in that order and per-bucket lower bounds.
__global__ void sjlt_plan_kernel(const int32_t *__restrict__ pos, const int8_t *__restrict__ sgn,
                                 int64_t n, int d, int alpha, int tk, int p2, int64_t bstride,
                                 int64_t estride, int pitch, uint16_t *__restrict__ bptr,
                                 uint4 *__restrict__ ent, int *err) {
    extern __shared__ uint32_t keys[];
    const int64_t c = blockIdx.x;
    const int64_t k0 = c * tk;
    const int kc = (int)(n - k0 < tk ? n - k0 : tk);
    const int cnt = kc * alpha;
    const int64_t q0 = k0 * alpha;
    for (int i = threadIdx.x; i < p2; i += blockDim.x) {
        uint32_t key = 0xFFFFFFFFu;
        if (i < cnt) {
            int p = pos[q0 + i];
            if (p < 0 || p >= d) {
                atomicOr(err, 1);
                p = p < 0 ? 0 : d - 1;
            }
            key = ((uint32_t)p << 12) | (uint32_t)i;
        }
        keys[i] = key;
    }
    __syncthreads();
    for (int k = 2; k <= p2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < p2; i += blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const uint32_t a = keys[i], b = keys[ixj];
                    if ((a > b) == ((i & k) == 0)) {
                        keys[i] = b;
                        keys[ixj] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
    uint4 *e_out = ent + c * estride;
    for (int e = threadIdx.x; e < estride; e += blockDim.x) {
        uint4 w = make_uint4(0, 0, 0, 0);
        if (e < cnt) {
            const int local = keys[e] & 4095;
            const uint32_t kk = (uint32_t)(local / alpha);
            const uint32_t g_hi = sgn[q0 + local] < 0 ? 0xBFF00000u : 0x3FF00000u;  // -1.0 / +1.0
            // .y: byte XOR of the S' tile swizzle (row ^ (kk mod 32))
            w = make_uint4(kk * pitch * 8, (kk & 31u) * 8u, 0, g_hi);
        }
        e_out[e] = w;
    }
    uint16_t *b_out = bptr + c * bstride;
    for (int64_t j = threadIdx.x; j < bstride; j += blockDim.x) {
        int lb = cnt;
        if (j < d) {  // number of keys with bucket < j
            const uint32_t target = (uint32_t)j << 12;
            int lo = 0, hi = cnt;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (keys[mid] < target) lo = mid + 1; else hi = mid;
            }
            lb = lo;
        }
        b_out[j] = (uint16_t)lb;
    }
}

// ------------------------------------------------------- consumer inner loop
// One bucket's entries [pe, pe_end) (shared byte addresses, 16 B each) folded
// into the lane's RPT accumulators.  Written in PTX so the loop branches are
// `bra.uni` (warp-uniform by construction: every lane walks the same entry
// list), which spares the per-bucket convergence barriers the compiler
// would otherwise emit.  Per entry: LDS.128 entry, IADD, LDS.128 tile, RPT
// DFMA with the pre-decoded +-1.0.
__device__ __forceinline__ void bucket_run2(uint32_t &pe, uint32_t pe_end, uint32_t sxl,
                                            double &a0, double &a1) {
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        ".reg .b32 o, z, gl, gh, ad;\n\t"
        ".reg .f64 x, y, g;\n\t"
        "setp.ge.u32 p, %2, %3;\n\t"
        "@p bra.uni DONE;\n\t"
        "LOOP:\n\t"
        "ld.shared.v4.b32 {o, z, gl, gh}, [%2];\n\t"
        "add.u32 ad, o, %4;\n\t"
        "ld.shared.v2.f64 {x, y}, [ad];\n\t"
        "mov.b64 g, {gl, gh};\n\t"
        "fma.rn.f64 %0, x, g, %0;\n\t"
        "fma.rn.f64 %1, y, g, %1;\n\t"
        "add.u32 %2, %2, 16;\n\t"
        "setp.lt.u32 p, %2, %3;\n\t"
        "@p bra.uni LOOP;\n\t"
        "DONE:\n\t"
        "}"
        : "+d"(a0), "+d"(a1), "+r"(pe)
        : "r"(pe_end), "r"(sxl)
        : "memory");
}

__device__ __forceinline__ void bucket_run4(uint32_t &pe, uint32_t pe_end, uint32_t sxl,
                                            double &a0, double &a1, double &a2, double &a3) {
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        ".reg .b32 o, z, gl, gh, ad;\n\t"
        ".reg .f64 x, y, u, v, g;\n\t"
        "setp.ge.u32 p, %4, %5;\n\t"
        "@p bra.uni DONE;\n\t"
        "LOOP:\n\t"
        "ld.shared.v4.b32 {o, z, gl, gh}, [%4];\n\t"
        "add.u32 ad, o, %6;\n\t"
        "ld.shared.v2.f64 {x, y}, [ad];\n\t"
        "ld.shared.v2.f64 {u, v}, [ad+16];\n\t"
        "mov.b64 g, {gl, gh};\n\t"
        "fma.rn.f64 %0, x, g, %0;\n\t"
        "fma.rn.f64 %1, y, g, %1;\n\t"
        "fma.rn.f64 %2, u, g, %2;\n\t"
        "fma.rn.f64 %3, v, g, %3;\n\t"
        "add.u32 %4, %4, 16;\n\t"
        "setp.lt.u32 p, %4, %5;\n\t"
        "@p bra.uni LOOP;\n\t"
        "DONE:\n\t"
        "}"
        : "+d"(a0), "+d"(a1), "+d"(a2), "+d"(a3), "+r"(pe)
        : "r"(pe_end), "r"(sxl)
        : "memory");
}

// S' tiles are stored swizzled: element (kk, row) lives at kk*TM + (row ^ (kk%32))
// so that the transposing 8-byte cp.async writes (lanes along kk) and the
// consumer reads (lanes along rows) are both conflict-free.  A lane owns
// rows lane + 32*r, r < RPT; entry .y holds the XOR term (kk%32)*8.
__device__ __forceinline__ void bucket_run_t2(uint32_t &pe, uint32_t pe_end, uint32_t st,
                                              uint32_t lane8, double &a0, double &a1) {
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        ".reg .b32 o, x, gl, gh, ad;\n\t"
        ".reg .f64 u, v, g;\n\t"
        "setp.ge.u32 p, %2, %3;\n\t"
        "@p bra.uni DONE;\n\t"
        "LOOP:\n\t"
        "ld.shared.v4.b32 {o, x, gl, gh}, [%2];\n\t"
        "xor.b32 ad, x, %5;\n\t"
        "add.u32 ad, ad, o;\n\t"
        "add.u32 ad, ad, %4;\n\t"
        "ld.shared.f64 u, [ad];\n\t"
        "ld.shared.f64 v, [ad+256];\n\t"
        "mov.b64 g, {gl, gh};\n\t"
        "fma.rn.f64 %0, u, g, %0;\n\t"
        "fma.rn.f64 %1, v, g, %1;\n\t"
        "add.u32 %2, %2, 16;\n\t"
        "setp.lt.u32 p, %2, %3;\n\t"
        "@p bra.uni LOOP;\n\t"
        "DONE:\n\t"
        "}"
        : "+d"(a0), "+d"(a1), "+r"(pe)
        : "r"(pe_end), "r"(st), "r"(lane8)
        : "memory");
}

__device__ __forceinline__ void bucket_run_t4(uint32_t &pe, uint32_t pe_end, uint32_t st,
                                              uint32_t lane8, double &a0, double &a1,
                                              double &a2, double &a3) {
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        ".reg .b32 o, x, gl, gh, ad;\n\t"
        ".reg .f64 u, v, w, y, g;\n\t"
        "setp.ge.u32 p, %4, %5;\n\t"
        "@p bra.uni DONE;\n\t"
        "LOOP:\n\t"
        "ld.shared.v4.b32 {o, x, gl, gh}, [%4];\n\t"
        "xor.b32 ad, x, %7;\n\t"
        "add.u32 ad, ad, o;\n\t"
        "add.u32 ad, ad, %6;\n\t"
        "ld.shared.f64 u, [ad];\n\t"
        "ld.shared.f64 v, [ad+256];\n\t"
        "ld.shared.f64 w, [ad+512];\n\t"
        "ld.shared.f64 y, [ad+768];\n\t"
        "mov.b64 g, {gl, gh};\n\t"
        "fma.rn.f64 %0, u, g, %0;\n\t"
        "fma.rn.f64 %1, v, g, %1;\n\t"
        "fma.rn.f64 %2, w, g, %2;\n\t"
        "fma.rn.f64 %3, y, g, %3;\n\t"
        "add.u32 %4, %4, 16;\n\t"
        "setp.lt.u32 p, %4, %5;\n\t"
        "@p bra.uni LOOP;\n\t"
        "DONE:\n\t"
        "}"
        : "+d"(a0), "+d"(a1), "+d"(a2), "+d"(a3), "+r"(pe)
        : "r"(pe_end), "r"(st), "r"(lane8)
        : "memory");
}

// ----------------------------------------------------------------- apply
struct ApplyArgs {
    const double *A;
    int64_t lda;
    int trans;
    int use_tma;
    int mode;       // 0: TMA tile (S), 1: swizzled transposing cp.async (S'), 2: cp.async (S)
    int ksplit;     // CTAs of a cluster splitting the k range (DSMEM reduction)
    int64_t m_out;  // output rows (rows of A for trans 0, cols of A for trans 1)
    int64_t n;      // input index extent (= op.n)
    int d, alpha, tk;
    int64_t nchunks, bstride, estride;
    const uint16_t *bptr;
    const uint4 *ent;
    double scale;
    double *S;
    int64_t lds, col0;
    int nslabs, stages, pitch;
    int stage_bytes, bp_off, en_off;
};

// Warp roles: warps [0, NW) consume (bucket owners), warps [NW, NW+PW)
// produce.  Lane l owns rows RPT*l .. RPT*l+RPT-1 of the TM-row tile.
template <int RPT, int DB, int NW, int PW, bool TRANS>
__global__ void __launch_bounds__((NW + PW) * 32, 1)
    sjlt_apply_kernel(const ApplyArgs p, const __grid_constant__ CUtensorMap tmap) {
    constexpr int TM = 32 * RPT;
    constexpr int SLAB = NW * DB;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);
    uint64_t *empty = full + 8;
    unsigned char *stage0 = smem + 128;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ks = p.ksplit;
    const int kr = (int)(blockIdx.x % ks);  // == %cluster_ctarank (cluster = ks consecutive CTAs)
    const int64_t bid = blockIdx.x / ks;
    const int slab = (int)(bid % p.nslabs);
    const int64_t tile = bid / p.nslabs;
    const int64_t r0 = tile * TM;
    const int j0 = slab * SLAB;
    // chunk range of this CTA
    const int64_t per = (p.nchunks + ks - 1) / ks;
    const int64_t c_begin = (int64_t)kr * per < p.nchunks ? (int64_t)kr * per : p.nchunks;
    const int64_t c_end = c_begin + per < p.nchunks ? c_begin + per : p.nchunks;
    const int64_t nloc = c_end - c_begin;
    const int mode = p.mode;

    if (threadIdx.x == 0) {
        const uint32_t fcount = mode == 0 ? 1u : mode == 1 ? 1u + 32u * PW : 32u * PW;  // S': bulk + noinc
        for (int s = 0; s < p.stages; ++s) {
            mbar_init(&full[s], fcount);
            mbar_init(&empty[s], NW);
        }
        fence_mbar_init();
        if (mode == 0) prefetch_tmap(&tmap);
    }
    __syncthreads();

    const int stages = p.stages;
    if (warp >= NW) {
        // ---------------------------------------------------- producers
        const int pw = warp - NW;
        const uint32_t bp_bytes = (SLAB + 8) * 2;
        const uint32_t en_bytes = (uint32_t)p.estride * 16;
        const uint32_t tile_bytes = (uint32_t)p.tk * TM * 8;
        int s = 0;
        uint32_t ph = 0;  // parity of the empty-barrier phase to wait for
        if (mode != 0 || pw == 0) {
            for (int64_t i = 0; i < nloc; ++i) {
                const int64_t c = c_begin + i;
                if (i >= stages) mbar_wait(&empty[s], ph ^ 1u);
                unsigned char *st = stage0 + (size_t)s * p.stage_bytes;
                double *sx = reinterpret_cast<double *>(st);
                uint16_t *sbp = reinterpret_cast<uint16_t *>(st + p.bp_off);
                uint4 *sen = reinterpret_cast<uint4 *>(st + p.en_off);
                const int64_t k0 = c * p.tk;
                const int kc = (int)(p.n - k0 < p.tk ? p.n - k0 : p.tk);
                const uint16_t *gbp = p.bptr + c * p.bstride + j0;
                const uint4 *gen = p.ent + c * p.estride;
                if (mode == 0) {
                    if (lane == 0) {
                        mbar_arrive_expect_tx(&full[s], tile_bytes + bp_bytes + en_bytes);
                        tma_load_2d(sx, &tmap, (int)r0, (int)k0, &full[s]);
                        bulk_g2s(sbp, gbp, bp_bytes, &full[s]);
                        bulk_g2s(sen, gen, en_bytes, &full[s]);
                    }
                    __syncwarp();
                } else if (TRANS) {
                    // S' tile: element (kk, rr) = A[k0+kk, r0+rr], stored at
                    // kk*TM + (rr ^ (kk%32)).  Lanes run along kk (256 B of one
                    // column of A per instruction); the swizzle spreads the
                    // 32 stores over all bank pairs.
                    if (pw == 0 && lane == 0) {
                        mbar_arrive_expect_tx(&full[s], bp_bytes + en_bytes);
                        bulk_g2s(sbp, gbp, bp_bytes, &full[s]);
                        bulk_g2s(sen, gen, en_bytes, &full[s]);
                    }
                    const int pl = pw * 32 + lane;
                    for (int idx = pl; idx < p.tk * TM; idx += 32 * PW) {
                        const int rr = idx / p.tk, kk = idx % p.tk;
                        const bool v = (kk < kc) && (r0 + rr < p.m_out);
                        const double *src = p.A + (r0 + rr) * p.lda + k0 + kk;
                        cp_async8(sx + kk * TM + (rr ^ (kk & 31)), v ? src : p.A, v);
                    }
                    cp_async_mbar_arrive(&full[s]);
                } else {
                    const int pl = pw * 32 + lane;  // producer lane id in [0, 32*PW)
                    for (uint32_t q = pl; q < bp_bytes / 16; q += 32 * PW)
                        cp_async16(sbp + q * 8, gbp + q * 8, true);
                    for (uint32_t q = pl; q < en_bytes / 16; q += 32 * PW)
                        cp_async16(sen + q, gen + q, true);
                    for (int idx = pl; idx < p.tk * TM; idx += 32 * PW) {
                        int kk, rr;
                        const double *src;
                        if (!p.trans) {  // lanes along rows: coalesced global
                            kk = idx / TM;
                            rr = idx % TM;
                            src = p.A + (k0 + kk) * p.lda + r0 + rr;
                        } else {         // lanes along k: coalesced global
                            rr = idx / p.tk;
                            kk = idx % p.tk;
                            src = p.A + (r0 + rr) * p.lda + k0 + kk;
                        }
                        const bool v = (kk < kc) && (r0 + rr < p.m_out);
                        cp_async8(sx + kk * p.pitch + rr, v ? src : p.A, v);
                    }
                    cp_async_mbar_arrive(&full[s]);
                }
                if (++s == stages) {
                    s = 0;
                    ph ^= 1u;
                }
            }
        }
        if (ks > 1) {  // match the consumers' barriers of the k-split reduction
            __syncthreads();
            cluster_sync();
            cluster_sync();
        }
        return;
    }

    // -------------------------------------------------------- consumers
    double acc[RPT][DB];
#pragma unroll
    for (int r = 0; r < RPT; ++r)
#pragma unroll
        for (int jj = 0; jj < DB; ++jj) acc[r][jj] = 0.0;
    {
        const uint32_t smem_base = smem_u32(stage0);
        int s = 0;
        uint32_t ph = 0;
        for (int64_t i = 0; i < nloc; ++i) {
            mbar_wait(&full[s], ph);
            const uint32_t st = smem_base + (uint32_t)s * p.stage_bytes;
            const uint32_t sxl = st + lane * RPT * 8;
            const uint16_t *sbp = reinterpret_cast<const uint16_t *>(
                                      stage0 + (size_t)s * p.stage_bytes + p.bp_off) + warp * DB;
            const uint32_t sen = st + p.en_off;
            uint32_t pe = sen + 16u * (uint32_t)sbp[0];
#pragma unroll
            for (int jj = 0; jj < DB; ++jj) {
                const uint32_t pe_end = sen + 16u * (uint32_t)sbp[jj + 1];
                if (TRANS) {
                    if (RPT == 2)
                        bucket_run_t2(pe, pe_end, st, lane * 8u, acc[0][jj], acc[1][jj]);
                    else
                        bucket_run_t4(pe, pe_end, st, lane * 8u, acc[0][jj], acc[1][jj],
                                      acc[RPT - 2][jj], acc[RPT - 1][jj]);
                } else if (RPT == 2) {
                    bucket_run2(pe, pe_end, sxl, acc[0][jj], acc[1][jj]);
                } else {
                    bucket_run4(pe, pe_end, sxl, acc[0][jj], acc[1][jj], acc[RPT - 2][jj],
                                acc[RPT - 1][jj]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (++s == stages) {
                s = 0;
                ph ^= 1u;
            }
        }
    }

    // ------------------------------------------- k-split: DSMEM reduction
    // Partial sums of the ks CTAs of a cluster are combined by rank 0 in
    // rank order (deterministic).  The stage ring is reused as the buffer.
    double *red = reinterpret_cast<double *>(stage0);
    if (ks > 1) {
        __syncthreads();  // every stage consumed: the ring is free
        if (kr > 0) {
#pragma unroll
            for (int jj = 0; jj < DB; ++jj)
#pragma unroll
                for (int r = 0; r < RPT; ++r)
                    red[((warp * DB + jj) * RPT + r) * 32 + lane] = acc[r][jj];
        }
        cluster_sync();
        if (kr == 0) {
            for (int q = 1; q < ks; ++q) {
#pragma unroll
                for (int jj = 0; jj < DB; ++jj)
#pragma unroll
                    for (int r = 0; r < RPT; ++r)
                        acc[r][jj] += ld_dsmem_f64(&red[((warp * DB + jj) * RPT + r) * 32 + lane], q);
            }
        }
        cluster_sync();
        if (kr > 0) return;
    }

    // epilogue: one final scaling, as the reference (`out *= scale`)
    const bool vec_ok = ((p.lds & 1) == 0) && ((reinterpret_cast<uintptr_t>(p.S) & 15) == 0);
#pragma unroll
    for (int jj = 0; jj < DB; ++jj) {
        const int j = j0 + warp * DB + jj;
        if (j < p.d) {
            double *col = p.S + (p.col0 + j) * p.lds;
            if (TRANS) {  // lane owns rows lane + 32 r
#pragma unroll
                for (int r = 0; r < RPT; ++r) {
                    const int64_t row = r0 + lane + 32 * r;
                    if (row < p.m_out) col[row] = acc[r][jj] * p.scale;
                }
            } else {      // lane owns rows RPT*lane + r
                const int64_t row = r0 + lane * RPT;
#pragma unroll
                for (int r = 0; r < RPT; r += 2) {
                    if (vec_ok && row + r + 1 < p.m_out) {
                        *reinterpret_cast<double2 *>(col + row + r) =
                            make_double2(acc[r][jj] * p.scale, acc[r + 1][jj] * p.scale);
                    } else {
                        if (row + r < p.m_out) col[row + r] = acc[r][jj] * p.scale;
                        if (row + r + 1 < p.m_out) col[row + r + 1] = acc[r + 1][jj] * p.scale;
                    }
                }
            }
        }
    }
}

template <int RPT, int DB, int NW>
static int launch(ApplyArgs a, const Geom &g, cudaStream_t st) {
    constexpr int TM = 32 * RPT;
    constexpr int SLAB = NW * DB;
    constexpr int PW = 2;  // producer warps (1 active on the TMA path)
    HSK_REQUIRE(g.tm == TM, HSK_EINVAL, "sjlt: plan/config mismatch");
    a.pitch = g.pitch;
    const bool aligned = a.use_tma != 0;  // 16-byte aligned columns (lda even)
    a.mode = a.trans ? 1 : (aligned ? 0 : 2);
    CUtensorMap tmap;
    memset(&tmap, 0, sizeof(tmap));
    if (a.mode == 0) {
        int rc = make_tmap_f64_2d(&tmap, a.A, (uint64_t)a.m_out, (uint64_t)a.n, (uint64_t)a.lda,
                                  TM, (uint32_t)a.tk);
        if (rc) return rc;
    }
    const int a_bytes = (int)roundup((int64_t)a.tk * a.pitch * 8, 128);
    const int bp_bytes = (int)roundup((SLAB + 8) * 2, 128);
    const int en_bytes = (int)roundup(a.estride * 16, 128);
    a.bp_off = a_bytes;
    a.en_off = a_bytes + bp_bytes;
    a.stage_bytes = a_bytes + bp_bytes + en_bytes;
    a.nslabs = (a.d + SLAB - 1) / SLAB;
    const int64_t tiles = (a.m_out + TM - 1) / TM;
    // k-split across a cluster when the tile grid cannot fill the GPU
    int ks = 1;
    const int64_t ctas = tiles * a.nslabs;
    if (ctas < sm_count()) {
        ks = (int)std::min<int64_t>(8, sm_count() / ctas);
        while (ks > 1 && a.nchunks / ks < 8) --ks;
        if (ks == 3 || ks == 5 || ks == 6 || ks == 7) ks = ks >= 4 ? 4 : 2;
    }
    a.ksplit = ks;
    const int per = (int)((a.nchunks + ks - 1) / ks);
    const int budget = 224 * 1024;
    a.stages = std::max(2, std::min(8, (budget - 128) / a.stage_bytes));
    if (per > 0 && a.stages > per) a.stages = std::max(2, per);
    int smem = 128 + a.stages * a.stage_bytes;
    if (ks > 1) smem = std::max(smem, 128 + NW * DB * RPT * 32 * 8);
    auto kern = a.trans ? sjlt_apply_kernel<RPT, DB, NW, PW, true>
                        : sjlt_apply_kernel<RPT, DB, NW, PW, false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return cuda_status(e, "sjlt: set smem attribute");
    const int64_t grid = tiles * a.nslabs * ks;
    HSK_REQUIRE(grid < (1ll << 31), HSK_EINVAL, "sjlt: grid too large");
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid, 1, 1);
    cfg.blockDim = dim3((NW + PW) * 32, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = ks;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, a, tmap);
    if (e != cudaSuccess) return cuda_status(e, "sjlt_apply_kernel launch");
    HSK_CHECK_LAUNCH("sjlt_apply_kernel");
    return HSK_OK;
}

}  // namespace sjlt
}  // namespace hsk

using namespace hsk;

extern "C" int64_t hsk_sjlt_plan_bytes(int64_t n, int32_t d, int32_t alpha) {
    if (n < 0 || d < 1 || alpha < 1 || d > sjlt::kMaxD || alpha > sjlt::kMaxChunkEntries)
        return HSK_EINVAL;
    return sjlt::geom(n, d, alpha).bytes;
}

extern "C" int hsk_sjlt_plan_build(const int32_t *pos, const int8_t *sgn, int64_t n, int32_t d,
                                   int32_t alpha, void *plan, int64_t plan_bytes, void *stream) {
    HSK_REQUIRE(n >= 0 && d >= 1 && alpha >= 1, HSK_EINVAL,
                "sjlt plan: need n >= 0, d >= 1, alpha >= 1 (n=%lld d=%d alpha=%d)",
                (long long)n, d, alpha);
    HSK_REQUIRE(d <= sjlt::kMaxD, HSK_EINVAL, "sjlt plan: d=%d exceeds %lld", d,
                (long long)sjlt::kMaxD);
    HSK_REQUIRE(alpha <= sjlt::kMaxChunkEntries, HSK_EINVAL, "sjlt plan: alpha=%d too large", alpha);
    HSK_REQUIRE(n < (1ll << 31), HSK_EINVAL, "sjlt plan: n too large");
    const sjlt::Geom g = sjlt::geom(n, d, alpha);
    HSK_REQUIRE(plan != nullptr && plan_bytes >= g.bytes, HSK_EINVAL,
                "sjlt plan: buffer of %lld bytes, need %lld", (long long)plan_bytes,
                (long long)g.bytes);
    HSK_REQUIRE(n == 0 || (pos != nullptr && sgn != nullptr), HSK_EINVAL, "sjlt plan: null pattern");
    cudaStream_t st = as_stream(stream);
    unsigned char *base = static_cast<unsigned char *>(plan);
    cudaError_t e = cudaMemsetAsync(base, 0, g.bytes, st);
    if (e != cudaSuccess) return cuda_status(e, "sjlt plan: memset");
    if (n > 0) {
        int p2 = 1;
        while (p2 < g.tk * alpha) p2 <<= 1;
        sjlt::sjlt_plan_kernel<<<(unsigned)g.nchunks, 256, p2 * sizeof(uint32_t), st>>>(
            pos, sgn, n, d, alpha, g.tk, p2, g.bstride, g.estride, g.pitch,
            reinterpret_cast<uint16_t *>(base + g.bptr_off),
            reinterpret_cast<uint4 *>(base + g.ent_off), reinterpret_cast<int *>(base + 28));
        HSK_CHECK_LAUNCH("sjlt_plan_kernel");
    }
    return HSK_OK;
}

extern "C" int hsk_sjlt_apply(const double *A, int64_t rows, int64_t cols, int64_t lda,
                              int32_t trans, const void *plan, int64_t n, int32_t d,
                              int32_t alpha, double scale, double *S, int64_t lds, int64_t col0,
                              void *stream) {
    HSK_REQUIRE(trans == 0 || trans == 1, HSK_EINVAL, "sjlt apply: trans must be 0 or 1");
    HSK_REQUIRE(rows >= 0 && cols >= 0 && lda >= std::max<int64_t>(rows, 1), HSK_EINVAL,
                "sjlt apply: bad A shape rows=%lld cols=%lld lda=%lld", (long long)rows,
                (long long)cols, (long long)lda);
    HSK_REQUIRE(d >= 1 && alpha >= 1 && d <= sjlt::kMaxD && alpha <= sjlt::kMaxChunkEntries,
                HSK_EINVAL, "sjlt apply: bad d=%d alpha=%d", d, alpha);
    const int64_t kdim = trans ? rows : cols;
    const int64_t m_out = trans ? cols : rows;
    if (kdim != n) {
        return set_error(HSK_EINVAL, "operator is over dimension %lld, matrix has %lld %s",
                         (long long)n, (long long)kdim, trans ? "rows" : "columns");
    }
    HSK_REQUIRE(lds >= std::max<int64_t>(m_out, 1) && col0 >= 0, HSK_EINVAL,
                "sjlt apply: bad output lds=%lld col0=%lld", (long long)lds, (long long)col0);
    if (m_out == 0) return HSK_OK;
    HSK_REQUIRE(plan != nullptr && S != nullptr && (A != nullptr || n == 0), HSK_EINVAL,
                "sjlt apply: null pointer");
    HSK_REQUIRE(m_out < (1ll << 31) && n < (1ll << 31), HSK_EINVAL, "sjlt apply: too large");
    const sjlt::Geom g = sjlt::geom(n, d, alpha);
    const unsigned char *base = static_cast<const unsigned char *>(plan);
    sjlt::ApplyArgs a{};
    a.A = A;
    a.lda = lda;
    a.trans = trans;
    a.use_tma = ((reinterpret_cast<uintptr_t>(A) & 15) == 0) && (lda % 2 == 0) && n > 0;
    a.m_out = m_out;
    a.n = n;
    a.d = d;
    a.alpha = alpha;
    a.tk = g.tk;
    a.nchunks = g.nchunks;
    a.bstride = g.bstride;
    a.estride = g.estride;
    a.bptr = reinterpret_cast<const uint16_t *>(base + g.bptr_off);
    a.ent = reinterpret_cast<const uint4 *>(base + g.ent_off);
    a.scale = scale;
    a.S = S;
    a.lds = lds;
    a.col0 = col0;
    cudaStream_t st = as_stream(stream);
    if (d <= 64) return sjlt::launch<4, 4, 16>(a, g, st);
    if (d <= 128) return sjlt::launch<2, 16, 8>(a, g, st);
    return sjlt::launch<2, 16, 16>(a, g, st);
}
