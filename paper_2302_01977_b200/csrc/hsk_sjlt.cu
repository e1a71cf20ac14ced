// hsk_sjlt.cu -- SJLT sketch S = A R^T and S' = A^T R^T on sm_100a.
//
// Replaces SjltBlock._build_storage / apply_right / apply_right_transposed
// (/root/reference/pkg/src/hsskit/sketching.py:292-351; PAPER.md §6).
//
// Design (DESIGN.md §SJLT):
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

// Per-direction sub-plan geometry.  One plan buffer holds a header, the S
// sub-plan (trans 0) and the S' sub-plan (trans 1): the best tile shape can
// differ per direction (measured): 128-row tiles for d <= 64, 64-row tiles
// (256-bucket slabs, TK 128) otherwise, except S with d > 512, which prefers
// 32-row tiles with 512-bucket slabs and TK = 256 (half the slab re-reads).
struct Geom {
    int rpt;           // rows per lane (tile rows tm = 32 * rpt)
    int tm;
    int pitch;         // tile pitch (doubles) = tm: TMA writes densely; the S'
                       // producer orders its transposing stores conflict-free
    int tk;            // input indices per chunk
    int64_t nchunks;
    int64_t bstride;   // uint16 per bucket-offset row
    int64_t estride;   // entries per chunk row (tk*alpha)
    int64_t bptr_off;  // bytes from the plan base
    int64_t ent_off;   // bytes from the plan base
    int64_t end;       // bytes from the plan base (end of this sub-plan)
};

static inline int64_t roundup(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

static inline int stage_bytes_for(int tk, int tm, int alpha) {
    return tk * tm * 8 + tm * 8 + 1152 + (tk * alpha + 1) * 16;
}

// largest power-of-two TK <= cap whose stage fits `per_stage` bytes
static inline int tk_fit(int alpha, int tm, int cap, int per_stage) {
    int tk = cap;
    while (tk > 1 && (tk * alpha > kMaxChunkEntries || stage_bytes_for(tk, tm, alpha) > per_stage))
        tk >>= 1;
    return tk;
}

static Geom geom_dir(int64_t n, int d, int alpha, int trans, int64_t base) {
    Geom g;
    int tk;
    // per-stage budgets: 3 stages (or 2) of the 226 KB ring
    constexpr int kStage3 = (226 * 1024 - 256) / 3, kStage2 = (226 * 1024 - 256) / 2;
    if (d <= 64) {                          // 128-row tiles, three or more stages
        g.rpt = 4;
        tk = tk_fit(alpha, 128, 128, kStage3);
    } else if (trans || d <= 512) {         // 64-row tiles, TK 128, three stages
        g.rpt = 2;
        tk = tk_fit(alpha, 64, 128, kStage3);
    } else {                                // S, d > 512: 32-row tiles (512-bucket slabs), TK 256
        g.rpt = 1;
        tk = tk_fit(alpha, 32, 256, kStage2);
    }
    if (const char *env = getenv(trans ? "HSK_SJLT_TK_T" : "HSK_SJLT_TK")) tk = atoi(env);
    if (const char *env = getenv(trans ? "HSK_SJLT_RPT_T" : "HSK_SJLT_RPT")) g.rpt = atoi(env);
    g.tm = 32 * g.rpt;
    g.pitch = g.tm;
    g.tk = tk;
    g.nchunks = (n + g.tk - 1) / g.tk;
    g.bstride = roundup(d, kPlanSlab) + 8;
    g.estride = (int64_t)g.tk * alpha;
    g.bptr_off = base;
    g.ent_off = roundup(g.bptr_off + (g.nchunks + 1) * g.bstride * 2, 128);
    g.end = g.ent_off + roundup((g.nchunks + 1) * g.estride * 16, 128);
    return g;
}

struct Plan {
    Geom s, t;
    int64_t bytes;
};

static Plan plan_geom(int64_t n, int d, int alpha) {
    Plan pl;
    pl.s = geom_dir(n, d, alpha, 0, kHeaderBytes);
    pl.t = geom_dir(n, d, alpha, 1, pl.s.end);
    pl.bytes = pl.t.end;
    return pl;
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

// ------------------------------------------------------------------ apply
//
// Stage layout in shared memory (per ring slot):
//   [A tile: TK rows of TM doubles][zero row: TM doubles][bucket bounds]
//   [entries: estride + 1 words of 16 B; the last is the null entry]
// The null entry {offset of the zero row, 0, +1.0} lets a warp fold the
// FIRST entry of every bucket in a batch without predication: empty
// buckets read the zero row and add +0.0.
//
// Lane -> tile rows.  S tiles (dense, TMA-written): RPT = 2 -> rows 2l, 2l+1
// (one LDS.128); RPT = 4 -> rows 2l, 2l+1, 64+2l, 64+2l+1 (two LDS.128, each
// a contiguous 512 B).  S' tiles (swizzled, element (kk,row) at
// kk*TM + (row ^ (kk%32))): rows l + 32 r (LDS.64 each, conflict-free).

// Entries [pe, pend) of one bucket (shared byte addresses), one per
// iteration: consecutive DFMAs on an accumulator are a full iteration (two
// shared loads) apart.  `bra.uni`: every lane walks the same list.
// run_*f: the bucket's first entry is passed in registers (prefetched while
// the previous bucket ran), so a bucket's chain starts at its tile load.
// run_s*: S tiles, rows {2l, 2l+1} at [sx + o] (and {64+2l, 64+2l+1} at +512).
// run_t*: S' tiles, rows l + 32 r at st + o + (x ^ lane8) + 256 r.
__device__ __forceinline__ void run_s2(uint32_t &pe, uint32_t pend, uint32_t sx, double &c0, double &c1) {
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 o0, x0, l0, h0, a0;\n\t.reg .f64 u0, v0, g0;\n\tsetp.ge.u32 p, %0, %3;\n\t@p bra.uni DONE;\n\tLOOP:\n\tld.shared.v4.b32 {o0, x0, l0, h0}, [%0];\n\tadd.u32 a0, o0, %4;\n\tld.shared.v2.f64 {u0, v0}, [a0];\n\tmov.b64 g0, {l0, h0};\n\tfma.rn.f64 %1, u0, g0, %1;\n\tfma.rn.f64 %2, v0, g0, %2;\n\tadd.u32 %0, %0, 16;\n\tsetp.lt.u32 p, %0, %3;\n\t@p bra.uni LOOP;\n\tDONE:\n\t}"
                 : "+r"(pe), "+d"(c0), "+d"(c1)
                 : "r"(pend), "r"(sx)
                 : "memory");
}

__device__ __forceinline__ void run_s2f(uint32_t &pe, uint32_t pend, uint32_t sx, uint4 f, double &c0, double &c1) {
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 o0, x0, l0, h0, a0;\n\t.reg .f64 u0, v0, g0;\n\tsetp.ge.u32 p, %0, %3;\n\t@p bra.uni DONE;\n\tadd.u32 a0, %5, %4;\n\tld.shared.v2.f64 {u0, v0}, [a0];\n\tmov.b64 g0, {%7, %8};\n\tfma.rn.f64 %1, u0, g0, %1;\n\tfma.rn.f64 %2, v0, g0, %2;\n\tadd.u32 %0, %0, 16;\n\tsetp.ge.u32 p, %0, %3;\n\t@p bra.uni DONE;\n\tLOOP:\n\tld.shared.v4.b32 {o0, x0, l0, h0}, [%0];\n\tadd.u32 a0, o0, %4;\n\tld.shared.v2.f64 {u0, v0}, [a0];\n\tmov.b64 g0, {l0, h0};\n\tfma.rn.f64 %1, u0, g0, %1;\n\tfma.rn.f64 %2, v0, g0, %2;\n\tadd.u32 %0, %0, 16;\n\tsetp.lt.u32 p, %0, %3;\n\t@p bra.uni LOOP;\n\tDONE:\n\t}"
                 : "+r"(pe), "+d"(c0), "+d"(c1)
                 : "r"(pend), "r"(sx), "r"(f.x), "r"(f.y), "r"(f.z), "r"(f.w)
                 : "memory");
}

__device__ __forceinline__ void run_t2(uint32_t &pe, uint32_t pend, uint32_t st, uint32_t lane8, double &c0, double &c1) {
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 o0, x0, l0, h0, a0;\n\t.reg .f64 u0, v0, g0;\n\tsetp.ge.u32 p, %0, %3;\n\t@p bra.uni DONE;\n\tLOOP:\n\tld.shared.v4.b32 {o0, x0, l0, h0}, [%0];\n\txor.b32 a0, x0, %5;\n\tadd.u32 a0, a0, o0;\n\tadd.u32 a0, a0, %4;\n\tld.shared.f64 u0, [a0];\n\tld.shared.f64 v0, [a0+256];\n\tmov.b64 g0, {l0, h0};\n\tfma.rn.f64 %1, u0, g0, %1;\n\tfma.rn.f64 %2, v0, g0, %2;\n\tadd.u32 %0, %0, 16;\n\tsetp.lt.u32 p, %0, %3;\n\t@p bra.uni LOOP;\n\tDONE:\n\t}"
                 : "+r"(pe), "+d"(c0), "+d"(c1)
                 : "r"(pend), "r"(st), "r"(lane8)
                 : "memory");
}

__device__ __forceinline__ void run_t2f(uint32_t &pe, uint32_t pend, uint32_t st, uint32_t lane8, uint4 f, double &c0, double &c1) {
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 o0, x0, l0, h0, a0;\n\t.reg .f64 u0, v0, g0;\n\tsetp.ge.u32 p, %0, %3;\n\t@p bra.uni DONE;\n\txor.b32 a0, %7, %5;\n\tadd.u32 a0, a0, %6;\n\tadd.u32 a0, a0, %4;\n\tld.shared.f64 u0, [a0];\n\tld.shared.f64 v0, [a0+256];\n\tmov.b64 g0, {%8, %9};\n\tfma.rn.f64 %1, u0, g0, %1;\n\tfma.rn.f64 %2, v0, g0, %2;\n\tadd.u32 %0, %0, 16;\n\tsetp.ge.u32 p, %0, %3;\n\t@p bra.uni DONE;\n\tLOOP:\n\tld.shared.v4.b32 {o0, x0, l0, h0}, [%0];\n\txor.b32 a0, x0, %5;\n\tadd.u32 a0, a0, o0;\n\tadd.u32 a0, a0, %4;\n\tld.shared.f64 u0, [a0];\n\tld.shared.f64 v0, [a0+256];\n\tmov.b64 g0, {l0, h0};\n\tfma.rn.f64 %1, u0, g0, %1;\n\tfma.rn.f64 %2, v0, g0, %2;\n\tadd.u32 %0, %0, 16;\n\tsetp.lt.u32 p, %0, %3;\n\t@p bra.uni LOOP;\n\tDONE:\n\t}"
                 : "+r"(pe), "+d"(c0), "+d"(c1)
                 : "r"(pend), "r"(st), "r"(lane8), "r"(f.x), "r"(f.y), "r"(f.z), "r"(f.w)
                 : "memory");
}

__device__ __forceinline__ void run_s4(uint32_t &pe, uint32_t pend, uint32_t sx, double &c0, double &c1, double &c2, double &c3) {
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 o0, x0, l0, h0, a0;\n\t.reg .f64 u0, v0, w0, y0, g0;\n\tsetp.ge.u32 p, %0, %5;\n\t@p bra.uni DONE;\n\tLOOP:\n\tld.shared.v4.b32 {o0, x0, l0, h0}, [%0];\n\tadd.u32 a0, o0, %6;\n\tld.shared.v2.f64 {u0, v0}, [a0];\n\tld.shared.v2.f64 {w0, y0}, [a0+512];\n\tmov.b64 g0, {l0, h0};\n\tfma.rn.f64 %1, u0, g0, %1;\n\tfma.rn.f64 %2, v0, g0, %2;\n\tfma.rn.f64 %3, w0, g0, %3;\n\tfma.rn.f64 %4, y0, g0, %4;\n\tadd.u32 %0, %0, 16;\n\tsetp.lt.u32 p, %0, %5;\n\t@p bra.uni LOOP;\n\tDONE:\n\t}"
                 : "+r"(pe), "+d"(c0), "+d"(c1), "+d"(c2), "+d"(c3)
                 : "r"(pend), "r"(sx)
                 : "memory");
}

__device__ __forceinline__ void run_s4f(uint32_t &pe, uint32_t pend, uint32_t sx, uint4 f, double &c0, double &c1, double &c2, double &c3) {
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 o0, x0, l0, h0, a0;\n\t.reg .f64 u0, v0, w0, y0, g0;\n\tsetp.ge.u32 p, %0, %5;\n\t@p bra.uni DONE;\n\tadd.u32 a0, %7, %6;\n\tld.shared.v2.f64 {u0, v0}, [a0];\n\tld.shared.v2.f64 {w0, y0}, [a0+512];\n\tmov.b64 g0, {%9, %10};\n\tfma.rn.f64 %1, u0, g0, %1;\n\tfma.rn.f64 %2, v0, g0, %2;\n\tfma.rn.f64 %3, w0, g0, %3;\n\tfma.rn.f64 %4, y0, g0, %4;\n\tadd.u32 %0, %0, 16;\n\tsetp.ge.u32 p, %0, %5;\n\t@p bra.uni DONE;\n\tLOOP:\n\tld.shared.v4.b32 {o0, x0, l0, h0}, [%0];\n\tadd.u32 a0, o0, %6;\n\tld.shared.v2.f64 {u0, v0}, [a0];\n\tld.shared.v2.f64 {w0, y0}, [a0+512];\n\tmov.b64 g0, {l0, h0};\n\tfma.rn.f64 %1, u0, g0, %1;\n\tfma.rn.f64 %2, v0, g0, %2;\n\tfma.rn.f64 %3, w0, g0, %3;\n\tfma.rn.f64 %4, y0, g0, %4;\n\tadd.u32 %0, %0, 16;\n\tsetp.lt.u32 p, %0, %5;\n\t@p bra.uni LOOP;\n\tDONE:\n\t}"
                 : "+r"(pe), "+d"(c0), "+d"(c1), "+d"(c2), "+d"(c3)
                 : "r"(pend), "r"(sx), "r"(f.x), "r"(f.y), "r"(f.z), "r"(f.w)
                 : "memory");
}

__device__ __forceinline__ void run_t4(uint32_t &pe, uint32_t pend, uint32_t st, uint32_t lane8, double &c0, double &c1, double &c2, double &c3) {
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 o0, x0, l0, h0, a0;\n\t.reg .f64 u0, v0, w0, y0, g0;\n\tsetp.ge.u32 p, %0, %5;\n\t@p bra.uni DONE;\n\tLOOP:\n\tld.shared.v4.b32 {o0, x0, l0, h0}, [%0];\n\txor.b32 a0, x0, %7;\n\tadd.u32 a0, a0, o0;\n\tadd.u32 a0, a0, %6;\n\tld.shared.f64 u0, [a0];\n\tld.shared.f64 v0, [a0+256];\n\tld.shared.f64 w0, [a0+512];\n\tld.shared.f64 y0, [a0+768];\n\tmov.b64 g0, {l0, h0};\n\tfma.rn.f64 %1, u0, g0, %1;\n\tfma.rn.f64 %2, v0, g0, %2;\n\tfma.rn.f64 %3, w0, g0, %3;\n\tfma.rn.f64 %4, y0, g0, %4;\n\tadd.u32 %0, %0, 16;\n\tsetp.lt.u32 p, %0, %5;\n\t@p bra.uni LOOP;\n\tDONE:\n\t}"
                 : "+r"(pe), "+d"(c0), "+d"(c1), "+d"(c2), "+d"(c3)
                 : "r"(pend), "r"(st), "r"(lane8)
                 : "memory");
}

__device__ __forceinline__ void run_t4f(uint32_t &pe, uint32_t pend, uint32_t st, uint32_t lane8, uint4 f, double &c0, double &c1, double &c2, double &c3) {
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 o0, x0, l0, h0, a0;\n\t.reg .f64 u0, v0, w0, y0, g0;\n\tsetp.ge.u32 p, %0, %5;\n\t@p bra.uni DONE;\n\txor.b32 a0, %9, %7;\n\tadd.u32 a0, a0, %8;\n\tadd.u32 a0, a0, %6;\n\tld.shared.f64 u0, [a0];\n\tld.shared.f64 v0, [a0+256];\n\tld.shared.f64 w0, [a0+512];\n\tld.shared.f64 y0, [a0+768];\n\tmov.b64 g0, {%10, %11};\n\tfma.rn.f64 %1, u0, g0, %1;\n\tfma.rn.f64 %2, v0, g0, %2;\n\tfma.rn.f64 %3, w0, g0, %3;\n\tfma.rn.f64 %4, y0, g0, %4;\n\tadd.u32 %0, %0, 16;\n\tsetp.ge.u32 p, %0, %5;\n\t@p bra.uni DONE;\n\tLOOP:\n\tld.shared.v4.b32 {o0, x0, l0, h0}, [%0];\n\txor.b32 a0, x0, %7;\n\tadd.u32 a0, a0, o0;\n\tadd.u32 a0, a0, %6;\n\tld.shared.f64 u0, [a0];\n\tld.shared.f64 v0, [a0+256];\n\tld.shared.f64 w0, [a0+512];\n\tld.shared.f64 y0, [a0+768];\n\tmov.b64 g0, {l0, h0};\n\tfma.rn.f64 %1, u0, g0, %1;\n\tfma.rn.f64 %2, v0, g0, %2;\n\tfma.rn.f64 %3, w0, g0, %3;\n\tfma.rn.f64 %4, y0, g0, %4;\n\tadd.u32 %0, %0, 16;\n\tsetp.lt.u32 p, %0, %5;\n\t@p bra.uni LOOP;\n\tDONE:\n\t}"
                 : "+r"(pe), "+d"(c0), "+d"(c1), "+d"(c2), "+d"(c3)
                 : "r"(pend), "r"(st), "r"(lane8), "r"(f.x), "r"(f.y), "r"(f.z), "r"(f.w)
                 : "memory");
}

// Whole-chunk consumers: one PTX block walks all DB buckets of the warp
// (bounds unpacked in-line, uniform branches, no convergence barriers
// between buckets): ~4 instructions per empty bucket, 8 per entry.
// one warp, one chunk, all 8 buckets, RPT = 2 (S tiles)
__device__ __forceinline__ void chunk_s_2x8(double (&acc)[2][8], uint32_t sen, uint32_t sx, const uint32_t (&bw)[5]) {
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 o, x, gl, gh, a, t, pe, pend;\n\t.reg .f64 u, v, w, y, g;\n\tand.b32 t, %18, 65535;\n\tmad.lo.u32 pe, t, 16, %16;\n\tshr.u32 t, %18, 16;\n\tmad.lo.u32 pend, t, 16, %16;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B0_DONE;\n\tB0_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %17;\n\tld.shared.v2.f64 {u, v}, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %0, u, g, %0;\n\tfma.rn.f64 %1, v, g, %1;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B0_LOOP;\n\tB0_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %19, 65535;\n\tmad.lo.u32 pend, t, 16, %16;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B1_DONE;\n\tB1_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %17;\n\tld.shared.v2.f64 {u, v}, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %2, u, g, %2;\n\tfma.rn.f64 %3, v, g, %3;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B1_LOOP;\n\tB1_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %19, 16;\n\tmad.lo.u32 pend, t, 16, %16;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B2_DONE;\n\tB2_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %17;\n\tld.shared.v2.f64 {u, v}, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %4, u, g, %4;\n\tfma.rn.f64 %5, v, g, %5;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B2_LOOP;\n\tB2_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %20, 65535;\n\tmad.lo.u32 pend, t, 16, %16;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B3_DONE;\n\tB3_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %17;\n\tld.shared.v2.f64 {u, v}, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %6, u, g, %6;\n\tfma.rn.f64 %7, v, g, %7;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B3_LOOP;\n\tB3_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %20, 16;\n\tmad.lo.u32 pend, t, 16, %16;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B4_DONE;\n\tB4_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %17;\n\tld.shared.v2.f64 {u, v}, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %8, u, g, %8;\n\tfma.rn.f64 %9, v, g, %9;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B4_LOOP;\n\tB4_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %21, 65535;\n\tmad.lo.u32 pend, t, 16, %16;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B5_DONE;\n\tB5_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %17;\n\tld.shared.v2.f64 {u, v}, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %10, u, g, %10;\n\tfma.rn.f64 %11, v, g, %11;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B5_LOOP;\n\tB5_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %21, 16;\n\tmad.lo.u32 pend, t, 16, %16;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B6_DONE;\n\tB6_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %17;\n\tld.shared.v2.f64 {u, v}, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %12, u, g, %12;\n\tfma.rn.f64 %13, v, g, %13;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B6_LOOP;\n\tB6_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %22, 65535;\n\tmad.lo.u32 pend, t, 16, %16;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B7_DONE;\n\tB7_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %17;\n\tld.shared.v2.f64 {u, v}, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %14, u, g, %14;\n\tfma.rn.f64 %15, v, g, %15;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B7_LOOP;\n\tB7_DONE:\n\tmov.b32 pe, pend;\n\t}"
                 : "+d"(acc[0][0]), "+d"(acc[1][0]), "+d"(acc[0][1]), "+d"(acc[1][1]), "+d"(acc[0][2]), "+d"(acc[1][2]), "+d"(acc[0][3]), "+d"(acc[1][3]), "+d"(acc[0][4]), "+d"(acc[1][4]), "+d"(acc[0][5]), "+d"(acc[1][5]), "+d"(acc[0][6]), "+d"(acc[1][6]), "+d"(acc[0][7]), "+d"(acc[1][7])
                 : "r"(sen), "r"(sx), "r"(bw[0]), "r"(bw[1]), "r"(bw[2]), "r"(bw[3]), "r"(bw[4])
                 : "memory");
}

// one warp, one chunk, all 4 buckets, RPT = 2 (S tiles)
__device__ __forceinline__ void chunk_s_2x4(double (&acc)[2][4], uint32_t sen, uint32_t sx, const uint32_t (&bw)[3]) {
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 o, x, gl, gh, a, t, pe, pend;\n\t.reg .f64 u, v, w, y, g;\n\tand.b32 t, %10, 65535;\n\tmad.lo.u32 pe, t, 16, %8;\n\tshr.u32 t, %10, 16;\n\tmad.lo.u32 pend, t, 16, %8;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B0_DONE;\n\tB0_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %9;\n\tld.shared.v2.f64 {u, v}, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %0, u, g, %0;\n\tfma.rn.f64 %1, v, g, %1;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B0_LOOP;\n\tB0_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %11, 65535;\n\tmad.lo.u32 pend, t, 16, %8;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B1_DONE;\n\tB1_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %9;\n\tld.shared.v2.f64 {u, v}, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %2, u, g, %2;\n\tfma.rn.f64 %3, v, g, %3;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B1_LOOP;\n\tB1_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %11, 16;\n\tmad.lo.u32 pend, t, 16, %8;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B2_DONE;\n\tB2_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %9;\n\tld.shared.v2.f64 {u, v}, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %4, u, g, %4;\n\tfma.rn.f64 %5, v, g, %5;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B2_LOOP;\n\tB2_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %12, 65535;\n\tmad.lo.u32 pend, t, 16, %8;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B3_DONE;\n\tB3_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %9;\n\tld.shared.v2.f64 {u, v}, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %6, u, g, %6;\n\tfma.rn.f64 %7, v, g, %7;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B3_LOOP;\n\tB3_DONE:\n\tmov.b32 pe, pend;\n\t}"
                 : "+d"(acc[0][0]), "+d"(acc[1][0]), "+d"(acc[0][1]), "+d"(acc[1][1]), "+d"(acc[0][2]), "+d"(acc[1][2]), "+d"(acc[0][3]), "+d"(acc[1][3])
                 : "r"(sen), "r"(sx), "r"(bw[0]), "r"(bw[1]), "r"(bw[2])
                 : "memory");
}

// one warp, one chunk, all 2 buckets, RPT = 4 (S tiles)
__device__ __forceinline__ void chunk_s_4x2(double (&acc)[4][2], uint32_t sen, uint32_t sx, const uint32_t (&bw)[2]) {
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 o, x, gl, gh, a, t, pe, pend;\n\t.reg .f64 u, v, w, y, g;\n\tand.b32 t, %10, 65535;\n\tmad.lo.u32 pe, t, 16, %8;\n\tshr.u32 t, %10, 16;\n\tmad.lo.u32 pend, t, 16, %8;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B0_DONE;\n\tB0_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %9;\n\tld.shared.v2.f64 {u, v}, [a];\n\tld.shared.v2.f64 {w, y}, [a+512];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %0, u, g, %0;\n\tfma.rn.f64 %1, v, g, %1;\n\tfma.rn.f64 %2, w, g, %2;\n\tfma.rn.f64 %3, y, g, %3;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B0_LOOP;\n\tB0_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %11, 65535;\n\tmad.lo.u32 pend, t, 16, %8;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B1_DONE;\n\tB1_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %9;\n\tld.shared.v2.f64 {u, v}, [a];\n\tld.shared.v2.f64 {w, y}, [a+512];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %4, u, g, %4;\n\tfma.rn.f64 %5, v, g, %5;\n\tfma.rn.f64 %6, w, g, %6;\n\tfma.rn.f64 %7, y, g, %7;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B1_LOOP;\n\tB1_DONE:\n\tmov.b32 pe, pend;\n\t}"
                 : "+d"(acc[0][0]), "+d"(acc[1][0]), "+d"(acc[2][0]), "+d"(acc[3][0]), "+d"(acc[0][1]), "+d"(acc[1][1]), "+d"(acc[2][1]), "+d"(acc[3][1])
                 : "r"(sen), "r"(sx), "r"(bw[0]), "r"(bw[1])
                 : "memory");
}

// one warp, one chunk, all 4 buckets, RPT = 4 (S tiles)
__device__ __forceinline__ void chunk_s_4x4(double (&acc)[4][4], uint32_t sen, uint32_t sx, const uint32_t (&bw)[3]) {
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 o, x, gl, gh, a, t, pe, pend;\n\t.reg .f64 u, v, w, y, g;\n\tand.b32 t, %18, 65535;\n\tmad.lo.u32 pe, t, 16, %16;\n\tshr.u32 t, %18, 16;\n\tmad.lo.u32 pend, t, 16, %16;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B0_DONE;\n\tB0_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %17;\n\tld.shared.v2.f64 {u, v}, [a];\n\tld.shared.v2.f64 {w, y}, [a+512];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %0, u, g, %0;\n\tfma.rn.f64 %1, v, g, %1;\n\tfma.rn.f64 %2, w, g, %2;\n\tfma.rn.f64 %3, y, g, %3;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B0_LOOP;\n\tB0_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %19, 65535;\n\tmad.lo.u32 pend, t, 16, %16;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B1_DONE;\n\tB1_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %17;\n\tld.shared.v2.f64 {u, v}, [a];\n\tld.shared.v2.f64 {w, y}, [a+512];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %4, u, g, %4;\n\tfma.rn.f64 %5, v, g, %5;\n\tfma.rn.f64 %6, w, g, %6;\n\tfma.rn.f64 %7, y, g, %7;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B1_LOOP;\n\tB1_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %19, 16;\n\tmad.lo.u32 pend, t, 16, %16;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B2_DONE;\n\tB2_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %17;\n\tld.shared.v2.f64 {u, v}, [a];\n\tld.shared.v2.f64 {w, y}, [a+512];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %8, u, g, %8;\n\tfma.rn.f64 %9, v, g, %9;\n\tfma.rn.f64 %10, w, g, %10;\n\tfma.rn.f64 %11, y, g, %11;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B2_LOOP;\n\tB2_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %20, 65535;\n\tmad.lo.u32 pend, t, 16, %16;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B3_DONE;\n\tB3_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %17;\n\tld.shared.v2.f64 {u, v}, [a];\n\tld.shared.v2.f64 {w, y}, [a+512];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %12, u, g, %12;\n\tfma.rn.f64 %13, v, g, %13;\n\tfma.rn.f64 %14, w, g, %14;\n\tfma.rn.f64 %15, y, g, %15;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B3_LOOP;\n\tB3_DONE:\n\tmov.b32 pe, pend;\n\t}"
                 : "+d"(acc[0][0]), "+d"(acc[1][0]), "+d"(acc[2][0]), "+d"(acc[3][0]), "+d"(acc[0][1]), "+d"(acc[1][1]), "+d"(acc[2][1]), "+d"(acc[3][1]), "+d"(acc[0][2]), "+d"(acc[1][2]), "+d"(acc[2][2]), "+d"(acc[3][2]), "+d"(acc[0][3]), "+d"(acc[1][3]), "+d"(acc[2][3]), "+d"(acc[3][3])
                 : "r"(sen), "r"(sx), "r"(bw[0]), "r"(bw[1]), "r"(bw[2])
                 : "memory");
}

// one warp, one chunk, all 16 buckets, RPT = 2 (S tiles)
__device__ __forceinline__ void chunk_s_2x16(double (&acc)[2][16], uint32_t sen, uint32_t sx, const uint32_t (&bw)[9]) {
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 o, x, gl, gh, a, t, pe, pend;\n\t.reg .f64 u, v, w, y, g;\n\tand.b32 t, %34, 65535;\n\tmad.lo.u32 pe, t, 16, %32;\n\tshr.u32 t, %34, 16;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B0_DONE;\n\tB0_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.v2.f64 {u, v}, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %0, u, g, %0;\n\tfma.rn.f64 %1, v, g, %1;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B0_LOOP;\n\tB0_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %35, 65535;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B1_DONE;\n\tB1_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.v2.f64 {u, v}, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %2, u, g, %2;\n\tfma.rn.f64 %3, v, g, %3;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B1_LOOP;\n\tB1_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %35, 16;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B2_DONE;\n\tB2_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.v2.f64 {u, v}, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %4, u, g, %4;\n\tfma.rn.f64 %5, v, g, %5;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B2_LOOP;\n\tB2_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %36, 65535;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B3_DONE;\n\tB3_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.v2.f64 {u, v}, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %6, u, g, %6;\n\tfma.rn.f64 %7, v, g, %7;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B3_LOOP;\n\tB3_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %36, 16;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B4_DONE;\n\tB4_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.v2.f64 {u, v}, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %8, u, g, %8;\n\tfma.rn.f64 %9, v, g, %9;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B4_LOOP;\n\tB4_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %37, 65535;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B5_DONE;\n\tB5_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.v2.f64 {u, v}, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %10, u, g, %10;\n\tfma.rn.f64 %11, v, g, %11;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B5_LOOP;\n\tB5_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %37, 16;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B6_DONE;\n\tB6_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.v2.f64 {u, v}, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %12, u, g, %12;\n\tfma.rn.f64 %13, v, g, %13;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B6_LOOP;\n\tB6_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %38, 65535;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B7_DONE;\n\tB7_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.v2.f64 {u, v}, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %14, u, g, %14;\n\tfma.rn.f64 %15, v, g, %15;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B7_LOOP;\n\tB7_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %38, 16;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B8_DONE;\n\tB8_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.v2.f64 {u, v}, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %16, u, g, %16;\n\tfma.rn.f64 %17, v, g, %17;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B8_LOOP;\n\tB8_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %39, 65535;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B9_DONE;\n\tB9_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.v2.f64 {u, v}, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %18, u, g, %18;\n\tfma.rn.f64 %19, v, g, %19;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B9_LOOP;\n\tB9_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %39, 16;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B10_DONE;\n\tB10_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.v2.f64 {u, v}, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %20, u, g, %20;\n\tfma.rn.f64 %21, v, g, %21;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B10_LOOP;\n\tB10_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %40, 65535;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B11_DONE;\n\tB11_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.v2.f64 {u, v}, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %22, u, g, %22;\n\tfma.rn.f64 %23, v, g, %23;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B11_LOOP;\n\tB11_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %40, 16;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B12_DONE;\n\tB12_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.v2.f64 {u, v}, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %24, u, g, %24;\n\tfma.rn.f64 %25, v, g, %25;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B12_LOOP;\n\tB12_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %41, 65535;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B13_DONE;\n\tB13_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.v2.f64 {u, v}, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %26, u, g, %26;\n\tfma.rn.f64 %27, v, g, %27;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B13_LOOP;\n\tB13_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %41, 16;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B14_DONE;\n\tB14_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.v2.f64 {u, v}, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %28, u, g, %28;\n\tfma.rn.f64 %29, v, g, %29;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B14_LOOP;\n\tB14_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %42, 65535;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B15_DONE;\n\tB15_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.v2.f64 {u, v}, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %30, u, g, %30;\n\tfma.rn.f64 %31, v, g, %31;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B15_LOOP;\n\tB15_DONE:\n\tmov.b32 pe, pend;\n\t}"
                 : "+d"(acc[0][0]), "+d"(acc[1][0]), "+d"(acc[0][1]), "+d"(acc[1][1]), "+d"(acc[0][2]), "+d"(acc[1][2]), "+d"(acc[0][3]), "+d"(acc[1][3]), "+d"(acc[0][4]), "+d"(acc[1][4]), "+d"(acc[0][5]), "+d"(acc[1][5]), "+d"(acc[0][6]), "+d"(acc[1][6]), "+d"(acc[0][7]), "+d"(acc[1][7]), "+d"(acc[0][8]), "+d"(acc[1][8]), "+d"(acc[0][9]), "+d"(acc[1][9]), "+d"(acc[0][10]), "+d"(acc[1][10]), "+d"(acc[0][11]), "+d"(acc[1][11]), "+d"(acc[0][12]), "+d"(acc[1][12]), "+d"(acc[0][13]), "+d"(acc[1][13]), "+d"(acc[0][14]), "+d"(acc[1][14]), "+d"(acc[0][15]), "+d"(acc[1][15])
                 : "r"(sen), "r"(sx), "r"(bw[0]), "r"(bw[1]), "r"(bw[2]), "r"(bw[3]), "r"(bw[4]), "r"(bw[5]), "r"(bw[6]), "r"(bw[7]), "r"(bw[8])
                 : "memory");
}

// one warp, one chunk, all 8 buckets, RPT = 4 (S tiles)
__device__ __forceinline__ void chunk_s_4x8(double (&acc)[4][8], uint32_t sen, uint32_t sx, const uint32_t (&bw)[5]) {
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 o, x, gl, gh, a, t, pe, pend;\n\t.reg .f64 u, v, w, y, g;\n\tand.b32 t, %34, 65535;\n\tmad.lo.u32 pe, t, 16, %32;\n\tshr.u32 t, %34, 16;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B0_DONE;\n\tB0_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.v2.f64 {u, v}, [a];\n\tld.shared.v2.f64 {w, y}, [a+512];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %0, u, g, %0;\n\tfma.rn.f64 %1, v, g, %1;\n\tfma.rn.f64 %2, w, g, %2;\n\tfma.rn.f64 %3, y, g, %3;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B0_LOOP;\n\tB0_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %35, 65535;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B1_DONE;\n\tB1_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.v2.f64 {u, v}, [a];\n\tld.shared.v2.f64 {w, y}, [a+512];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %4, u, g, %4;\n\tfma.rn.f64 %5, v, g, %5;\n\tfma.rn.f64 %6, w, g, %6;\n\tfma.rn.f64 %7, y, g, %7;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B1_LOOP;\n\tB1_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %35, 16;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B2_DONE;\n\tB2_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.v2.f64 {u, v}, [a];\n\tld.shared.v2.f64 {w, y}, [a+512];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %8, u, g, %8;\n\tfma.rn.f64 %9, v, g, %9;\n\tfma.rn.f64 %10, w, g, %10;\n\tfma.rn.f64 %11, y, g, %11;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B2_LOOP;\n\tB2_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %36, 65535;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B3_DONE;\n\tB3_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.v2.f64 {u, v}, [a];\n\tld.shared.v2.f64 {w, y}, [a+512];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %12, u, g, %12;\n\tfma.rn.f64 %13, v, g, %13;\n\tfma.rn.f64 %14, w, g, %14;\n\tfma.rn.f64 %15, y, g, %15;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B3_LOOP;\n\tB3_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %36, 16;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B4_DONE;\n\tB4_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.v2.f64 {u, v}, [a];\n\tld.shared.v2.f64 {w, y}, [a+512];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %16, u, g, %16;\n\tfma.rn.f64 %17, v, g, %17;\n\tfma.rn.f64 %18, w, g, %18;\n\tfma.rn.f64 %19, y, g, %19;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B4_LOOP;\n\tB4_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %37, 65535;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B5_DONE;\n\tB5_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.v2.f64 {u, v}, [a];\n\tld.shared.v2.f64 {w, y}, [a+512];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %20, u, g, %20;\n\tfma.rn.f64 %21, v, g, %21;\n\tfma.rn.f64 %22, w, g, %22;\n\tfma.rn.f64 %23, y, g, %23;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B5_LOOP;\n\tB5_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %37, 16;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B6_DONE;\n\tB6_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.v2.f64 {u, v}, [a];\n\tld.shared.v2.f64 {w, y}, [a+512];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %24, u, g, %24;\n\tfma.rn.f64 %25, v, g, %25;\n\tfma.rn.f64 %26, w, g, %26;\n\tfma.rn.f64 %27, y, g, %27;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B6_LOOP;\n\tB6_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %38, 65535;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B7_DONE;\n\tB7_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.v2.f64 {u, v}, [a];\n\tld.shared.v2.f64 {w, y}, [a+512];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %28, u, g, %28;\n\tfma.rn.f64 %29, v, g, %29;\n\tfma.rn.f64 %30, w, g, %30;\n\tfma.rn.f64 %31, y, g, %31;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B7_LOOP;\n\tB7_DONE:\n\tmov.b32 pe, pend;\n\t}"
                 : "+d"(acc[0][0]), "+d"(acc[1][0]), "+d"(acc[2][0]), "+d"(acc[3][0]), "+d"(acc[0][1]), "+d"(acc[1][1]), "+d"(acc[2][1]), "+d"(acc[3][1]), "+d"(acc[0][2]), "+d"(acc[1][2]), "+d"(acc[2][2]), "+d"(acc[3][2]), "+d"(acc[0][3]), "+d"(acc[1][3]), "+d"(acc[2][3]), "+d"(acc[3][3]), "+d"(acc[0][4]), "+d"(acc[1][4]), "+d"(acc[2][4]), "+d"(acc[3][4]), "+d"(acc[0][5]), "+d"(acc[1][5]), "+d"(acc[2][5]), "+d"(acc[3][5]), "+d"(acc[0][6]), "+d"(acc[1][6]), "+d"(acc[2][6]), "+d"(acc[3][6]), "+d"(acc[0][7]), "+d"(acc[1][7]), "+d"(acc[2][7]), "+d"(acc[3][7])
                 : "r"(sen), "r"(sx), "r"(bw[0]), "r"(bw[1]), "r"(bw[2]), "r"(bw[3]), "r"(bw[4])
                 : "memory");
}

// RPT = 1 variants (32-row tiles): lane l owns row l.
__device__ __forceinline__ void chunk_s_1x16(double (&acc)[1][16], uint32_t sen, uint32_t sx, const uint32_t (&bw)[9]) {
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 o, x, gl, gh, a, t, pe, pend;\n\t.reg .f64 u, g;\n\tand.b32 t, %18, 65535;\n\tmad.lo.u32 pe, t, 16, %16;\n\tshr.u32 t, %18, 16;\n\tmad.lo.u32 pend, t, 16, %16;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B0_DONE;\n\tB0_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %17;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %0, u, g, %0;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B0_LOOP;\n\tB0_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %19, 65535;\n\tmad.lo.u32 pend, t, 16, %16;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B1_DONE;\n\tB1_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %17;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %1, u, g, %1;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B1_LOOP;\n\tB1_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %19, 16;\n\tmad.lo.u32 pend, t, 16, %16;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B2_DONE;\n\tB2_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %17;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %2, u, g, %2;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B2_LOOP;\n\tB2_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %20, 65535;\n\tmad.lo.u32 pend, t, 16, %16;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B3_DONE;\n\tB3_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %17;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %3, u, g, %3;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B3_LOOP;\n\tB3_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %20, 16;\n\tmad.lo.u32 pend, t, 16, %16;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B4_DONE;\n\tB4_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %17;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %4, u, g, %4;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B4_LOOP;\n\tB4_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %21, 65535;\n\tmad.lo.u32 pend, t, 16, %16;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B5_DONE;\n\tB5_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %17;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %5, u, g, %5;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B5_LOOP;\n\tB5_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %21, 16;\n\tmad.lo.u32 pend, t, 16, %16;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B6_DONE;\n\tB6_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %17;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %6, u, g, %6;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B6_LOOP;\n\tB6_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %22, 65535;\n\tmad.lo.u32 pend, t, 16, %16;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B7_DONE;\n\tB7_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %17;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %7, u, g, %7;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B7_LOOP;\n\tB7_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %22, 16;\n\tmad.lo.u32 pend, t, 16, %16;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B8_DONE;\n\tB8_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %17;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %8, u, g, %8;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B8_LOOP;\n\tB8_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %23, 65535;\n\tmad.lo.u32 pend, t, 16, %16;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B9_DONE;\n\tB9_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %17;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %9, u, g, %9;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B9_LOOP;\n\tB9_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %23, 16;\n\tmad.lo.u32 pend, t, 16, %16;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B10_DONE;\n\tB10_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %17;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %10, u, g, %10;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B10_LOOP;\n\tB10_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %24, 65535;\n\tmad.lo.u32 pend, t, 16, %16;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B11_DONE;\n\tB11_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %17;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %11, u, g, %11;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B11_LOOP;\n\tB11_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %24, 16;\n\tmad.lo.u32 pend, t, 16, %16;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B12_DONE;\n\tB12_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %17;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %12, u, g, %12;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B12_LOOP;\n\tB12_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %25, 65535;\n\tmad.lo.u32 pend, t, 16, %16;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B13_DONE;\n\tB13_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %17;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %13, u, g, %13;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B13_LOOP;\n\tB13_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %25, 16;\n\tmad.lo.u32 pend, t, 16, %16;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B14_DONE;\n\tB14_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %17;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %14, u, g, %14;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B14_LOOP;\n\tB14_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %26, 65535;\n\tmad.lo.u32 pend, t, 16, %16;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B15_DONE;\n\tB15_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %17;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %15, u, g, %15;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B15_LOOP;\n\tB15_DONE:\n\tmov.b32 pe, pend;\n\t}"
                 : "+d"(acc[0][0]), "+d"(acc[0][1]), "+d"(acc[0][2]), "+d"(acc[0][3]), "+d"(acc[0][4]), "+d"(acc[0][5]), "+d"(acc[0][6]), "+d"(acc[0][7]), "+d"(acc[0][8]), "+d"(acc[0][9]), "+d"(acc[0][10]), "+d"(acc[0][11]), "+d"(acc[0][12]), "+d"(acc[0][13]), "+d"(acc[0][14]), "+d"(acc[0][15])
                 : "r"(sen), "r"(sx), "r"(bw[0]), "r"(bw[1]), "r"(bw[2]), "r"(bw[3]), "r"(bw[4]), "r"(bw[5]), "r"(bw[6]), "r"(bw[7]), "r"(bw[8])
                 : "memory");
}
__device__ __forceinline__ void chunk_s_1x32(double (&acc)[1][32], uint32_t sen, uint32_t sx, const uint32_t (&bw)[17]) {
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 o, x, gl, gh, a, t, pe, pend;\n\t.reg .f64 u, g;\n\tand.b32 t, %34, 65535;\n\tmad.lo.u32 pe, t, 16, %32;\n\tshr.u32 t, %34, 16;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B0_DONE;\n\tB0_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %0, u, g, %0;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B0_LOOP;\n\tB0_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %35, 65535;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B1_DONE;\n\tB1_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %1, u, g, %1;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B1_LOOP;\n\tB1_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %35, 16;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B2_DONE;\n\tB2_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %2, u, g, %2;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B2_LOOP;\n\tB2_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %36, 65535;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B3_DONE;\n\tB3_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %3, u, g, %3;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B3_LOOP;\n\tB3_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %36, 16;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B4_DONE;\n\tB4_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %4, u, g, %4;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B4_LOOP;\n\tB4_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %37, 65535;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B5_DONE;\n\tB5_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %5, u, g, %5;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B5_LOOP;\n\tB5_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %37, 16;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B6_DONE;\n\tB6_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %6, u, g, %6;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B6_LOOP;\n\tB6_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %38, 65535;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B7_DONE;\n\tB7_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %7, u, g, %7;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B7_LOOP;\n\tB7_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %38, 16;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B8_DONE;\n\tB8_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %8, u, g, %8;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B8_LOOP;\n\tB8_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %39, 65535;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B9_DONE;\n\tB9_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %9, u, g, %9;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B9_LOOP;\n\tB9_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %39, 16;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B10_DONE;\n\tB10_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %10, u, g, %10;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B10_LOOP;\n\tB10_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %40, 65535;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B11_DONE;\n\tB11_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %11, u, g, %11;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B11_LOOP;\n\tB11_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %40, 16;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B12_DONE;\n\tB12_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %12, u, g, %12;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B12_LOOP;\n\tB12_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %41, 65535;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B13_DONE;\n\tB13_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %13, u, g, %13;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B13_LOOP;\n\tB13_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %41, 16;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B14_DONE;\n\tB14_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %14, u, g, %14;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B14_LOOP;\n\tB14_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %42, 65535;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B15_DONE;\n\tB15_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %15, u, g, %15;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B15_LOOP;\n\tB15_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %42, 16;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B16_DONE;\n\tB16_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %16, u, g, %16;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B16_LOOP;\n\tB16_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %43, 65535;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B17_DONE;\n\tB17_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %17, u, g, %17;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B17_LOOP;\n\tB17_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %43, 16;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B18_DONE;\n\tB18_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %18, u, g, %18;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B18_LOOP;\n\tB18_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %44, 65535;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B19_DONE;\n\tB19_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %19, u, g, %19;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B19_LOOP;\n\tB19_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %44, 16;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B20_DONE;\n\tB20_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %20, u, g, %20;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B20_LOOP;\n\tB20_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %45, 65535;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B21_DONE;\n\tB21_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %21, u, g, %21;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B21_LOOP;\n\tB21_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %45, 16;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B22_DONE;\n\tB22_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %22, u, g, %22;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B22_LOOP;\n\tB22_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %46, 65535;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B23_DONE;\n\tB23_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %23, u, g, %23;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B23_LOOP;\n\tB23_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %46, 16;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B24_DONE;\n\tB24_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %24, u, g, %24;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B24_LOOP;\n\tB24_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %47, 65535;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B25_DONE;\n\tB25_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %25, u, g, %25;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B25_LOOP;\n\tB25_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %47, 16;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B26_DONE;\n\tB26_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %26, u, g, %26;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B26_LOOP;\n\tB26_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %48, 65535;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B27_DONE;\n\tB27_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %27, u, g, %27;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B27_LOOP;\n\tB27_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %48, 16;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B28_DONE;\n\tB28_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %28, u, g, %28;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B28_LOOP;\n\tB28_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %49, 65535;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B29_DONE;\n\tB29_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %29, u, g, %29;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B29_LOOP;\n\tB29_DONE:\n\tmov.b32 pe, pend;\n\tshr.u32 t, %49, 16;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B30_DONE;\n\tB30_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %30, u, g, %30;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B30_LOOP;\n\tB30_DONE:\n\tmov.b32 pe, pend;\n\tand.b32 t, %50, 65535;\n\tmad.lo.u32 pend, t, 16, %32;\n\tsetp.ge.u32 p, pe, pend;\n\t@p bra.uni B31_DONE;\n\tB31_LOOP:\n\tld.shared.v4.b32 {o, x, gl, gh}, [pe];\n\tadd.u32 a, o, %33;\n\tld.shared.f64 u, [a];\n\tmov.b64 g, {gl, gh};\n\tfma.rn.f64 %31, u, g, %31;\n\tadd.u32 pe, pe, 16;\n\tsetp.lt.u32 p, pe, pend;\n\t@p bra.uni B31_LOOP;\n\tB31_DONE:\n\tmov.b32 pe, pend;\n\t}"
                 : "+d"(acc[0][0]), "+d"(acc[0][1]), "+d"(acc[0][2]), "+d"(acc[0][3]), "+d"(acc[0][4]), "+d"(acc[0][5]), "+d"(acc[0][6]), "+d"(acc[0][7]), "+d"(acc[0][8]), "+d"(acc[0][9]), "+d"(acc[0][10]), "+d"(acc[0][11]), "+d"(acc[0][12]), "+d"(acc[0][13]), "+d"(acc[0][14]), "+d"(acc[0][15]), "+d"(acc[0][16]), "+d"(acc[0][17]), "+d"(acc[0][18]), "+d"(acc[0][19]), "+d"(acc[0][20]), "+d"(acc[0][21]), "+d"(acc[0][22]), "+d"(acc[0][23]), "+d"(acc[0][24]), "+d"(acc[0][25]), "+d"(acc[0][26]), "+d"(acc[0][27]), "+d"(acc[0][28]), "+d"(acc[0][29]), "+d"(acc[0][30]), "+d"(acc[0][31])
                 : "r"(sen), "r"(sx), "r"(bw[0]), "r"(bw[1]), "r"(bw[2]), "r"(bw[3]), "r"(bw[4]), "r"(bw[5]), "r"(bw[6]), "r"(bw[7]), "r"(bw[8]), "r"(bw[9]), "r"(bw[10]), "r"(bw[11]), "r"(bw[12]), "r"(bw[13]), "r"(bw[14]), "r"(bw[15]), "r"(bw[16])
                 : "memory");
}
__device__ __forceinline__ void run_s1(uint32_t &pe, uint32_t pend, uint32_t sx, double &c0) {
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 o0, x0, l0, h0, a0;\n\t.reg .f64 u0, g0;\n\tsetp.ge.u32 p, %0, %2;\n\t@p bra.uni DONE;\n\tLOOP:\n\tld.shared.v4.b32 {o0, x0, l0, h0}, [%0];\n\tadd.u32 a0, o0, %3;\n\tld.shared.f64 u0, [a0];\n\tmov.b64 g0, {l0, h0};\n\tfma.rn.f64 %1, u0, g0, %1;\n\tadd.u32 %0, %0, 16;\n\tsetp.lt.u32 p, %0, %2;\n\t@p bra.uni LOOP;\n\tDONE:\n\t}"
                 : "+r"(pe), "+d"(c0)
                 : "r"(pend), "r"(sx)
                 : "memory");
}
__device__ __forceinline__ void run_s1f(uint32_t &pe, uint32_t pend, uint32_t sx, uint4 f, double &c0) {
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 o0, x0, l0, h0, a0;\n\t.reg .f64 u0, g0;\n\tsetp.ge.u32 p, %0, %2;\n\t@p bra.uni DONE;\n\tadd.u32 a0, %4, %3;\n\tld.shared.f64 u0, [a0];\n\tmov.b64 g0, {%6, %7};\n\tfma.rn.f64 %1, u0, g0, %1;\n\tadd.u32 %0, %0, 16;\n\tsetp.ge.u32 p, %0, %2;\n\t@p bra.uni DONE;\n\tLOOP:\n\tld.shared.v4.b32 {o0, x0, l0, h0}, [%0];\n\tadd.u32 a0, o0, %3;\n\tld.shared.f64 u0, [a0];\n\tmov.b64 g0, {l0, h0};\n\tfma.rn.f64 %1, u0, g0, %1;\n\tadd.u32 %0, %0, 16;\n\tsetp.lt.u32 p, %0, %2;\n\t@p bra.uni LOOP;\n\tDONE:\n\t}"
                 : "+r"(pe), "+d"(c0)
                 : "r"(pend), "r"(sx), "r"(f.x), "r"(f.y), "r"(f.z), "r"(f.w)
                 : "memory");
}
__device__ __forceinline__ void run_t1(uint32_t &pe, uint32_t pend, uint32_t st, uint32_t lane8, double &c0) {
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 o0, x0, l0, h0, a0;\n\t.reg .f64 u0, g0;\n\tsetp.ge.u32 p, %0, %2;\n\t@p bra.uni DONE;\n\tLOOP:\n\tld.shared.v4.b32 {o0, x0, l0, h0}, [%0];\n\txor.b32 a0, x0, %4;\n\tadd.u32 a0, a0, o0;\n\tadd.u32 a0, a0, %3;\n\tld.shared.f64 u0, [a0];\n\tmov.b64 g0, {l0, h0};\n\tfma.rn.f64 %1, u0, g0, %1;\n\tadd.u32 %0, %0, 16;\n\tsetp.lt.u32 p, %0, %2;\n\t@p bra.uni LOOP;\n\tDONE:\n\t}"
                 : "+r"(pe), "+d"(c0)
                 : "r"(pend), "r"(st), "r"(lane8)
                 : "memory");
}
__device__ __forceinline__ void run_t1f(uint32_t &pe, uint32_t pend, uint32_t st, uint32_t lane8, uint4 f, double &c0) {
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 o0, x0, l0, h0, a0;\n\t.reg .f64 u0, g0;\n\tsetp.ge.u32 p, %0, %2;\n\t@p bra.uni DONE;\n\txor.b32 a0, %6, %4;\n\tadd.u32 a0, a0, %5;\n\tadd.u32 a0, a0, %3;\n\tld.shared.f64 u0, [a0];\n\tmov.b64 g0, {%7, %8};\n\tfma.rn.f64 %1, u0, g0, %1;\n\tadd.u32 %0, %0, 16;\n\tsetp.ge.u32 p, %0, %2;\n\t@p bra.uni DONE;\n\tLOOP:\n\tld.shared.v4.b32 {o0, x0, l0, h0}, [%0];\n\txor.b32 a0, x0, %4;\n\tadd.u32 a0, a0, o0;\n\tadd.u32 a0, a0, %3;\n\tld.shared.f64 u0, [a0];\n\tmov.b64 g0, {l0, h0};\n\tfma.rn.f64 %1, u0, g0, %1;\n\tadd.u32 %0, %0, 16;\n\tsetp.lt.u32 p, %0, %2;\n\t@p bra.uni LOOP;\n\tDONE:\n\t}"
                 : "+r"(pe), "+d"(c0)
                 : "r"(pend), "r"(st), "r"(lane8), "r"(f.x), "r"(f.y), "r"(f.z), "r"(f.w)
                 : "memory");
}

__device__ __forceinline__ uint4 lds_u4(uint32_t addr) {
    uint4 w;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w) : "r"(addr) : "memory");
    return w;
}

struct ApplyArgs {
    const double *A;
    int64_t lda;
    int trans;
    int use_tma;
    int mode;       // 0: TMA tile (S), 1: swizzled transposing cp.async (S'), 2: cp.async (S)
    int ksplit;     // CTAs of a cluster splitting the k range (DSMEM reduction)
    int64_t m_out;  // output rows (rows of A for trans 0, cols of A for trans 1)
    int64_t n;      // input index extent (= op.n)
    int d, alpha, tk, log2tk;
    int64_t nchunks, bstride, estride;
    const uint16_t *bptr;
    const uint4 *ent;
    double scale;
    double *S;
    int64_t lds, col0;
    int nslabs, stages;
    int stage_bytes, zero_off, bp_off, en_off;
};

// All NW warps own buckets (NW*DB per CTA slab) and share the producer work:
// warp 0 / lane 0 issues TMA + bulk copies (mode 0); in modes 1/2 every lane
// issues its share of 8-byte cp.async for the chunk STAGES-1 ahead.
template <int RPT, int DB, int NW, bool TRANS, bool BATCH, bool PROD, bool WHOLE = true>
__global__ void __launch_bounds__((NW + (PROD ? (TRANS ? 4 : 1) : 0)) * 32, 1)
    sjlt_apply_kernel(const ApplyArgs p, const __grid_constant__ CUtensorMap tmap) {
    constexpr int TM = 32 * RPT;
    constexpr int SLAB = NW * DB;
    constexpr int G = DB < 4 ? DB : 4;  // buckets whose first entries are folded as one batch
    static_assert(DB % G == 0, "DB must be a multiple of the batch");
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);
    uint64_t *empty = full + 8;
    unsigned *done = reinterpret_cast<unsigned *>(full + 16);  // per-slot finished-warp counters
    unsigned char *stage0 = smem + 256;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ks = p.ksplit;
    const int kr = (int)(blockIdx.x % ks);  // == %cluster_ctarank (cluster = ks consecutive CTAs)
    const int64_t bid = blockIdx.x / ks;
    const int slab = (int)(bid % p.nslabs);
    const int64_t tile = bid / p.nslabs;
    const int64_t r0 = tile * TM;
    const int j0 = slab * SLAB;
    const int64_t per = (p.nchunks + ks - 1) / ks;
    const int64_t c_begin = (int64_t)kr * per < p.nchunks ? (int64_t)kr * per : p.nchunks;
    const int64_t c_end = c_begin + per < p.nchunks ? c_begin + per : p.nchunks;
    const int nloc = (int)(c_end - c_begin);
    const int mode = p.mode;
    const int stages = p.stages;
    const uint32_t bp_bytes = (SLAB + 8) * 2;
    const uint32_t en_bytes = (uint32_t)p.estride * 16;
    const uint32_t tile_bytes = (uint32_t)p.tk * TM * 8;

    // zero rows + null entries, barriers
    for (int s = 0; s < stages; ++s) {
        unsigned char *st = stage0 + (size_t)s * p.stage_bytes;
        double *zr = reinterpret_cast<double *>(st + p.zero_off);
        for (int q = threadIdx.x; q < TM; q += blockDim.x) zr[q] = 0.0;
        if (threadIdx.x == 0)
            reinterpret_cast<uint4 *>(st + p.en_off)[p.estride] =
                make_uint4((uint32_t)p.zero_off, 0u, 0u, 0x3FF00000u);
    }
    if (threadIdx.x == 0) {
        constexpr int PW = PROD ? (TRANS ? 4 : 1) : 0;  // dedicated producer warps
        const uint32_t fcount = mode == 0 ? 1u : 1u + 32u * (PROD ? PW : NW);
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], fcount);
            mbar_init(&empty[s], NW);
            done[s] = 0;
        }
        fence_mbar_init();
        if (mode == 0) prefetch_tmap(&tmap);
    }
    __syncthreads();

    // ---- producer helpers
    auto stage_of = [&](int j) { return stage0 + (size_t)(j % stages) * p.stage_bytes; };
    auto issue_tma = [&](int j) {  // warp 0, lane 0
        unsigned char *st = stage_of(j);
        uint64_t *bar = &full[j % stages];
        const int64_t c = c_begin + j;
        mbar_arrive_expect_tx(bar, tile_bytes + bp_bytes + en_bytes);
        tma_load_2d(st, &tmap, (int)r0, (int)(c * p.tk), bar);
        bulk_g2s(st + p.bp_off, p.bptr + c * p.bstride + j0, bp_bytes, bar);
        bulk_g2s(st + p.en_off, p.ent + c * p.estride, en_bytes, bar);
    };
    auto issue_coop = [&](int j, int ptid, int pnt) {  // threads [0, pnt) of the producer set
        unsigned char *st = stage_of(j);
        uint64_t *bar = &full[j % stages];
        const int64_t c = c_begin + j;
        const int64_t k0 = c * p.tk;
        const int kc = (int)(p.n - k0 < p.tk ? p.n - k0 : p.tk);
        if (ptid == 0) {
            mbar_arrive_expect_tx(bar, bp_bytes + en_bytes);
            bulk_g2s(st + p.bp_off, p.bptr + c * p.bstride + j0, bp_bytes, bar);
            bulk_g2s(st + p.en_off, p.ent + c * p.estride, en_bytes, bar);
        }
        double *sx = reinterpret_cast<double *>(st);
        const int nel = p.tk * TM;
        if (TRANS) {
            // element (kk, rr) = A[k0+kk, r0+rr] -> sx[kk*TM + (rr ^ (kk%32))];
            // lanes along kk: coalesced reads, conflict-free swizzled writes.
            // Thread t owns columns kk = t, t + pnt, ... and walks all TM rows
            // with pointer increments (lanes along kk: 256 B per instruction).
            const int tk = p.tk;
            const bool full_rows = r0 + TM <= p.m_out;
            for (int kk = ptid; kk < tk; kk += pnt) {
                const int sw = kk & 31;
                const double *src = p.A + r0 * p.lda + k0 + kk;
                double *dbase = sx + kk * TM;
                if (kk < kc && full_rows) {
#pragma unroll 8
                    for (int rr = 0; rr < TM; ++rr, src += p.lda) cp_async8(dbase + (rr ^ sw), src, true);
                } else {
                    const bool vk = kk < kc;
                    for (int rr = 0; rr < TM; ++rr, src += p.lda) {
                        const bool v = vk && (r0 + rr < p.m_out);
                        cp_async8(dbase + (rr ^ sw), v ? src : p.A, v);
                    }
                }
            }
        } else {
            for (int idx = ptid; idx < nel; idx += pnt) {
                const int kk = idx / TM, rr = idx % TM;
                const bool v = (kk < kc) && (r0 + rr < p.m_out);
                const double *src = p.A + (k0 + kk) * p.lda + r0 + rr;
                cp_async8(sx + kk * TM + rr, v ? src : p.A, v);
            }
        }
        cp_async_mbar_arrive(bar);
    };

    int issued = 0;
    if (PROD) {
        // dedicated producer warp(s): refill a slot as soon as every consumer
        // warp has released it (mode 0: one TMA-issuing lane; modes 1/2: the
        // producer warps share the 8-byte transposing copies)
        if (warp >= NW) {
            constexpr int PW = TRANS ? 4 : 1;
            if (mode == 0) {
                if (lane == 0 && warp == NW) {
                    for (int j = 0; j < nloc; ++j) {
                        if (j >= stages) mbar_wait(&empty[j % stages], (uint32_t)((j / stages) - 1) & 1u);
                        issue_tma(j);
                    }
                }
            } else {
                const int ptid = threadIdx.x - NW * 32;
                for (int j = 0; j < nloc; ++j) {
                    if (j >= stages) mbar_wait(&empty[j % stages], (uint32_t)((j / stages) - 1) & 1u);
                    issue_coop(j, ptid, PW * 32);
                }
            }
            __syncwarp();
            if (ks > 1) {  // match the consumers' barriers of the k-split reduction
                __syncthreads();
                cluster_sync();
                cluster_sync();
            }
            return;
        }
    } else if (mode == 0) {
        if (warp == 0 && lane == 0)
            for (; issued < nloc && issued < stages; ++issued) issue_tma(issued);
    } else {
        for (; issued < nloc && issued < stages - 1; ++issued) issue_coop(issued, threadIdx.x, NW * 32);
    }

    double acc[RPT][DB];
#pragma unroll
    for (int r = 0; r < RPT; ++r)
#pragma unroll
        for (int jj = 0; jj < DB; ++jj) acc[r][jj] = 0.0;

    const uint32_t smem_base = smem_u32(stage0);
    const uint32_t lane8 = lane * 8u;
    const uint32_t lane_off = TRANS ? 0u : lane * 8u * (RPT == 1 ? 1u : 2u);  // S: rows 2l,2l+1 (+64) / l
    int cs = 0;
    uint32_t cph = 0;
    for (int i = 0; i < nloc; ++i) {
        // ---- producer duty (modes 1/2): chunk i + stages - 1 into the slot of
        // chunk i - 1, once every warp has finished chunk i - 1
        if (!PROD && mode != 0 && issued < nloc) {
            const int j = issued;
            if (j >= stages) mbar_wait(&empty[j % stages], (uint32_t)((j / stages) - 1) & 1u);
            issue_coop(j, threadIdx.x, NW * 32);
            ++issued;
        }

        // ---- consume chunk i
        const int s = cs;
        mbar_wait(&full[s], cph);
        const uint32_t st = smem_base + (uint32_t)s * p.stage_bytes;
        const uint32_t sx = st + lane_off;
        const uint32_t sen = st + p.en_off;
        const uint16_t *sbp = reinterpret_cast<const uint16_t *>(
                                  stage0 + (size_t)s * p.stage_bytes + p.bp_off) + warp * DB;
        const uint32_t nul = (uint32_t)p.estride;
        // the warp's DB+1 bucket bounds, preloaded (packed u16 pairs) so no
        // bucket waits on a shared-memory load of its own bound
        constexpr int NBW = DB / 2 + 1;
        uint32_t bw[NBW];
        {
            const uint32_t *src = reinterpret_cast<const uint32_t *>(sbp);
#pragma unroll
            for (int q = 0; q < NBW; ++q) bw[q] = src[q];
        }
        auto bound = [&](int jj) -> uint32_t {
            return (jj & 1) ? (bw[jj >> 1] >> 16) : (bw[jj >> 1] & 0xffffu);
        };
        if (!BATCH && !TRANS && WHOLE) {
            if constexpr (RPT == 1 && DB == 16) chunk_s_1x16(acc, sen, sx, bw);
            else if constexpr (RPT == 1 && DB == 32) chunk_s_1x32(acc, sen, sx, bw);
            else if constexpr (RPT == 2 && DB == 8) chunk_s_2x8(acc, sen, sx, bw);
            else if constexpr (RPT == 2 && DB == 4) chunk_s_2x4(acc, sen, sx, bw);
            else if constexpr (RPT == 2 && DB == 16) chunk_s_2x16(acc, sen, sx, bw);
            else if constexpr (RPT == 4 && DB == 2) chunk_s_4x2(acc, sen, sx, bw);
            else if constexpr (RPT == 4 && DB == 4) chunk_s_4x4(acc, sen, sx, bw);
            else if constexpr (RPT == 4 && DB == 8) chunk_s_4x8(acc, sen, sx, bw);
        } else if (!BATCH) {
            // per-bucket loops; the first entry of bucket jj+1 is loaded while
            // bucket jj runs (index <= estride: the null entry keeps it in range)
            uint32_t pe = sen + 16u * bound(0);
            uint4 wn = lds_u4(pe);
#pragma unroll
            for (int jj = 0; jj < DB; ++jj) {
                const uint32_t pend = sen + 16u * bound(jj + 1);
                const uint4 w = wn;
                if (jj + 1 < DB) wn = lds_u4(pend);
                if constexpr (RPT == 1) {
                    if (TRANS) run_t1f(pe, pend, st, lane8, w, acc[0][jj]);
                    else run_s1f(pe, pend, sx, w, acc[0][jj]);
                } else if constexpr (RPT == 2) {
                    if (TRANS) run_t2f(pe, pend, st, lane8, w, acc[0][jj], acc[1][jj]);
                    else run_s2f(pe, pend, sx, w, acc[0][jj], acc[1][jj]);
                } else {
                    if (TRANS) run_t4f(pe, pend, st, lane8, w, acc[0][jj], acc[1][jj],
                                       acc[RPT - 2][jj], acc[RPT - 1][jj]);
                    else run_s4f(pe, pend, sx, w, acc[0][jj], acc[1][jj], acc[RPT - 2][jj],
                                 acc[RPT - 1][jj]);
                }
                pe = pend;
            }
        }
#pragma unroll
        for (int g0 = 0; g0 < (BATCH ? DB : 0); g0 += G) {
            uint32_t b[G + 1];
#pragma unroll
            for (int t = 0; t <= G; ++t) b[t] = bound(g0 + t);
            // batch: first entry of each of the G buckets (null if empty)
            uint4 w[G];
#pragma unroll
            for (int t = 0; t < G; ++t) {
                const uint32_t idx = b[t + 1] > b[t] ? b[t] : nul;
                asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(w[t].x), "=r"(w[t].y), "=r"(w[t].z), "=r"(w[t].w)
                             : "r"(sen + 16u * idx) : "memory");
            }
#pragma unroll
            for (int t = 0; t < G; ++t) {
                const double g = __hiloint2double((int)w[t].w, (int)w[t].z);
                const int jj = g0 + t;
                if (TRANS) {
                    const uint32_t ad = st + w[t].x + (w[t].y ^ lane8);
#pragma unroll
                    for (int r = 0; r < RPT; ++r) {
                        double u;
                        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(u) : "r"(ad + 256u * r) : "memory");
                        acc[r][jj] = fma(u, g, acc[r][jj]);
                    }
                } else if constexpr (RPT == 1) {
                    double u;
                    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(u) : "r"(sx + w[t].x) : "memory");
                    acc[0][jj] = fma(u, g, acc[0][jj]);
                } else {
                    const uint32_t ad = sx + w[t].x;
#pragma unroll
                    for (int h = 0; h < RPT / 2; ++h) {
                        double u, v;
                        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(u), "=d"(v)
                                     : "r"(ad + 512u * h) : "memory");
                        acc[2 * h][jj] = fma(u, g, acc[2 * h][jj]);
                        acc[2 * h + 1][jj] = fma(v, g, acc[2 * h + 1][jj]);
                    }
                }
            }
            // remaining entries of each bucket
#pragma unroll
            for (int t = 0; t < G; ++t) {
                const int jj = g0 + t;
                uint32_t pe = sen + 16u * (b[t] + 1);
                const uint32_t pend = sen + 16u * b[t + 1];
                if constexpr (RPT == 1) {
                    if (TRANS) run_t1(pe, pend, st, lane8, acc[0][jj]);
                    else run_s1(pe, pend, sx, acc[0][jj]);
                } else if constexpr (RPT == 2) {
                    if (TRANS) run_t2(pe, pend, st, lane8, acc[0][jj], acc[1][jj]);
                    else run_s2(pe, pend, sx, acc[0][jj], acc[1][jj]);
                } else {
                    if (TRANS) run_t4(pe, pend, st, lane8, acc[0][jj], acc[1][jj], acc[RPT - 2][jj],
                                      acc[RPT - 1][jj]);
                    else run_s4(pe, pend, sx, acc[0][jj], acc[1][jj], acc[RPT - 2][jj],
                                acc[RPT - 1][jj]);
                }
            }
        }
        __syncwarp();
        if (lane == 0) {
            if (mode == 0 && !PROD) {
                // the last warp to finish chunk i refills its slot with chunk i + stages
                if (atomicAdd(&done[s], 1u) == NW - 1) {
                    done[s] = 0;
                    if (i + stages < nloc) issue_tma(i + stages);
                }
            } else {
                mbar_arrive(&empty[s]);
            }
        }
        if (++cs == stages) {
            cs = 0;
            cph ^= 1u;
        }
    }

    // ------------------------------------------- k-split: DSMEM reduction
    // Partial sums of the ks CTAs of a cluster are combined by rank 0 in
    // rank order (deterministic).  The stage ring is reused as the buffer.
    if (ks > 1) {
        double *red = reinterpret_cast<double *>(stage0);
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
            } else if constexpr (RPT == 1) {
                const int64_t row = r0 + lane;
                if (row < p.m_out) col[row] = acc[0][jj] * p.scale;
            } else {      // lane owns rows 2l, 2l+1 (+64 for RPT 4)
#pragma unroll
                for (int h = 0; h < RPT / 2; ++h) {
                    const int64_t row = r0 + 64 * h + 2 * lane;
                    const double x0 = acc[2 * h][jj] * p.scale, x1 = acc[2 * h + 1][jj] * p.scale;
                    if (vec_ok && row + 1 < p.m_out) {
                        *reinterpret_cast<double2 *>(col + row) = make_double2(x0, x1);
                    } else {
                        if (row < p.m_out) col[row] = x0;
                        if (row + 1 < p.m_out) col[row + 1] = x1;
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
    HSK_REQUIRE(g.tm == TM, HSK_EINVAL, "sjlt: plan/config mismatch");
    const bool aligned = a.use_tma != 0;  // 16-byte aligned columns (lda even)
    a.mode = a.trans ? 1 : (aligned ? 0 : 2);
    a.log2tk = 0;
    while ((1 << a.log2tk) < a.tk) ++a.log2tk;
    CUtensorMap tmap;
    memset(&tmap, 0, sizeof(tmap));
    if (a.mode == 0) {
        int rc = make_tmap_f64_2d(&tmap, a.A, (uint64_t)a.m_out, (uint64_t)a.n, (uint64_t)a.lda,
                                  TM, (uint32_t)a.tk);
        if (rc) return rc;
    }
    const int a_bytes = a.tk * TM * 8;
    a.zero_off = a_bytes;
    a.bp_off = (int)roundup(a_bytes + TM * 8, 128);
    a.en_off = (int)roundup(a.bp_off + (SLAB + 8) * 2, 128);
    a.stage_bytes = (int)roundup(a.en_off + (a.estride + 1) * 16, 128);
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
    const int budget = 226 * 1024;
    a.stages = std::max(2, std::min(8, (budget - 256) / a.stage_bytes));
    if (const char *env = getenv("HSK_SJLT_STAGES")) a.stages = std::max(2, std::min(a.stages, atoi(env)));
    if (per > 0 && a.stages > per + 1) a.stages = std::max(2, per + 1);
    int smem = 256 + a.stages * a.stage_bytes;
    if (ks > 1) smem = std::max(smem, 256 + NW * DB * RPT * 32 * 8);
    // batched first-entry folding pays off when buckets hold several entries
    // per chunk (lambda = tk*alpha/d); HSK_SJLT_BATCH=0/1 overrides
    bool batch = (int64_t)a.tk * a.alpha >= 4 * (int64_t)a.d;
    if (const char *env = getenv("HSK_SJLT_BATCH")) batch = env[0] == '1';
    // dedicated producer warp (TMA path only; 17 warps -> 96-register budget,
    // so it pairs with the unbatched consumer loops)
    bool prod = NW < 32;  // a 33rd warp would cut the register budget to 56
    if (const char *env = getenv("HSK_SJLT_PROD")) prod = env[0] == '1';
    prod = prod && (a.mode == 0 || a.mode == 1) && NW + (a.trans ? 4 : 1) <= 32;
    if (prod) batch = false;
    bool whole = true;
    if (const char *env = getenv("HSK_SJLT_WHOLE")) whole = env[0] == '1';
    auto kern = a.trans ? (prod ? sjlt_apply_kernel<RPT, DB, NW, true, false, true>
                                : batch ? sjlt_apply_kernel<RPT, DB, NW, true, true, false>
                                        : sjlt_apply_kernel<RPT, DB, NW, true, false, false>)
                        : (prod ? sjlt_apply_kernel<RPT, DB, NW, false, false, true>
                                : batch ? sjlt_apply_kernel<RPT, DB, NW, false, true, false>
                                        : whole ? sjlt_apply_kernel<RPT, DB, NW, false, false, false, true>
                                                : sjlt_apply_kernel<RPT, DB, NW, false, false, false, false>);
    const int nthreads = (NW + (prod ? (a.trans ? 4 : 1) : 0)) * 32;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return cuda_status(e, "sjlt: set smem attribute");
    const int64_t grid = tiles * a.nslabs * ks;
    HSK_REQUIRE(grid < (1ll << 31), HSK_EINVAL, "sjlt: grid too large");
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid, 1, 1);
    cfg.blockDim = dim3(nthreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = ks;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = ks > 1 ? 1 : 0;  // plain launch unless the k-split needs a cluster
    if (const char *env = getenv("HSK_SJLT_FORCE_CLUSTER")) cfg.numAttrs = env[0] == '1' ? 1 : cfg.numAttrs;
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
    return sjlt::plan_geom(n, d, alpha).bytes;
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
    const sjlt::Plan pl = sjlt::plan_geom(n, d, alpha);
    HSK_REQUIRE(plan != nullptr && plan_bytes >= pl.bytes, HSK_EINVAL,
                "sjlt plan: buffer of %lld bytes, need %lld", (long long)plan_bytes,
                (long long)pl.bytes);
    HSK_REQUIRE(n == 0 || (pos != nullptr && sgn != nullptr), HSK_EINVAL, "sjlt plan: null pattern");
    cudaStream_t st = as_stream(stream);
    unsigned char *base = static_cast<unsigned char *>(plan);
    cudaError_t e = cudaMemsetAsync(base, 0, pl.bytes, st);
    if (e != cudaSuccess) return cuda_status(e, "sjlt plan: memset");
    if (n > 0) {
        for (const sjlt::Geom *g : {&pl.s, &pl.t}) {
            int p2 = 1;
            while (p2 < g->tk * alpha) p2 <<= 1;
            sjlt::sjlt_plan_kernel<<<(unsigned)g->nchunks, 256, p2 * sizeof(uint32_t), st>>>(
                pos, sgn, n, d, alpha, g->tk, p2, g->bstride, g->estride, g->pitch,
                reinterpret_cast<uint16_t *>(base + g->bptr_off),
                reinterpret_cast<uint4 *>(base + g->ent_off), reinterpret_cast<int *>(base + 28));
            HSK_CHECK_LAUNCH("sjlt_plan_kernel");
        }
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
    const sjlt::Plan pl = sjlt::plan_geom(n, d, alpha);
    const sjlt::Geom &g = trans ? pl.t : pl.s;
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
    // S: 32 warps x (DB/2) buckets -- twice the warps to hide the shared-memory
    // latency of the entry -> tile -> DFMA chain (<= 64 registers per thread).
    // S': 16 warps (its cp.async producer work is shared by all warps).
    bool w32 = !trans;
    if (const char *env = getenv("HSK_SJLT_W32")) w32 = env[0] == '1';
    if (g.rpt == 1) {  // 32-row tiles, 512-bucket slabs
        if (w32) return sjlt::launch<1, 16, 32>(a, g, st);
        return sjlt::launch<1, 32, 16>(a, g, st);
    }
    if (g.rpt == 4) {  // 128-row tiles, 64-bucket slabs
        if (w32) return sjlt::launch<4, 2, 32>(a, g, st);
        return sjlt::launch<4, 4, 16>(a, g, st);
    }
    if (w32) {          // 64-row tiles
        if (d <= 128) return sjlt::launch<2, 4, 32>(a, g, st);
        return sjlt::launch<2, 8, 32>(a, g, st);
    }
    if (d <= 128) return sjlt::launch<2, 8, 16>(a, g, st);
    return sjlt::launch<2, 16, 16>(a, g, st);
}
