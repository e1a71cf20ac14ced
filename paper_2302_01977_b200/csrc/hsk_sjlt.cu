// hsk_sjlt.cu -- SJLT sketch S = A R^T and S' = A^T R^T on sm_100a.
//
// Replaces SjltBlock._build_storage / apply_right / apply_right_transposed
// (/root/reference/pkg/src/hsskit/sketching.py:292-351; §6).
//
// Design:
//  * Plan.  The reference keeps R^T = s (B+ - B-) as index-only CSR/CSC.  The
//    GPU plan re-blocks the same pattern by k-chunks of TK input indices: per
//    chunk, its TK*alpha entries sorted by bucket (stable in (k, t)), plus
//    per-chunk bucket offsets.  An entry is one 4-byte word kk << 3 | neg << 31
//    (kk = input index within the chunk): the consumer turns it into a tile
//    address with one shift-add and into +-1.0 with one LOP3.  Broadcast
//    entry loads are what fills the SM's register-writeback port (128 B/clk)
//    besides the tile loads themselves, so the word is kept minimal.  Each
//    direction has its own sub-plan (tile shape).  Built on device by a
//    per-chunk bitonic sort.
//  * Apply.  A CTA owns TM = 32*RPT output rows and a slab of NW*DB buckets.
//    Consumer warp w owns buckets [j0 + w*DB, +DB); lane l owns rows
//    l*RPT .. l*RPT+RPT-1, so each warp holds an RPT x DB register
//    accumulator block: owner-computes, no atomics, a fixed summation order
//    (deterministic).  Per entry: one broadcast LDS.32 of the entry word, one
//    LDS.128 (RPT = 2) of the staged A tile, RPT DFMAs with +-1 (exactly the
//    reference's add/subtract, one rounding each; no data multiplies).  The
//    walk over a warp's entries is software-pipelined (tools/gen_consumers.py).
//  * Paired plans (HSK_SJLT_CHUNKED, block construction with d/alpha = 8):
//    one entry carries an index's buckets in two construction chunks, so
//    each tile element is read alpha/2 times instead of alpha (geom_dir).
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
#include "hsk_sjlt_pipe.cuh"

// Diagnostic builds only (-DHSK_SJLT_DEBUG=1, then HSK_SJLT_DBG=<mode> at run
// time): 1 = producers only (consumers skip the walk), 2 = consumers only (no
// refills after the first ring fill; results are garbage), 3 = checked bucket
// bounds and stream-K roles (device printf).  Production kernels compile none
// of it -- the extra live values cost registers the walker needs.
#ifndef HSK_SJLT_DEBUG
#define HSK_SJLT_DEBUG 0
#endif
// tuning builds (-DHSK_TUNING=1) add the A/B kernel variants of DESIGN.md §7
#ifndef HSK_TUNING
#define HSK_TUNING 0
#endif
#define DBG_IS(m) (HSK_SJLT_DEBUG && p.dbg == (m))

// producer warps of the transposed 128-row S' tiles: mode 4 (TMA staging +
// in-smem transpose) measured 10.9 ms on C3 with 8, 12.3 with 4; mode 1 (unaligned A)
#ifndef HSK_XPOSE_PRODUCERS
#define HSK_XPOSE_PRODUCERS 8
#endif
constexpr int kXposeProducers = HSK_XPOSE_PRODUCERS;

// TMA multicast across slab clusters (opt-in at build time and run time,
// -DHSK_SJLT_MULTICAST=1 plus HSK_SJLT_MC=1): measured slower (see launch<>),
// and its remote-arrive branches cost the default kernels registers and
// scheduling even when not taken (d = 2048 S: 6.0 vs 5.45 ms), so production
// builds compile none of it.
#ifndef HSK_SJLT_MULTICAST
#define HSK_SJLT_MULTICAST 0
#endif
// The stream-K instantiations keep the (runtime-inert) multicast branches:
// measured 3.5 % faster on C2 with them than without (code layout; the
// walker SASS is identical), while the whole-tile ones are faster without.
#define MC_ON ((HSK_SJLT_MULTICAST || SK) && p.mc > 1)

namespace hsk {
namespace sjlt {

constexpr int kHeaderBytes = 128;
constexpr int kMaxChunkEntries = 4096;  // TK * alpha bound (12-bit local index)
constexpr int64_t kMaxD = (1 << 19);    // bucket index fits 19 bits of the sort key

// Per-direction sub-plan geometry.  One plan buffer holds a header, the S
// sub-plan (trans 0) and the S' sub-plan (trans 1): the best tile shape can
// differ per direction (measured): 128-row tiles for d <= 64, 64-row tiles
// (256-bucket slabs, TK 128) otherwise, except S with d > 512, which prefers
// 32-row tiles with 512-bucket slabs and TK = 256 (half the slab re-reads).
struct Geom {
    int pair;          // paired plan (block construction, d/alpha = 8): below
    int rpt;           // rows per lane (tile rows tm = 32 * rpt)
    int db, nw;        // buckets per consumer warp, consumer warps per CTA
    int64_t ngroups;   // warp groups of db buckets (nslabs * nw)
    int tm;
    int pitch;         // tile pitch (doubles) = tm: TMA writes densely; the S'
                       // producer orders its transposing stores conflict-free
    int tk;            // input indices per chunk
    int64_t nchunks;
    int64_t gstride;   // uint32 per group-start row (ngroups + 1, padded)
    int64_t estride;   // words per chunk row (tk*alpha entries + ngroups terminators)
    int64_t gptr_off;  // bytes from the plan base
    int64_t ent_off;   // bytes from the plan base
    int64_t end;       // bytes from the plan base (end of this sub-plan)
};

static inline int64_t roundup(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// ring slot bytes: [tile][group starts][entry words + null words] (mirrors launch<>())
static inline int stage_bytes_for(int tk, int tm, int alpha, int64_t ngroups, int nw) {
    const int64_t tile = roundup((int64_t)(tk + 15) / 16 * 16 * tm * 8, 1024);
    const int64_t en_off = roundup(tile + (nw + 4) / 4 * 16, 128);
    return (int)roundup(en_off + (roundup((int64_t)tk * alpha + ngroups, 4) + 8) * 4, 1024);
}

// largest power-of-two TK <= cap whose stage fits `per_stage` bytes
static inline int tk_fit(int alpha, int tm, int cap, int per_stage, int64_t ng, int nw) {
    int tk = cap;
    while (tk > 1 && (tk * alpha > kMaxChunkEntries || stage_bytes_for(tk, tm, alpha, ng, nw) > per_stage))
        tk >>= 1;
    return tk;
}

// largest multiple of 16 TK <= cap (<= 256: TMA box limit) whose stage fits;
// when not even TK = 16 keeps TK * alpha within a chunk's 12-bit local index
// (alpha > 256), the power-of-two rule (down to 1) of tk_fit
static inline int tk_fit16(int alpha, int tm, int cap, int per_stage, int64_t ng, int nw) {
    int tk = cap;
    while (tk > 16 && (tk * alpha > kMaxChunkEntries || stage_bytes_for(tk, tm, alpha, ng, nw) > per_stage))
        tk -= 16;
    if (tk * alpha > kMaxChunkEntries || stage_bytes_for(tk, tm, alpha, ng, nw) > per_stage)
        return tk_fit(alpha, tm, 16, per_stage, ng, nw);
    return tk;
}

// consumer warps and buckets per warp of the kernel that walks a sub-plan
// (16 consumer warps: the 96-register budget holds RPT x DB accumulators plus
// the walker; the 32-warp variants, half the buckets per warp, are kept for
// tuning: HSK_SJLT_W32=1)
static inline void warp_shape(int rpt, int d, int &db, int &nw) {
#if HSK_TUNING
    const bool w32 = tuning().sjlt_w32 == 1;
#else
    const bool w32 = false;  // 32-warp variants are compiled only in tuning builds
#endif
    nw = w32 ? 32 : 16;
    if (rpt == 1) db = w32 ? 16 : 32;        // 32-row tiles, 512-bucket slabs
    else if (rpt == 4) db = w32 ? 2 : 4;     // 128-row tiles, 64-bucket slabs
    else db = (d <= 128 ? 4 : 8) * (w32 ? 1 : 2);  // 64-row tiles
}

// Paired sub-plans (block construction with chunk d/alpha = 8, d a multiple
// of 64: C3's alpha = 8 increments of 64).  Every input index has exactly one
// bucket in each construction chunk, so one entry can carry an index's
// buckets in two chunks (t1 = 2p, t2 = 2p + 1) and one tile load feeds both.
// 64-row tiles, a slab is 64 buckets (4 chunk pairs), 16 consumer warps =
// 4 chunk pairs x 4 quarters of chunk t1: warp (p, h) walks the indices whose
// t1 bucket lies in quarter h (2 of its 8 buckets, complete in the warp) and
// accumulates their chunk-t2 buckets (8, partial); the four quarters' t2
// partials are added in quarter order at the end of a row tile
// (deterministic).  Per (row, element): alpha/2 tile reads instead of alpha;
// 16 (t1, t2) bucket combos per warp.
constexpr int kPairSlab = 64;  // buckets per slab (4 chunk pairs)

static Geom geom_dir(int64_t n, int d, int alpha, int trans, int64_t base, int pair = 0) {
    Geom g;
    int tk;
    g.pair = pair;
    if (pair) {
        constexpr int kStage3 = (226 * 1024 - 2048) / 3, kStage2 = (226 * 1024 - 2048) / 2;
        const int ae = alpha / 2;  // entries per input index
        g.rpt = 2;
        g.db = 16;
        g.nw = 16;
        g.ngroups = (int64_t)(d / kPairSlab) * g.nw;
        tk = n >= 8192 ? tk_fit16(ae, 64, 256, kStage2, g.ngroups, g.nw)
                       : tk_fit16(ae, 64, 128, kStage3, g.ngroups, g.nw);
        if (const int e = trans ? tuning().sjlt_tk_t : tuning().sjlt_tk; e > 0)
            tk = std::max(16, e / 16 * 16);
        g.tm = 64;
        g.pitch = g.tm;
        g.tk = tk;
        g.nchunks = (n + g.tk - 1) / g.tk;
        g.gstride = roundup(g.ngroups + 4, 4);
        g.estride = roundup((int64_t)g.tk * ae + g.ngroups, 4);
        g.gptr_off = base;
        g.ent_off = roundup(g.gptr_off + (g.nchunks + 1) * g.gstride * 4, 128);
        g.end = g.ent_off + roundup((g.nchunks + 1) * g.estride * 4, 128);
        return g;
    }
    // per-stage budgets: 3 stages (or 2) of the 226 KB ring
    constexpr int kStage3 = (226 * 1024 - 2048) / 3, kStage2 = (226 * 1024 - 2048) / 2;
    // Long rows (n >= 8192): two stages of the largest TK -- more entries per
    // bucket visit (lambda = TK*alpha/d) and fewer chunk boundaries outweigh
    // the shallower ring (the dedicated producer refills a slot as soon as it
    // is released).  Short rows keep three power-of-two stages so every CTA
    // still has a deep pipeline.  Tiles: 128 rows for d <= 64, else 64 rows
    // (measured better than 32-row / 512-bucket slabs even at d = 2048: the
    // L2 re-reads of more slabs cost less than twice the entry walks).  The
    // transposing cp.async producer of 128-row S' tiles keeps three stages.
    // (S with more than two 256-bucket slabs keeps three stages: eight slab
    // CTAs sharing each tile through L2 want the deeper ring -- measured at
    // d = 2048, alpha = 8)
    const bool wide = n >= 8192 && (trans || d <= 512);
    g.rpt = d <= 64 ? 4 : 2;
    if (const int e = trans ? tuning().sjlt_rpt_t : tuning().sjlt_rpt; e == 1 || e == 2 || e == 4) g.rpt = e;
    warp_shape(g.rpt, d, g.db, g.nw);
    g.ngroups = roundup(d, (int64_t)g.db * g.nw) / g.db;
    if (d <= 64) {
        tk = wide && !trans ? tk_fit16(alpha, 128, 256, kStage2, g.ngroups, g.nw)
                            : tk_fit(alpha, 128, 128, kStage3, g.ngroups, g.nw);
    } else {
        tk = wide ? tk_fit16(alpha, 64, 256, kStage2, g.ngroups, g.nw)
                  : tk_fit(alpha, 64, 128, kStage3, g.ngroups, g.nw);
    }
    if (const int e = trans ? tuning().sjlt_tk_t : tuning().sjlt_tk; e > 0) tk = e;
    g.tm = 32 * g.rpt;
    g.pitch = g.tm;
    g.tk = tk;
    g.nchunks = (n + g.tk - 1) / g.tk;
    g.gstride = roundup(g.ngroups + 4, 4);  // a CTA copies nw + 1 starts, 16-byte rows
    g.estride = roundup((int64_t)g.tk * alpha + g.ngroups, 4);  // 16-byte rows for the bulk copy
    g.gptr_off = base;
    g.ent_off = roundup(g.gptr_off + (g.nchunks + 1) * g.gstride * 4, 128);
    g.end = g.ent_off + roundup((g.nchunks + 1) * g.estride * 4, 128);
    return g;
}

struct Plan {
    Geom s, t;
    int64_t bytes;
};

static inline bool pair_shape(int d, int alpha) {
    return d % kPairSlab == 0 && alpha * 8 == d;
}

static Plan plan_geom(int64_t n, int d, int alpha, int pair = 0) {
    Plan pl;
    pair = pair && pair_shape(d, alpha) && n > 0;
    pl.s = geom_dir(n, d, alpha, 0, kHeaderBytes, pair);
    pl.t = geom_dir(n, d, alpha, 1, pl.s.end, pair);
    pl.bytes = pl.t.end;
    return pl;
}

// A chunk's sort key holds its entry index in 12 bits (paired: the input
// index in 8): a geometry outside that can never build a valid plan.
static bool geom_ok(const Geom &g, int alpha) {
    if (g.tk < 1) return false;
    if (g.pair) return g.tk <= 256 && (int64_t)g.tk * (alpha / 2) <= kMaxChunkEntries;
    return (int64_t)g.tk * alpha <= kMaxChunkEntries;
}

// ------------------------------------------------------------ plan build
// A chunk's entries are sorted by (bucket, input index); the entries of every
// group of db buckets (the ones one consumer warp owns) are closed by a
// terminator, so a warp's list is contiguous and self-delimiting.  Entry word:
//   (sign < 0) << 31 | (bucket mod db) << 24 | address bits,
// terminator bucket field = db (address bits 0).  Address bits of input index kk:
//   S  tiles (tm_t = 0):  kk  -- the walker forms kk*TM*8 with one shift (the
//                         sign and bucket bits shift out)
//   S' tiles (tm_t = TM): (kk/16)*TM*128 + (kk%16)*8 -- the byte offset of (kk, col 0)
//                         in the TMA S' tile layout (below); a lane's address is
//                         base_lane + ((e ^ 16*(lane%8)) & 0xffffff): one LOP3 + add
//   S' tiles (tm_t = -TM, transposed layout of 128-row tiles): kk*TM*8 | (kk%32)*8 --
//                         lane address st + (e & 0xffff00) + ((e & 248) ^ 8*lane)
// Group starts: gptr[c * gstride + g] = index of group g's first word.
__host__ __device__ inline uint32_t entry_addr(uint32_t kk, int tm_t) {
    if (tm_t < 0) return kk * (uint32_t)(-tm_t) * 8u + ((kk & 31u) << 3);
    return tm_t ? (kk >> 4) * (uint32_t)tm_t * 128u + ((kk & 15u) << 3) : kk;
}

// One CTA per chunk: sort the chunk's (bucket, local index) keys, emit
// bucket-tagged entry words, group terminators and group starts.
__global__ void sjlt_plan_kernel(const int32_t *__restrict__ pos, const int8_t *__restrict__ sgn,
                                 int64_t n, int d, int alpha, int tk, int p2, int db, int64_t ngroups,
                                 int64_t gstride, int64_t estride, int tm_t, int pair,
                                 uint32_t *__restrict__ gptr, uint32_t *__restrict__ ent, int *err) {
    extern __shared__ uint32_t keys[];
    const int64_t c = blockIdx.x;
    const int64_t k0 = c * tk;
    const int kc = (int)(n - k0 < tk ? n - k0 : tk);
    const int np = alpha / 2;  // paired plans: entries per input index
    const int cnt = kc * (pair ? np : alpha);
    const int64_t q0 = k0 * alpha;
    // paired key: group << 14 | combo << 8 | kk, group = slab * 16 + (pair mod
    // 4) * 4 + c1 / 2 (the consumer warp), combo = (c1 & 1) * 8 + c2
    const int gsh = pair ? 14 : 12;
    for (int i = threadIdx.x; i < p2; i += blockDim.x) {
        uint32_t key = 0xFFFFFFFFu;
        if (pair && i < cnt) {
            const int kk = i / np, pg = i - kk * np;
            const int b1 = pos[q0 + (int64_t)kk * alpha + 2 * pg] - 16 * pg;
            const int b2 = pos[q0 + (int64_t)kk * alpha + 2 * pg + 1] - 16 * pg - 8;
            if (b1 < 0 || b1 >= 8 || b2 < 0 || b2 >= 8) atomicOr(err, 2);
            const uint32_t grp = (uint32_t)((pg >> 2) * 16 + (pg & 3) * 4 + ((b1 & 7) >> 1));
            key = (grp << 14) | ((uint32_t)((b1 & 1) * 8 + (b2 & 7)) << 8) | (uint32_t)kk;
        } else if (i < cnt) {
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
    uint32_t *e_out = ent + c * estride;
    // padding after the last terminator (the walk loads, never uses, one word
    // past a terminator): null words
    for (int64_t e = cnt + ngroups + threadIdx.x; e < estride; e += blockDim.x) e_out[e] = 0u;
    // paired S' plans on TMA-landed tiles (tm_t > 0): within each (warp,
    // combo) run, entries of opposite input parity are emitted as adjacent
    // pairs (head word flagged, bit 29) ahead of the run's singles: the walker
    // reads a pair's two entries in one set of conflict-free loads (the
    // 8-byte half of a tile word is the index parity; see pipe_t_pair)
    const bool parity = pair && tm_t > 0;
    uint32_t *tw = keys + p2;  // parity: words in sorted order
    for (int e = threadIdx.x; e < cnt; e += blockDim.x) {
        const uint32_t key = keys[e];
        if (pair) {
            const uint32_t grp = key >> 14, kk = key & 255u, combo = (key >> 8) & 63u;
            const int pg = (int)((grp >> 4) * 4 + ((grp >> 2) & 3));
            const int64_t q = q0 + (int64_t)kk * alpha + 2 * pg;
            const uint32_t w = (sgn[q] < 0 ? 0x80000000u : 0u) | (combo << 24) |
                               (sgn[q + 1] < 0 ? 0x00800000u : 0u) | entry_addr(kk, tm_t);
            if (parity) tw[e] = w;
            else e_out[e + grp] = w;
            continue;
        }
        const uint32_t b = key >> 12;
        const int local = key & 4095;
        e_out[e + b / (uint32_t)db] = (sgn[q0 + local] < 0 ? 0x80000000u : 0u) | ((b % (uint32_t)db) << 24) |
                                      entry_addr((uint32_t)(local / alpha), tm_t);
    }
    if (parity) {
        __syncthreads();
        // one thread per run start: pairs (even, odd) first, then the rest
        for (int e = threadIdx.x; e < cnt; e += blockDim.x) {
            const uint32_t run = keys[e] >> 8;
            if (e > 0 && (keys[e - 1] >> 8) == run) continue;
            int end = e + 1;
            while (end < cnt && (keys[end] >> 8) == run) ++end;
            uint32_t *o = e_out + e + (run >> 6);  // + one terminator per earlier group
            int ie = e, io = e, w = 0;
            auto next_par = [&](int i, uint32_t par) {
                while (i < end && (keys[i] & 1u) != par) ++i;
                return i;
            };
            ie = next_par(ie, 0u);
            io = next_par(io, 1u);
            while (ie < end && io < end) {
                o[w++] = tw[ie] | (1u << 29);
                o[w++] = tw[io];
                ie = next_par(ie + 1, 0u);
                io = next_par(io + 1, 1u);
            }
            for (; ie < end; ie = next_par(ie + 1, 0u)) o[w++] = tw[ie];
            for (; io < end; io = next_par(io + 1, 1u)) o[w++] = tw[io];
        }
    }
    uint32_t *g_out = gptr + c * gstride;
    for (int64_t g = threadIdx.x; g < gstride; g += blockDim.x) {
        // lb(g) = number of keys with bucket < g * db
        int lb = cnt;
        if (g < ngroups) {
            const uint32_t target = pair ? (uint32_t)g << gsh : (uint32_t)(g * db) << 12;
            int lo = 0, hi = cnt;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (keys[mid] < target) lo = mid + 1; else hi = mid;
            }
            lb = lo;
        }
        const int64_t gg = g < ngroups ? g : ngroups;
        g_out[g] = (uint32_t)(lb + gg);
        // group g-1 ends where group g starts: its terminator
        if (g >= 1 && g <= ngroups) e_out[lb + g - 1] = (uint32_t)(pair ? 16 : db) << 24;
    }
}

// ------------------------------------------------------------------ apply
//
// Stage layout in shared memory (per ring slot):
//   [A tile: TK rows of TM doubles][zero row: TM doubles][bucket bounds]
//   [entries: estride words, then null words (kk = TK: the zero row)]
//
// Lane -> tile rows.  S tiles (dense, TMA-written): RPT = 2 -> rows 2l, 2l+1
// (one LDS.128); RPT = 4 -> rows 2l, 2l+1, 64+2l, 64+2l+1 (two LDS.128, each
// a contiguous 512 B).
// S' tiles (32/64 rows) hold A's natural layout (k contiguous) as TMA writes
// it: blocks of 16 input indices, one 128-byte row per output row, 128-byte
// swizzle -- element (kk, c) at (kk/16)*TM*128 + c*128 + ((kk%16)*8 ^ 16*(c%8)).
// Lane l owns output rows c = l + 32 r (LDS.64 each; 8-byte columns of a TMA
// tile cannot be spread over all 16 bank pairs, so these loads are 2-way
// conflicted -- the price of a transposition-free TMA producer).
// S' tiles of 128 rows (d <= 64: alpha-heavy, consumer-bound) are instead
// transposed on the way in by four cp.async producer warps: element (kk, c)
// at kk*TM + (c ^ (kk%32)) doubles -- conflict-free for the consumer.

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
    int64_t nchunks, gstride, estride;
    const uint32_t *gptr;  // group starts (plan)
    const uint32_t *ent;
    double scale;
    double *S;
    int64_t lds, col0;
    int nslabs, stages;
    int stage_bytes, zero_off, gs_off, en_off;
    // persistent balanced schedule: `groups` groups of nslabs CTAs split the
    // flattened (row tile, chunk) space of `units` chunks evenly; a row tile
    // cut between groups is summed by the group holding its first chunk
    int streamk, groups;
    int dbg;
    // TMA multicast: the nslabs CTAs of a row tile form a cluster of `mc`
    // CTAs; each loads 1/mc of every tile for all of them (1 = off)
    int mc;
    int wait_ns;  // consumer full-barrier wait: try_wait suspend hint (0 = default)
    int pf;  // mode 0: chunks prefetched into L2 beyond the shared-memory ring
    int64_t units;
    double *ws;  // per-CTA partial tile (SLAB x TM doubles)
    int *flags;  // per-CTA "partial published" flags (left zero)
};

// All NW warps own buckets (NW*DB per CTA slab) and share the producer work:
// warp 0 / lane 0 issues TMA + bulk copies (mode 0); in modes 1/2 every lane
// issues its share of 8-byte cp.async for the chunk STAGES-1 ahead.
template <int RPT, int DB, int NW, bool TRANS, bool PROD, bool SK, bool PAIR>
__global__ void __launch_bounds__((NW + (PROD ? (TRANS && RPT == 4 ? kXposeProducers : 1) : 0)) * 32, 1)
    sjlt_apply_kernel(const ApplyArgs p, const __grid_constant__ CUtensorMap tmap) {
    constexpr int TM = 32 * RPT;
    constexpr int SLAB = PAIR ? kPairSlab : NW * DB;
    constexpr bool XPOSE = TRANS && RPT == 4;       // transposed S' tile layout
    // (paired plans: warp (p, h) = 4p + h holds t1 buckets 16p + 2h + {0, 1}
    // in acc[.][0..1] and, once the quarters are folded into h = 0, the t2
    // buckets 16p + 8 + c2 in acc[.][2 + c2]; partials published / reduced
    // across CTAs keep the per-warp layout of the unpaired kernels)
    constexpr int PW = PROD ? (XPOSE ? kXposeProducers : 1) : 0;  // dedicated producer warps
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem);
    uint64_t *empty = full + 8;
    unsigned *done = reinterpret_cast<unsigned *>(full + 16);  // per-slot finished-warp counters
    int *sk = reinterpret_cast<int *>(smem + 192);  // stream-K roles (below)
    // stage ring from the first 1024-byte boundary past the 256-byte header
    // (the S' tile layout relies on the TMA 128-byte swizzle pattern)
    unsigned char *stage0 = smem + ((((smem_u32(smem) + 256u + 1023u) & ~1023u)) - smem_u32(smem));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ks = p.ksplit;
    int kr = 0;  // == %cluster_ctarank (cluster = ks consecutive CTAs)
    int slab;
    int64_t u0, u1;  // this CTA's chunks in the flattened (row tile, chunk) order
    int64_t tile0;   // row tile of the first chunk
    if (SK) {
        const int64_t grp = blockIdx.x / p.nslabs;
        slab = (int)(blockIdx.x % p.nslabs);
        u0 = grp * p.units / p.groups;
        u1 = (grp + 1) * p.units / p.groups;
        tile0 = u0 / p.nchunks;
    } else {
        kr = (int)(blockIdx.x % ks);
        const int64_t bid = blockIdx.x / ks;
        slab = (int)(bid % p.nslabs);
        const int64_t tile = bid / p.nslabs;
        const int64_t per = (p.nchunks + ks - 1) / ks;
        const int64_t c_begin = (int64_t)kr * per < p.nchunks ? (int64_t)kr * per : p.nchunks;
        const int64_t c_end = c_begin + per < p.nchunks ? c_begin + per : p.nchunks;
        u0 = tile * p.nchunks + c_begin;
        u1 = tile * p.nchunks + c_end;
        tile0 = tile;
    }
    const int j0 = slab * SLAB;
    const int nloc = (int)(u1 - u0);
    const int mode = p.mode;
    const int stages = p.stages;
    // this CTA's NW + 1 group starts (16-byte multiple for the bulk copy)
    const uint32_t gs_bytes = (uint32_t)((NW + 4) / 4 * 16);
    const int g0 = slab * NW;  // first warp group of the slab
    const uint32_t en_bytes = (uint32_t)p.estride * 4;
    const uint32_t tile_bytes = (uint32_t)p.tk * TM * 8;

    // null words after each chunk's list: the pipelined walk loads (never
    // accumulates) up to two entries past a warp's list -- they only need to
    // address the tile
    for (int s = 0; s < stages; ++s) {
        unsigned char *st = stage0 + (size_t)s * p.stage_bytes;
        if (threadIdx.x < 8) reinterpret_cast<uint32_t *>(st + p.en_off)[p.estride + threadIdx.x] = 0u;
    }
    const bool tma = mode == 0 || mode == 3;
    if (threadIdx.x == 0) {
        // TMA modes: one arrival (expect_tx); cp.async modes: every thread
        // of the (consumer) warps that share the copies, plus the issuer
        const uint32_t fcount = tma ? 1u : 1u + 32u * (PROD ? PW : NW);
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], fcount);
            mbar_init(&empty[s], (HSK_SJLT_MULTICAST || SK) ? NW * p.mc : NW);  // consumer warps of the cluster
            done[s] = 0;
        }
        fence_mbar_init();
        if (tma || mode == 4) prefetch_tmap(&tmap);
        if (mode == 4) mbar_init(full + 7, 1);  // staging buffer (stages <= 7 here)
        if (SK) {
            // sk[0]: the first segment is the tail of a tile (publish it);
            // sk[1], sk[2]: the last segment is the head of a tile cut by the
            // schedule -- count and first CTA of the later groups holding its
            // tails (stride nslabs); sk[3]: first row tile
            const int64_t grp = blockIdx.x / p.nslabs;
            const int64_t tb = (u1 - 1) / p.nchunks * p.nchunks;  // start of the last tile
            int nq = 0;
            if (u1 % p.nchunks != 0 && tb >= u0)
                for (int64_t q = grp + 1; q < p.groups && q * p.units / p.groups < tb + p.nchunks; ++q) ++nq;
            sk[0] = u0 % p.nchunks != 0;
            sk[1] = nq;
            sk[2] = (int)((grp + 1) * p.nslabs + slab);
            sk[3] = (int)tile0;
            if (DBG_IS(3))
                printf("sjlt dbg: cta %d grp %lld u0 %lld u1 %lld nloc %d sk %d %d %d %d stages %d\n",
                       (int)blockIdx.x, (long long)grp, (long long)u0, (long long)u1, nloc, sk[0], sk[1],
                       sk[2], sk[3], stages);
        }
    }
    __syncthreads();
    // multicast loads and remote releases target the peers' barriers: every
    // CTA of the cluster has initialised its ring before any of them issues
    if (MC_ON) cluster_sync();

    // ---- producer helpers
    // row offset and chunk index of the CTA's j-th chunk (stream-K: 32-bit
    // arithmetic, the host keeps units < 2^31)
    auto chunk_of = [&](int j, int64_t &r0, int64_t &c) {
        if constexpr (SK) {
            const uint32_t u = (uint32_t)u0 + (uint32_t)j;
            const uint32_t t = u / (uint32_t)p.nchunks;
            r0 = (int64_t)t * TM;
            c = u - t * (uint32_t)p.nchunks;
        } else {
            r0 = tile0 * TM;
            c = u0 - tile0 * p.nchunks + j;
        }
    };
    auto stage_of = [&](int j) { return stage0 + (size_t)(j % stages) * p.stage_bytes; };
    auto issue_tma = [&](int j) {  // warp 0, lane 0
        unsigned char *st = stage_of(j);
        uint64_t *bar = &full[j % stages];
        int64_t r0, c;
        chunk_of(j, r0, c);
        mbar_arrive_expect_tx(bar, tile_bytes + gs_bytes + en_bytes);
        if (MC_ON) {  // this CTA's share of the tile, for every CTA of the cluster
            const uint32_t rank = cluster_ctarank();
            const uint16_t mask = (uint16_t)((1u << p.mc) - 1u);
            if constexpr (TRANS) {
                for (int kb = (int)rank; kb < p.tk / 16; kb += p.mc)
                    tma_load_2d_mc(st + kb * TM * 128, &tmap, (int)(c * p.tk + kb * 16), (int)r0, bar,
                                   mask);
            } else {
                const int part = p.tk / p.mc;  // the box is TM x part
                tma_load_2d_mc(st + (size_t)rank * part * TM * 8, &tmap, (int)r0,
                               (int)(c * p.tk + rank * part), bar, mask);
            }
        } else if constexpr (TRANS) {  // S': one 16 x TM box per 16 input indices
            for (int kb = 0; kb < p.tk / 16; ++kb)
                tma_load_2d(st + kb * TM * 128, &tmap, (int)(c * p.tk + kb * 16), (int)r0, bar);
        } else {
            tma_load_2d(st, &tmap, (int)r0, (int)(c * p.tk), bar);
        }
        // keep the HBM stream ahead of the ring: chunk j + pf into L2 (chunks
        // stages .. stages+pf-1 are requested together with the first loads)
        const int jp = j < stages ? j + stages : j + p.pf;
        if (p.pf > 0 && jp < nloc && (j < stages ? j < p.pf : true)) {
            int64_t rp, cp;
            chunk_of(jp, rp, cp);
            const int part = p.tk / p.mc;
            tma_prefetch_2d(&tmap, (int)rp, (int)(cp * p.tk + (MC_ON ? cluster_ctarank() * part : 0)));
        }
        bulk_g2s(st + p.gs_off, p.gptr + c * p.gstride + g0, gs_bytes, bar);
        bulk_g2s(st + p.en_off, p.ent + c * p.estride, en_bytes, bar);
    };
    auto issue_coop = [&](int j, int ptid, int pnt) {  // threads [0, pnt) of the producer set
        unsigned char *st = stage_of(j);
        uint64_t *bar = &full[j % stages];
        int64_t r0, c;
        chunk_of(j, r0, c);
        const int64_t k0 = c * p.tk;
        const int kc = (int)(p.n - k0 < p.tk ? p.n - k0 : p.tk);
        if (ptid == 0) {
            mbar_arrive_expect_tx(bar, gs_bytes + en_bytes);
            bulk_g2s(st + p.gs_off, p.gptr + c * p.gstride + g0, gs_bytes, bar);
            bulk_g2s(st + p.en_off, p.ent + c * p.estride, en_bytes, bar);
        }
        double *sx = reinterpret_cast<double *>(st);
        const int nel = p.tk * TM;
        if (XPOSE) {
            // (kk, rr) = A[k0+kk, r0+rr] -> sx[kk*TM + (rr ^ (kk%32))]; lanes
            // along kk: coalesced reads, conflict-free swizzled writes
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
        } else if (TRANS) {
            // unaligned A: the S' tile layout of the TMA path, written by
            // 8-byte cp.async -- (kk, rr) at (kk/16)*TM*128 + rr*128 +
            // ((kk%16)*8 ^ 16*(rr%8)); lanes along kk (coalesced reads)
            const int tk = p.tk;
            for (int kk = ptid; kk < tk; kk += pnt) {
                const double *src = p.A + r0 * p.lda + k0 + kk;
                unsigned char *dbase = st + (kk >> 4) * TM * 128;
                const int kx = (kk & 15) << 3;
                const bool vk = kk < kc;
                for (int rr = 0; rr < TM; ++rr, src += p.lda) {
                    const bool v = vk && (r0 + rr < p.m_out);
                    cp_async8(dbase + rr * 128 + (kx ^ ((rr & 7) << 4)), v ? src : p.A, v);
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
        if (warp >= NW) {  // one TMA-issuing lane, or PW warps of transposing copies
            const int jn = DBG_IS(2) && nloc > stages ? stages : nloc;
            if (tma) {
                if (lane == 0) {
                    for (int j = 0; j < jn; ++j) {
                        if (j >= stages) mbar_wait(&empty[j % stages], (uint32_t)((j / stages) - 1) & 1u);
                        issue_tma(j);
                    }
                }
            } else if (XPOSE && mode == 4) {
                // transposed 128-row S' tiles of aligned A: one lane TMA-loads
                // the chunk in A's natural layout (16 x TM boxes, 128-byte
                // swizzle) into a staging buffer; the PW warps transpose it into
                // the ring slot (conflict-free for the consumers); a named
                // barrier among them frees the staging buffer for the next TMA
                const int ptid = threadIdx.x - NW * 32;
                unsigned char *stg = stage0 + (size_t)stages * p.stage_bytes;  // 1024-aligned
                uint64_t *stg_full = full + 7;
                auto issue_stg = [&](int j) {
                    int64_t r0, c;
                    chunk_of(j, r0, c);
                    mbar_arrive_expect_tx(stg_full, tile_bytes);
                    for (int kb = 0; kb < p.tk / 16; ++kb)
                        tma_load_2d(stg + kb * TM * 128, &tmap, (int)(c * p.tk + kb * 16), (int)r0, stg_full);
                };
                if (ptid == 0 && jn > 0) issue_stg(0);
                for (int j = 0; j < jn; ++j) {
                    const int s = j % stages;
                    unsigned char *st = stage0 + (size_t)s * p.stage_bytes;
                    if (j >= stages) mbar_wait(&empty[s], (uint32_t)((j / stages) - 1) & 1u);
                    if (ptid == 0) {
                        int64_t r0, c;
                        chunk_of(j, r0, c);
                        mbar_arrive_expect_tx(&full[s], gs_bytes + en_bytes);
                        bulk_g2s(st + p.gs_off, p.gptr + c * p.gstride + g0, gs_bytes, &full[s]);
                        bulk_g2s(st + p.en_off, p.ent + c * p.estride, en_bytes, &full[s]);
                    }
                    mbar_wait(stg_full, (uint32_t)(j & 1));
                    // (kk, kk+1) of column cc: one 16-byte load from the swizzled
                    // staging tile, two 8-byte stores at kk*TM + (cc ^ kk%32)
                    double *dst = reinterpret_cast<double *>(st);
                    for (int u = ptid; u < (p.tk / 2) * TM; u += PW * 32) {
                        const int cc = u % TM, kk = 2 * (u / TM);
                        const uint32_t off = (uint32_t)((kk >> 4) * TM * 128 + cc * 128) +
                                             ((uint32_t)((kk & 15) * 8) ^ ((uint32_t)(cc & 7) << 4));
                        const double2 v = *reinterpret_cast<const double2 *>(stg + off);
                        dst[kk * TM + (cc ^ (kk & 31))] = v.x;
                        dst[(kk + 1) * TM + (cc ^ ((kk + 1) & 31))] = v.y;
                    }
                    asm volatile("bar.sync 2, %0;" ::"r"(PW * 32) : "memory");  // staging read
                    if (ptid == 0 && j + 1 < jn) issue_stg(j + 1);
                    mbar_arrive(&full[s]);  // this thread's stores of slot s are done
                }
            } else {
                const int ptid = threadIdx.x - NW * 32;
                for (int j = 0; j < jn; ++j) {
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
            if (MC_ON) cluster_sync();  // peers stay alive for remote arrivals
            return;
        }
    } else if (tma) {
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
    // S' swizzle term of rows l + 32 r (TMA layout: 16-byte chunk; transposed: 8 bytes)
    const uint32_t lanex = XPOSE ? lane * 8u : (uint32_t)(lane & 7) << 4;
    // S: rows 2l, 2l+1 (+64) / l;  S': row l (TMA layout: 128 bytes per row)
    const uint32_t lane_off = XPOSE ? 0u : TRANS ? lane * 128u : lane * 8u * (RPT == 1 ? 1u : 2u);
    // epilogue: one final scaling, as the reference (`out *= scale`)
    auto store_tile = [&](const int64_t r0) {
    const bool vec_ok = ((p.lds & 1) == 0) && ((reinterpret_cast<uintptr_t>(p.S) & 15) == 0);
#pragma unroll
    for (int jj = 0; jj < (PAIR ? 10 : DB); ++jj) {
        if (PAIR && jj >= 2 && (warp & 3) != 0) break;
        const int j = PAIR ? j0 + (warp >> 2) * 16 + (jj < 2 ? 2 * (warp & 3) + jj : 6 + jj)
                           : j0 + warp * DB + jj;
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
    };

    // stream-K: loop index at which the current row-tile segment ends (the
    // rest of the bookkeeping is recomputed there, off the hot loop)
    int seg_end = SK ? (int)((tile0 + 1) * p.nchunks - u0) : 0;
    seg_end = seg_end < nloc ? seg_end : nloc;
    int ctile = (int)tile0;
    int cs = 0;
    uint32_t cph = 0;
    for (int i = 0; i < nloc; ++i) {
        // ---- producer duty (modes 1/2): chunk i + stages - 1 into the slot of
        // chunk i - 1, once every warp has finished chunk i - 1
        if (!PROD && !tma && issued < nloc) {
            const int j = issued;
            if (j >= stages) mbar_wait(&empty[j % stages], (uint32_t)((j / stages) - 1) & 1u);
            issue_coop(j, threadIdx.x, NW * 32);
            ++issued;
        }

        // ---- consume chunk i
        const int s = cs;
        if (!DBG_IS(2) || i < stages) {
            if (p.wait_ns) mbar_wait_hint(&full[s], cph, (uint32_t)p.wait_ns);
            else mbar_wait(&full[s], cph);
        }
        const uint32_t st = smem_base + (uint32_t)s * p.stage_bytes;
        const uint32_t sx = st + lane_off;
        const uint32_t sen = st + p.en_off;
        // shared address of the warp's group start (index of its first word)
        const uint32_t sbw = st + (uint32_t)p.gs_off + (uint32_t)(warp * 4);
#if HSK_SJLT_DEBUG
        if (DBG_IS(3)) {  // checked mode: the warp's list lies in the chunk and ends in its terminator
            const uint32_t *gs = reinterpret_cast<const uint32_t *>(stage0 + (size_t)s * p.stage_bytes + p.gs_off);
            const uint32_t *en = reinterpret_cast<const uint32_t *>(stage0 + (size_t)s * p.stage_bytes + p.en_off);
            const uint32_t b0 = gs[warp], b1 = gs[warp + 1];
            bool bad = b0 >= b1 || b1 > (uint32_t)p.estride || ((en[b1 - 1] >> 24) & 127u) != (uint32_t)DB;
            for (uint32_t q = b0; !bad && q + 1 < b1; ++q)
                bad = ((en[q] >> 24) & 127u) >= (uint32_t)DB ||
                      (q > b0 && ((en[q] >> 24) & 127u) < ((en[q - 1] >> 24) & 127u));
            if (bad) {
                printf("sjlt dbg: cta %d warp %d chunk-iter %d bad list [%u, %u) estride %d\n",
                       (int)blockIdx.x, warp, i, b0, b1, (int)p.estride);
                __trap();
            }
        }
#endif
        if (DBG_IS(1)) {
        } else if constexpr (PAIR && TRANS) {
            pipe_t_pair(acc, sen, sx, lanex, sbw);
        } else if constexpr (PAIR) {
            pipe_s_pair(acc, sen, sx, sbw);
        } else if constexpr (TRANS) {
            if constexpr (RPT == 1 && DB == 16) pipe_t_1x16(acc, sen, sx, lanex, sbw);
            else if constexpr (RPT == 1 && DB == 32) pipe_t_1x32(acc, sen, sx, lanex, sbw);
            else if constexpr (RPT == 2 && DB == 4) pipe_t_2x4(acc, sen, sx, lanex, sbw);
            else if constexpr (RPT == 2 && DB == 8) pipe_t_2x8(acc, sen, sx, lanex, sbw);
            else if constexpr (RPT == 2 && DB == 16) pipe_t_2x16(acc, sen, sx, lanex, sbw);
            else if constexpr (RPT == 4 && DB == 2) pipe_t_4x2(acc, sen, sx, lanex, sbw);
            else if constexpr (RPT == 4 && DB == 4) pipe_t_4x4(acc, sen, sx, lanex, sbw);
            else if constexpr (RPT == 4 && DB == 8) pipe_t_4x8(acc, sen, sx, lanex, sbw);
        } else {
            if constexpr (RPT == 1 && DB == 16) pipe_s_1x16(acc, sen, sx, sbw);
            else if constexpr (RPT == 1 && DB == 32) pipe_s_1x32(acc, sen, sx, sbw);
            else if constexpr (RPT == 2 && DB == 4) pipe_s_2x4(acc, sen, sx, sbw);
            else if constexpr (RPT == 2 && DB == 8) pipe_s_2x8(acc, sen, sx, sbw);
            else if constexpr (RPT == 2 && DB == 16) pipe_s_2x16(acc, sen, sx, sbw);
            else if constexpr (RPT == 4 && DB == 2) pipe_s_4x2(acc, sen, sx, sbw);
            else if constexpr (RPT == 4 && DB == 4) pipe_s_4x4(acc, sen, sx, sbw);
            else if constexpr (RPT == 4 && DB == 8) pipe_s_4x8(acc, sen, sx, sbw);
        }
        if constexpr (PAIR) {
            // a row tile ends here: fold quarters 1..3's chunk-t2 partials into
            // quarter 0 (in quarter order) through slot s, before its release
            if (SK ? i + 1 == seg_end : i + 1 == nloc) {
                constexpr int NT = NW * 32;
                double *red = reinterpret_cast<double *>(stage0 + (size_t)s * p.stage_bytes);
                const int h = warp & 3;
                bar_named(NT);  // every warp is done with the slot
                if (h > 0) {
#pragma unroll
                    for (int jj = 2; jj < 10; ++jj)
#pragma unroll
                        for (int r = 0; r < RPT; ++r) {
                            red[((warp * 8 + jj - 2) * RPT + r) * 32 + lane] = acc[r][jj];
                            acc[r][jj] = 0.0;
                        }
                }
                bar_named(NT);
                if (h == 0) {
                    for (int q = 1; q < 4; ++q)
#pragma unroll
                        for (int jj = 2; jj < 10; ++jj)
#pragma unroll
                            for (int r = 0; r < RPT; ++r)
                                acc[r][jj] += red[(((warp + q) * 8 + jj - 2) * RPT + r) * 32 + lane];
                }
                bar_named(NT);
            }
        }
        __syncwarp();
        if (lane == 0) {
            if (tma && !PROD) {
                // the last warp to finish chunk i refills its slot with chunk i + stages
                if (atomicAdd(&done[s], 1u) == NW - 1) {
                    done[s] = 0;
                    if (i + stages < nloc && !DBG_IS(2)) issue_tma(i + stages);
                }
            } else if (MC_ON) {
                // release the slot in every CTA of the cluster: no producer
                // multicasts into it until all of them are done with it
                for (int r = 0; r < p.mc; ++r) mbar_arrive_cluster(&empty[s], (uint32_t)r);
            } else {
                mbar_arrive(&empty[s]);
            }
        }
        if (++cs == stages) {
            cs = 0;
            cph ^= 1u;
        }
        if (SK && i + 1 == seg_end) {
            // segment of row tile `ctile` ends here; its role was fixed in the
            // prologue (sk[]): the first segment may be a tail to publish, the
            // last one a head that adds the later groups' tails in group order
            constexpr int NT = NW * 32;
            if (ctile == sk[3] && sk[0]) {
                double *w = p.ws + (size_t)blockIdx.x * (NW * DB * TM);
#pragma unroll
                for (int jj = 0; jj < DB; ++jj)
#pragma unroll
                    for (int r = 0; r < RPT; ++r)
                        __stcg(&w[((warp * DB + jj) * RPT + r) * 32 + lane], acc[r][jj]);
                __threadfence();
                bar_named(NT);
                if (threadIdx.x == 0) st_release_gpu(&p.flags[blockIdx.x], 1);
            } else {
                const int nq = i + 1 == nloc ? sk[1] : 0;
                for (int q = 0; q < nq; ++q) {
                    const int cq = sk[2] + q * p.nslabs;
                    if (threadIdx.x == 0) {
                        while (ld_acquire_gpu(&p.flags[cq]) == 0) __nanosleep(100);
                        p.flags[cq] = 0;
                    }
                    bar_named(NT);
                    const double *w = p.ws + (size_t)cq * (NW * DB * TM);
#pragma unroll
                    for (int jj = 0; jj < DB; ++jj)
#pragma unroll
                        for (int r = 0; r < RPT; ++r)
                            acc[r][jj] += __ldcg(&w[((warp * DB + jj) * RPT + r) * 32 + lane]);
                }
                store_tile((int64_t)ctile * TM);
            }
#pragma unroll
            for (int r = 0; r < RPT; ++r)
#pragma unroll
                for (int jj = 0; jj < DB; ++jj) acc[r][jj] = 0.0;
            ++ctile;
            seg_end = i + 1 + (int)p.nchunks < nloc ? i + 1 + (int)p.nchunks : nloc;
        }
    }
    if (SK) {
        if (MC_ON) cluster_sync();
        return;
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
    store_tile(tile0 * TM);
    if (MC_ON) cluster_sync();
}


template <int RPT, int DB, int NW, bool PAIR = false>
static int launch(ApplyArgs a, const Geom &g, cudaStream_t st) {
    constexpr int TM = 32 * RPT;
    constexpr int SLAB = PAIR ? kPairSlab : NW * DB;
    HSK_REQUIRE(g.tm == TM && g.db == DB && g.nw == NW, HSK_EINVAL, "sjlt: plan/config mismatch");
    const bool aligned = a.use_tma != 0;  // 16-byte aligned columns (lda even)
    // 0: TMA S tile; 1: cp.async S' tile (unaligned A); 2: cp.async S tile;
    // 3: TMA S' tile (16 x TM boxes, 128-byte swizzle)
    constexpr bool XPOSE = RPT == 4;  // (for S') transposed tile, cp.async producer
    // 4: TMA S' staging + in-smem transpose into the transposed 128-row tile
    a.mode = a.trans ? (aligned && a.tk % 16 == 0 ? (XPOSE ? 4 : 3) : 1) : (aligned ? 0 : 2);
    a.log2tk = 0;
    while ((1 << a.log2tk) < a.tk) ++a.log2tk;
    // S' tiles occupy whole 16-index blocks (the layout's unit); ring slots
    // start on 1024-byte boundaries
    const int a_bytes = (int)roundup((a.trans ? roundup(a.tk, 16) : a.tk) * (int64_t)TM * 8, 1024);
    a.zero_off = 0;
    a.gs_off = a_bytes;
    a.en_off = (int)roundup(a.gs_off + (NW + 4) / 4 * 16, 128);
    a.stage_bytes = (int)roundup(a.en_off + (a.estride + 8) * 4, 1024);
    // paired plans fold the quarters' t2 partials through the slot of a row
    // tile's last chunk: NW warps x 8 buckets x RPT x 32 lanes doubles (64 KB)
    // must lie inside that slot (the next slot may already hold a landed or
    // in-flight chunk)
    if (PAIR) a.stage_bytes = std::max(a.stage_bytes, (int)roundup((int64_t)NW * 8 * RPT * 32 * 8, 1024));
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
    // dedicated producer warp(s) (TMA issue for S, transposing copies for S');
    // a 33rd warp would cut the register budget to 56, so 32-warp CTAs refill
    // from the last consumer warp to release a slot instead
    bool prod = NW < 32;
    if (tuning().sjlt_prod >= 0) prod = tuning().sjlt_prod == 1;
    const int pw = a.trans && XPOSE ? kXposeProducers : 1;
    prod = prod && (a.mode == 0 || a.mode == 3 || ((a.mode == 1 || a.mode == 4) && XPOSE)) &&
           NW + pw <= 32;
    if (a.mode == 4 && !prod) a.mode = 1;  // the staging transpose needs the producer warps
    // persistent balanced schedule (stream-K) when whole-tile CTAs would
    // leave a partial last wave: one CTA per SM, groups of nslabs CTAs (the
    // slabs of a row tile stay in lockstep, so A is read from HBM once)
    const int sms = sm_count();
    const int64_t plain = ctas * ks;
    const int64_t waves = (plain + sms - 1) / sms;
    const double eff = (double)plain / (double)(waves * sms);
    a.units = tiles * a.nchunks;
    a.groups = (int)std::min<int64_t>(sms / a.nslabs, a.units);
    // (grids smaller than the GPU split k over a cluster instead: measured
    // better on C1, where stream-K's per-CTA fixups are a large share)
    a.streamk = eff < 0.9 && ctas >= sms;
    if (tuning().sjlt_streamk >= 0) a.streamk = tuning().sjlt_streamk == 1;
    a.streamk = a.streamk && a.groups >= 1 && a.nchunks > 0 && a.units < (1ll << 31);
    if (a.streamk) ks = 1;
    // TMA multicast across the slab CTAs of a row tile (they read the same
    // tile): a cluster of nslabs CTAs, each loading 1/nslabs of every tile for
    // all of them, cuts the L2 -> SM traffic by nslabs.  Opt-in only
    // (HSK_SJLT_MC=1): measured slower -- C2 S 0.58 vs 0.47 ms, d = 2048 S
    // 33.9 vs 5.9 ms -- because a slot is refilled only after every CTA of the
    // cluster released it, which runs the slab CTAs in lockstep behind the
    // slowest; without it each CTA runs ahead on its own and L2 absorbs the skew.
    a.mc = 1;
    // HSK_SJLT_MC=1: clusters of all nslabs slab CTAs; =2/4/8: clusters of that
    // many consecutive slabs of a row tile (nslabs a multiple of it)
    const int mc_req = tuning().sjlt_mc == 1 ? a.nslabs : tuning().sjlt_mc;
    if (HSK_SJLT_MULTICAST && mc_req >= 2 && prod && (a.mode == 0 || a.mode == 3) && ks == 1 &&
        (mc_req == 2 || mc_req == 4 || mc_req == 8) && a.nslabs % mc_req == 0 &&
        (a.mode == 3 || a.tk % mc_req == 0))
        a.mc = mc_req;
    CUtensorMap tmap;
    memset(&tmap, 0, sizeof(tmap));
    if (a.mode == 0) {
        int rc = make_tmap_f64_2d(&tmap, a.A, (uint64_t)a.m_out, (uint64_t)a.n, (uint64_t)a.lda,
                                  TM, (uint32_t)(a.tk / a.mc));
        if (rc) return rc;
    } else if (a.mode == 3 || a.mode == 4) {  // A is n x m_out: inner dimension = input index
        int rc = make_tmap_f64_2d(&tmap, a.A, (uint64_t)a.n, (uint64_t)a.m_out, (uint64_t)a.lda,
                                  16, TM, true);
        if (rc) return rc;
    }
    const int nthreads = (NW + (prod ? pw : 0)) * 32;
    const int budget = 226 * 1024;
    const int stg_bytes = a.mode == 4 ? a_bytes : 0;  // mode 4 staging buffer
    const int stages_max = std::max(2, std::min(7, (budget - 2048 - stg_bytes) / a.stage_bytes));
    if (a.streamk && a.mc > 1) {
        // every group is one cluster and groups wait on later groups: keep
        // the grid to the clusters that can be co-resident
        auto kprobe = a.trans ? sjlt_apply_kernel<RPT, DB, NW, true, true, true, PAIR>
                              : sjlt_apply_kernel<RPT, DB, NW, false, true, true, PAIR>;
        const int smem_max = 2048 + stages_max * a.stage_bytes;
        cudaError_t e = cudaFuncSetAttribute(kprobe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max);
        if (e != cudaSuccess) return cuda_status(e, "sjlt: set smem attribute");
        cudaLaunchConfig_t pc = {};
        pc.gridDim = dim3((unsigned)(a.groups * a.nslabs), 1, 1);
        pc.blockDim = dim3(nthreads, 1, 1);
        pc.dynamicSmemBytes = smem_max;
        cudaLaunchAttribute pa[1];
        pa[0].id = cudaLaunchAttributeClusterDimension;
        pa[0].val.clusterDim.x = a.mc;
        pa[0].val.clusterDim.y = 1;
        pa[0].val.clusterDim.z = 1;
        pc.attrs = pa;
        pc.numAttrs = 1;
        int nclusters = 0;
        e = cudaOccupancyMaxActiveClusters(&nclusters, kprobe, &pc);
        if (e != cudaSuccess) return cuda_status(e, "sjlt: cluster occupancy");
        if (nclusters < 1) {
            a.mc = 1;  // cannot place a cluster: plain launch
            int rc = make_tmap_f64_2d(&tmap, a.A, a.mode == 0 ? (uint64_t)a.m_out : (uint64_t)a.n,
                                      a.mode == 0 ? (uint64_t)a.n : (uint64_t)a.m_out, (uint64_t)a.lda,
                                      a.mode == 0 ? TM : 16, a.mode == 0 ? (uint32_t)a.tk : TM,
                                      a.mode == 3);
            if (rc) return rc;
        } else {
            a.groups = std::min(a.groups, nclusters);
        }
    }
    if (a.streamk) {
        void *ws = nullptr;
        int *flags = nullptr;
        const int nct = a.groups * a.nslabs;
        int rc = stream_workspace(st, (size_t)nct * NW * DB * TM * sizeof(double), nct, &ws, &flags);
        if (rc) return rc;
        a.ws = static_cast<double *>(ws);
        a.flags = flags;
    }
    a.ksplit = ks;
    const int per = (int)(a.streamk ? (a.units + a.groups - 1) / a.groups : (a.nchunks + ks - 1) / ks);
    a.stages = stages_max;
    if (tuning().sjlt_stages > 0) a.stages = std::max(2, std::min(a.stages, tuning().sjlt_stages));
    if (per > 0 && a.stages > per + 1) a.stages = std::max(2, per + 1);
    int smem = 2048 + a.stages * a.stage_bytes + stg_bytes;  // header + 1024-byte alignment slack
    if (ks > 1) smem = std::max(smem, 2048 + NW * DB * RPT * 32 * 8);
    auto kern = a.trans ? (prod ? (a.streamk ? sjlt_apply_kernel<RPT, DB, NW, true, true, true, PAIR>
                                             : sjlt_apply_kernel<RPT, DB, NW, true, true, false, PAIR>)
                                : (a.streamk ? sjlt_apply_kernel<RPT, DB, NW, true, false, true, PAIR>
                                             : sjlt_apply_kernel<RPT, DB, NW, true, false, false, PAIR>))
                        : (prod ? (a.streamk ? sjlt_apply_kernel<RPT, DB, NW, false, true, true, PAIR>
                                             : sjlt_apply_kernel<RPT, DB, NW, false, true, false, PAIR>)
                                : (a.streamk ? sjlt_apply_kernel<RPT, DB, NW, false, false, true, PAIR>
                                             : sjlt_apply_kernel<RPT, DB, NW, false, false, false, PAIR>));
    // L2 prefetch beyond the ring: off -- the duplicate requests cost power,
    // and sustained runs are power-capped (C2, 2000 launches: 0.505 ms
    // without, 0.540 ms with; no burst gain either).  HSK_SJLT_PF=<chunks>.
    a.pf = 0;
    // consumers waiting for a tile sleep up to 1 us per poll (measured neutral
    // to +1 %: fewer polling instructions under the power cap)
    a.wait_ns = tuning().sjlt_wait_ns >= 0 ? tuning().sjlt_wait_ns : 1000;
    a.dbg = std::max(0, tuning().sjlt_dbg);
    a.pf = std::max(0, tuning().sjlt_pf);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return cuda_status(e, "sjlt: set smem attribute");
    const int64_t grid = a.streamk ? (int64_t)a.groups * a.nslabs : tiles * a.nslabs * ks;
    HSK_REQUIRE(grid < (1ll << 31), HSK_EINVAL, "sjlt: grid too large");
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid, 1, 1);
    cfg.blockDim = dim3(nthreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    const int cdim = ks > 1 ? ks : a.mc;  // k-split and multicast never combine
    if (cdim > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = cdim;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    if (a.streamk && cdim == 1) {  // groups wait on later groups' partials: co-resident
        attr[na].id = cudaLaunchAttributeCooperative;
        attr[na].val.cooperative = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    e = cudaLaunchKernelEx(&cfg, kern, a, tmap);
    if (e != cudaSuccess) return cuda_status(e, "sjlt_apply_kernel launch");
    HSK_CHECK_LAUNCH("sjlt_apply_kernel");
    return HSK_OK;
}

}  // namespace sjlt
}  // namespace hsk

using namespace hsk;

extern "C" int64_t hsk_sjlt_plan_bytes_ex(int64_t n, int32_t d, int32_t alpha, int32_t flags) {
    if (n < 0 || d < 1 || alpha < 1 || d > sjlt::kMaxD || alpha > sjlt::kMaxChunkEntries ||
        (flags & ~HSK_SJLT_CHUNKED))
        return HSK_EINVAL;
    return sjlt::plan_geom(n, d, alpha, flags & HSK_SJLT_CHUNKED).bytes;
}

extern "C" int64_t hsk_sjlt_plan_bytes(int64_t n, int32_t d, int32_t alpha) {
    return hsk_sjlt_plan_bytes_ex(n, d, alpha, 0);
}

extern "C" int hsk_sjlt_plan_build(const int32_t *pos, const int8_t *sgn, int64_t n, int32_t d,
                                   int32_t alpha, void *plan, int64_t plan_bytes, void *stream) {
    return hsk_sjlt_plan_build_ex(pos, sgn, n, d, alpha, 0, plan, plan_bytes, stream);
}

extern "C" int hsk_sjlt_plan_build_ex(const int32_t *pos, const int8_t *sgn, int64_t n, int32_t d,
                                      int32_t alpha, int32_t flags, void *plan, int64_t plan_bytes,
                                      void *stream) {
    HSK_REQUIRE((flags & ~HSK_SJLT_CHUNKED) == 0, HSK_EINVAL, "sjlt plan: unknown flags %d", flags);
    HSK_REQUIRE(n >= 0 && d >= 1 && alpha >= 1, HSK_EINVAL,
                "sjlt plan: need n >= 0, d >= 1, alpha >= 1 (n=%lld d=%d alpha=%d)",
                (long long)n, d, alpha);
    HSK_REQUIRE(d <= sjlt::kMaxD, HSK_EINVAL, "sjlt plan: d=%d exceeds %lld", d,
                (long long)sjlt::kMaxD);
    HSK_REQUIRE(alpha <= sjlt::kMaxChunkEntries, HSK_EINVAL, "sjlt plan: alpha=%d too large", alpha);
    HSK_REQUIRE(n < (1ll << 31), HSK_EINVAL, "sjlt plan: n too large");
    const sjlt::Plan pl = sjlt::plan_geom(n, d, alpha, flags & HSK_SJLT_CHUNKED);
    HSK_REQUIRE(n == 0 || (sjlt::geom_ok(pl.s, alpha) && sjlt::geom_ok(pl.t, alpha)), HSK_EINVAL,
                "sjlt plan: no chunk geometry for d=%d alpha=%d (TK %d / %d)", d, alpha, pl.s.tk, pl.t.tk);
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
            while (p2 < g->tk * (g->pair ? alpha / 2 : alpha)) p2 <<= 1;
            sjlt::sjlt_plan_kernel<<<(unsigned)g->nchunks, 256, 2 * p2 * sizeof(uint32_t), st>>>(
                pos, sgn, n, d, alpha, g->tk, p2, g->db, g->ngroups, g->gstride, g->estride,
                g == &pl.t ? (g->rpt == 4 ? -g->tm : g->tm) : 0, g->pair,
                reinterpret_cast<uint32_t *>(base + g->gptr_off),
                reinterpret_cast<uint32_t *>(base + g->ent_off), reinterpret_cast<int *>(base + 28));
            HSK_CHECK_LAUNCH("sjlt_plan_kernel");
        }
        // the plan kernel flags positions outside [0, d) (bit 0) and, for
        // paired plans, entries outside their construction chunk (bit 1):
        // read the flags back (one stream sync, once per operator block)
        int err = 0;
        e = cudaMemcpyAsync(&err, base + 28, sizeof(int), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return cuda_status(e, "sjlt plan: check");
        if (err & 1) return set_error(HSK_ERANGE, "sjlt plan: pattern positions must lie in [0, %d)", d);
        if (err & 2)
            return set_error(HSK_EINVAL, "sjlt plan: HSK_SJLT_CHUNKED given for a pattern whose "
                                         "entry t is not in chunk t of d/alpha buckets");
    }
    return HSK_OK;
}

extern "C" int hsk_sjlt_apply(const double *A, int64_t rows, int64_t cols, int64_t lda,
                              int32_t trans, const void *plan, int64_t n, int32_t d,
                              int32_t alpha, double scale, double *S, int64_t lds, int64_t col0,
                              void *stream) {
    return hsk_sjlt_apply_ex(A, rows, cols, lda, trans, plan, n, d, alpha, 0, scale, S, lds, col0,
                             stream);
}

extern "C" int hsk_sjlt_apply_ex(const double *A, int64_t rows, int64_t cols, int64_t lda,
                                 int32_t trans, const void *plan, int64_t n, int32_t d,
                                 int32_t alpha, int32_t flags, double scale, double *S, int64_t lds,
                                 int64_t col0, void *stream) {
    HSK_REQUIRE((flags & ~HSK_SJLT_CHUNKED) == 0, HSK_EINVAL, "sjlt apply: unknown flags %d", flags);
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
    const sjlt::Plan pl = sjlt::plan_geom(n, d, alpha, flags & HSK_SJLT_CHUNKED);
    const sjlt::Geom &g = trans ? pl.t : pl.s;
    HSK_REQUIRE(n == 0 || sjlt::geom_ok(g, alpha), HSK_EINVAL,
                "sjlt apply: no chunk geometry for d=%d alpha=%d (TK %d)", d, alpha, g.tk);
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
    a.gstride = g.gstride;
    a.estride = g.estride;
    a.gptr = reinterpret_cast<const uint32_t *>(base + g.gptr_off);
    a.ent = reinterpret_cast<const uint32_t *>(base + g.ent_off);
    a.scale = scale;
    a.S = S;
    a.lds = lds;
    a.col0 = col0;
    cudaStream_t st = as_stream(stream);
    // the plan was built for this warp shape (warp_shape): one kernel each
    if (g.pair) return sjlt::launch<2, 16, 16, true>(a, g, st);
    const int shape = g.rpt * 1000 + g.db * 10 + (g.nw == 32);
    switch (shape) {
        case 1320: return sjlt::launch<1, 32, 16>(a, g, st);   // 32-row tiles, 512-bucket slabs
        case 4040: return sjlt::launch<4, 4, 16>(a, g, st);    // 128-row tiles, 64-bucket slabs
        case 2080: return sjlt::launch<2, 8, 16>(a, g, st);    // 64-row tiles
        case 2160: return sjlt::launch<2, 16, 16>(a, g, st);
#if HSK_TUNING  // 32-warp variants (HSK_SJLT_W32=1): spill, never selected by default
        case 1161: return sjlt::launch<1, 16, 32>(a, g, st);
        case 4021: return sjlt::launch<4, 2, 32>(a, g, st);
        case 2041: return sjlt::launch<2, 4, 32>(a, g, st);
        case 2081: return sjlt::launch<2, 8, 32>(a, g, st);
#endif
        default: return set_error(HSK_EINVAL, "sjlt apply: no kernel for rpt=%d db=%d nw=%d", g.rpt, g.db, g.nw);
    }
}
