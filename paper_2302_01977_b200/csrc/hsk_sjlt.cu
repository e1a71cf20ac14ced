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
// producer warps of the S' tiles transposed into the S layout (mode 5 / 6, below)
#ifndef HSK_XP2_PRODUCERS
#define HSK_XP2_PRODUCERS 4
#endif
constexpr int kXp2Producers = HSK_XP2_PRODUCERS;
// ... of 128-row tiles (their 4 x 4 accumulator blocks leave the registers for 24 warps)
#ifndef HSK_XP2_WIDE_DB
#define HSK_XP2_WIDE_DB 0
#endif
#ifndef HSK_XP2_PRODUCERS4
#define HSK_XP2_PRODUCERS4 8
#endif
constexpr int kXp2Producers4 = HSK_XP2_PRODUCERS4;
// (128-row tiles' 4 x 4 accumulator blocks leave the registers for 24 warps: eight producer
// warps measured 4-7 % faster than four -- n = 16384 d = 64 alpha = 4 S' 0.517 -> 0.493 ms,
// n = 65536 8.16 -> 7.65; 64-row tiles' 2 x 16 need the 96 registers of 20 warps, and 2 x 8
// (HSK_XP2_WIDE_DB=8) gains under 2 % from eight)
constexpr int xp2_pw(int rpt, int db) { return rpt == 4 || db <= HSK_XP2_WIDE_DB ? kXp2Producers4 : kXp2Producers; }
// mode 6 copy mapping: consecutive inputs per warp instruction (x 32 / KQ rows)
#ifndef HSK_XP6_KQ
#define HSK_XP6_KQ 4
#endif

// TMA multicast across slab clusters (opt-in at build time and run time,
// -DHSK_SJLT_MULTICAST=1 plus HSK_SJLT_MC=1): measured slower (see launch<>),
// and its remote-arrive branches cost the default kernels registers and
// scheduling even when not taken (d = 2048 S: 6.0 vs 5.45 ms), so production
// builds compile none of it.
#ifndef HSK_SJLT_MULTICAST
#define HSK_SJLT_MULTICAST 0
#endif
#define MC_ON (HSK_SJLT_MULTICAST && p.mc > 1)

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
    int even;          // group lists start at even words (S' on 64-row tiles: the
                       // walker fetches entry words in 8-byte pairs)
    int xp;            // S' on 64-row tiles transposed in shared memory into the S
                       // layout and walked by the S walkers (xp_rule below)
    int rpt;           // rows per lane (tile rows tm = 32 * rpt)
    int db, nw;        // buckets per consumer warp, consumer warps per CTA
    int64_t ngroups;   // warp groups of db buckets (nslabs * nw)
    int tm;
    int pitch;         // tile pitch (doubles) = tm: TMA writes densely; the S'
                       // producer orders its transposing stores conflict-free
    int tk;            // input indices per chunk
    int64_t nchunks;
    int64_t gstride;   // uint32 per group-start row (ngroups + 1, padded)
    int64_t estride;   // words per chunk row (tk*alpha entries + group terminators;
                       // even: every group list starts at an even word, so up to
                       // 2 * ngroups + 1 words besides the entries)
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
static inline void warp_shape(int rpt, int d, int trans, int &db, int &nw) {
#if HSK_TUNING
    const bool w32 = tuning().sjlt_w32 == 1;
#else
    const bool w32 = false;  // 32-warp variants are compiled only in tuning builds
#endif
    // S on 64-row tiles: more, narrower consumer warps hide more of the
    // walker's latency (slabs of 260 / 264 buckets; measured r02):
    // 20 x 13 for d <= 512, 24 x 11 above.  S' keeps 16 x 16 (its walk is
    // bound by the shared-memory port, and more warps measured slower).
    // HSK_SJLT_W32 = 16 / 20 / 24 forces a shape (28: tuning builds).
    const int ws = tuning().sjlt_w32;
    // 256 < d <= 384 (a light second slab): 128-bucket slabs (16 x 8) split
    // the buckets evenly -- with stream-K the CTAs of a light slab idle while
    // the full ones set the time.  Measured (n = 16384, S / S' ms): d = 300
    // 0.517 / 0.824 vs 0.715 / 1.034 on 256-bucket slabs, d = 320 0.521 / 0.806
    // vs 0.696 / 0.956, d = 384 0.536 / 0.678 vs 0.637 / 0.859; not for d in
    // (512, 640]: 0.742 vs 0.712.  HSK_SJLT_W32 = 8 forces it, 16 / 20 / 24
    // the wide shapes.
    if (rpt == 2 && d > 128 && !w32 && (ws == 8 || (ws < 16 && d > 256 && d <= 384))) {
        nw = 16;
        db = 8;
        return;
    }
    if (rpt == 2 && d > 128 && !w32 && ws != 16 && (!trans || (HSK_TUNING && ws >= 20))) {
        const int pick = ws >= 20 ? ws : d > 512 ? 24 : 20;
        if (pick == 20) { nw = 20; db = 13; return; }
        if (pick == 24) { nw = 24; db = 11; return; }
#if HSK_TUNING
        if (pick == 28) { nw = 28; db = 10; return; }
#endif
    }
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

// S' tiles transposed in shared memory (modes 5 / 6).  In shared-memory passes
// per staged element and slab CTA, with a = the element's entries in that slab:
// a TMA-landed natural-layout tile costs 1 + 2a (its 8-byte column reads are
// 2-way conflicted), a tile transposed into the S layout 3 + a (staging write,
// the transposer's read and write, conflict-free 16-byte reads).  S' is bound
// by that port, so the transposed tile wins from a = 4 on -- measured r02q,
// n = 16384, S' ms natural / transposed: d = 128 alpha = 4 0.536 / 0.494,
// d = 256 alpha = 8 1.062 / 0.757 (the 11 / 17 pass ratio); not the paired
// plans (C3: 8.39 / 8.73 -- their walk is issue-bound and loses more to the
// smaller chunk than the passes save) and not a <= 3 (d = 96 / 192 alpha = 3:
// 0.418 / 0.443 and 0.436 / 0.466; d = 128 alpha = 2: 0.348 / 0.433; C2, C5).
// 128-row tiles (d <= 64) always: their earlier producers (mode 4: one staging
// tile, the transposed XOR layout read with 8-byte loads) measured 7-14 %
// slower (n = 16384, S' ms: d = 64 alpha = 4 0.558 / 0.515, alpha = 2
// 0.499 / 0.429, d = 32 alpha = 4 0.571 / 0.497; n = 65536 d = 64 alpha = 4
// 8.09 / 7.48); mode 4 / 1 stay for HSK_SJLT_XP = 0.
// HSK_SJLT_XP = 0 / 1 forces the choice for every S' plan.
static inline int xp_rule(int trans, int rpt, int a_per_slab, int pair) {
    if (!trans || (rpt != 2 && rpt != 4)) return 0;
    if (tuning().sjlt_xp >= 0) return tuning().sjlt_xp != 0;
    return rpt == 4 || (!pair && a_per_slab >= 4);
}

static Geom geom_dir(int64_t n, int d, int alpha, int trans, int64_t base, int pair = 0) {
    Geom g;
    int tk;
    g.pair = pair;
    g.even = 0;
    g.xp = 0;
    if (pair) {
        constexpr int kStage3 = (226 * 1024 - 2048) / 3, kStage2 = (226 * 1024 - 2048) / 2;
        const int ae = alpha / 2;  // entries per input index
        g.rpt = 2;
        g.db = 16;
        g.nw = 16;
        g.ngroups = (int64_t)(d / kPairSlab) * g.nw;
        g.xp = xp_rule(trans, g.rpt, ae, 1);
        // (transposed S' tiles: two ring slots and the staging copy share the 226 KB)
        tk = g.xp ? tk_fit16(ae, 64, 256, kStage3, g.ngroups, g.nw)
           : n >= 8192 ? tk_fit16(ae, 64, 256, kStage2, g.ngroups, g.nw)
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
    // (even-start entry rows: 2 * ngroups + 1 words besides the entries --
    // passed to the TK fit as its group-word count)
    if (const int e = trans ? tuning().sjlt_rpt_t : tuning().sjlt_rpt; e == 2 || e == 4 || (HSK_TUNING && e == 1))
        g.rpt = e;
    warp_shape(g.rpt, d, trans, g.db, g.nw);
    g.ngroups = roundup(d, (int64_t)g.db * g.nw) / g.db;
    g.xp = xp_rule(trans, g.rpt, alpha / (int)(g.ngroups / g.nw), 0);
    g.even = trans && g.rpt == 2 && !g.xp;
    const int64_t gw = g.even ? 2 * g.ngroups + 1 : g.ngroups;
    if (d <= 64) {
        tk = wide && !trans ? tk_fit16(alpha, 128, 256, kStage2, gw, g.nw)
                            : tk_fit(alpha, 128, 128, kStage3, gw, g.nw);
    } else if (g.xp) {
        tk = tk_fit16(alpha, 64, 256, kStage3, gw, g.nw);
    } else {
        // (S on the 20 x 13 warps: TK 128 x 3 stages measured faster in bursts,
        // C2 0.439 vs 0.449 ms over 20 launches, but slower under the power cap,
        // 0.514 vs 0.494 ms over 2000: two stages of TK 208 kept)
        tk = wide ? tk_fit16(alpha, 64, 256, kStage2, gw, g.nw)
                  : tk_fit(alpha, 64, 128, kStage3, gw, g.nw);
    }
    if (const int e = trans ? tuning().sjlt_tk_t : tuning().sjlt_tk; e > 0) tk = e;
    g.tm = 32 * g.rpt;
    g.pitch = g.tm;
    g.tk = tk;
    g.nchunks = (n + g.tk - 1) / g.tk;
    g.gstride = roundup(g.ngroups + 4, 4);  // a CTA copies nw + 1 starts, 16-byte rows
    g.estride = roundup((int64_t)g.tk * alpha + gw, 4);  // 16-byte rows for the bulk copy
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
// Even plans (S' on 64-row tiles) start every group at an even word,
// (lb(g) + 2g + 1) & ~1 with lb(g) = entries of the chunk in groups < g (a
// list of cnt_g entries and its terminator ends at or before the next start),
// so the walker fetches entry words in 8-byte pairs; the gaps stay null words.
__host__ __device__ inline uint32_t entry_addr(uint32_t kk, int tm_t) {
    if (tm_t < 0) return kk * (uint32_t)(-tm_t) * 8u + ((kk & 31u) << 3);
    return tm_t ? (kk >> 4) * (uint32_t)tm_t * 128u + ((kk & 15u) << 3) : kk;
}

// One CTA per chunk: sort the chunk's (bucket, local index) keys, emit
// bucket-tagged entry words, group terminators and group starts.
__global__ void sjlt_plan_kernel(const int32_t *__restrict__ pos, const int8_t *__restrict__ sgn,
                                 int64_t n, int d, int alpha, int tk, int p2, int db, int64_t ngroups,
                                 int64_t gstride, int64_t estride, int tm_t, int pair, int even,
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
    // padding after the last terminator (the walk loads, never uses, up to two
    // words past a terminator): null words (the host zero-fills the plan; the
    // even rows' gaps stay null)
    if (!even)
        for (int64_t e = cnt + ngroups + threadIdx.x; e < estride; e += blockDim.x) e_out[e] = 0u;
    // first key index of group g (keys sorted; unpaired plans)
    auto lb_of = [&](int64_t g) {
        const uint32_t target = (uint32_t)(g * db) << 12;
        int lo = 0, hi = cnt;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (keys[mid] < target) lo = mid + 1; else hi = mid;
        }
        return lo;
    };
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
        const uint32_t grp = b / (uint32_t)db;
        int64_t at = e + grp;
        if (even) {
            const int lb = lb_of(grp);
            at = ((lb + 2 * (int64_t)grp + 1) & ~(int64_t)1) + (e - lb);
        }
        e_out[at] =
            (sgn[q0 + local] < 0 ? 0x80000000u : 0u) | ((b % (uint32_t)db) << 24) |
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
        if (!even) {
            g_out[g] = (uint32_t)(lb + gg);
            // group g-1 ends where group g starts: its terminator
            if (g >= 1 && g <= ngroups) e_out[lb + g - 1] = (uint32_t)(pair ? 16 : db) << 24;
        } else {
            g_out[g] = (uint32_t)((lb + 2 * gg + 1) & ~(int64_t)1);
            // group g's terminator after its entries
            if (g < ngroups) {
                const int64_t st = (lb + 2 * g + 1) & ~(int64_t)1;
                e_out[st + (lb_of(g + 1) - lb)] = (uint32_t)db << 24;
            }
        }
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

constexpr int kMaxGroups = 160;  // stream-K groups (<= SMs)

// n / d for 0 <= n < 2^31 by multiply-high and shift (d = 1: m = 0, the
// identity): the kernel prologue divides with it so its values stay on the
// warp-uniform datapath (a division routine's results land in per-lane
// registers, and a chunk loop bounded by them is divergent to ptxas)
struct FastDiv {
    uint32_t d, m, s;
};

static inline FastDiv make_fastdiv(uint32_t d) {
    FastDiv f{d, 0u, 0u};
    if (d > 1) {
        uint32_t l = 0;
        while ((1ull << l) < d) ++l;  // ceil(log2 d)
        const uint32_t p = 31 + l;
        f.m = (uint32_t)(((1ull << p) + d - 1) / d);
        f.s = p - 32;
    }
    return f;
}

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv &f) {
    return f.d == 1 ? n : __umulhi(n, f.m) >> f.s;
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
    int wait_ns;  // consumer full-barrier wait: try_wait suspend hint (ns)
    int pf;  // mode 0: chunks prefetched into L2 beyond the shared-memory ring
    int nbox, gbox;  // mode 5: staging groups, boxes (16 input indices x TM rows) per group
    int64_t units;
    FastDiv div_slabs, div_ks;
    int32_t per;                   // whole-tile CTAs: chunks per k-split rank
    // stream-K, per group g (host-computed): first chunk, first row tile,
    // chunks in the first segment, segments, and roles (bit 0: the first
    // segment is the tail of a cut tile; bits 1..: count of later groups
    // holding the tails of the tile the last segment heads)
    int32_t sk_g[kMaxGroups + 1][4];
    double *ws;  // per-CTA partial tile (SLAB x TM doubles)
    int *flags;  // per-CTA "partial published" flags (left zero)
};

// Control flow of the apply kernel (measured on C2 S: 72 BSSY in the round-1
// kernel, a chain link 6 instructions, 4 of them reconvergence markers).
// ptxas brackets a branch with BSSY/BSYNC reconvergence markers unless it can
// prove the predicate warp-uniform; it ignores bra.uni, and a word loaded from
// shared memory is per-lane to it, so every chain link and loop-back branch of
// a walker got brackets.  The 64-row walkers therefore pass their branch
// predicates through vote.sync.any (tools/gen_consumers.py), and the kernel
// keeps every loop around a walker provably uniform: chunk and segment counts
// come from launch constants through 32-bit fast divisions and host-computed
// stream-K tables (a 64-bit division is a called routine with a per-lane fast
// path), the chunk loop restarts its own counter per segment (an inner loop
// that continues the outer loop's counter is divergent to ptxas), the producer
// role test reads a broadcast warp index, and the consumers' epilogue stores
// through selected addresses (out-of-range rows and buckets go to a sink) with
// the k-split and paired-fold exchanges done by every warp.
// Per-CTA ring bookkeeping shared by the producer and consumer paths.
struct Ring {
    unsigned char *stage0;  // first ring slot (1024-byte aligned)
    uint64_t *full, *empty;
    int64_t u0, u1, tile0;  // chunk range in the flattened (row tile, chunk) order
    int nloc, stages, g0, slab;
    uint32_t gs_bytes, en_bytes, tile_bytes;
};

// sink of the epilogue's out-of-range stores
__device__ double g_sjlt_sink[32];

// row offset and chunk index of the CTA's j-th chunk (stream-K: 32-bit
// arithmetic, the host keeps units < 2^31)
template <int TM, bool SK>
__device__ __forceinline__ void chunk_of(const ApplyArgs &p, const Ring &R, int j, int64_t &r0, int64_t &c) {
    if constexpr (SK) {
        const uint32_t u = (uint32_t)R.u0 + (uint32_t)j;
        const uint32_t t = u / (uint32_t)p.nchunks;
        r0 = (int64_t)t * TM;
        c = u - t * (uint32_t)p.nchunks;
    } else {
        r0 = R.tile0 * TM;
        c = R.u0 - R.tile0 * p.nchunks + j;
    }
}

// one TMA tile (S) or 16 x TM boxes (S') plus the chunk's plan slice into
// the slot of chunk j, completing on its full barrier (one issuing lane)
template <int TM, bool TRANS, bool SK>
__device__ __forceinline__ void issue_tma(const ApplyArgs &p, const CUtensorMap *tmap, const Ring &R, int j) {
    unsigned char *st = R.stage0 + (size_t)(j % R.stages) * p.stage_bytes;
    uint64_t *bar = &R.full[j % R.stages];
    int64_t r0, c;
    chunk_of<TM, SK>(p, R, j, r0, c);
    mbar_arrive_expect_tx(bar, R.tile_bytes + R.gs_bytes + R.en_bytes);
    uint32_t mc_off = 0;
#if HSK_SJLT_MULTICAST
    if (p.mc > 1) {  // this CTA's share of the tile, for every CTA of the cluster
        const uint32_t rank = cluster_ctarank();
        const uint16_t mask = (uint16_t)((1u << p.mc) - 1u);
        if constexpr (TRANS) {
            for (int kb = (int)rank; kb < p.tk / 16; kb += p.mc)
                tma_load_2d_mc(st + kb * TM * 128, tmap, (int)(c * p.tk + kb * 16), (int)r0, bar, mask);
        } else {
            const int part = p.tk / p.mc;  // the box is TM x part
            tma_load_2d_mc(st + (size_t)rank * part * TM * 8, tmap, (int)r0, (int)(c * p.tk + rank * part),
                           bar, mask);
        }
        mc_off = rank * (uint32_t)(p.tk / p.mc);
    } else
#endif
    if constexpr (TRANS) {  // S': one 16 x TM box per 16 input indices
        for (int kb = 0; kb < p.tk / 16; ++kb)
            tma_load_2d(st + kb * TM * 128, tmap, (int)(c * p.tk + kb * 16), (int)r0, bar);
    } else {
        tma_load_2d(st, tmap, (int)r0, (int)(c * p.tk), bar);
    }
    // keep the HBM stream ahead of the ring: chunk j + pf into L2 (chunks
    // stages .. stages+pf-1 are requested together with the first loads)
    const int jp = j < R.stages ? j + R.stages : j + p.pf;
    if (p.pf > 0 && jp < R.nloc && (j < R.stages ? j < p.pf : true)) {
        int64_t rp, cp;
        chunk_of<TM, SK>(p, R, jp, rp, cp);
        tma_prefetch_2d(tmap, (int)rp, (int)(cp * p.tk + mc_off));
    }
    bulk_g2s(st + p.gs_off, p.gptr + c * p.gstride + R.g0, R.gs_bytes, bar);
    bulk_g2s(st + p.en_off, p.ent + c * p.estride, R.en_bytes, bar);
}

// cp.async producer of chunk j: threads [0, pnt) of the producer set
template <int TM, bool TRANS, bool XPOSE, bool SK, bool XP2 = false>
__device__ __forceinline__ void issue_coop(const ApplyArgs &p, const Ring &R, int j, int ptid, int pnt) {
    unsigned char *st = R.stage0 + (size_t)(j % R.stages) * p.stage_bytes;
    uint64_t *bar = &R.full[j % R.stages];
    int64_t r0, c;
    chunk_of<TM, SK>(p, R, j, r0, c);
    const int64_t k0 = c * p.tk;
    const int kc = (int)(p.n - k0 < p.tk ? p.n - k0 : p.tk);
    if (ptid == 0) {
        mbar_arrive_expect_tx(bar, R.gs_bytes + R.en_bytes);
        bulk_g2s(st + p.gs_off, p.gptr + c * p.gstride + R.g0, R.gs_bytes, bar);
        bulk_g2s(st + p.en_off, p.ent + c * p.estride, R.en_bytes, bar);
    }
    double *sx = reinterpret_cast<double *>(st);
    const int nel = p.tk * TM;
    if (XP2) {
        // mode 6 (unaligned A):
        // (kk, rr) = A[k0+kk, r0+rr] -> sx[kk*TM + rr], the dense S layout.  A warp copies 4 consecutive inputs x 8 consecutive rows
        // per instruction: every 32-byte sector it reads is used whole, and its
        // stores are four 64-byte runs (2-way conflicts; lanes along kk alone
        // would put all 32 stores on one bank pair)
        const int tk = p.tk;
        constexpr int KQ = HSK_XP6_KQ, RQ = 32 / KQ;  // inputs x rows per warp instruction
        const int kq = ptid % KQ, rq = (ptid / KQ) % RQ, pw = ptid >> 5, npw = pnt >> 5;
        const int nkg = (tk + KQ - 1) / KQ;
        const bool full_rows = r0 + TM <= p.m_out;
        for (int kg = pw; kg < nkg; kg += npw) {
            const int kk = kg * KQ + kq;
            if (kk >= tk) continue;
            const double *src = p.A + (r0 + rq) * p.lda + k0 + kk;
            double *dst = sx + kk * TM + rq;
            const int64_t step = (int64_t)RQ * p.lda;
            if (kk < kc && full_rows) {
#pragma unroll
                for (int rg = 0; rg < TM / RQ; ++rg, src += step, dst += RQ) cp_async8(dst, src, true);
            } else {
                const bool vk = kk < kc;
                for (int rg = 0; rg < TM / RQ; ++rg, src += step, dst += RQ) {
                    const bool v = vk && (r0 + rq + rg * RQ < p.m_out);
                    cp_async8(dst, v ? src : p.A, v);
                }
            }
        }
    } else if (XPOSE) {
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
}

// Barrier set-up (thread 0) and the null words after each slot's entry list.
__device__ __forceinline__ void ring_setup(const ApplyArgs &p, const CUtensorMap *tmap, const Ring R,
                                        uint32_t fcount, uint32_t ecount) {
    unsigned *done = reinterpret_cast<unsigned *>(R.full + 16);  // per-slot finished-warp counters
    // null words after each chunk's list: the pipelined walk loads (never
    // accumulates) up to two entries past a warp's list -- they only need to
    // address the tile
    for (int s = 0; s < R.stages; ++s) {
        unsigned char *st = R.stage0 + (size_t)s * p.stage_bytes;
        if (threadIdx.x < 8) reinterpret_cast<uint32_t *>(st + p.en_off)[p.estride + threadIdx.x] = 0u;
    }
    if (threadIdx.x != 0) return;
    for (int s = 0; s < R.stages; ++s) {
        mbar_init(&R.full[s], fcount);
        mbar_init(&R.empty[s], ecount);
        done[s] = 0;
    }
    mbar_init(R.empty + 7, ecount);  // sink of deferred releases (stages <= 7)
    if (p.mode == 5)
        for (int b = 0; b < p.nbox; ++b) mbar_init(R.full + 24 + b, 1);  // staging boxes
    fence_mbar_init();
    if (p.mode == 0 || p.mode == 3 || p.mode == 4 || p.mode == 5) prefetch_tmap(tmap);
    if (p.mode == 4) mbar_init(R.full + 7, 1);  // staging buffer (stages <= 7 here)
}

// Dedicated producer warp(s): refill a slot as soon as every consumer warp
// has released it (modes 0 / 3: one TMA-issuing lane; mode 4: TMA staging +
// PW transposing warps; mode 1: PW warps of transposing cp.async copies).
template <int TM, int PW, bool TRANS, bool XPOSE, bool SK, bool XP2 = false>
__device__ __forceinline__ void producer_warps(const ApplyArgs &p, const CUtensorMap *tmap, const Ring R) {
    const int lane = threadIdx.x & 31;
    const int ptid = threadIdx.x - (blockDim.x - PW * 32);
    const int jn = DBG_IS(2) && R.nloc > R.stages ? R.stages : R.nloc;
    const int stages = R.stages;
    if (p.mode == 0 || p.mode == 3) {
        if (lane == 0) {
            for (int j = 0; j < jn; ++j) {
                if (j >= stages) mbar_wait(&R.empty[j % stages], (uint32_t)((j / stages) - 1) & 1u);
                issue_tma<TM, TRANS, SK>(p, tmap, R, j);
            }
        }
    } else if (XP2 && p.mode == 5) {
        if constexpr (XP2) {
            // S' tiles in the S layout (64-row tiles, aligned A).  One lane
            // TMA-loads A's natural layout (boxes of 16 input indices x TM output
            // rows, 128-byte swizzle) into a staging ring of p.nbox groups of
            // p.gbox boxes that runs ahead of the slots: a group is refilled as
            // soon as it has been read (its boxes issued back to back: gbox x
            // 128 contiguous bytes per output row), so the loads in flight do
            // not depend on the chunk size.  The PW warps copy group after group
            // into the ring slot as [kk][row] with the rows contiguous, and the
            // consumers run the S walkers (one conflict-free 16-byte load per
            // entry).  Thread -> output row cc and index pairs q = ph + NPH i of
            // a box: a quarter-warp's 16-byte loads hit eight different chunks
            // of eight rows (conflict-free), a half-warp's 8-byte stores one
            // 128-byte line.
            constexpr int NPH = PW * 32 / TM;  // threads per output row
            constexpr int NP = 8 / NPH;        // index pairs per thread and box
            static_assert(PW * 32 % TM == 0 && 8 % NPH == 0, "xp2 transposer mapping");
            constexpr int BOX = TM * 128;      // bytes per staging box
            unsigned char *stg = R.stage0 + (size_t)stages * p.stage_bytes;  // 1024-aligned
            uint64_t *grp_full = R.full + 24;  // p.nbox barriers (<= 16)
            const int gb = p.gbox;             // boxes per group
            const int gpc = p.tk / (16 * gb);  // groups per chunk
            const int ngrp = p.nbox;
            const int total = jn * gpc;        // groups of this CTA's chunks
            // group g of the CTA's sequence -> chunk g / gpc, boxes (g % gpc) * gb ..
            auto issue_group = [&](int g, int buf) {
                const int j = g / gpc, q = g - j * gpc;
                int64_t r0, c;
                chunk_of<TM, SK>(p, R, j, r0, c);
                mbar_arrive_expect_tx(&grp_full[buf], (uint32_t)(gb * BOX));
                for (int i = 0; i < gb; ++i)
                    tma_load_2d(stg + (size_t)(buf * gb + i) * BOX, tmap, (int)(c * p.tk + (q * gb + i) * 16),
                                (int)r0, &grp_full[buf]);
            };
            if (ptid == 0)
                for (int g = 0; g < ngrp && g < total; ++g) issue_group(g, g);
            const int cc = ptid % TM, ph = ptid / TM;
            uint32_t so[NP];
#pragma unroll
            for (int i = 0; i < NP; ++i) so[i] = (uint32_t)(cc * 128 + (((ph + NPH * i) ^ (cc & 7)) << 4));
            int s = 0, buf = 0, g = 0;
            uint32_t eph = 1u;  // parity of the slot's previous release (first round: none)
            uint32_t bph = 0u;  // parity of the staging ring's current round
            for (int j = 0; j < jn; ++j) {
                unsigned char *st = R.stage0 + (size_t)s * p.stage_bytes;
                if (j >= stages) mbar_wait(&R.empty[s], eph);
                if (ptid == 0) {
                    int64_t r0, c;
                    chunk_of<TM, SK>(p, R, j, r0, c);
                    mbar_arrive_expect_tx(&R.full[s], R.gs_bytes + R.en_bytes);
                    bulk_g2s(st + p.gs_off, p.gptr + c * p.gstride + R.g0, R.gs_bytes, &R.full[s]);
                    bulk_g2s(st + p.en_off, p.ent + c * p.estride, R.en_bytes, &R.full[s]);
                }
                double *dst = reinterpret_cast<double *>(st) + cc;
                for (int q = 0; q < gpc; ++q, ++g) {
                    mbar_wait(&grp_full[buf], bph);
                    const unsigned char *src = stg + (size_t)buf * gb * BOX;
#pragma unroll 2
                    for (int b = 0; b < gb; ++b, src += BOX, dst += 16 * TM) {
                        double2 v[NP];
#pragma unroll
                        for (int i = 0; i < NP; ++i) v[i] = *reinterpret_cast<const double2 *>(src + so[i]);
#pragma unroll
                        for (int i = 0; i < NP; ++i) {
                            dst[(2 * (ph + NPH * i)) * TM] = v[i].x;
                            dst[(2 * (ph + NPH * i) + 1) * TM] = v[i].y;
                        }
                    }
                    asm volatile("bar.sync 2, %0;" ::"r"(PW * 32) : "memory");  // group read by every thread
                    if (ptid == 0 && g + ngrp < total) issue_group(g + ngrp, buf);
                    if (++buf == ngrp) {
                        buf = 0;
                        bph ^= 1u;
                    }
                }
                mbar_arrive(&R.full[s]);  // this thread's stores of slot s are done
                if (++s == stages) {
                    s = 0;
                    eph ^= 1u;
                }
            }
        }
    } else if (XPOSE && p.mode == 4) {
        // transposed 128-row S' tiles of aligned A: one lane TMA-loads the
        // chunk in A's natural layout (16 x TM boxes, 128-byte swizzle) into a
        // staging buffer; the PW warps transpose it into the ring slot
        // (conflict-free for the consumers); a named barrier among them frees
        // the staging buffer for the next TMA
        unsigned char *stg = R.stage0 + (size_t)stages * p.stage_bytes;  // 1024-aligned
        uint64_t *stg_full = R.full + 7;
        auto issue_stg = [&](int j) {
            int64_t r0, c;
            chunk_of<TM, SK>(p, R, j, r0, c);
            mbar_arrive_expect_tx(stg_full, R.tile_bytes);
            for (int kb = 0; kb < p.tk / 16; ++kb)
                tma_load_2d(stg + kb * TM * 128, tmap, (int)(c * p.tk + kb * 16), (int)r0, stg_full);
        };
        if (ptid == 0 && jn > 0) issue_stg(0);
        for (int j = 0; j < jn; ++j) {
            const int s = j % stages;
            unsigned char *st = R.stage0 + (size_t)s * p.stage_bytes;
            if (j >= stages) mbar_wait(&R.empty[s], (uint32_t)((j / stages) - 1) & 1u);
            if (ptid == 0) {
                int64_t r0, c;
                chunk_of<TM, SK>(p, R, j, r0, c);
                mbar_arrive_expect_tx(&R.full[s], R.gs_bytes + R.en_bytes);
                bulk_g2s(st + p.gs_off, p.gptr + c * p.gstride + R.g0, R.gs_bytes, &R.full[s]);
                bulk_g2s(st + p.en_off, p.ent + c * p.estride, R.en_bytes, &R.full[s]);
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
            mbar_arrive(&R.full[s]);  // this thread's stores of slot s are done
        }
    } else {
        for (int j = 0; j < jn; ++j) {
            if (j >= stages) mbar_wait(&R.empty[j % stages], (uint32_t)((j / stages) - 1) & 1u);
            issue_coop<TM, TRANS, XPOSE, SK, XP2>(p, R, j, ptid, PW * 32);
        }
    }
    __syncwarp();
    if (!SK) {  // match the consumers' barriers of the (k-split) epilogue
        __syncthreads();
        if (p.ksplit > 1) {
            cluster_sync();
            cluster_sync();
        }
    }
    if (MC_ON) cluster_sync();  // peers stay alive for remote arrivals
}

// stream-K hand-off of a cut row tile's partials (thread 0): wait for the
// flag of CTA cq and clear it for the next launch / publish this CTA's
__device__ __noinline__ void sk_take_flag(int *flag) {
    if (threadIdx.x == 0) {
        while (ld_acquire_gpu(flag) == 0) __nanosleep(100);
        *flag = 0;
    }
}
__device__ __noinline__ void sk_post_flag(int *flag, int pub) {
    if (pub && threadIdx.x == 0) st_release_gpu(flag, 1);
}

// All NW warps own buckets (NW*DB per CTA slab); PROD adds dedicated
// producer warps (TMA issue, or transposing copies for 128-row S' tiles);
// without them the consumers share the producer work (modes 1/2: every lane
// issues its share of 8-byte cp.async for the chunk STAGES-1 ahead).
// XP2: S' whose tiles the producer warps transpose into the S layout (modes
// 5 / 6): the producer side is S' (tensor map, chunk coordinates), the consumer
// side -- walker, lane -> row mapping, epilogue -- is S's.
template <int RPT, int DB, int NW, bool TRANS, bool PROD, bool SK, bool PAIR, bool XP2 = false>
__global__ void __launch_bounds__((NW + (PROD ? (XP2 ? xp2_pw(RPT, DB) : TRANS && RPT == 4 ? kXposeProducers : 1) : 0)) * 32, 1)
    sjlt_apply_kernel(const __grid_constant__ ApplyArgs p, const __grid_constant__ CUtensorMap tmap) {
    static_assert(!XP2 || (TRANS && PROD && (RPT == 2 || RPT == 4)), "xp2 kernels: S' on 64- / 128-row tiles with producer warps");
    constexpr int TM = 32 * RPT;
    constexpr int SLAB = PAIR ? kPairSlab : NW * DB;
    constexpr bool XPOSE = TRANS && RPT == 4 && !XP2;  // transposed S' tile layout (128-row tiles)
    constexpr bool CT = TRANS && !XP2;                 // consumers read an S' tile layout
    // (paired plans: warp (p, h) = 4p + h holds t1 buckets 16p + 2h + {0, 1}
    // in acc[.][0..1] and, once the quarters are folded into h = 0, the t2
    // buckets 16p + 8 + c2 in acc[.][2 + c2]; partials published / reduced
    // across CTAs keep the per-warp layout of the unpaired kernels)
    constexpr int PW = PROD ? (XP2 ? xp2_pw(RPT, DB) : XPOSE ? kXposeProducers : 1) : 0;  // dedicated producer warps
    constexpr int NT = NW * 32;
    constexpr int NJ = PAIR ? 10 : DB;  // accumulator columns in use
    // slot release: lane 0 of each consumer warp arrives (PROD: inline; the
    // other paths through release_lane0)
    constexpr bool LANE_REL = !PROD || HSK_SJLT_MULTICAST;
    extern __shared__ __align__(128) unsigned char smem[];
    Ring R;
    R.full = reinterpret_cast<uint64_t *>(smem);
    R.empty = R.full + 8;
    unsigned *done = reinterpret_cast<unsigned *>(R.full + 16);
    // stage ring from the first 1024-byte boundary past the 512-byte header
    // (the S' tile layout relies on the TMA 128-byte swizzle pattern)
    R.stage0 = smem + ((((smem_u32(smem) + 512u + 1023u) & ~1023u)) - smem_u32(smem));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ks = p.ksplit;
    int kr = 0;  // == %cluster_ctarank (cluster = ks consecutive CTAs)
    // (32-bit index arithmetic on launch constants: fast divisions and host
    // tables instead of a division routine; the chunk and segment loops must
    // be warp-uniform to ptxas -- a loop whose bound may differ between lanes
    // is divergent, and so is every walker branch inside it)
    const uint32_t bx = blockIdx.x, nch = (uint32_t)p.nchunks;
    int grp = 0, nloc, nseg, seg_end;
    int sk_tail = 0, sk_nq = 0;
    if (SK) {
        grp = (int)fdiv(bx, p.div_slabs);
        R.slab = (int)(bx - (uint32_t)grp * p.div_slabs.d);
        R.u0 = p.sk_g[grp][0];
        R.u1 = p.sk_g[grp + 1][0];
        R.tile0 = p.sk_g[grp][1];
        seg_end = p.sk_g[grp][2];
        nseg = p.sk_g[grp][3] & 0xffff;
        sk_tail = (p.sk_g[grp][3] >> 16) & 1;
        sk_nq = p.sk_g[grp][3] >> 17;
        nloc = (int)(R.u1 - R.u0);
    } else {
        const uint32_t bid = fdiv(bx, p.div_ks);
        kr = (int)(bx - bid * (uint32_t)ks);
        const uint32_t tile = fdiv(bid, p.div_slabs);
        R.slab = (int)(bid - tile * p.div_slabs.d);
        const uint32_t per = (uint32_t)p.per;
        const uint32_t kb = (uint32_t)kr * per;
        const uint32_t c_begin = kb < nch ? kb : nch;
        const uint32_t c_end = c_begin + per < nch ? c_begin + per : nch;
        R.u0 = (int64_t)tile * nch + c_begin;
        R.u1 = (int64_t)tile * nch + c_end;
        R.tile0 = tile;
        nloc = (int)(c_end - c_begin);
        nseg = 1;
        seg_end = nloc;
    }
    // loop bounds broadcast from lane 0: warp-uniform to ptxas whatever
    // datapath computed them
    nloc = __shfl_sync(0xffffffffu, nloc, 0);
    nseg = __shfl_sync(0xffffffffu, nseg, 0);
    seg_end = __shfl_sync(0xffffffffu, seg_end, 0);
    sk_nq = __shfl_sync(0xffffffffu, sk_nq, 0);
    const int j0 = R.slab * SLAB;
    R.nloc = nloc;
    const int stages = p.stages;
    R.stages = stages;
    R.g0 = R.slab * NW;  // first warp group of the slab
    // this CTA's NW + 1 group starts (16-byte multiple for the bulk copy)
    R.gs_bytes = (uint32_t)((NW + 4) / 4 * 16);
    R.en_bytes = (uint32_t)p.estride * 4;
    R.tile_bytes = (uint32_t)p.tk * TM * 8;
    const int64_t tile0 = R.tile0;
    const bool tma = p.mode == 0 || p.mode == 3;
    // stream-K: the later groups holding the tails of the tile this CTA's
    // last segment heads start at CTA sk_cq (stride nslabs)
    const int sk_cq = (grp + 1) * p.nslabs + R.slab;
    if (SK && DBG_IS(3) && threadIdx.x == 0)
        printf("sjlt dbg: cta %d grp %d u0 %lld u1 %lld nloc %d nseg %d seg0 %d tail %d nq %d stages %d\n",
               (int)blockIdx.x, grp, (long long)R.u0, (long long)R.u1, nloc, nseg, seg_end, sk_tail, sk_nq,
               p.stages);
    {
        // TMA modes: one arrival (expect_tx); cp.async modes: every thread
        // of the (consumer) warps that share the copies, plus the issuer
        const uint32_t fcount = tma ? 1u : 1u + 32u * (PROD ? PW : NW);
        const uint32_t ecount = (uint32_t)(NW * p.mc);  // consumer warps of the cluster
        ring_setup(p, &tmap, R, fcount, ecount);
    }
    __syncthreads();
    // multicast loads and remote releases target the peers' barriers: every
    // CTA of the cluster has initialised its ring before any of them issues
    if (MC_ON) cluster_sync();

    if constexpr (PROD) {
        // (role test on a broadcast warp index: warp-uniform to ptxas)
        if (__shfl_sync(0xffffffffu, warp, 0) >= NW) {
            producer_warps<TM, PW, TRANS, XPOSE, SK, XP2>(p, &tmap, R);
            return;
        }
    }
    int issued = 0;
    if constexpr (!PROD) {
        if (tma) {
            if (warp == 0 && lane == 0)
                for (; issued < nloc && issued < stages; ++issued) issue_tma<TM, TRANS, SK>(p, &tmap, R, issued);
        } else {
            for (; issued < nloc && issued < stages - 1; ++issued)
                issue_coop<TM, TRANS, XPOSE, SK, XP2>(p, R, issued, threadIdx.x, NT);
        }
    }

    double acc[RPT][DB];
#pragma unroll
    for (int r = 0; r < RPT; ++r)
#pragma unroll
        for (int jj = 0; jj < DB; ++jj) acc[r][jj] = 0.0;

    const uint32_t smem_base = smem_u32(R.stage0);
    // S' swizzle term of rows l + 32 r (TMA layout: 16-byte chunk; transposed: 8 bytes)
    const uint32_t lanex = XPOSE ? lane * 8u : (uint32_t)(lane & 7) << 4;
    // S: rows 2l, 2l+1 (+64) / l;  S': row l (TMA layout: 128 bytes per row)
    const uint32_t lane_off = XPOSE ? 0u : CT ? lane * 128u : lane * 8u * (RPT == 1 ? 1u : 2u);

    // Epilogue: one store per accumulator, every one executed: to S scaled
    // once (the reference's `out *= scale`) -- rows past m_out and buckets
    // past d (or a paired quarter's folded-away t2 buckets) to the sink --
    // or, pubw != nullptr, the raw partial into the CTA's stream-K slot.
    auto store_acc = [&](const int64_t r0, double *pubw) {
        const bool pub = pubw != nullptr;
#pragma unroll
        for (int jj = 0; jj < NJ; ++jj) {
            const int j = PAIR ? j0 + (warp >> 2) * 16 + (jj < 2 ? 2 * (warp & 3) + jj : 6 + jj)
                               : j0 + warp * DB + jj;
            const bool jok = j < p.d && (!PAIR || jj < 2 || (warp & 3) == 0);
            double *col = p.S + (p.col0 + j) * p.lds;
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
                int64_t row;
                if (CT) row = r0 + lane + 32 * r;                // lane owns rows lane + 32 r
                else if (RPT == 1) row = r0 + lane;
                else row = r0 + 64 * (r >> 1) + 2 * lane + (r & 1);  // rows 2l, 2l+1 (+64)
                double *dst = pub ? pubw + ((warp * DB + jj) * RPT + r) * 32 + lane
                                  : (jok && row < p.m_out ? col + row : g_sjlt_sink + lane);
                __stcg(dst, pub ? acc[r][jj] : acc[r][jj] * p.scale);
            }
        }
    };
    // lane-0 slot release (paths with LANE_REL): arrive, or (no dedicated
    // producer, TMA) let the last warp to finish chunk ic refill its slot
    auto release_lane0 = [&](const int s, const int ic) {
        __syncwarp();
        if (lane == 0) {
            if (tma && !PROD) {
                if (atomicAdd(&done[s], 1u) == NW - 1) {
                    done[s] = 0;
                    if (ic + stages < nloc && !DBG_IS(2)) issue_tma<TM, TRANS, SK>(p, &tmap, R, ic + stages);
                }
            } else if (MC_ON) {
                // release the slot in every CTA of the cluster: no producer
                // multicasts into it until all of them are done with it
                for (int q = 0; q < p.mc; ++q) mbar_arrive_cluster(&R.empty[s], (uint32_t)q);
            } else {
                mbar_arrive(&R.empty[s]);
            }
        }
    };

    // Segments: stream-K CTAs walk consecutive row tiles (the first may be
    // the tail of a tile cut by the schedule, the last its head); whole-tile
    // CTAs one tile.
    int cs = 0;
    uint32_t cph = 0;
    int i = 0;  // chunks consumed before the current segment
    // (the chunk loop restarts its own counter per segment: an inner loop
    // continuing the outer loop's counter is divergent to ptxas)
#pragma unroll 1
    for (int seg = 0; seg < nseg; ++seg) {
        const int seg_len = seg == 0 ? seg_end : (nloc - i < (int)nch ? nloc - i : (int)nch);
#pragma unroll 1
        for (int k = 0; k < seg_len; ++k) {
            const int ic = i + k;  // chunk index
            // ---- producer duty (no producer warps, modes 1/2): chunk
            // i + stages - 1 into the slot of chunk i - 1, once every warp
            // has finished chunk i - 1
            if constexpr (!PROD) {
                if (!tma && issued < nloc) {
                    const int j = issued;
                    if (j >= stages) mbar_wait(&R.empty[j % stages], (uint32_t)((j / stages) - 1) & 1u);
                    issue_coop<TM, TRANS, XPOSE, SK, XP2>(p, R, j, threadIdx.x, NT);
                    ++issued;
                }
            }
            // ---- consume chunk i
            const int s = cs;
            if (!DBG_IS(2) || ic < stages) mbar_wait_hint(&R.full[s], cph, (uint32_t)p.wait_ns);
            const uint32_t st = smem_base + (uint32_t)s * p.stage_bytes;
            const uint32_t sx = st + lane_off;
            const uint32_t sen = st + p.en_off;
            // shared address of the warp's group start (index of its first word)
            const uint32_t sbw = st + (uint32_t)p.gs_off + (uint32_t)(warp * 4);
#if HSK_SJLT_DEBUG
            if (DBG_IS(3)) {  // checked mode: the warp's list lies in the chunk and ends in its terminator
                const uint32_t *gs = reinterpret_cast<const uint32_t *>(R.stage0 + (size_t)s * p.stage_bytes + p.gs_off);
                const uint32_t *en = reinterpret_cast<const uint32_t *>(R.stage0 + (size_t)s * p.stage_bytes + p.en_off);
                const uint32_t b0 = gs[warp], b1 = gs[warp + 1];
                // (unpaired lists start at even words: a null word may follow
                // the terminator)
                uint32_t q = b0;
                bool bad = b0 >= b1 || b1 > (uint32_t)p.estride;
                for (; !bad && q < b1 && ((en[q] >> 24) & 127u) != (uint32_t)DB; ++q)
                    bad = ((en[q] >> 24) & 127u) > (uint32_t)DB ||
                          (q > b0 && ((en[q] >> 24) & 127u) < ((en[q - 1] >> 24) & 127u));
                bad = bad || q >= b1 || (CT && RPT == 2 && !PAIR && (b0 & 1u));
                if (bad) {
                    printf("sjlt dbg: cta %d warp %d chunk-iter %d bad list [%u, %u) estride %d\n",
                           (int)blockIdx.x, warp, ic, b0, b1, (int)p.estride);
                    __trap();
                }
            }
#endif
            if (DBG_IS(1)) {
            } else if constexpr (PAIR && CT) {
                pipe_t_pair(acc, sen, sx, lanex, sbw);
            } else if constexpr (PAIR) {
                pipe_s_pair(acc, sen, sx, sbw);
            } else if constexpr (CT) {
                if constexpr (RPT == 1 && DB == 16) pipe_t_1x16(acc, sen, sx, lanex, sbw);
                else if constexpr (RPT == 1 && DB == 32) pipe_t_1x32(acc, sen, sx, lanex, sbw);
                else if constexpr (RPT == 2 && DB == 4) pipe_t_2x4(acc, sen, sx, lanex, sbw);
                else if constexpr (RPT == 2 && DB == 8) pipe_t_2x8(acc, sen, sx, lanex, sbw);
                else if constexpr (RPT == 2 && DB == 16) pipe_t_2x16(acc, sen, sx, lanex, sbw);
                else if constexpr (RPT == 2 && DB == 10) pipe_t_2x10(acc, sen, sx, lanex, sbw);
                else if constexpr (RPT == 2 && DB == 11) pipe_t_2x11(acc, sen, sx, lanex, sbw);
                else if constexpr (RPT == 2 && DB == 13) pipe_t_2x13(acc, sen, sx, lanex, sbw);
                else if constexpr (RPT == 4 && DB == 2) pipe_t_4x2(acc, sen, sx, lanex, sbw);
                else if constexpr (RPT == 4 && DB == 4) pipe_t_4x4(acc, sen, sx, lanex, sbw);
                else if constexpr (RPT == 4 && DB == 8) pipe_t_4x8(acc, sen, sx, lanex, sbw);
            } else {
                if constexpr (RPT == 1 && DB == 16) pipe_s_1x16(acc, sen, sx, sbw);
                else if constexpr (RPT == 1 && DB == 32) pipe_s_1x32(acc, sen, sx, sbw);
                else if constexpr (RPT == 2 && DB == 4) pipe_s_2x4(acc, sen, sx, sbw);
                else if constexpr (RPT == 2 && DB == 8) pipe_s_2x8(acc, sen, sx, sbw);
                else if constexpr (RPT == 2 && DB == 16) pipe_s_2x16(acc, sen, sx, sbw);
                else if constexpr (RPT == 2 && DB == 10) pipe_s_2x10(acc, sen, sx, sbw);
                else if constexpr (RPT == 2 && DB == 11) pipe_s_2x11(acc, sen, sx, sbw);
                else if constexpr (RPT == 2 && DB == 13) pipe_s_2x13(acc, sen, sx, sbw);
                else if constexpr (RPT == 4 && DB == 2) pipe_s_4x2(acc, sen, sx, sbw);
                else if constexpr (RPT == 4 && DB == 4) pipe_s_4x4(acc, sen, sx, sbw);
                else if constexpr (RPT == 4 && DB == 8) pipe_s_4x8(acc, sen, sx, sbw);
            }
            // ---- release the slot (a paired plan folds its quarters through
            // the slot of a row tile's last chunk: that release waits for the
            // fold; meanwhile lane 0 arrives on the sink barrier)
            if constexpr (!LANE_REL) {
                __syncwarp();
                if (lane == 0) mbar_arrive(PAIR && k + 1 == seg_len ? R.empty + 7 : &R.empty[s]);
            } else {
                if (!PAIR || k + 1 < seg_len) release_lane0(s, ic);
            }
            if (++cs == stages) {
                cs = 0;
                cph ^= 1u;
            }
        }
        i += seg_len;
        if constexpr (PAIR) {
            // a row tile ends here: fold quarters 1..3's chunk-t2 partials into
            // quarter 0 (in quarter order) through the slot of the tile's last
            // chunk, then release it.  Every warp stores and loads (quarter 0's
            // stores are never read; the other quarters add nothing).
            const int sl = cs == 0 ? stages - 1 : cs - 1;
            double *red = reinterpret_cast<double *>(R.stage0 + (size_t)sl * p.stage_bytes);
            const int h = warp & 3;
            bar_named(NT);  // every warp is done with the slot
#pragma unroll
            for (int jj = 2; jj < 10; ++jj)
#pragma unroll
                for (int r = 0; r < RPT; ++r) {
                    red[((warp * 8 + jj - 2) * RPT + r) * 32 + lane] = acc[r][jj];
                    acc[r][jj] = h > 0 ? 0.0 : acc[r][jj];
                }
            bar_named(NT);
            for (int q = 1; q < 4; ++q)
#pragma unroll
                for (int jj = 2; jj < 10; ++jj)
#pragma unroll
                    for (int r = 0; r < RPT; ++r) {
                        const double v = red[((((warp & ~3) + q) * 8 + jj - 2) * RPT + r) * 32 + lane];
                        acc[r][jj] += h == 0 ? v : 0.0;
                    }
            bar_named(NT);
            if constexpr (!LANE_REL) { if (lane == 0) mbar_arrive(&R.empty[sl]); }
            else release_lane0(sl, i - 1);
        }
        if constexpr (SK) {
            // segment of row tile tile0 + seg ends here: the first segment may
            // be a tail to publish, the last one a head that adds the later
            // groups' tails in group order
            const int pub = seg == 0 && sk_tail;
            const int nq = seg == nseg - 1 && !pub ? sk_nq : 0;
            for (int q = 0; q < nq; ++q) {
                const int cq = sk_cq + q * p.nslabs;
                sk_take_flag(&p.flags[cq]);
                bar_named(NT);
                const double *w = p.ws + (size_t)cq * (NW * DB * TM);
#pragma unroll
                for (int jj = 0; jj < NJ; ++jj)
#pragma unroll
                    for (int r = 0; r < RPT; ++r)
                        acc[r][jj] += __ldcg(&w[((warp * DB + jj) * RPT + r) * 32 + lane]);
            }
            store_acc((tile0 + seg) * TM, pub ? p.ws + (size_t)blockIdx.x * (NW * DB * TM) : nullptr);
            __threadfence();
            bar_named(NT);
            sk_post_flag(&p.flags[blockIdx.x], pub);
#pragma unroll
            for (int r = 0; r < RPT; ++r)
#pragma unroll
                for (int jj = 0; jj < DB; ++jj) acc[r][jj] = 0.0;
        }
    }
    if constexpr (SK) {
        if (MC_ON) cluster_sync();
        return;
    }

    // ------------------------------------------- k-split: DSMEM reduction
    // Partial sums of the ks CTAs of a cluster are combined by rank 0 in
    // rank order (deterministic).  The stage ring is reused as the buffer.
    // Every CTA stores its partial and reads its peers' (rank 0 adds them;
    // with ks = 1 the cluster is the CTA itself and nothing is read).
    {
        double *red = reinterpret_cast<double *>(R.stage0);
        __syncthreads();  // every stage consumed: the ring is free
#pragma unroll
        for (int jj = 0; jj < DB; ++jj)
#pragma unroll
            for (int r = 0; r < RPT; ++r) red[((warp * DB + jj) * RPT + r) * 32 + lane] = acc[r][jj];
        if (ks > 1) cluster_sync();
        for (int q = 1; q < ks; ++q) {
#pragma unroll
            for (int jj = 0; jj < DB; ++jj)
#pragma unroll
                for (int r = 0; r < RPT; ++r) {
                    const double v = ld_dsmem_f64(&red[((warp * DB + jj) * RPT + r) * 32 + lane], (uint32_t)q);
                    acc[r][jj] += kr == 0 ? v : 0.0;
                }
        }
        if (ks > 1) cluster_sync();
        if (kr > 0) return;
    }
    store_acc(tile0 * TM, nullptr);
    if (MC_ON) cluster_sync();
}


// SONLY: the shape serves S only (no S' kernels are instantiated for it)
template <int RPT, int DB, int NW, bool PAIR = false, bool SONLY = false>
static int launch(ApplyArgs a, const Geom &g, cudaStream_t st) {
    // a slab's group starts are bulk-copied from word slab * NW: 16-byte aligned
    static_assert(NW % 4 == 0, "consumer warps per CTA must be a multiple of 4");
    if (SONLY && a.trans) return set_error(HSK_EINVAL, "sjlt apply: no S' kernel for rpt=%d db=%d nw=%d", RPT, DB, NW);
    constexpr int TM = 32 * RPT;
    constexpr int SLAB = PAIR ? kPairSlab : NW * DB;
    HSK_REQUIRE(g.tm == TM && g.db == DB && g.nw == NW, HSK_EINVAL, "sjlt: plan/config mismatch");
    const bool aligned = a.use_tma != 0;  // 16-byte aligned columns (lda even)
    // 0: TMA S tile; 1: cp.async S' tile (unaligned A); 2: cp.async S tile;
    // 3: TMA S' tile (16 x TM boxes, 128-byte swizzle)
    constexpr bool XPOSE = RPT == 4;  // (for S') transposed tile, cp.async producer
    // 4: TMA S' staging + in-smem transpose into the transposed 128-row tile
    // 5: TMA S' staging + in-smem copy into the S layout (64-row tiles, plans
    // with g.xp); 6: the same tile written by 8-byte cp.async (unaligned A)
    constexpr bool XP2_OK = (RPT == 2 || RPT == 4) && NW == 16 && !SONLY;  // the shapes with xp2 kernels
    const bool xp = a.trans && g.xp;
    if (xp && !XP2_OK) return set_error(HSK_EINVAL, "sjlt apply: no transposed-tile S' kernel for rpt=%d db=%d nw=%d", RPT, DB, NW);
    a.mode = a.trans ? (aligned && a.tk % 16 == 0 ? (xp ? 5 : XPOSE ? 4 : 3) : (xp ? 6 : 1)) : (aligned ? 0 : 2);
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
    const int pw = xp ? xp2_pw(RPT, DB) : a.trans && XPOSE ? kXposeProducers : 1;
    // (mode 6, the 8-byte copies of an unaligned operand, runs at ~1.5 ms on
    // n = 16384 whoever issues them -- the four producer warps or all consumer
    // warps, 2 to 32 inputs per warp instruction -- against 0.7-1.0 ms for the
    // natural / XOR layouts of mode 1: the price of the dense layout on the rare
    // odd-ld operand; DeviceMatrix pads every leading dimension to even)
    prod = (xp || prod) && (a.mode == 0 || a.mode == 3 || ((a.mode == 1 || a.mode == 4) && XPOSE) || xp) &&
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
    a.streamk = a.streamk && a.groups >= 1 && a.groups <= kMaxGroups && a.nchunks > 0 && a.units < (1ll << 31);
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
    } else if (a.mode == 3 || a.mode == 4 || a.mode == 5) {  // A is n x m_out: inner dimension = input index
        int rc = make_tmap_f64_2d(&tmap, a.A, (uint64_t)a.n, (uint64_t)a.m_out, (uint64_t)a.lda,
                                  16, TM, true);
        if (rc) return rc;
    }
    const int nthreads = (NW + (prod ? pw : 0)) * 32;
    const int budget = 226 * 1024;
    // staging of the transposing producers: mode 4 one tile; mode 5 two ring
    // slots and as many staging groups as fit beside them (<= 16)
    int stg_bytes = a.mode == 4 ? a_bytes : 0;
    int stages_max = std::max(2, std::min(7, (budget - 2048 - stg_bytes) / a.stage_bytes));
    a.nbox = a.gbox = 0;
    if (a.mode == 5) {
        // two slots (HSK_SJLT_STAGES asks for more: they must leave room for a group)
        stages_max = std::max(2, std::min(tuning().sjlt_stages, (budget - 2048 - 32768) / a.stage_bytes));
        // groups of gbox boxes (default 32 KB: 4 boxes of 64 rows, 512 contiguous
        // bytes per output row and TMA issue; the largest divisor of the chunk's
        // boxes not above it)
        const int nb = a.tk / 16;
        int gb = tuning().sjlt_xp_gb > 0 ? tuning().sjlt_xp_gb : 32768 / (TM * 128);
        gb = std::max(1, std::min(gb, nb));
        while (nb % gb) --gb;
        a.gbox = gb;
        a.nbox = std::min(16, (budget - 2048 - stages_max * a.stage_bytes) / (gb * TM * 128));
        HSK_REQUIRE(a.nbox >= 1, HSK_EINVAL, "sjlt: no room for the S' staging groups (TK %d)", a.tk);
        stg_bytes = a.nbox * gb * TM * 128;
    }
    if (a.streamk && a.mc > 1) {
        // every group is one cluster and groups wait on later groups: keep
        // the grid to the clusters that can be co-resident
        auto kprobe = sjlt_apply_kernel<RPT, DB, NW, false, true, true, PAIR>;
        if constexpr (!SONLY)
            if (a.trans) kprobe = sjlt_apply_kernel<RPT, DB, NW, true, true, true, PAIR>;
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
        for (int g = 0; g <= a.groups; ++g) a.sk_g[g][0] = (int32_t)(g * a.units / a.groups);
        for (int g = 0; g < a.groups; ++g) {
            const int64_t u0 = a.sk_g[g][0], u1 = a.sk_g[g + 1][0], nch = a.nchunks;
            const int64_t tile0 = u0 / nch, tb = (u1 - 1) / nch * nch;  // start of the last tile
            int nq = 0;
            if (u1 % nch != 0 && tb >= u0)
                for (int q = g + 1; q < a.groups && a.sk_g[q][0] < tb + nch; ++q) ++nq;
            a.sk_g[g][1] = (int32_t)tile0;
            a.sk_g[g][2] = (int32_t)std::min((tile0 + 1) * nch - u0, u1 - u0);
            a.sk_g[g][3] = (int32_t)(((u1 - 1) / nch - tile0 + 1) | (u0 % nch != 0) << 16 | nq << 17);
        }
        void *ws = nullptr;
        int *flags = nullptr;
        const int nct = a.groups * a.nslabs;
        int rc = stream_workspace(st, (size_t)nct * NW * DB * TM * sizeof(double), nct, &ws, &flags);
        if (rc) return rc;
        a.ws = static_cast<double *>(ws);
        a.flags = flags;
    }
    a.ksplit = ks;
    a.div_slabs = make_fastdiv((uint32_t)a.nslabs);
    a.div_ks = make_fastdiv((uint32_t)ks);
    a.per = (int32_t)((a.nchunks + ks - 1) / ks);
    const int per = (int)(a.streamk ? (a.units + a.groups - 1) / a.groups : (a.nchunks + ks - 1) / ks);
    a.stages = stages_max;
    if (tuning().sjlt_stages > 0) a.stages = std::max(2, std::min(a.stages, tuning().sjlt_stages));
    if (per > 0 && a.stages > per + 1) a.stages = std::max(2, per + 1);
    int smem = 2048 + a.stages * a.stage_bytes + stg_bytes;  // header + 1024-byte alignment slack
    // whole-tile CTAs stage their partial in the ring for the (k-split) epilogue
    if (!a.streamk) smem = std::max(smem, 2048 + NW * DB * RPT * 32 * 8);
    auto kern = prod ? (a.streamk ? sjlt_apply_kernel<RPT, DB, NW, false, true, true, PAIR>
                                  : sjlt_apply_kernel<RPT, DB, NW, false, true, false, PAIR>)
                     : (a.streamk ? sjlt_apply_kernel<RPT, DB, NW, false, false, true, PAIR>
                                  : sjlt_apply_kernel<RPT, DB, NW, false, false, false, PAIR>);
    if constexpr (!SONLY)
        if (a.trans)
            kern = prod ? (a.streamk ? sjlt_apply_kernel<RPT, DB, NW, true, true, true, PAIR>
                                     : sjlt_apply_kernel<RPT, DB, NW, true, true, false, PAIR>)
                        : (a.streamk ? sjlt_apply_kernel<RPT, DB, NW, true, false, true, PAIR>
                                     : sjlt_apply_kernel<RPT, DB, NW, true, false, false, PAIR>);
    if constexpr (XP2_OK)
        if (xp)
            kern = a.streamk ? sjlt_apply_kernel<RPT, DB, NW, true, true, true, PAIR, true>
                             : sjlt_apply_kernel<RPT, DB, NW, true, true, false, PAIR, true>;
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
                g == &pl.t && !g->xp ? (g->rpt == 4 ? -g->tm : g->tm) : 0, g->pair, g->even,
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
        case 4040: return sjlt::launch<4, 4, 16>(a, g, st);    // 128-row tiles, 64-bucket slabs
        case 2080: return sjlt::launch<2, 8, 16>(a, g, st);    // 64-row tiles
        case 2160: return sjlt::launch<2, 16, 16>(a, g, st);
        case 2130:  // S: 20 x 13 (S' only when forced in a tuning build)
#if HSK_TUNING
            if (trans) return sjlt::launch<2, 13, 20>(a, g, st);
#endif
            return sjlt::launch<2, 13, 20, false, true>(a, g, st);
        case 2110:  // S: 24 x 11
#if HSK_TUNING
            if (trans) return sjlt::launch<2, 11, 24>(a, g, st);
#endif
            return sjlt::launch<2, 11, 24, false, true>(a, g, st);
#if HSK_TUNING  // 32-row tiles (HSK_SJLT_RPT=1) and the 32-warp variants (HSK_SJLT_W32=1): never selected by default
        case 1320: return sjlt::launch<1, 32, 16>(a, g, st);   // 32-row tiles, 512-bucket slabs
        case 2100: return sjlt::launch<2, 10, 28>(a, g, st);   // HSK_SJLT_W32 = 28
        case 1161: return sjlt::launch<1, 16, 32>(a, g, st);
        case 4021: return sjlt::launch<4, 2, 32>(a, g, st);
        case 2041: return sjlt::launch<2, 4, 32>(a, g, st);
        case 2081: return sjlt::launch<2, 8, 32>(a, g, st);
#endif
        default: return set_error(HSK_EINVAL, "sjlt apply: no kernel for rpt=%d db=%d nw=%d", g.rpt, g.db, g.nw);
    }
}
