#!/usr/bin/env python
"""Generate csrc/hsk_sjlt_pipe.cuh: software-pipelined whole-chunk SJLT walkers.

One PTX block walks every entry of the DB buckets a warp owns in one k-chunk.
The plan sorts a chunk's entries by (bucket, input index) and closes the
entries of every group of DB buckets (one warp's) with a terminator word, so a
warp's list is contiguous and self-delimiting.  Entry words are

    e = negative << 31 | bucket mod DB << 24 | address bits,

terminator bucket field = DB.  The loop of bucket jj adds U * (+-1.0) into the
bucket's accumulators (one rounding: exactly the reference's add / subtract)
and exits when the next word's bucket field differs; it falls into a chain of
bucket tests (one compare-and-branch per bucket) that enters the next non-empty
bucket or ends the walk -- no bucket bounds are loaded.  (Splitting buckets by
sign into separate add / subtract loops saves the +-1.0 operand but doubles the
chain's branches: measured slower, C2 S 0.493 vs 0.463 ms.)

Two-stage software pipeline; at a loop top
    U, G = tile values and +-1.0 of entry pe,  E = word of entry pe + 1
    body:  acc += U * G ; U, G = tile(E), sign(E) ; k = E & 0x7f000000 ;
           pe += 4 ; E = word pe + 1 ; loop while k == jj << 24
so every load is consumed one iteration after it was issued.  The walk reads
one word past the warp's terminator: the kernel keeps null words after each
chunk's list.

Address bits (the sign and bucket bits never reach an address):
  S  tiles (dense, TMA):  e = kk;  row 2l(+1) of lane l at  sx + (e << log2(TM*8))
  S' tiles (TMA, 128-B swizzle): (kk, c) at (kk/16)*TM*128 + 128c + ((kk%16)*8 ^ 16(c%8))
                          e = (kk/16)*TM*128 + (kk%16)*8;
                          row c = l + 32r at st + 128l + ((e ^ 16(l%8)) & 0xffffff) + 4096r
  S' 128-row tiles (transposed, cp.async): (kk, c) at kk*TM*8 + 8(c ^ kk%32);
                          e = kk*TM*8 | 8(kk%32);
                          row c = l + 32r at st + (e & 0xffff00) + ((e & 248) ^ 8l) + 256r

Paired walkers (pipe_{s,t}_pair; block construction with d/alpha = 8): the
four warps of chunk pair (t1 = 2p, t2 = 2p + 1) split chunk t1's 8 buckets into
quarters; warp h walks every input index whose t1 bucket c1 lies in quarter h,
with one entry carrying both of its buckets,

    e = neg1 << 31 | ((c1 & 1) * 8 + c2) << 24 | neg2 << 23 | address bits,

(c1, c2 = bucket mod 8 in chunks t1, t2; terminator combo field = 16): one tile
load feeds two buckets, and the chain runs over 16 combos.  Accumulators: the
warp's two t1 buckets in acc[.][0..1] (complete), chunk t2's 8 buckets in
acc[.][2..9] (partial over the quarter; the kernel folds the four warps).

Uniform branches (VOTE_DOC).  ptxas does not trust bra.uni: a predicate
computed from a shared-memory word is per-lane to its divergence analysis, so
every chain link and loop-back branch of a walker that sits in a loop gets
BSSY/BSYNC reconvergence brackets -- a chain link then costs six instructions
(ISETP, BRA, 2 BSSY, 2 BSYNC) instead of two.  vote.sync.any on the predicate
(all lanes hold the same word, so it is the predicate itself) makes it
warp-uniform to ptxas: no brackets, at one VOTE per branch -- a link costs
three instructions, an entry one more.  That pays where entries per bucket
and chunk are few (64-row tiles: C1 ~2, C2 1.6, C5 0.5) and not on the
alpha-heavy 128-row tiles (C3: 16), which keep plain branches.

Usage: python tools/gen_consumers.py > paper_2302_01977_b200/csrc/hsk_sjlt_pipe.cuh
"""
import sys

S_CONFIGS = [(1, 16), (1, 32), (2, 4), (2, 8), (2, 10), (2, 11), (2, 13), (2, 16), (4, 2), (4, 4), (4, 8)]
T_CONFIGS = [(1, 16), (1, 32), (2, 4), (2, 8), (2, 10), (2, 11), (2, 13), (2, 16), (4, 2), (4, 4), (4, 8)]


def log2(x):
    return x.bit_length() - 1


def gen(rpt, db, trans, vote=None):
    # vote: make every branch predicate warp-uniform with vote.sync.any (see
    # VOTE_DOC); by default on the 64-row tiles (rpt 2: C1, C2, C5 -- few
    # entries per bucket and chunk), off for the alpha-heavy 128-row tiles
    if vote is None:
        vote = rpt == 2
    nacc = rpt * db
    sh = log2(32 * rpt * 8)  # e << sh == kk * TM * 8 (the state byte shifts out)
    L = []
    a = L.append
    sen, base = nacc, nacc + 1
    lane8 = nacc + 2 if trans else None
    sgs = nacc + (3 if trans else 2)  # shared address of the warp's group start (entries)
    a(".reg .pred q;")
    a(".reg .b32 pe, t, ad, e, k, gh, zero, one;")
    a(".reg .f64 " + ", ".join(f"u{r}" for r in range(rpt)) + ", g;")
    a("mov.b32 zero, 0;")
    a("mov.b32 one, 1072693248;")

    def load_tile():
        if trans and rpt == 4:
            # transposed layout: independent and/xor terms (measured faster
            # than a single LOP3 form)
            out = ["and.b32 t, e, 16776960;", "and.b32 ad, e, 248;", f"xor.b32 ad, ad, %{lane8};",
                   "add.u32 ad, ad, t;", f"add.u32 ad, ad, %{base};"]
            out += [f"ld.shared.f64 u{r}, [ad+{256 * r}];" for r in range(rpt)]
        elif trans:
            # (e ^ 16*(lane%8)) & 0xffffff in one LOP3 (lut 0x28); base = tile +
            # 128*lane; rows l + 32 r at +4096 r
            out = [f"lop3.b32 ad, e, %{lane8}, 16777215, 0x28;", f"add.u32 ad, ad, %{base};"]
            out += [f"ld.shared.f64 u{r}, [ad+{4096 * r}];" for r in range(rpt)]
        else:
            out = [f"shl.b32 t, e, {sh};", f"add.u32 ad, t, %{base};"]
            if rpt == 1:
                out += ["ld.shared.f64 u0, [ad];"]
            else:
                out += [f"ld.shared.v2.f64 {{u{2 * h}, u{2 * h + 1}}}, [ad+{512 * h}];"
                        for h in range(rpt // 2)]
        # gh = (e & 0x80000000) | 0x3FF00000 in one LOP3 (lut 0xEA: (a & b) | c)
        out += ["lop3.b32 gh, e, -2147483648, one, 0xEA;", "mov.b64 g, {zero, gh};"]
        return out

    # prologue: U, G = tile / sign of the first word, k = its bucket field,
    # E = the next word
    a(f"ld.shared.b32 t, [%{sgs}];")
    a(f"mad.lo.u32 pe, t, 4, %{sen};")
    a("ld.shared.b32 e, [pe];")
    L.extend(load_tile())
    a("and.b32 k, e, 2130706432;")
    a("ld.shared.b32 e, [pe+4];")
    uni = ["vote.sync.any.pred q, q, -1;"] if vote else []
    for jj in range(db):
        nxt = f"T{jj + 1}" if jj + 1 < db else "DONE"
        a(f"T{jj}:")
        a(f"setp.ne.u32 q, k, {jj << 24};")
        L.extend(uni)
        a(f"@q bra.uni {nxt};")
        a(f"S{jj}:")
        for r in range(rpt):
            acc = jj * rpt + r
            a(f"fma.rn.f64 %{acc}, u{r}, g, %{acc};")
        L.extend(load_tile())
        a("and.b32 k, e, 2130706432;")
        a("add.u32 pe, pe, 4;")
        a("ld.shared.b32 e, [pe+4];")
        a(f"setp.eq.u32 q, k, {jj << 24};")
        L.extend(uni)
        a(f"@q bra.uni S{jj};")
    a("DONE:")
    txt = "\\n\\t".join(L)
    outs = ", ".join(f'"+d"(acc[{k % rpt}][{k // rpt}])' for k in range(nacc))
    ins = ['"r"(sen)', '"r"(base)'] + (['"r"(lanex)'] if trans else []) + ['"r"(sgs)']
    name = f"pipe_{'t' if trans else 's'}_{rpt}x{db}"
    sig = "uint32_t sen, uint32_t base, " + ("uint32_t lanex, " if trans else "")
    return (f"__device__ __forceinline__ void {name}(double (&acc)[{rpt}][{db}], {sig}"
            f"uint32_t sgs) {{\n"
            f'    asm volatile("{{\\n\\t{txt}\\n\\t}}"\n'
            f"                 : {outs}\n"
            f"                 : {', '.join(ins)}\n"
            f'                 : "memory");\n}}\n')


def gen_tw(rpt, db, trans):
    """S' walker of 64-row TMA tiles (REL_DOC): one-instruction bucket tests,
    unrolled by two, entry words fetched in 8-byte pairs.

    * The loop test of bucket jj is a LOP3 with a predicate output,
          k = (E ^ jj << 24) & 0x7f000000,  q = k != 0,
      instead of k = E & mask plus a compare.  k is the next word's bucket
      relative to jj, so every bucket loop exits into its own chain, whose
      links compare k with (b ^ jj) << 24 for b = jj + 1 .. DB - 1 and branch
      into loop b on a match (the next bucket, the common case, first).
    * Unrolled by two with the next-word register alternating between e0 and
      e1: half A of loop jj holds the current entry at pe and the next word in
      e0, half B the current entry at pe + 4 and the next word in e1; an exit
      from A leaves the B state (its chain enters B halves), an exit from B the
      A state.
    * Group lists start at even words (plan kernel, Geom::even), so half A
      (current entry at an even word) loads the next two words with one
      ld.shared.v2 and half B loads none: one broadcast wavefront per two
      entries.  The walk reads up to two words past its terminator.
    Measured (same box, ms): C2 S' 0.611 -> 0.589, C1 S' 55.7 -> 53.4 us, C5
    shard S' equal; on S the same walker is slower (C2 0.449 -> 0.454, C5
    shard 8.7 -> 9.3: S is not bound by the word loads), so S keeps gen()."""
    nacc = rpt * db
    sh = log2(32 * rpt * 8)
    L = []
    a = L.append
    sen, base = nacc, nacc + 1
    lane8 = nacc + 2 if trans else None
    sgs = nacc + (3 if trans else 2)
    a(".reg .pred q, pz;")
    a(".reg .b32 pe, t, ad, e, e0, e1, k, gh, zero, one;")
    a(".reg .f64 " + ", ".join(f"u{r}" for r in range(rpt)) + ", g;")
    a("mov.b32 zero, 0;")
    a("mov.b32 one, 1072693248;")
    a("setp.ne.u32 pz, zero, zero;")

    def load_tile(e):
        if trans:
            out = [f"lop3.b32 ad, {e}, %{lane8}, 16777215, 0x28;", f"add.u32 ad, ad, %{base};"]
            out += [f"ld.shared.f64 u{r}, [ad+{4096 * r}];" for r in range(rpt)]
        else:
            out = [f"shl.b32 t, {e}, {sh};", f"add.u32 ad, t, %{base};"]
            out += [f"ld.shared.v2.f64 {{u{2 * h}, u{2 * h + 1}}}, [ad+{512 * h}];" for h in range(rpt // 2)]
        out += [f"lop3.b32 gh, {e}, -2147483648, one, 0xEA;", "mov.b64 g, {zero, gh};"]
        return out

    def chain(jj, half):
        rel = 0 if jj < 0 else jj
        for b in range(jj + 1, db):
            a(f"setp.eq.u32 q, k, {(b ^ rel) << 24};")
            a("vote.sync.any.pred q, q, -1;")
            a(f"@q bra.uni {half}{b};")
        a("bra.uni DONE;")

    def fma(jj):
        for r in range(rpt):
            acc = jj * rpt + r
            a(f"fma.rn.f64 %{acc}, u{r}, g, %{acc};")

    a(f"ld.shared.b32 t, [%{sgs}];")
    a(f"mad.lo.u32 pe, t, 4, %{sen};")
    a("ld.shared.v2.b32 {e, e0}, [pe];")
    L.extend(load_tile("e"))
    a("and.b32 k, e, 2130706432;")
    chain(-1, "WA")
    for jj in range(db):
        a(f"WA{jj}:")
        fma(jj)
        L.extend(load_tile("e0"))
        a(f"lop3.or.b32 k|q, e0, {jj << 24}, 2130706432, 0x28, pz;")
        a("ld.shared.v2.b32 {e1, e0}, [pe+8];")
        a("vote.sync.any.pred q, q, -1;")
        a(f"@q bra.uni WX{jj};")
        a(f"WB{jj}:")
        fma(jj)
        L.extend(load_tile("e1"))
        a(f"lop3.or.b32 k|q, e1, {jj << 24}, 2130706432, 0x28, pz;")
        a("add.u32 pe, pe, 8;")
        a("vote.sync.any.pred q, !q, -1;")
        a(f"@q bra.uni WA{jj};")
        chain(jj, "WA")
        a(f"WX{jj}:")
        chain(jj, "WB")
    a("DONE:")
    txt = "\\n\\t".join(L)
    outs = ", ".join(f'"+d"(acc[{k % rpt}][{k // rpt}])' for k in range(nacc))
    ins = ['"r"(sen)', '"r"(base)'] + (['"r"(lanex)'] if trans else []) + ['"r"(sgs)']
    name = f"pipe_{'t' if trans else 's'}_{rpt}x{db}"
    sig = "uint32_t sen, uint32_t base, " + ("uint32_t lanex, " if trans else "")
    return (f"__device__ __forceinline__ void {name}(double (&acc)[{rpt}][{db}], {sig}"
            f"uint32_t sgs) {{\n"
            f'    asm volatile("{{\\n\\t{txt}\\n\\t}}"\n'
            f"                 : {outs}\n"
            f"                 : {', '.join(ins)}\n"
            f'                 : "memory");\n}}\n')


def gen_pair(trans):
    """RPT = 2 rows per lane, 16 buckets = two chunks of 8 (see the docstring)."""
    rpt, nacc = 2, 20
    L = []
    a = L.append
    sen, base = nacc, nacc + 1
    lane8 = nacc + 2 if trans else None
    sgs = nacc + (3 if trans else 2)
    a(".reg .pred q;")
    a(".reg .b32 pe, t, t2, ad, e, k, gh, gh2, zero, one;")
    a(".reg .f64 u0, u1, g, g2;")
    a("mov.b32 zero, 0;")
    a("mov.b32 one, 1072693248;")

    def load_tile():
        if trans:
            # neg2 (bit 23) stays out of the address: mask 0x7fffff
            out = [f"lop3.b32 ad, e, %{lane8}, 8388607, 0x28;", f"add.u32 ad, ad, %{base};",
                   "ld.shared.f64 u0, [ad];", "ld.shared.f64 u1, [ad+4096];"]
        else:
            out = ["shl.b32 t, e, 9;", f"add.u32 ad, t, %{base};", "ld.shared.v2.f64 {u0, u1}, [ad];"]
        out += ["lop3.b32 gh, e, -2147483648, one, 0xEA;", "mov.b64 g, {zero, gh};",
                "shl.b32 t2, e, 8;", "lop3.b32 gh2, t2, -2147483648, one, 0xEA;",
                "mov.b64 g2, {zero, gh2};"]
        return out

    a(f"ld.shared.b32 t, [%{sgs}];")
    a(f"mad.lo.u32 pe, t, 4, %{sen};")
    a("ld.shared.b32 e, [pe];")
    L.extend(load_tile())
    a("and.b32 k, e, 2130706432;")
    a("ld.shared.b32 e, [pe+4];")
    for cc in range(16):
        nxt = f"T{cc + 1}" if cc + 1 < 16 else "DONE"
        c1, c2 = cc // 8, cc % 8
        a(f"T{cc}:")
        a(f"setp.ne.u32 q, k, {cc << 24};")
        a(f"@q bra.uni {nxt};")
        a(f"S{cc}:")
        for r in range(rpt):
            k1, k2 = c1 * rpt + r, (2 + c2) * rpt + r
            a(f"fma.rn.f64 %{k1}, u{r}, g, %{k1};")
            a(f"fma.rn.f64 %{k2}, u{r}, g2, %{k2};")
        L.extend(load_tile())
        a("and.b32 k, e, 2130706432;")
        a("add.u32 pe, pe, 4;")
        a("ld.shared.b32 e, [pe+4];")
        a(f"setp.eq.u32 q, k, {cc << 24};")
        a(f"@q bra.uni S{cc};")
    a("DONE:")
    txt = "\\n\\t".join(L)
    outs = ", ".join(f'"+d"(acc[{k % rpt}][{k // rpt}])' for k in range(nacc))
    ins = ['"r"(sen)', '"r"(base)'] + (['"r"(lanex)'] if trans else []) + ['"r"(sgs)']
    name = f"pipe_{'t' if trans else 's'}_pair"
    sig = "uint32_t sen, uint32_t base, " + ("uint32_t lanex, " if trans else "")
    return (f"__device__ __forceinline__ void {name}(double (&acc)[{rpt}][16], {sig}"
            f"uint32_t sgs) {{\n"
            f'    asm volatile("{{\\n\\t{txt}\\n\\t}}"\n'
            f"                 : {outs}\n"
            f"                 : {', '.join(ins)}\n"
            f'                 : "memory");\n}}\n')


def gen_pair_t():
    """Paired S' walker on TMA-landed tiles with parity pairs.

    A combo's entries come as (even, odd) input-index pairs -- head word
    flagged with bit 29 -- followed by the leftover singles.  In a pair
    iteration lanes with (lane & 8) == 0 load entry a for their rows and
    lanes with (lane & 8) != 0 entry b, then the other way round: each
    half-warp's 64-bit loads cover 8 rows at an even index and 8 at an odd
    one, i.e. all 16 bank pairs (a single entry's loads are 2-way
    conflicted: the tile's 128-byte swizzle cannot move an element's 8-byte
    half).  Singles walk as in pipe_t_pair.  Registers: h = the current
    item's head word; the pair loop prefetches the next two words (E2, F2);
    entering a pair loop from the chain, or leaving it for singles, issues
    that item's loads without the one-iteration lead (once per combo)."""
    rpt, nacc = 2, 20
    L = []
    a = L.append
    sen, base, lane8, sgs = nacc, nacc + 1, nacc + 2, nacc + 3
    PF = 1 << 29
    a(".reg .pred q, lo, sp;")
    a(".reg .b32 pe, t, t2, ad, e, k, gh, gh2, gy, gy2, zero, one, h, wa, wb, wx, wy, E2, F2;")
    a(".reg .f64 u0, u1, v0, v1, g, g2, gx, gx2;")
    a("mov.b32 zero, 0;")
    a("mov.b32 one, 1072693248;")
    a("mov.u32 t, %laneid;")
    a("and.b32 t, t, 8;")
    a("setp.eq.u32 lo, t, 0;")

    def signs(w, hi, hi2, d1, d2):
        return [f"lop3.b32 {hi}, {w}, -2147483648, one, 0xEA;", f"mov.b64 {d1}, {{zero, {hi}}};",
                f"shl.b32 t2, {w}, 8;", f"lop3.b32 {hi2}, t2, -2147483648, one, 0xEA;",
                f"mov.b64 {d2}, {{zero, {hi2}}};"]

    def load_single():  # from e: rows l, l + 32 of entry e
        # skipped when e heads a pair: the chain then enters that combo's pair
        # loop, which loads the pair itself (no wasted 2-way-conflicted loads)
        out = ["and.b32 t, e, 536870912;", "setp.eq.u32 sp, t, 0;",
               f"lop3.b32 ad, e, %{lane8}, 8388607, 0x28;", f"add.u32 ad, ad, %{base};",
               "@sp ld.shared.f64 u0, [ad];", "@sp ld.shared.f64 u1, [ad+4096];"]
        return out + signs("e", "gh", "gh2", "g", "g2")

    def load_pair():  # from (wa, wb): X = own half's entry, Y = the other
        out = ["selp.b32 wx, wa, wb, lo;", "selp.b32 wy, wb, wa, lo;",
               f"lop3.b32 ad, wx, %{lane8}, 8388607, 0x28;", f"add.u32 ad, ad, %{base};",
               "ld.shared.f64 u0, [ad];", "ld.shared.f64 u1, [ad+4096];",
               f"lop3.b32 ad, wy, %{lane8}, 8388607, 0x28;", f"add.u32 ad, ad, %{base};",
               "ld.shared.f64 v0, [ad];", "ld.shared.f64 v1, [ad+4096];"]
        return out + signs("wx", "gh", "gh2", "g", "g2") + signs("wy", "gy", "gy2", "gx", "gx2")

    def fma(c1, c2, u, gg, gg2):
        out = []
        for r in range(rpt):
            k1, k2 = c1 * rpt + r, (2 + c2) * rpt + r
            out += [f"fma.rn.f64 %{k1}, {u}{r}, {gg}, %{k1};", f"fma.rn.f64 %{k2}, {u}{r}, {gg2}, %{k2};"]
        return out

    a(f"ld.shared.b32 t, [%{sgs}];")
    a(f"mad.lo.u32 pe, t, 4, %{sen};")
    a("ld.shared.b32 e, [pe];")
    a("mov.b32 h, e;")
    L.extend(load_single())
    a("and.b32 k, e, 2130706432;")
    a("ld.shared.b32 e, [pe+4];")
    for cc in range(16):
        nxt = f"T{cc + 1}" if cc + 1 < 16 else "DONE"
        c1, c2 = cc // 8, cc % 8
        a(f"T{cc}:")
        a(f"setp.ne.u32 q, k, {(cc << 24) | PF};")
        a(f"@q bra.uni U{cc};")
        # pair entry: head h at pe, second word e
        a("mov.b32 wa, h;")
        a("mov.b32 wb, e;")
        L.extend(load_pair())
        a("ld.shared.b32 E2, [pe+8];")
        a("ld.shared.b32 F2, [pe+12];")
        a(f"P{cc}:")
        L.extend(fma(c1, c2, "u", "g", "g2"))
        L.extend(fma(c1, c2, "v", "gx", "gx2"))
        a("mov.b32 wa, E2;")
        a("mov.b32 wb, F2;")
        a("and.b32 k, wa, 2130706432;")
        a("add.u32 pe, pe, 8;")
        a(f"setp.ne.u32 q, k, {(cc << 24) | PF};")
        a(f"@q bra.uni X{cc};")
        L.extend(load_pair())
        a("ld.shared.b32 E2, [pe+8];")
        a("ld.shared.b32 F2, [pe+12];")
        a(f"bra.uni P{cc};")
        a(f"X{cc}:")  # next item (head wa at pe) is not a pair of this combo
        a("mov.b32 h, wa;")
        a("mov.b32 e, wa;")
        L.extend(load_single())
        a("mov.b32 e, wb;")
        a(f"U{cc}:")
        a(f"setp.ne.u32 q, k, {cc << 24};")
        a(f"@q bra.uni {nxt};")
        a(f"S{cc}:")
        L.extend(fma(c1, c2, "u", "g", "g2"))
        a("mov.b32 h, e;")
        L.extend(load_single())
        a("and.b32 k, e, 2130706432;")
        a("add.u32 pe, pe, 4;")
        a("ld.shared.b32 e, [pe+4];")
        a(f"setp.eq.u32 q, k, {cc << 24};")
        a(f"@q bra.uni S{cc};")
    a("DONE:")
    txt = "\\n\\t".join(L)
    outs = ", ".join(f'"+d"(acc[{k % rpt}][{k // rpt}])' for k in range(nacc))
    ins = ['"r"(sen)', '"r"(base)', '"r"(lanex)', '"r"(sgs)']
    return (f"__device__ __forceinline__ void pipe_t_pair(double (&acc)[{rpt}][16], uint32_t sen, "
            f"uint32_t base, uint32_t lanex, uint32_t sgs) {{\n"
            f'    asm volatile("{{\\n\\t{txt}\\n\\t}}"\n'
            f"                 : {outs}\n"
            f"                 : {', '.join(ins)}\n"
            f'                 : "memory");\n}}\n')


def main():
    out = ["// GENERATED by tools/gen_consumers.py -- do not edit by hand.",
           "// Software-pipelined whole-chunk SJLT walkers (state-tagged entries); see the generator.",
           "#pragma once", "#include <cstdint>", ""]
    for rpt, db in S_CONFIGS:
        out.append(gen(rpt, db, False))
    for rpt, db in T_CONFIGS:
        out.append(gen_tw(rpt, db, True) if rpt == 2 else gen(rpt, db, True))
    out.append(gen_pair(False))
    out.append(gen_pair_t())
    sys.stdout.write("\n".join(out))


if __name__ == "__main__":
    main()
