#!/usr/bin/env python
"""Generate csrc/hsk_sjlt_pipe.cuh: software-pipelined whole-chunk SJLT walkers.

One PTX block walks every entry of the DB buckets a warp owns in one k-chunk.
The warp's entries are contiguous in shared memory (sorted by bucket), so the
walk is one pointer `pe` crossing bucket boundaries; only the accumulator
changes.  Entries are 4-byte words  e = kk << 3 | neg << 31  (kk = input index
within the chunk), so a broadcast entry load costs one register-writeback
cycle instead of four (the writeback port, 128 B/clk/SM, is what the entry
walk saturates first).

Two-stage software pipeline; at a loop top
    U, G = tile values and +-1.0 of entry pe,   E = entry word pe + 1
    body:  acc += U * G ; pe += 4 ; U, G = tile(E), sign(E) ; E = word pe + 1
so every load is consumed one iteration after it was issued.  The walk reads
one word past the warp's list: the kernel keeps null words (pointing at a zero
row) after each chunk's list.

  S  tiles (dense, TMA):  row 2l(+1) of lane l at  sx + kk*TM*8          (RPT 2)
                          entry word e = kk << 3 | sign << 31
  S' tiles (TMA, 128-B swizzle): (kk, c) at (kk/16)*TM*128 + 128c + ((kk%16)*8 ^ 16(c%8))
                          entry word e = (kk/16)*TM*128 + (kk%16)*8 | sign << 31;
                          row c = l + 32r at st + 128l + ((e ^ 16(l%8)) & 0x7fffffff) + 4096r
  S' 128-row tiles (transposed, cp.async): (kk, c) at kk*TM*8 + 8(c ^ kk%32);
                          e = kk*TM*8 | 8(kk%32) | sign << 31;
                          row c = l + 32r at st + ((e ^ 8l) & 0x7fffffff) + 256r

Usage: python tools/gen_consumers.py > paper_2302_01977_b200/csrc/hsk_sjlt_pipe.cuh
"""
import sys

S_CONFIGS = [(1, 16), (1, 32), (2, 4), (2, 8), (2, 16), (4, 2), (4, 4), (4, 8)]
T_CONFIGS = [(1, 16), (1, 32), (2, 4), (2, 8), (2, 16), (4, 2), (4, 4), (4, 8)]


def log2(x):
    return x.bit_length() - 1


def gen(rpt, db, trans, vote=False):
    nacc = rpt * db
    sh = log2(32 * rpt * 8) - 3  # e << sh == kk * TM * 8 (the sign bit shifts out)
    L = []
    a = L.append
    sen, base = nacc, nacc + 1
    lane8 = nacc + 2 if trans else None
    sbw = nacc + (3 if trans else 2)  # shared address of the warp's packed u16 bounds
    nw = db // 2 + 1                  # bound words (bounds 2q, 2q+1 in word q)
    a(".reg .pred p, q;")
    a(".reg .b32 pe, pend, pnx, t, ad, e, gh, zero, one;")
    a(".reg .b32 " + ", ".join(f"w{k}" for k in range(nw)) + ";")
    a(".reg .f64 " + ", ".join(f"u{r}" for r in range(rpt)) + ", g;")
    a("mov.b32 zero, 0;")
    a("mov.b32 one, 1072693248;")

    def load_tile():
        if trans and rpt == 4:
            # transposed layout: measured faster with the independent and/xor
            # terms than with the single LOP3 (C3 S' 11.0 vs 11.4 ms)
            out = [f"and.b32 t, e, 2147483647;", f"and.b32 ad, e, 248;", f"xor.b32 ad, ad, %{lane8};",
                   "and.b32 t, t, -256;", "add.u32 ad, ad, t;", f"add.u32 ad, ad, %{base};"]
            out += [f"ld.shared.f64 u{r}, [ad+{256 * r}];" for r in range(rpt)]
        elif trans:
            # e = (kk/16)*TM*128 + (kk%16)*8 | sign: (e ^ 16*(lane%8)) & 0x7fffffff in
            # one LOP3 (lut 0x28); base = tile + 128*lane; rows l + 32 r at +4096 r
            out = [f"lop3.b32 ad, e, %{lane8}, 2147483647, 0x28;", f"add.u32 ad, ad, %{base};"]
            # 128-row S' tiles use the transposed layout (rows l + 32 r at +256 r)
            stride = 256 if rpt == 4 else 4096
            out += [f"ld.shared.f64 u{r}, [ad+{stride * r}];" for r in range(rpt)]
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

    def bound_to(dst, b):  # dst = sen + 4 * bound(b); bound(b) in word b >> 1, lo/hi half
        w = f"w{b >> 1}"
        return [(f"and.b32 t, {w}, 65535;" if b % 2 == 0 else f"shr.u32 t, {w}, 16;"),
                f"mad.lo.u32 {dst}, t, 4, %{sen};"]

    def branch(pred, label):
        if vote:
            return [f"vote.sync.any.pred {pred}, {pred}, -1;", f"@{pred} bra.uni {label};"]
        return [f"@{pred} bra.uni {label};"]

    # bound words stream in two buckets ahead of use: word q is first needed at
    # bucket 2q - 2 (as bound 2q, the end of bucket 2q - 1) and is loaded at
    # the start of bucket 2q - 4 (words 0 and 1 in the prologue)
    a(f"ld.shared.b32 w0, [%{sbw}];")
    if nw > 1:
        a(f"ld.shared.b32 w1, [%{sbw}+4];")
    # prologue: U, G = entry pe; E = word pe + 1; pend = end of bucket 0
    L.extend(bound_to("pe", 0))
    a("ld.shared.b32 e, [pe];")
    L.extend(load_tile())
    a("ld.shared.b32 e, [pe+4];")
    L.extend(bound_to("pend", 1))
    for jj in range(db):
        if jj % 2 == 0 and jj // 2 + 2 < nw:
            qn = jj // 2 + 2
            a(f"ld.shared.b32 w{qn}, [%{sbw}+{4 * qn}];")
        # end of the next bucket, computed off the critical path
        if jj + 1 < db:
            L.extend(bound_to("pnx", jj + 2))
        a("setp.ge.u32 p, pe, pend;")
        L.extend(branch("p", f"B{jj}_END"))
        a(f"B{jj}_LOOP:")
        a("add.u32 pe, pe, 4;")
        a("setp.lt.u32 q, pe, pend;")
        for r in range(rpt):
            a(f"fma.rn.f64 %{jj * rpt + r}, u{r}, g, %{jj * rpt + r};")
        L.extend(load_tile())
        a("ld.shared.b32 e, [pe+4];")
        L.extend(branch("q", f"B{jj}_LOOP"))
        a(f"B{jj}_END:")
        if jj + 1 < db:
            a("mov.b32 pend, pnx;")
    txt = "\\n\\t".join(L)
    outs = ", ".join(f'"+d"(acc[{k % rpt}][{k // rpt}])' for k in range(nacc))
    ins = ['"r"(sen)', '"r"(base)'] + (['"r"(lanex)'] if trans else []) + ['"r"(sbw)']
    name = f"pipe_{'t' if trans else 's'}_{rpt}x{db}"
    sig = "uint32_t sen, uint32_t base, " + ("uint32_t lanex, " if trans else "")
    return (f"__device__ __forceinline__ void {name}(double (&acc)[{rpt}][{db}], {sig}"
            f"uint32_t sbw) {{\n"
            f'    asm volatile("{{\\n\\t{txt}\\n\\t}}"\n'
            f"                 : {outs}\n"
            f"                 : {', '.join(ins)}\n"
            f'                 : "memory");\n}}\n')


def main():
    out = ["// GENERATED by tools/gen_consumers.py -- do not edit by hand.",
           "// Software-pipelined whole-chunk SJLT walkers (4-byte entries); see the generator.",
           "#pragma once", "#include <cstdint>", ""]
    vote = "--vote" in sys.argv
    for rpt, db in S_CONFIGS:
        out.append(gen(rpt, db, False, vote))
    for rpt, db in T_CONFIGS:
        out.append(gen(rpt, db, True, vote))
    sys.stdout.write("\n".join(out))


if __name__ == "__main__":
    main()
