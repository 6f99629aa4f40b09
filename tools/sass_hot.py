"""Where a kernel's instructions and stall samples go, from the ncu source page
(--page source --csv --print-source sass, gzipped by tools/profile_all.sh):
contiguous address blocks ranked by instructions executed, with their opcode mix.
Usage: python tools/sass_hot.py gpurun_out/prof/k3_series.sass.csv.gz [block=64]"""
import collections
import csv
import gzip
import sys

path = sys.argv[1]
blk = int(sys.argv[2]) if len(sys.argv) > 2 else 64
rows = list(csv.reader(gzip.open(path, "rt")))
hdr = rows[1]
ia, isrc, iex, ismp = (hdr.index("Address"), hdr.index("Source"),
                       hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)"))
ins = []
for r in rows[2:]:
    try:
        ins.append((r[isrc].strip(), int(r[iex] or 0), int(r[ismp] or 0)))
    except (ValueError, IndexError):
        pass
tot = sum(e for _, e, _ in ins) or 1
tots = sum(s for _, _, s in ins) or 1
print(f"{len(ins)} instructions, {tot:.3e} executed, {tots} stall samples")
blocks = []
for b0 in range(0, len(ins), blk):
    seg = ins[b0:b0 + blk]
    ex = sum(e for _, e, _ in seg)
    sm = sum(s for _, _, s in seg)
    mix = collections.Counter()
    for s, e, _ in seg:
        op = s.split()[0] if not s.startswith("@") else s.split()[1]
        mix[op.split(".")[0]] += e
    blocks.append((ex, sm, b0, mix))
for ex, sm, b0, mix in sorted(blocks, reverse=True)[:12]:
    top = ", ".join(f"{k}:{v / ex:.0%}" for k, v in mix.most_common(5))
    print(f"instr {b0:5d}-{b0 + blk - 1:5d}: {ex / tot:6.1%} of executed, {sm / tots:6.1%} of stalls | {top}")
