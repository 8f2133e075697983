"""Histogram of SASS opcodes (executed warp instructions and stall samples) from an ncu source-page csv."""
import csv, sys, collections, re
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; i_src = hdr.index("Source"); i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_e = hdr.index("Instructions Executed")
ops = collections.Counter(); st = collections.Counter(); tot_e = 0; tot_s = 0
for r in rows[2:]:
    if len(r) <= i_e: continue
    src = r[i_src].strip()
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", src)
    if not m: continue
    op = m.group(2) + (m.group(3) or "")
    try:
        e = int(r[i_e]); s = int(r[i_s])
    except ValueError:
        continue
    ops[op] += e; st[op] += s; tot_e += e; tot_s += s
print(f"total warp inst {tot_e/1e6:.1f}M, samples {tot_s}")
for op, e in ops.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    print(f"{op:28s} {e/1e6:8.2f}M {100*e/tot_e:5.1f}%  stall-samples {100*st[op]/max(tot_s,1):5.1f}%")
