"""Per-CUDA-source-line executed warp instructions + stall samples from `ncu --page source --print-source cuda,sass --csv`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hdr_i]
i_e = hdr.index("Instructions Executed"); i_s = hdr.index("Warp Stall Sampling (All Samples)")
items = []; tot = 0
for r in rows[hdr_i + 1:]:
    if r and r[0] and r[0] != "":
        try:
            e = int(r[i_e]); s = int(r[i_s])
        except (ValueError, IndexError):
            continue
        items.append((e, s, r[0], r[1].strip()[:100])); tot += e
items.sort(reverse=True)
print(f"total {tot/1e6:.1f}M warp inst")
for e, s, l, src in items[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{e/1e6:7.2f}M {100*e/tot:5.1f}% st{s:6d} L{l:>4s} {src}")
