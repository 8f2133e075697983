"""Per-source-line executed warp instructions and stall samples of one kernel
from `ncu -i REP --page source --csv --print-source cuda,sass --kernel-name regex:K`.
usage: tools/ncu_src_lines.py CSV [top]"""
import csv, sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
fname, ie, isx, items, te, ts = "", None, None, [], 0, 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        ie = r.index("Instructions Executed")
        isx = r.index("Warp Stall Sampling (All Samples)")
        continue
    if ie is None or not r[0].isdigit():
        continue
    try:
        e, s = int(r[ie]), int(r[isx])
    except ValueError:
        continue
    items.append((e, s, f"{fname}:{r[0]}", r[1].strip()[:80]))
    te += e
    ts += s
items.sort(reverse=True)
print(f"total {te / 1e6:.1f}M warp instructions, {ts} stall samples")
for e, s, loc, src in items[:top]:
    print(f"{e / 1e6:7.2f}M {100 * e / max(te, 1):5.1f}%  st {100 * s / max(ts, 1):5.1f}%  {loc:>22s}  {src}")
