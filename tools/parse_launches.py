"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel."""
import csv, collections, sys, io

def load(path):
    txt = open(path).read().splitlines()
    start = next(i for i, l in enumerate(txt) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(txt[start:]))))
    agg = collections.OrderedDict()
    for r in rows:
        k = r['Kernel Name'].split('(')[0].replace('(anonymous namespace)::', '').replace('hs::', '')
        d = agg.setdefault((int(r['ID']), k), {})
        d[r['Metric Name']] = float(r['Metric Value'].replace(',', ''))
    return agg

if __name__ == "__main__":
    agg = load(sys.argv[1])
    tot = collections.OrderedDict()
    for (i, k), d in agg.items():
        t = tot.setdefault(k, [0, 0.0, 0.0, 0.0])
        t[0] += 1; t[1] += d.get('gpu__time_duration.sum', 0) / 1e3
        t[2] += d.get('dram__bytes_read.sum', 0) / 1e6; t[3] += d.get('dram__bytes_write.sum', 0) / 1e6
    all_t = sum(v[1] for v in tot.values())
    print(f"{'kernel':44s} {'n':>3s} {'us/launch':>10s} {'share':>6s} {'rdMB':>8s} {'wrMB':>8s}")
    for k, (n, t, r, w) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:44]:44s} {n:3d} {t/n:10.1f} {100*t/all_t:5.1f}% {r/n:8.1f} {w/n:8.1f}")
