"""profiles/traffic.json: DRAM bytes (read + write) per launch of each bench kernel slot, from one
`ncu --set full` report (tools/gpu_check.sh).  usage: python tools/make_traffic.py REPORT [OUT]"""
import csv, io, json, subprocess, sys

SLOTS = {  # kernel-name fragment -> bench.py stage slots it serves
    "raster_bwd_tile1w": ["raster_bwd"], "raster_fwd_kernel": ["raster_fwd"],
    "ssim_loss_kernel": ["loss_ssim"], "pcols_fwd": ["cols_fwd"], "pcols_bwd": ["cols_bwd"],
    "srows_fwd": ["rows_fwd", "rows_fwd_bwd"], "srows_inv": ["rows_inv", "rows_inv_bwd"],
}
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

def main(rep, out, workload="cfg2"):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u = rows[0], rows[1]
    ir, iw, ik = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum"), h.index("Kernel Name")
    res = {}
    for r in rows[2:]:
        b = float(r[ir].replace(",", "")) * SCALE[u[ir]] + float(r[iw].replace(",", "")) * SCALE[u[iw]]
        for frag, slots in SLOTS.items():
            if frag in r[ik]:
                for s in slots:
                    res.setdefault(s, []).append(b)
    res = {k: sum(v) / len(v) for k, v in res.items()}
    json.dump({"source": rep, "workload": workload,
               "unit": "bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum)", **res},
              open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))

if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "profiles/traffic.json",
         sys.argv[3] if len(sys.argv) > 3 else "cfg2")
