"""Key metrics per kernel from an ncu --set full report (raw page)."""
import csv, io, subprocess, sys
METRICS = [
    ("gpu__time_duration.sum", "us", 1),
    ("dram__bytes_read.sum", "rdMB", 1),
    ("dram__bytes_write.sum", "wrMB", 1),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM%", 1),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem%", 1),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1%", 1),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2%", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%", 1),
    ("smsp__inst_executed.sum", "Minst", 1e-6),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma%", 1),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu%", 1),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu%", 1),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64%", 1),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%", 1),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "bankcf(M)", 1e-6),
    ("launch__registers_per_thread", "regs", 1),
    ("launch__occupancy_limit_registers", "occ_reg", 1),
]
STALLS = "smsp__average_warps_issue_stalled_"
def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    units = rows[1]
    data = rows[2:]
    SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}
    idx = {h: i for i, h in enumerate(hdr)}
    for r in data:
        name = r[idx["Kernel Name"]].split("(")[0].replace("(anonymous namespace)::", "")[:50]
        vals = []
        for m, lab, sc in METRICS:
            if m in idx:
                try:
                    v = float(r[idx[m]].replace(',', '')) * sc
                    if m.startswith(("dram__bytes", "gpu__time")):
                        v = v * SCALE.get(units[idx[m]], 1.0)
                    vals.append(f"{lab}={v:.1f}")
                except ValueError:
                    pass
        print(name); print("   " + " ".join(vals))
        st = []
        for h, i in idx.items():
            if h.startswith(STALLS) and h.endswith("_per_issue_active.ratio"):
                try:
                    st.append((float(r[i].replace(',', '')), h[len(STALLS):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        st.sort(reverse=True)
        print("   stalls: " + ", ".join(f"{n}={v:.2f}" for v, n in st[:7]))
if __name__ == "__main__":
    main(sys.argv[1])
