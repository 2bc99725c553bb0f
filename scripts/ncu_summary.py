"""Summarises an ncu --set full report: one line per kernel launch with the
metrics that bound a straight-line walk (duration, FP64 pipe, issue, cache
hit rates, top stall reasons, spills, DRAM bytes).

  python scripts/ncu_summary.py report.ncu-rep [more.ncu-rep ...]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "ms", 1e-6),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64%", 1),
    ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue%", 1),
    ("smsp__inst_executed.sum", "inst", 1),
    ("sm__icc_request_hit_rate.pct", "icc_hit%", 1),
    ("idc__request_hit_rate.pct", "idc_hit%", 1),
    ("launch__registers_per_thread", "regs", 1),
    ("smsp__sass_inst_executed_op_local_ld.sum", "lcl_ld", 1),
    ("dram__bytes_read.sum", "dram_rd", 1),
    ("dram__bytes_write.sum", "dram_wr", 1),
]
STALLS = ["short_scoreboard", "long_scoreboard", "math_pipe_throttle", "mio_throttle", "wait",
          "not_selected", "no_instruction", "barrier", "lg_throttle", "dispatch_stall", "branch_resolving"]

for path in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    for row in rows[2:]:
        d = dict(zip(head, row))
        u = dict(zip(head, units))
        parts = [d.get("Kernel Name", "")[:28]]
        for k, label, scale in KEYS:
            v = d.get(k)
            if v is None or v == "":
                continue
            x = float(v.replace(",", ""))
            unit = u.get(k, "")
            if k.startswith("gpu__time"):
                x = x * {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(unit, 1e-6)
            elif k.startswith("dram__bytes"):
                x = x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1) / 1e6
                label += "MB"
            parts.append(f"{label}={x:.4g}")
        st = []
        for s in STALLS:
            v = d.get(f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio")
            if v:
                st.append((float(v), s))
        st.sort(reverse=True)
        parts.append("stalls=" + ",".join(f"{s}:{v:.2f}" for v, s in st[:4]))
        print(path.split("/")[-1], " ".join(parts))
