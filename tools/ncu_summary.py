"""One line per kernel of an `ncu --set full` report: time, DRAM bytes, issue/occupancy,
FMA pipe, shared-memory wavefronts and conflicts, and the top warp-stall reasons per issue.

  python tools/ncu_summary.py gpurun_out/TAG/passes.ncu-rep > profiles/TAG_ncu_full_passes.txt
"""
import csv
import io
import subprocess
import sys

M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
     "launch__registers_per_thread", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
     "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
     "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
ST = ["wait", "short_scoreboard", "math_pipe_throttle", "mio_throttle", "barrier", "long_scoreboard",
      "no_instruction", "not_selected", "lg_throttle"]
SM = [f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio" for s in ST]
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
ci = {h: i for i, h in enumerate(hdr)}
print("# kernel | time_ms | dram_read_GB | dram_write_GB | " + " | ".join(m.split(".")[0] if "pct" not in m else m.split(".avg")[0] for m in M[3:])
      + " | stalls/issue: " + " ".join(ST))
for r in rows[2:]:
    def g(m):
        v = r[ci[m]] if m in ci else ""
        try:
            return float(v.replace(",", ""))
        except ValueError:
            return float("nan")
    name = r[ci["Kernel Name"]]
    vals = [g(m) for m in M]
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "msecond": 1.0, "ms": 1.0,
             "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}
    for k in range(3):                           # -> ms, GB, GB
        vals[k] *= scale.get(rows[1][ci[M[k]]], 1.0)
    print(f"{name} | " + " | ".join(f"{v:.6g}" for v in vals) + " | " + " ".join(f"{g(s):.3f}" for s in SM))
