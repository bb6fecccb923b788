"""Key counters + top stall reasons per kernel from an .ncu-rep (read here, no GPU)."""
import csv
import io
import subprocess
import sys

rep, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", f"regex:{pat}"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
KEYS = ["gpu__time_duration.sum", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "smsp__cycles_elapsed.avg.per_second",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread"]
for d in rows[2:]:
    print("==", d[hdr.index("Kernel Name")][:70])
    for k in KEYS:
        if k in hdr:
            print(f"   {k:95s} {d[hdr.index(k)]} {units[hdr.index(k)]}")
    st = {}
    for h, v in zip(hdr, d):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                st[h[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(v)
            except ValueError:
                pass
    tot = sum(st.values()) or 1
    print("   stalls:", ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]))
