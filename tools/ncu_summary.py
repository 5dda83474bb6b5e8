"""Summarise an .ncu-rep (one block per profiled kernel launch) for profiles/: duration, DRAM
bytes and throughput, SM / tensor-pipe activity, registers, grid. Usage: ncu_summary.py REP [title]"""
import csv
import io
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
           "launch__registers_per_thread", "launch__grid_size", "sm__cycles_elapsed.avg.per_second"]

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
if len(sys.argv) > 2:
    print(sys.argv[2])
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    print(name[:90])
    for m in METRICS:
        if m in hdr:
            i = hdr.index(m)
            print(f"   {m} = {r[i]} {units[i]}")
