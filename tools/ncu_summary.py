"""Summarise an ncu report: key raw metrics per kernel and the hottest SASS lines."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kfilter = sys.argv[2] if len(sys.argv) > 2 else None
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size",
           "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_bytes.sum"]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
for r in rows[2:]:
    name = r[h.index("Kernel Name")]
    if kfilter and kfilter not in name:
        continue
    print(name[:70])
    for m in METRICS:
        if m in h:
            print(f"   {m} = {r[h.index(m)]} {rows[1][h.index(m)]}")
if kfilter:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kfilter}"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    hh = rows[1]
    data = [x for x in rows[2:] if len(x) == len(hh) and x[0] != hh[0]]
    si = hh.index("Warp Stall Sampling (All Samples)")
    ii = hh.index("Instructions Executed")
    sc = hh.index("Source")
    tot = sum(float(x[si] or 0) for x in data)
    print("stall samples:", tot)
    for x in sorted(data, key=lambda x: -float(x[si] or 0))[:int(sys.argv[3]) if len(sys.argv) > 3 else 20]:
        print(f"  {x[0][-5:]} {float(x[si] or 0)/tot*100:5.1f}% exec={x[ii]:>10} {x[sc][:80]}")
