"""Per-kernel durations of the last search in an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import csv
import sys

for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h, data = rows[hi], rows[hi + 1:]
    kn, mv = h.index("Kernel Name"), h.index("Metric Value")
    ks = [(r[kn], float(r[mv].replace(",", ""))) for r in data if len(r) > mv and "read_stream" not in r[kn]]
    # the last search starts at the last qsplit/row_norms launch pair
    starts = [i for i, (n, _) in enumerate(ks) if "row_norms" in n or "qprep" in n]
    last = ks[starts[-1]:] if starts else ks
    print(path, f"{sum(t for _, t in last) / 1000:.1f} us in {len(last)} launches")
    for n, t in last:
        print(f"  {t / 1000:8.1f} us  {n.split('(')[0].replace('(anonymous namespace)::', '')[:70]}")
