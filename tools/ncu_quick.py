"""Summarise an ncu report: key metrics + top stall sites (source page).
  python tools/ncu_quick.py gpurun_out/x.ncu-rep [n_top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 20
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h = r[0]
keys = ["Kernel Name", "gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "launch__grid_size", "launch__registers_per_thread",
        "sm__cycles_elapsed.avg.per_second", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
for row in r[2:]:
    d = dict(zip(h, row))
    for k in keys:
        if k in d:
            print(f"  {k} = {d[k][:100]}  {r[1][h.index(k)]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(io.StringIO(src)))
hi = next(i for i, x in enumerate(r) if "Warp Stall Sampling (All Samples)" in x)
h = r[hi]
si = h.index("Warp Stall Sampling (All Samples)")
rows = [x for x in r[hi + 1:] if len(x) > si and x[si].replace(".", "").isdigit()]
tot = sum(float(x[si]) for x in rows)
print("  stall samples", tot)
order = sorted(range(len(rows)), key=lambda i: -float(rows[i][si]))
for i in order[:ntop]:
    x = rows[i]
    prev = rows[i - 1][1].strip()[:60] if i > 0 else ""
    print(f"  {float(x[si]) / tot * 100:5.1f}%  {x[1].strip()[:80]:80s} | prev: {prev}")
