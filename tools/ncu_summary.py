"""Summarise an ncu report (--page raw) into profiles/<name>.md and, for K1,
profiles/k1_traffic.json (dram bytes per launch, read by bench.py)."""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__grid_size",
    "launch__block_size", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tensor_op_hmma.sum", "lts__t_bytes.sum", "l1tex__t_bytes.sum",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
]


def main(rep: str, name: str, alg_log: str = "", first: int = 400):
    """alg_log: the SPEX_ATTN_LOG file of the profiled command (launch index,
    algorithmic bytes, ms); the ncu capture skipped `first` K1 launches, so its
    launches are alg_log lines first, first+1, ..."""
    alg = []
    if alg_log:
        rows = [ln.split() for ln in open(alg_log) if ln.strip()]
        alg = [float(r[1]) for r in rows if first <= int(r[0])]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    launches = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:90]}
        for w in WANT:
            if w in hdr:
                v = r[hdr.index(w)].replace(",", "")
                try:
                    d[w] = float(v)
                except ValueError:
                    d[w] = v
                d[w + ".unit"] = units[hdr.index(w)]
        launches.append(d)
    md = [f"# ncu summary: {name}", "", f"source: `{rep}` (--set full, --clock-control none)", ""]
    for i, d in enumerate(launches):
        md.append(f"## launch {i}: `{d['kernel']}`")
        for w in WANT:
            if w in d:
                md.append(f"- {w}: {d[w]} {d.get(w + '.unit', '')}")
        md.append("")
    (ROOT / "profiles" / f"{name}.md").write_text("\n".join(md))
    if launches:
        def to_bytes(d, k):
            u = d.get(k + ".unit", "byte")
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            return d.get(k, 0.0) * mult
        traffic = sum(to_bytes(d, "dram__bytes_read.sum") + to_bytes(d, "dram__bytes_write.sum")
                      for d in launches) / len(launches)
        out = {"dram_bytes_per_launch": traffic, "launches": launches}
        if alg:
            k = min(len(alg), len(launches))
            out["alg_bytes_per_launch"] = sum(alg[:k]) / k
            out["dram_over_alg"] = traffic / out["alg_bytes_per_launch"]
            md.append(f"algorithmic bytes per launch (same launches): {out['alg_bytes_per_launch']:.4g}; "
                      f"DRAM/algorithmic = {out['dram_over_alg']:.3f}")
            (ROOT / "profiles" / f"{name}.md").write_text("\n".join(md))
        (ROOT / "profiles" / f"{name}.json").write_text(json.dumps(out, indent=1))
    print("\n".join(md[:40]))


if __name__ == "__main__":
    main(*sys.argv[1:3], *(sys.argv[3:4]), *([int(sys.argv[4])] if len(sys.argv) > 4 else []))
