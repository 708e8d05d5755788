"""Aggregate an ncu --metrics gpu__time_duration.sum launch list (CSV) by kernel."""
import collections
import csv
import sys


def main(path, out=None):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        name = r[ki].split("(")[0][:70]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(t for _, t in agg.values())
    lines = [f"# launch list {path}: {sum(n for n, _ in agg.values())} launches, {tot / 1e6:.2f} ms "
             "(ncu, serialised, cold cache: compare shares)"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{t / 1e6:10.2f} ms {100 * t / tot:5.1f}% n={n:6d} avg={t / n / 1e3:9.1f} us  {k}")
    text = "\n".join(lines)
    if out:
        open(out, "w").write(text + "\n")
    print(text)


if __name__ == "__main__":
    main(*sys.argv[1:])
