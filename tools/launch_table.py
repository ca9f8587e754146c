"""Aggregates an ncu --metrics gpu__time_duration.sum CSV launch list: time per kernel name."""
import collections, csv, sys
def main(path, builds=1):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]; ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0]); tot = 0.0
    for r in rows[h + 1:]:
        if len(r) <= vi: continue
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1e-3)
        name = r[ki].split("(")[0].replace("void ", "")[:60]
        agg[name][0] += 1; agg[name][1] += v; tot += v
    print(f"{'us/build':>10} {'launches':>8}  kernel")
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        if v / builds > 5: print(f"{v / builds:10.1f} {c // builds:8d}  {k}")
    print(f"total kernel time per build: {tot / builds / 1e3:.2f} ms")
if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)
