"""Per-source-line warp-stall samples from an ncu report (--page source --print-source cuda,sass).

usage: python tools/ncu_lines.py REPORT.ncu-rep [top]"""
import collections
import csv
import subprocess
import sys


def main(path, top=30):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
    fname, hdr, tot = "?", None, 0.0
    for r in csv.reader(out.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            wi = hdr.index("Warp Stall Sampling (All Samples)")
            ii = hdr.index("Instructions Executed")
            continue
        if hdr is None or len(r) <= wi or not r[0].strip().isdigit():
            continue
        key = (fname, int(r[0]))
        try:
            w = float(r[wi] or 0)
            ie = float(r[ii] or 0)
        except ValueError:
            continue
        agg[key][0] += w
        agg[key][1] += ie
        agg[key][2] = r[1][:100]
        tot += w
    print(f"total stall samples {tot:.0f}")
    for (f, ln), (w, ie, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{w:8.0f} {100 * w / max(tot, 1):5.1f}% {f}:{ln:<4} inst={ie:10.0f}  {src.strip()}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
