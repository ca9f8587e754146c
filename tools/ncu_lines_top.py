"""Top source lines of an ncu report by warp-stall samples (source page, cuda+sass view): which
lines of which file hold the kernel's time.  Usage: ncu_lines_top.py report.ncu-rep [N]"""
import collections, csv, subprocess, sys


def main(path, top=30):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    agg = collections.defaultdict(lambda: [0, 0, ""])
    f, hdr = "?", None
    tot = 0
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "Function Name" or not r[0].isdigit():
            continue
        try:
            smp = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
            ins = int(r[hdr.index("Instructions Executed")])
        except (ValueError, IndexError):
            continue
        key = (f, int(r[0]))
        agg[key][0] += smp
        agg[key][1] += ins
        agg[key][2] = r[1][:90]
        tot += smp
    print(f"total samples {tot}")
    for (fn, ln), (s, i, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{100.0 * s / max(tot, 1):5.1f}% {i:>10} {fn}:{ln}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
