"""Top stall-sampled SASS lines of one kernel in an ncu report.
    python tools/ncu_top_lines.py REPORT KERNEL_REGEX [N]"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--kernel-name", "regex:" + kern, "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hi = [j for j, x in enumerate(r) if "Source" in x and "Address" in x][0]
    h = r[hi]
    rows = [x for x in r[hi + 1:] if len(x) == len(h)]
    i, s = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")

    def num(x):
        try:
            return int(x)
        except ValueError:
            return 0
    seen = set()
    rows = [x for x in rows if not (x[0] in seen or seen.add(x[0]))]
    print("total samples", sum(num(x[i]) for x in rows))
    for x in sorted(rows, key=lambda x: -num(x[i]))[:n]:
        print(f"{x[i]:>6} {x[0][-5:]} {x[s][:100]}")


if __name__ == "__main__":
    main()
