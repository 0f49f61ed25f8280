"""Per-opcode instruction mix and stall share of one kernel from
`ncu --page source --print-source sass --csv` (tools/gpu_profiles_r02.sh)."""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    data = rows[2:]
    isrc, iss, iex = (hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"),
                      hdr.index("Instructions Executed"))
    tot = sum(float(r[iss] or 0) for r in data) or 1.0
    ex = sum(float(r[iex] or 0) for r in data) or 1.0
    agg = defaultdict(lambda: [0.0, 0.0])
    for r in data:
        t = r[isrc].split()
        if not t:
            continue
        op = (t[1] if t[0].startswith("@") and len(t) > 1 else t[0]).split(".")[0]
        agg[op][0] += float(r[iex] or 0)
        agg[op][1] += float(r[iss] or 0)
    print(f"warp instructions executed: {ex:.6g}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:30]:
        print(f"{k:12s} {v[0] / ex * 100:6.2f}% of instructions  {v[1] / tot * 100:6.2f}% of stall samples")


if __name__ == "__main__":
    main(sys.argv[1])
