"""Instruction mix of one kernel from `ncu --page source --print-source sass --csv`."""
import csv
import sys


def main(path, points):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ie, src = hdr.index("Instructions Executed"), hdr.index("Source")
    tot, ops = 0.0, {}
    for r in rows[2:]:
        try:
            n = float(r[ie])
        except (ValueError, IndexError):
            continue
        tot += n
        toks = r[src].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        op = op.split(".")[0]
        ops[op] = ops.get(op, 0) + n
    print(f"total warp instructions {tot:.4g}; per point {tot * 32 / points:.1f}")
    for k, v in sorted(ops.items(), key=lambda x: -x[1])[:40]:
        print(f"{k:12s} {v / tot * 100:6.2f}%  per-point {v * 32 / points:6.2f}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]))
