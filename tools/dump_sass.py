"""SASS listing of every kernel in libdivuq_b200.so -> profiles/sass/.

cuobjdump -sass the in-tree library, split it per function, demangle, and
write (a) SUMMARY.txt: one line per function with the instruction classes that
prove the design (UTMALDG = TMA loads, SYNCS = mbarrier, MUFU, fp64 ops, local
spills; HMMA/UTC* would be tensor-core ops -- none by design), and (b) one
.sass file per kernel family holding the instantiations the bench/tests use.

    python tools/dump_sass.py
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2510_01190_b200", "libdivuq_b200.so")
OUT = os.path.join(ROOT, "profiles", "sass")

CLASSES = [
    ("UTMALDG", r"\bUTMALDG"), ("UBLKCP", r"\bUBLKCP"), ("SYNCS", r"\bSYNCS"),
    ("LDS", r"\bLDS\b|\bLDS\."), ("LDG", r"\bLDG"), ("STG", r"\bSTG"), ("SHFL", r"\bSHFL"),
    ("MUFU", r"\bMUFU"), ("DFMA/DMUL/DADD", r"\bD(FMA|MUL|ADD)\b"),
    ("HMMA/UTC", r"\bHMMA|\bUTC"), ("STL/LDL", r"\bSTL|\bLDL"),
]


def demangle(names):
    res = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return res.stdout.splitlines()


def ptxas_table():
    path = os.path.join(ROOT, "paper_2510_01190_b200", "csrc", "ptxas.log")
    if not os.path.exists(path):
        return ["(ptxas.log absent: build with __graft_entry__.build(force=True))"]
    out, name = [], None
    mangled, stats = [], {}
    for ln in open(path):
        m = re.search(r"Compiling entry function '([^']+)'", ln)
        if m:
            name = m.group(1)
            mangled.append(name)
            stats[name] = ["", ""]
            continue
        if name and "spill stores" in ln:
            stats[name][0] = ln.strip()
        if name and "Used" in ln and "registers" in ln:
            stats[name][1] = re.sub(r"^ptxas info\s*:\s*", "", ln.strip())
    for m, pretty in zip(mangled, demangle(mangled)):
        short = re.sub(r"^void |\(anonymous namespace\)::|divuq::", "", pretty).split("(")[0]
        out.append(f"{short:60s} {stats[m][1]}; {stats[m][0]}")
    return sorted(out)


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    blocks = re.split(r"\n\s*Function : ", sass)[1:]
    funcs = []
    for b in blocks:
        name, body = b.split("\n", 1)
        instr = [ln for ln in body.splitlines() if re.match(r"\s+/\*[0-9a-f]{4,}\*/\s", ln)]
        funcs.append((name.strip(), instr))
    pretty = demangle([f[0] for f in funcs])
    os.makedirs(OUT, exist_ok=True)
    for f in os.listdir(OUT):
        if f.endswith(".sass"):
            os.remove(os.path.join(OUT, f))
    fam = collections.defaultdict(list)
    lines = []
    for (mangled, instr), pname in zip(funcs, pretty):
        short = re.sub(r"^void ", "", pname)
        short = re.sub(r"\(anonymous namespace\)::", "", short)
        family = re.sub(r"<.*", "", short).split("(")[0].replace("divuq::", "")
        short = short.split("(")[0].replace("divuq::", "")
        cnt = {k: sum(1 for ln in instr if re.search(rx, ln)) for k, rx in CLASSES}
        lines.append(f"{short:60s} instr={len(instr):5d} " +
                     " ".join(f"{k}={v:3d}" for k, v in cnt.items()))
        fam[family].append((short, instr))
    with open(os.path.join(OUT, "SUMMARY.txt"), "w") as fh:
        fh.write("SASS of libdivuq_b200.so (sm_100a, nvcc 12.9, cuobjdump -sass); tools/dump_sass.py\n")
        fh.write("UTMALDG = cp.async.bulk.tensor (TMA) loads; SYNCS = mbarrier ops; "
                 "HMMA/UTC = tensor-core ops (none by design: no contraction).\n\n")
        fh.write("\n".join(sorted(lines)) + "\n")
        fh.write("\nptxas -v (registers, spills) per function, from the same build "
                 "(paper_2510_01190_b200/csrc/ptxas.log):\n")
        fh.write("\n".join(ptxas_table()) + "\n")
    for family, items in fam.items():
        # keep the file small: at most 4 instantiations per family
        with open(os.path.join(OUT, f"{family}.sass"), "w") as fh:
            for short, instr in items[:4]:
                fh.write(f"// ===== {short}  ({len(instr)} instructions)\n")
                fh.write("\n".join(instr) + "\n\n")
    print(f"{len(funcs)} functions, {len(fam)} families -> {OUT}")


if __name__ == "__main__":
    sys.exit(main())
