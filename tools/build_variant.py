"""Build a variant of libdivuq_b200.so with extra -D flags into tools/variants/
(git-ignored scratch; select it with DIVUQ_LIB_PATH).  Usage:
    python tools/build_variant.py NAME -DFOO=1 [-DBAR=2 ...]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as g  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(ROOT, "tools", "variants", name + ".so")
os.makedirs(os.path.dirname(out), exist_ok=True)
cmd = [g.NVCC, *g.NVCC_FLAGS, *defs, "-o", out, os.path.join(g.CSRC, "capi.cu")]
res = subprocess.run(cmd, capture_output=True, text=True)
if res.returncode:
    sys.exit(res.stderr[-3000:])
for ln in res.stdout.splitlines() + res.stderr.splitlines():
    if "mc_chunk" in ln or ("Used" in ln and "mc_chunk" in ln):
        pass
print(out)
