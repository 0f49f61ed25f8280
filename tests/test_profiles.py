"""Committed evidence stays in step with the code (CPU tests).

* every ``__global__`` kernel in csrc/ has a committed SASS listing in
  profiles/sass/ (tools/dump_sass.py), and SUMMARY.txt lists it;
* every kernel in a committed ncu launch list (profiles/*/launches_*.csv)
  has a listing;
* no binary ncu reports are tracked (the summaries are).
"""

import csv
import glob
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2510_01190_b200", "csrc")
SASS = os.path.join(ROOT, "profiles", "sass")


def _kernels():
    names = set()
    for path in glob.glob(os.path.join(CSRC, "*.cu*")):
        src = open(path).read()
        for m in re.finditer(r"__global__\s+void\s+(?:__launch_bounds__\([^)]*\)\s*)?(\w+)\s*\(", src):
            names.add(m.group(1))
    return names


def test_every_kernel_has_a_sass_listing():
    kernels = _kernels()
    assert len(kernels) >= 20, sorted(kernels)
    summary = open(os.path.join(SASS, "SUMMARY.txt")).read()
    for k in sorted(kernels):
        assert os.path.exists(os.path.join(SASS, f"{k}.sass")), f"no SASS listing for {k}"
        assert re.search(rf"^{k}\b", summary, re.M), f"{k} missing from SUMMARY.txt"


def test_launched_kernels_have_listings():
    lists = glob.glob(os.path.join(ROOT, "profiles", "*", "launches_*.csv"))
    assert lists, "no committed ncu launch lists"
    for path in lists:
        rows = [r for r in csv.reader(open(path)) if r]
        hdr = next(r for r in rows if "Kernel Name" in r)
        ki = hdr.index("Kernel Name")
        for r in rows[rows.index(hdr) + 1:]:
            if len(r) <= ki or not r[ki] or r[ki] == "Kernel Name":
                continue
            name = re.sub(r"^(void )?(divuq::)?(\(anonymous namespace\)::)?", "", r[ki])
            name = re.split(r"[<(]", name)[0]
            if "::" in name:      # torch's own kernels (L2 flush, dtype casts): not ours
                continue
            assert os.path.exists(os.path.join(SASS, f"{name}.sass")), (path, name)


def test_no_binary_reports_tracked():
    out = subprocess.run(["git", "ls-files", "profiles"], cwd=ROOT, capture_output=True, text=True)
    if out.returncode != 0:
        return
    assert not [f for f in out.stdout.split() if f.endswith(".ncu-rep")]
