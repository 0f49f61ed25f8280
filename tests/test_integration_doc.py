"""INTEGRATION.md lists every symbol include/divuq_b200.h exports (CPU test)."""

import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_every_header_symbol_is_documented():
    hdr = open(os.path.join(ROOT, "include", "divuq_b200.h")).read()
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    syms = sorted(set(re.findall(r"\b(divuq_[a-z0-9_]+)\s*\(", hdr)))
    assert len(syms) >= 50, syms
    missing = [s for s in syms if f"`{s}`" not in doc]
    assert not missing, missing
