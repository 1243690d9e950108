"""Shared test helpers (paths, fixture readers)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def read_golden_text(fn):
    with open(os.path.join(GOLDEN, fn)) as f:
        return f.read()


def csv_of(history):
    """residuals.csv bytes in the reference's schema (cli.cpp:87-94)."""
    lines = ["iteration,rrn,explicit"] + [f"{i},{r:.17g},{1 if e else 0}" for i, r, e in history]
    return "\n".join(lines) + "\n"
