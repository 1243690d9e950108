"""Regenerate the committed golden fixtures from the UNMODIFIED reference.

Run here (the reference is mounted read-only at /root/reference):
    make -C oracle all ref && python tests/golden/make_golden.py

Every fixture is produced by oracle/_ref/libcbgref.so, i.e. the reference's
own compress / write_frsz2_file / gmres_solve compiled from
/root/reference/proj/src, so the GPU parity tests (which cannot read
/root/reference on the GPU box) compare against the reference itself.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import pyoracle as po  # noqa: E402


def residuals_csv(history):
    """cli.cpp:87-94 schema: iteration,rrn(%.17g),explicit."""
    lines = ["iteration,rrn,explicit"]
    for it, rrn, ex in history:
        lines.append(f"{it},{rrn:.17g},{1 if ex else 0}")
    return "\n".join(lines) + "\n"


def main():
    assert po.Ref.available(), "build oracle/_ref first (make -C oracle ref)"
    R, P = po.Ref(), po.Port()
    meta = {"containers": {}, "solves": {}}
    # 1) codec containers on the corner-case generators
    inputs = {
        "mixed_4099_s7": po.mixed_values(4099, 7),
        "wide_5000_s11": po.wide_values(5000, 11, -60, 0),
        "uniform_1000_s3": po.uniform_values(1000, 3, -100.0, 100.0),
    }
    for name, v in inputs.items():
        np.save(os.path.join(HERE, f"in_{name}.npy"), v)
        for l in (16, 21, 32):
            c = R.container(v, l)
            fn = f"c_{name}_l{l}.frsz2"
            with open(os.path.join(HERE, fn), "wb") as f:
                f.write(c)
            meta["containers"][fn] = hashlib.sha256(c).hexdigest()
    # 2) 2^24 uniform[-1,1) mt19937_64(42) -- hashes only
    big = po.uniform_values(1 << 24, 42)
    meta["uniform_2p24_s42_input_sha256"] = hashlib.sha256(big.tobytes()).hexdigest()
    meta["uniform_2p24_s42_container_sha256"] = {
        str(l): hashlib.sha256(R.container(big, l)).hexdigest() for l in (16, 21, 32)}
    # 3) solver histories (residuals.csv bytes) on small instances
    cases = {
        "convdiff100_pe1": ("convdiff", (100, 100, 1.0, 0.0), ["f64", "frsz2-32", "f32", "frsz2-16", "frsz2-21"], 100),
        "convdiff8_pe1_rs12": ("convdiff", (8, 8, 1.0, 12.0), ["frsz2-32"], 100),
        "convdiff12_pe1_m20": ("convdiff", (12, 12, 1.0, 0.0), ["frsz2-32", "f64"], 20),
        "p7_16": ("stencil", (0, 16, 16, 16, 0.0), ["f64", "frsz2-32", "frsz2-16", "frsz2-21"], 100),
        "cd7_12_pe1": ("stencil", (1, 12, 12, 12, 1.0), ["f64", "frsz2-32"], 30),
        "p27_10": ("stencil", (2, 10, 10, 10, 0.0), ["f64", "frsz2-32"], 100),
    }
    for name, (kind, args, fmts, restart) in cases.items():
        if kind == "convdiff":
            rp, ci, va = P.convdiff(args[0], args[1], args[2], decades=args[3])
        else:
            rp, ci, va = P.stencil(args[0], args[1], args[2], args[3], pe=args[4])
        b, _ = R_generate(R, P, rp, ci, va)
        for fmt in fmts:
            r = R.gmres(rp, ci, va, b, fmt=fmt, restart=restart)
            fn = f"res_{name}_{fmt}.csv"
            with open(os.path.join(HERE, fn), "w") as f:
                f.write(residuals_csv(r["history"]))
            meta["solves"][f"{name}/{fmt}"] = dict(
                kind=kind, args=list(args), restart=restart, fmt=fmt,
                converged=r["converged"], iterations=r["iterations"], restarts=r["restarts"],
                final_rrn=r["final_rrn"], residuals=fn,
                solution_sha256=hashlib.sha256(r["x"].tobytes()).hexdigest())
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", len(meta["containers"]), "containers,", len(meta["solves"]), "solves")


def R_generate(R, P, rp, ci, va):
    n = rp.size - 1
    b = np.zeros(n)
    x = np.zeros(n)
    assert R.lib.ref_generate_problem(n, rp, ci, va, b, x) == 0
    return b, x


if __name__ == "__main__":
    main()
