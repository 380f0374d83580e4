"""Write the recorded-trace fixtures under tests/golden/ from the CPU oracle.

Only calls oracle/ (the committed, pinned CPU oracle) and workloads/ (inputs);
nothing comes from the CUDA path.  Run: python scripts/make_traces.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import workloads as W  # noqa: E402


def main():
    ctl = W.Control()   # A = +10 deg, theta0 = 0, dt = 1 ms, 100 steps
    rec = oracle.positions(W.truth_opc(), ctl)
    path = os.path.join(ROOT, "tests", "golden", "trace_truth_A10_dt1_n100.txt")
    with open(path, "w") as f:
        f.write("# Clean recorded trace for the bench / smoke workload (SURVEY 8(d) TRUTH):\n"
                "# oracle.positions(TRUTH = Table 1 defaults with PW = 40 ms, A = +10 deg,\n"
                "# theta0 = 0, dt = 1 ms, n_steps = 100), written by scripts/make_traces.py\n"
                "# (CPU oracle only).  101 samples, degrees, %.17g.\n")
        for v in rec:
            f.write("%.17g\n" % v)
    print("wrote", path)


if __name__ == "__main__":
    main()
