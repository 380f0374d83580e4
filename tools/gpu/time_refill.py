"""Lane refill (kernel_variant 5) against the default kernel
(variant 1): kernel time of a 10^6-candidate S_paper fit at n = 100 / 150 /
300 steps, fp64 and fp32, median of 9 launches (opmm_last_kernel_ms), plus
the fraction of candidates that end at +inf.
    python tools/gpu/time_refill.py [pkg_dir]
pkg_dir: the package build to time (REFILL_MIN / REFILL_SEG sweeps)."""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
pkg = sys.argv[1] if len(sys.argv) > 1 else ROOT
sys.path.insert(0, ROOT)
sys.path.insert(0, pkg)
import torch  # noqa: E402
import workloads as W  # noqa: E402
from paper_2007_09884_b200 import opmm  # noqa: E402
sys.path.insert(0, os.path.join(ROOT, "tools"))
from synth_trace import truth_trace  # noqa: E402

tag = os.path.basename(pkg.rstrip("/")) if pkg != ROOT else "repo"
n = 10**6
with opmm.opmm_create(0, kernel_timing=True) as h:
    for n_steps in (100, 150, 300):
        ctl = W.Control(n_steps=n_steps)
        rec = truth_trace(opmm, h, ctl)
        sp = W.paper_space(n_steps=n_steps)
        recd = torch.as_tensor(rec, device="cuda")
        out = torch.zeros(ctypes.sizeof(opmm.FitResult), dtype=torch.uint8, device="cuda")
        line = []
        for prec in (0, 1):
            t = {}
            for kv in (1, 5):
                o = opmm.fit_options(cpu_check=0, precision=prec, kernel_variant=kv)
                for _ in range(3):
                    opmm.opmm_fit_async(h, recd, ctl, sp, n, out, o)
                ts = []
                for _ in range(9):
                    opmm.opmm_fit_async(h, recd, ctl, sp, n, out, o)
                    ts.append(opmm.opmm_last_kernel_ms(h))
                torch.cuda.ExternalStream(h.stream).synchronize()
                r = opmm.decode_result(bytes(out.cpu().numpy()))
                t[kv] = (1e3 * sorted(ts)[4], r["best_index"], r["n_finite"])
            assert t[1][1:] == t[5][1:], (t, "refill must give the same argmin and n_finite")
            line.append(f"{'fp64' if prec == 0 else 'fp32'}: v1 {t[1][0]:7.1f} us  refill {t[5][0]:7.1f} us "
                        f"(x{t[1][0] / t[5][0]:.3f})")
        print(f"{tag:>6} n={n_steps:3d} inf {1 - t[1][2] / n:.3f} | " + " | ".join(line), flush=True)
