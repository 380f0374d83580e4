"""Kernel time of the fit modes on the bench workload (10^6 S_paper
candidates, n = 100), median of 9 launches (opmm_last_kernel_ms):
    python tools/gpu/time_modes.py [pkg_dir] [n]
pkg_dir: directory holding the paper_2007_09884_b200 package to time (A/B
against another build); default the repo's."""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
pkg = sys.argv[1] if len(sys.argv) > 1 and sys.argv[1] != "-" else ROOT
n = int(float(sys.argv[2])) if len(sys.argv) > 2 else 10**6
sys.path.insert(0, ROOT)
sys.path.insert(0, pkg)
import torch  # noqa: E402
import workloads as W  # noqa: E402
from paper_2007_09884_b200 import opmm  # noqa: E402

rec = np.loadtxt(os.path.join(ROOT, "tests/golden/trace_truth_A10_dt1_n100.txt")) + W.noise(101)
ctl, sp = W.Control(), W.paper_space()
new_api = "top_k" in [f[0] for f in opmm.FitOptions._fields_]
modes = [("fp64", dict(precision=0)), ("fp32", dict(precision=1)),
         ("fp32 certify", dict(precision=1, certify=1))]
if new_api:
    modes += [("fp64 top1", dict(precision=0, top_k=1)), ("fp64 top8", dict(precision=0, top_k=8)),
              ("fp64 top32", dict(precision=0, top_k=32)), ("fp32 certify K=32", dict(precision=1, certify=1, top_k=32)),
              ("fp64 nosort", dict(precision=0, flags=1)), ("fp64 block 192", dict(precision=0, block_size=192)),
              ("fp64 block 128", dict(precision=0, block_size=128))]
with opmm.opmm_create(0, kernel_timing=True) as h:
    recd = torch.as_tensor(rec, device="cuda")
    out = torch.zeros(ctypes.sizeof(opmm.FitResult), dtype=torch.uint8, device="cuda")
    for name, kw in modes:
        o = opmm.fit_options(cpu_check=0, **kw)
        for _ in range(3):
            opmm.opmm_fit_async(h, recd, ctl, sp, n, out, o)
        ts = []
        for _ in range(9):
            opmm.opmm_fit_async(h, recd, ctl, sp, n, out, o)
            ts.append(opmm.opmm_last_kernel_ms(h))
        torch.cuda.ExternalStream(h.stream).synchronize()
        r = opmm.decode_result(bytes(out.cpu().numpy()))
        print(f"{os.path.basename(pkg.rstrip('/')):>8} {name:18s} {1e3 * sorted(ts)[4]:8.1f} us  "
              f"best {r['best_index']} certified {r['certified']}", flush=True)
