"""Kernel time of a 10^6-candidate S_paper fit (fp64 and fp32) per trace length,
median of 7 launches:   python tools/gpu/time_steps.py [pkg_dir|-] n1 n2 ..."""
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
pkg = sys.argv[1] if len(sys.argv) > 1 and sys.argv[1] != "-" else ROOT
sys.path.insert(0, ROOT)
sys.path.insert(0, pkg)
import torch, workloads as W
from paper_2007_09884_b200 import opmm
sys.path.insert(0, os.path.join(ROOT, "tools"))
from synth_trace import truth_trace
tag = os.path.basename(pkg.rstrip("/")) if pkg != ROOT else "repo"
with opmm.opmm_create(0, kernel_timing=True) as h:
    out = torch.zeros(ctypes.sizeof(opmm.FitResult), dtype=torch.uint8, device="cuda")
    for n_steps in (int(x) for x in sys.argv[2:]):
        ctl = W.Control(n_steps=n_steps)
        rec = torch.as_tensor(truth_trace(opmm, h, ctl), device="cuda")
        sp = W.paper_space(n_steps=n_steps)
        line = []
        for prec in (0, 1):
            o = opmm.fit_options(cpu_check=0, precision=prec)
            ts = []
            for r in range(10):
                opmm.opmm_fit_async(h, rec, ctl, sp, 10**6, out, o)
                if r >= 3:
                    ts.append(opmm.opmm_last_kernel_ms(h))
            torch.cuda.ExternalStream(h.stream).synchronize()
            line.append(f"{'fp64' if prec == 0 else 'fp32'} {1e3 * sorted(ts)[3]:8.1f} us")
        print(f"{tag:>6} n={n_steps:5d}  " + "  ".join(line), flush=True)
