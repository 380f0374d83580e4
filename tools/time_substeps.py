"""Fit kernel time and finite fraction vs RK4 substeps (GPU box): python tools/time_substeps.py"""
import ctypes, os, sys
import torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import workloads as W
from paper_2007_09884_b200 import opmm
with opmm.opmm_create(0, kernel_timing=True) as h:
    out = torch.zeros(ctypes.sizeof(opmm.FitResult), dtype=torch.uint8, device="cuda")
    rec = torch.linspace(0, 10, 101, dtype=torch.float64, device="cuda")
    for s in (0, 2, 4, 16, 64):
        ctl = W.Control(substeps=s)
        o = opmm.fit_options(cpu_check=0)
        ts = []
        for _ in range(6):
            opmm.opmm_fit_async(h, rec, ctl, W.paper_space(), 10**6, out, o)
            ts.append(opmm.opmm_last_kernel_ms(h))
        torch.cuda.ExternalStream(h.stream).synchronize()
        r = opmm.decode_result(bytes(out.cpu().numpy()))
        print(f"substeps {s:3d}: {sorted(ts)[3]*1e3:7.1f} us  n_finite {r['n_finite']}", flush=True)
