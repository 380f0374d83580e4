"""One fp64 fit of 10^6 S_paper candidates per trace length (n_steps from
argv), for an ncu capture of how the fp64 pipe utilisation splits between
the setup-dominated (n = 1) and the loop-dominated (large n) regimes.
    python tools/gpu/prof_steps.py 1 100 1000"""
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch, workloads as W
from paper_2007_09884_b200 import opmm
sys.path.insert(0, os.path.join(ROOT, "tools"))
from synth_trace import truth_trace
with opmm.opmm_create(0, kernel_timing=True) as h:
    out = torch.zeros(ctypes.sizeof(opmm.FitResult), dtype=torch.uint8, device="cuda")
    for n_steps in (int(x) for x in sys.argv[1:]):
        ctl = W.Control(n_steps=n_steps)
        rec = torch.as_tensor(truth_trace(opmm, h, ctl), device="cuda")
        opmm.opmm_fit_async(h, rec, ctl, W.paper_space(n_steps=n_steps), 10**6, out, opmm.fit_options(cpu_check=0))
        torch.cuda.ExternalStream(h.stream).synchronize()
        print(n_steps, opmm.opmm_last_kernel_ms(h), flush=True)
