import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import workloads as W
from paper_2007_09884_b200 import opmm
with opmm.opmm_create(0) as h:
    out = torch.zeros(ctypes.sizeof(opmm.FitResult), dtype=torch.uint8, device="cuda")
    ctl = W.Control(n_steps=100)
    rec = torch.linspace(0, 10, 101, dtype=torch.float64, device="cuda")
    for _ in range(5):
        opmm.opmm_fit_async(h, rec, ctl, W.paper_space(), 32, out, opmm.fit_options(cpu_check=0))
    torch.cuda.synchronize()
