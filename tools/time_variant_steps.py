"""fit1 vs fit3 (warp-specialised) kernel time at several trace lengths (GPU box)."""
import ctypes, os, sys
import torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import workloads as W
from paper_2007_09884_b200 import opmm
N = 10**6
with opmm.opmm_create(0, kernel_timing=True) as h:
    out = torch.zeros(ctypes.sizeof(opmm.FitResult), dtype=torch.uint8, device="cuda")
    for kv in (1, 3):
        line = []
        for ns in (1, 50, 100, 200):
            ctl = W.Control(n_steps=ns)
            rec = torch.linspace(0, 10, ns + 1, dtype=torch.float64, device="cuda")
            o = opmm.fit_options(cpu_check=0, kernel_variant=kv)
            ts = []
            for _ in range(6):
                opmm.opmm_fit_async(h, rec, ctl, W.paper_space(n_steps=100), N, out, o)
                ts.append(opmm.opmm_last_kernel_ms(h))
            line.append(f"n={ns}: {sorted(ts)[3]*1e3:6.1f}")
        print(f"variant {kv}: " + "  ".join(line), flush=True)
