"""Host-side cost of the fit entry points at N = 1000 (GPU box): python tools/time_host.py"""
import ctypes, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import workloads as W
from paper_2007_09884_b200 import opmm
rec = torch.as_tensor(np.loadtxt("tests/golden/trace_truth_A10_dt1_n100.txt") + W.noise(101)).pin_memory().numpy()
ctl, sp = W.Control(), W.paper_space()
with opmm.opmm_create(0) as h:
    recd = torch.as_tensor(rec, device="cuda")
    out = torch.zeros(ctypes.sizeof(opmm.FitResult), dtype=torch.uint8, device="cuda")
    o = opmm.fit_options(cpu_check=0)
    s = torch.cuda.ExternalStream(h.stream)
    for name, fn in [("fit_async dev rec", lambda: opmm.opmm_fit_async(h, recd, ctl, sp, 1000, out, o)),
                     ("fit sync host rec", lambda: opmm.opmm_fit(h, rec, ctl, sp, 1000, o)),
                     ("fit sync dev rec", lambda: opmm.opmm_fit(h, recd, ctl, sp, 1000, o))]:
        for _ in range(20): fn(); s.synchronize()
        ts = []
        for _ in range(50):
            s.synchronize()
            t0 = time.perf_counter(); fn(); t1 = time.perf_counter()
            ts.append(t1 - t0)
        print(f"{name:20s} call {np.median(ts)*1e6:7.1f} us", flush=True)
    # python binding overhead: marshal structs only
    t0 = time.perf_counter()
    for _ in range(1000): opmm._space(sp); opmm._ctl(ctl)
    print("marshal", (time.perf_counter()-t0)*1e3, "us/call")
