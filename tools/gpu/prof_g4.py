"""One G4 fit (10^8, superposition kernel, default options) for an ncu capture."""
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch, workloads as W
from paper_2007_09884_b200 import opmm
rec = np.loadtxt(os.path.join(ROOT, "tests/golden/trace_truth_A10_dt1_n100.txt"))
ctl, sp = W.Control(), W.g4_space(100)
with opmm.opmm_create(0) as h:
    recd = torch.as_tensor(rec, device="cuda")
    out = torch.zeros(ctypes.sizeof(opmm.FitResult), dtype=torch.uint8, device="cuda")
    opmm.opmm_fit_async(h, recd, ctl, sp, sp.n_grid(), out, opmm.fit_options(cpu_check=0))
    torch.cuda.ExternalStream(h.stream).synchronize()
    print(opmm.decode_result(bytes(out.cpu().numpy()))["best_index"])
