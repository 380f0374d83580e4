"""Two fit launches for an ncu A/B capture: the given option sets, in order
(10^6 S_paper candidates, n = 100).   python tools/gpu/prof_fit_modes.py "top_k=0" "top_k=32" """
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch, workloads as W
from paper_2007_09884_b200 import opmm
rec = np.loadtxt(os.path.join(ROOT, "tests/golden/trace_truth_A10_dt1_n100.txt")) + W.noise(101)
ctl, sp = W.Control(), W.paper_space()
with opmm.opmm_create(0) as h:
    recd = torch.as_tensor(rec, device="cuda")
    out = torch.zeros(ctypes.sizeof(opmm.FitResult), dtype=torch.uint8, device="cuda")
    for spec in sys.argv[1:]:
        kw = {k: int(v) for k, v in (x.split("=") for x in spec.split(",") if x)}
        opmm.opmm_fit_async(h, recd, ctl, sp, 10**6, out, opmm.fit_options(cpu_check=0, **kw))
        torch.cuda.ExternalStream(h.stream).synchronize()
        print(spec, opmm.decode_result(bytes(out.cpu().numpy()))["best_index"], flush=True)
