"""Per-block start/end spread of the fit kernel (GPU box; needs a build with
-DOPMM_EXP_BLOCKTIME, e.g. via tools/ab_variants.sh or build_variant).
    OPMM_LIB=build/variants/libopmm_bt.so python tools/time_blocks.py"""
import ctypes, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from paper_2007_09884_b200 import opmm  # noqa: E402
N = 10**6
with opmm.opmm_create(0) as h:
    rec = torch.linspace(0, 10, 101, dtype=torch.float64, device="cuda")
    err = torch.zeros(N, dtype=torch.float64, device="cuda")
    out = torch.zeros(ctypes.sizeof(opmm.FitResult), dtype=torch.uint8, device="cuda")
    for prec in (0, 1):
        for _ in range(3):
            opmm.opmm_fit_async(h, rec, W.Control(), W.paper_space(), N, out,
                                opmm.fit_options(precision=prec, cpu_check=0, err_out=err))
        torch.cuda.ExternalStream(h.stream).synchronize()
        t = err[:296].cpu().numpy().reshape(-1, 2)
        t0 = t[:, 0].min()
        st, en = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
        print(f"{'fp64' if prec == 0 else 'fp32'}: kernel {opmm.opmm_last_kernel_ms(h)*1e3:.1f} us; "
              f"block start max {st.max():.1f} us; end min/median/max {en.min():.1f}/"
              f"{np.median(en):.1f}/{en.max():.1f} us")
