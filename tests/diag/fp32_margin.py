"""fp32 vs fp64 per-sample trajectory difference over 3e4 RK4-stable S_paper candidates (GPU box)."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import oracle, workloads as W
from oracle import referee
from paper_2007_09884_b200 import opmm
ctl = W.Control(amplitude_deg=10.0)
sp = W.paper_space()
n = 30000
c = oracle.generate_batch(sp, 0, n)
rho = np.array([referee.rk4_spectral_radius(p, 1.0) for p in c])
stable = rho < 1.0
with opmm.opmm_create(0) as h:
    opc = torch.as_tensor(np.ascontiguousarray(c.T), device="cuda")
    t64 = torch.zeros((101, n), dtype=torch.float64, device="cuda")
    t32 = torch.zeros((101, n), dtype=torch.float32, device="cuda")
    opmm.opmm_simulate(h, opc, n, ctl, t64, precision=0, stream=torch.cuda.current_stream())
    opmm.opmm_simulate(h, opc, n, ctl, t32, precision=1, stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    d = (t32.double() - t64).abs().cpu().numpy()
    T64 = t64.cpu().numpy()
fin = np.all(np.isfinite(T64), axis=0) & (np.abs(T64).sum(0) < 1e20)
sel = stable & fin
print("stable finite", sel.sum(), "max |diff| deg", d[:, sel].max(), "99.99pct", np.quantile(d[:, sel].max(0), 0.9999))
