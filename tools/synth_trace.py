"""Synthetic recorded traces for the timing tools: TRUTH simulated by the
library itself (opmm_simulate), plus the seeded workload noise.  Measurement
input only -- the oracle is test infrastructure (tests/, smoke, bench's CPU
baseline) and the tools do not import it."""
import numpy as np
import torch

import workloads as W


def truth_trace(opmm, h, ctl, noisy=True):
    opc = torch.as_tensor(np.ascontiguousarray(W.truth_opc().reshape(-1, 1)), device="cuda")
    traj = torch.zeros((ctl.n_steps + 1, 1), dtype=torch.float64, device="cuda")
    opmm.opmm_simulate(h, opc, 1, ctl, traj, stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    rec = traj[:, 0].cpu().numpy().copy()
    return rec + W.noise(ctl.n_steps + 1) if noisy else rec
