"""f2 lane-refill model: the crossing-step
distribution of diverged S_paper candidates (oracle trajectories) and the
throughput of refilling dead lanes in batches of R, with the measured costs
(setup ~80 step-equivalents per warp-wide batch: 100 us of setup against
1.26 us per step per 10^6 candidates).   python tests/diag/model_refill.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402  (test infrastructure: trajectories for the model's input)
import workloads as W  # noqa: E402

ctl, sp = W.Control(), W.paper_space()
rec = np.loadtxt(os.path.join(ROOT, "tests/golden/trace_truth_A10_dt1_n100.txt"), comments="#") + W.noise(101)
rel, _, Ap = oracle.relativize(rec, ctl.amplitude_deg)
N = 20000
P = oracle.generate_batch(sp, 0, N)
life = np.empty(N, dtype=int)
for i in range(N):
    d = oracle.simulate(P[i], 1.0, 100, Ap, 40.0)
    with np.errstate(all="ignore"):
        bad = ~(np.cumsum(np.abs(d - rel)) < 1e20)
    life[i] = np.argmax(bad) if bad.any() else 100
div = life < 100
print(f"diverged {div.mean():.3f}; crossing step median {np.median(life[div]):.0f} mean {life[div].mean():.1f}; "
      f"by step 20: {(life[div] <= 20).mean():.2f}; loop work removable {(100 - life).sum() / (100 * N):.3f}")
S, rng = 80.0, np.random.default_rng(0)


def refill(R, chunk=2, warps=200):
    tot = done = 0.0
    for _ in range(warps):
        q = list(rng.choice(life, size=2000))
        rem = np.array([q.pop() for _ in range(32)], float)
        alive = np.ones(32, bool)
        t = S
        while len(q) >= 32:
            order = np.sort(rem[alive])
            need = max(R - (32 - alive.sum()), 1)
            adv = np.ceil((order[need - 1] if need <= len(order) else order[-1]) / chunk) * chunk
            t += adv
            rem -= adv
            alive &= ~(rem <= 0)
            dead = np.flatnonzero(~alive)
            for lane in dead:
                rem[lane] = q.pop()
                alive[lane] = True
            t += S
            done += len(dead)
        tot += t
    return tot / done


base = (S + 100) / 32
for R in (4, 8, 12, 16, 20, 24, 28, 32):
    print(f"refill when {R:2d} lanes are dead: {base / refill(R):.2f}x the current throughput")
