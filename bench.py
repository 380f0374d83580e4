"""bench.py -- OPC candidate-simulation throughput of libopmm on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl libopmm|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N

A step = one pass of the whole hot path over one batch:
opmm_fit of the synthetic 10 deg saccade (1 kHz, 100 ms) over 10^6 random OPC
candidates per GPU from S_paper (BASELINE.json configs[1]): generate ->
simulate -> score -> argmin, plus for N > 1 the one NCCL all-gather of the
per-rank (E, index) pairs.  Candidates are sharded disjointly per rank, so
per-GPU work is fixed as N grows ("scaling": "weak").

value  : candidates/s over all ranks, inputs resident in HBM (opmm_fit_async),
         device time from CUDA events on the launching stream, max over ranks;
         L2 flushed (512 MiB write) between timed steps, outside the events.
e2e    : the same metric through the synchronous C-ABI call opmm_fit with the
         trace in pinned HOST memory, H2D + kernel + D2H + CPU_check timed.
roofline: the fused fit kernel vs the FP64 SIMT peak.
cpu_baseline: the CPU oracle (oracle/, as it stands) on a bounded sample.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

N_STEPS = 100
PER_GPU = 10**6
# Algorithmic FP64 work of the fit kernel per candidate:
# the RK4 map in two-step propagator blocks is 32 FMA + 2 score adds per two
# steps = 34 flop per step; generation + per-candidate setup = 1285 flop
# (ncu op counts dfma/dadd/dmul at n = 100 minus the loop's exact count,
# profiles/r01_fit_kernel_fp64_opcounts.txt).
FLOP_PER_STEP = 34
FLOP_SETUP = 1285
FP64_INST_PER_STEP = 18    # fp64-pipe instructions per step (loop)
FP64_INST_SETUP = 797      # fp64-pipe instructions per candidate outside the loop (ncu)
SMS, FP64_LANES, FP32_LANES, SM_MAX_MHZ = 148, 64, 128, 1965.0
FP64_PEAK_TFLOPS = SMS * FP64_LANES * 2 * SM_MAX_MHZ * 1e6 / 1e12   # 37.23
FP32_PEAK_TFLOPS = SMS * FP32_LANES * 2 * SM_MAX_MHZ * 1e6 / 1e12   # 74.45
# DFMA / FFMA microbenchmark (tools/fma_peak.cu, profiles/r02_fma_peak.txt) in
# the fit loop's operand form (every operand a distinct register): DFMA
# 36.90 TFLOP/s (99% of nominal), FFMA 45.64 TFLOP/s -- all-register FFMAs
# issue at ~0.61 of the nominal FP32 rate (the constant-operand form reaches
# 70.76), so 45.64 is the FP32 roofline of the fp32 loop.
FP64_MEASURED_TFLOPS = 36.90
FP32_MEASURED_TFLOPS = 45.64


def ncu_traffic_bytes(kernel="fit_kernel<double, 0, 0, 0>"):
    """dram__bytes_read.sum + dram__bytes_write.sum of a fit kernel from the
    committed `ncu --set full` capture summary (profiles/), per launch."""
    units = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    path = os.path.join(ROOT, "profiles", "r02_fit_kernels_ncu_full.txt")
    try:
        tot, on = 0.0, False
        for line in open(path):
            if line.startswith("kernel:"):
                on = kernel in line
                continue
            parts = line.split()
            if on and parts and parts[0] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                tot += float(parts[1]) * units[parts[2]]
        return tot or None
    except OSError:
        return None


def fp32_roofline(per_gpu, kernel_ms):
    """The fp32 fit kernel (uncertified, the kernel the fp32 leg's time is
    spent in) against both pipes it uses: the fp32 loop's executed flops
    (34 per step) vs the nominal FP32 peak, and the fp64
    generation + setup flops (1285 per candidate) vs the nominal FP64 peak.
    The two pipes share the warp schedulers' issue slots, so frac = the sum
    of the two fractions; ncu's issue utilisation is in profiles/."""
    t = kernel_ms * 1e-3
    f32 = FLOP_PER_STEP * N_STEPS * per_gpu / t / 1e12
    f64 = FLOP_SETUP * per_gpu / t / 1e12
    return {"bound": "alu", "unit": "TFLOP/s", "kernel": "fit_kernel<float, propagator, L1>",
            "kernel_ms": kernel_ms, "achieved": f32, "peak": FP32_MEASURED_TFLOPS,
            "fp32_frac": f32 / FP32_MEASURED_TFLOPS, "fp32_frac_of_nominal": f32 / FP32_PEAK_TFLOPS,
            "fp64_setup_tflops": f64, "fp64_frac": f64 / FP64_PEAK_TFLOPS,
            "frac": f32 / FP32_MEASURED_TFLOPS + f64 / FP64_PEAK_TFLOPS,
            "traffic": ncu_traffic_bytes("fit_kernel<float, 0, 0, 0>"),
            "peak_basis": "measured all-register FFMA rate (profiles/r02_fma_peak.txt); nominal "
                          "148 SM x 128 FP32 lanes x 2 x 1965 MHz = 74.4 for context; fp64 setup "
                          "vs nominal 37.2"}


def workload_config(per_gpu, world):
    """The workload keys both arms' `config` share (configs[1])."""
    return {"workload": workload_name(per_gpu, world), "n_candidates": per_gpu * world,
            "per_gpu": per_gpu, "n_steps": N_STEPS, "dt_ms": 1.0, "metric": "L1"}


def workload_name(per_gpu, world):
    return (f"configs[1]: single synthetic 10 deg horizontal saccade, 1 kHz, 100 ms, "
            f"{per_gpu:.0e} random OPC candidates per GPU over S_paper (x{world} GPUs)")


def make_trace():
    """Recorded trace: stored fixture written by scripts/make_traces.py from
    the CPU oracle (TRUTH at A = 10 deg) plus seeded N(0, 0.02 deg) noise."""
    path = os.path.join(ROOT, "tests", "golden", "trace_truth_A10_dt1_n100.txt")
    rec = np.loadtxt(path, comments="#")
    assert rec.shape == (N_STEPS + 1,)
    return rec + W.noise(N_STEPS + 1)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.2)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def host_info():
    """CPU model and the oracle's compiler, for the cpu_baseline record."""
    model = None
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except OSError:
        pass
    try:
        cc = subprocess.run(["gcc", "--version"], capture_output=True, text=True).stdout.splitlines()[0]
    except (OSError, IndexError):
        cc = "gcc"
    import oracle
    return {"cpu_model": model, "compiler": f"{cc}; {' '.join(oracle.CFLAGS)}"}


def cpu_baseline(target_s=12.0, sample_cap=3 * 10**6, single_n=20000):
    """The oracle as it stands on the host: one thread on a 2*10^4-candidate
    sample, then all cores (OpenMP) on a bounded sample of the same workload
    (same trace, same candidate stream)."""
    import oracle
    ctl = W.Control()
    rec = make_trace()
    sp = W.paper_space()
    cores = len(os.sched_getaffinity(0))
    t0 = time.perf_counter()
    oracle.fit(rec, ctl, sp, 0, single_n, nthreads=1)
    single = single_n / (time.perf_counter() - t0)
    t0 = time.perf_counter()
    oracle.fit(rec, ctl, sp, 0, 20000, nthreads=cores)
    rate0 = 20000 / (time.perf_counter() - t0)
    n = int(min(sample_cap, max(20000, rate0 * target_s)))
    t0 = time.perf_counter()
    oracle.fit(rec, ctl, sp, 0, n, nthreads=cores)
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": "candidate sims/s", "cores": cores, "threads": cores,
            "kind": "oracle", "single_thread_value": single,
            "sample": f"all cores: candidates [0, {n}) of the bench workload (same trace and Philox "
                      f"stream), {dt:.1f} s, OpenMP static chunks; single thread: [0, {single_n})",
            **host_info()}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    ctl = W.Control()
    rec = make_trace()
    sp = W.paper_space()
    cores = len(os.sched_getaffinity(0))
    n_total = args.per_gpu * args.gpus
    sample = min(200000, n_total)
    # step s scores candidates [b, b + sample) of the workload's [0, n_total),
    # wrapping around: every sample lies inside the workload the config names
    starts = [((k * sample) % n_total) if (k * sample) % n_total + sample <= n_total else 0
              for k in range(args.warmup + args.steps)]
    for s in range(args.warmup):
        oracle.fit(rec, ctl, sp, starts[s], starts[s] + sample, nthreads=cores)
    times = []
    for s in range(args.steps):
        b = starts[args.warmup + s]
        t0 = time.perf_counter()
        oracle.fit(rec, ctl, sp, b, b + sample, nthreads=cores)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * sum(times) / len(times)
    value = sample / (ms * 1e-3)
    line = {"impl": "reference", "metric": "OPC candidate sims/s", "value": value,
            "unit": "candidate sims/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {**workload_config(args.per_gpu, args.gpus),
                       "integrator": "rk4-classical (oracle)",
                       "n_candidates_timed": sample * args.steps,
                       "reference_step": f"{sample} candidates of the workload per step (bounded sample), "
                                         f"index ranges {sorted(set(starts[args.warmup:]))} + {sample}, "
                                         f"inside [0, {n_total})"},
            "cpu_baseline": {"value": value, "unit": "candidate sims/s", "cores": cores,
                             "threads": cores, "kind": "oracle",
                             "sample": f"{sample} candidates per step x {args.steps} steps",
                             **host_info()},
            "e2e": {"value": value, "unit": "candidate sims/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def population_traces(h, opmm, torch, S, n_steps):
    """Config-5 population (workloads.population): each saccade simulated at its
    own amplitude with opmm_simulate (input generation), plus N(0, 0.02 deg)."""
    amp, pw, truths = W.population(S)
    ctls = [W.Control(n_steps=n_steps, amplitude_deg=float(a), pw_default_ms=float(p))
            for a, p in zip(amp, pw)]
    opc = torch.as_tensor(np.ascontiguousarray(truths.T), device="cuda")
    traj = torch.zeros((n_steps + 1, S), dtype=torch.float64, device="cuda")
    opmm.opmm_simulate_batch(h, opc, S, ctls, traj, stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    recs = traj.cpu().numpy().T.copy()
    recs += np.random.default_rng(W.SEED_NOISE).normal(0.0, 0.02, size=recs.shape)
    return ctls, recs


def population_leg(h, opmm, torch, args, max_over_ranks=lambda x: x, world=1):
    """Config 5 (BASELINE.json configs[4]): S synthetic saccades x n_per
    candidates each through opmm_fit_batch (S_paper over n_steps = 150,
    Philox counter word 2 = saccade), saccades sharded over the N GPUs.
    Device time of the fit kernel (CUDA events, max over ranks), 1 warm-up + 2
    timed launches."""
    S, n_per, n_steps = args.pop_saccades, args.pop_candidates, 150
    ctls, recs = population_traces(h, opmm, torch, S, n_steps)
    sp = W.paper_space(n_steps=n_steps)
    opts = opmm.fit_options(cpu_check=0)
    ms, wall = [], []
    for rep in range(3):
        t0 = time.perf_counter()
        res = opmm.opmm_fit_batch(h, recs, ctls, sp, n_per, opts)
        wall.append(time.perf_counter() - t0)
        if rep > 0:
            ms.append(opmm.opmm_last_kernel_ms(h))
    # N > 1: saccades are sharded over the ranks (opmm_fit_batch, no
    # collective); the time is the max over ranks, the residual this rank's
    kern = max_over_ranks(sum(ms) / len(ms))
    f = np.array([r["opt_err"] for r in res if r is not None])
    e2e_s = max_over_ranks(min(wall[1:]))
    return {"metric": "OPC candidate sims/s (population)", "value": S * n_per / (kern * 1e-3),
            "e2e_value": S * n_per / e2e_s, "e2e_api": "opmm_fit_batch from Python, host traces",
            "saccades": S, "candidates_per_saccade": n_per, "n_steps": n_steps, "n_gpus": world,
            "kernel_ms": kern, "saccades_per_s": S / (kern * 1e-3),
            "mean_best_residual_deg_per_sample": float(np.mean(f / (n_steps + 1)))}


def latency_leg(h, opmm, torch, rec, world, max_over_ranks):
    """Config 3 (real-time mode): wall-clock latency of one synchronous
    opmm_fit (trace in pinned host memory, H2D + kernel + D2H + CPU_check) at
    10^5..10^8 candidates in total over the ranks, median (and p95) of 100
    calls after warm-up (20 / 10 at 10^7 / 10^8); the real-time bar is the
    trace's own duration, 100 ms.  Cold start separately: a
    fresh single-GPU handle (opmm_create: workspaces, exp table) and its first
    10^6-candidate fit (graph capture, first launches)."""
    rec_np = torch.as_tensor(rec, dtype=torch.float64).pin_memory().numpy()
    ctl_c, sp_c = opmm.control(W.Control()), opmm.search_space(W.paper_space())
    opts = opmm.fit_options(cpu_check=1)
    out = {}
    for n, reps in ((10**5, 100), (10**6, 100), (10**7, 20), (10**8, 10)):
        for _ in range(2):
            opmm.opmm_fit(h, rec_np, ctl_c, sp_c, n, opts)
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            opmm.opmm_fit(h, rec_np, ctl_c, sp_c, n, opts)
            ts.append(time.perf_counter() - t0)
        ms = max_over_ranks(1e3 * statistics.median(ts))
        p95 = max_over_ranks(1e3 * float(np.percentile(ts, 95)))
        out[f"{n:.0e}"] = {"ms": ms, "p95_ms": p95, "calls": reps, "realtime_factor": 100.0 / ms}
    t0 = time.perf_counter()
    hc = opmm.opmm_create(torch.cuda.current_device())
    t1 = time.perf_counter()
    opmm.opmm_fit(hc, rec_np, ctl_c, sp_c, 10**6, opts)
    t2 = time.perf_counter()
    opmm.opmm_destroy(hc)
    cold = {"create_ms": max_over_ranks(1e3 * (t1 - t0)), "first_fit_1e6_ms": max_over_ranks(1e3 * (t2 - t1))}
    return {"metric": "fit latency (sync opmm_fit, host trace, CPU_check on), median of 100 (1e7: 20, 1e8: 10)",
            "n_gpus": world, "candidates": out, "cold_start": cold}


def score_leg(h, opmm, torch, max_over_ranks, n=4 * 10**6, n_samples=101):
    """opmm_score, the one HBM-bound entry point: stored fp64
    trajectories [n_samples][n] (time-major) against one trace; GB/s of bytes
    moved (trajectories + errors) against the measured HBM copy bandwidth."""
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    traj = torch.randn((n_samples, n), dtype=torch.float64, device="cuda")
    rec = torch.randn(n_samples, dtype=torch.float64, device="cuda")
    err = torch.empty(n, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream()
    for _ in range(3):
        opmm.opmm_score(h, traj, n, n_samples, rec, err, stream=st)
    ms = []
    for _ in range(10):
        opmm.opmm_score(h, traj, n, n_samples, rec, err, stream=st)
        ms.append(opmm.opmm_last_kernel_ms(h))
    t = max_over_ranks(statistics.median(ms))
    gbs = (traj.numel() * 8 + n * 8) / (t * 1e-3) / 1e9
    del traj
    return {"kernel": "score_kernel<double, L1>", "candidates": n, "n_samples": n_samples,
            "kernel_ms": t, "achieved_gbs": gbs, "peak_gbs": peak, "frac": gbs / peak,
            "peak_basis": "MEASURED_PEAKS.json hbm_gbs (copy, read+write)"}


def g4_leg(h, opmm, torch, max_over_ranks, reps=5):
    """Config 4's planted grid G4: 100^4 = 10^8 candidates over
    {K_SE_AG, B_AG, N_SAC_AG, PW}, sharded over the ranks.  The default fit
    (kernel_variant 0) takes the superposition kernel here (100 N_SAC_AG
    levels per node); the direct one-candidate-per-thread kernel
    (variant 1) is timed beside it.  Both must return the planted index."""
    ctl, sp = W.Control(), W.g4_space(100)
    n = sp.n_grid()
    rec_dev = torch.as_tensor(clean_trace(), dtype=torch.float64, device="cuda")
    out = torch.zeros(ctypes.sizeof(opmm.FitResult), dtype=torch.uint8, device="cuda")
    st = torch.cuda.ExternalStream(h.stream)
    res = {}
    for kv in (0, 1):
        o = opmm.fit_options(cpu_check=0, kernel_variant=kv)
        for _ in range(2):
            opmm.opmm_fit_async(h, rec_dev, ctl, sp, n, out, o)
        ms = []
        for _ in range(reps):
            opmm.opmm_fit_async(h, rec_dev, ctl, sp, n, out, o)
            ms.append(opmm.opmm_last_kernel_ms(h))
        st.synchronize()
        r = opmm.decode_result(bytes(out.cpu().numpy()))
        res[kv] = (max_over_ranks(statistics.median(ms)), r)
    # fp32 superposition (fp32 columns and level loop; fp64 integration)
    o32 = opmm.fit_options(cpu_check=0, precision=opmm.FP32)
    for _ in range(2):
        opmm.opmm_fit_async(h, rec_dev, ctl, sp, n, out, o32)
    ms32 = []
    for _ in range(reps):
        opmm.opmm_fit_async(h, rec_dev, ctl, sp, n, out, o32)
        ms32.append(opmm.opmm_last_kernel_ms(h))
    st.synchronize()
    r32 = opmm.decode_result(bytes(out.cpu().numpy()))
    t32 = max_over_ranks(statistics.median(ms32))
    planted = W.g4_planted_index()
    return {"metric": "OPC candidate sims/s (G4 planted grid)", "candidates": n,
            "fp32_kernel_ms": t32, "fp32_value": n / (t32 * 1e-3),
            "fp32_best_index": r32["best_index"],
            "value": n / (res[0][0] * 1e-3), "kernel_ms": res[0][0],
            "kernel": "fit_super_kernel<L1> (auto: superposition over 100 N_SAC_AG levels)",
            "direct_kernel_ms": res[1][0], "direct_value": n / (res[1][0] * 1e-3),
            "speedup_vs_direct": res[1][0] / res[0][0],
            "best_index": res[0][1]["best_index"], "planted_index": planted,
            "planted_found": res[0][1]["best_index"] == planted == res[1][1]["best_index"]
            == r32["best_index"],
            "opt_err": res[0][1]["opt_err"]}


def clean_trace():
    """G4 is scored against the clean TRUTH trace (the stored fixture, no noise)."""
    return np.loadtxt(os.path.join(ROOT, "tests", "golden", "trace_truth_A10_dt1_n100.txt"),
                      comments="#")


def nm_leg(h, opmm, torch, args, max_over_ranks=lambda x: x, sum_over_ranks=lambda x: x):
    """The paper's own estimator (batched parallel Nelder-Mead)
    on a synthetic population (SURVEY 8(d) config 5 recipe: A ~ U[5, 30] deg,
    PW = 2.2 A + 15 ms, truths = defaults +-20% on K_SE_AG, B_AG, N_SAC_AG;
    n_steps = 150 at 1 kHz, noise 0.02 deg).  Traces are simulated on the GPU
    with opmm_simulate (input generation).  Throughput in NM-fitted saccades/s
    -- the unit of the paper's Table 3 -- kernel time
    (CUDA events) and end-to-end through the synchronous opmm_estimate_batch."""
    S, n_steps = args.nm_saccades, 150
    ctls, recs = population_traces(h, opmm, torch, S, n_steps)
    opts = opmm.nm_options(cpu_check=0)
    # warm-up at the full size (the handle's workspaces are sized on first use), then two timed calls
    opmm.opmm_estimate_batch(h, recs, ctls, options=opts)
    walls = []
    for _ in range(2):
        t0 = time.perf_counter()
        res = opmm.opmm_estimate_batch(h, recs, ctls, options=opts)
        walls.append(time.perf_counter() - t0)
    e2e_s = min(walls)
    # N > 1: saccades are sharded over the ranks (opmm_estimate_batch); the
    # statistics below are this rank's share, the times the max over ranks
    kern_ms = max_over_ranks(opmm.opmm_last_kernel_ms(h))
    e2e_s = max_over_ranks(e2e_s)
    res = [r for r in res if r is not None]
    its = np.array([r["iterations"] for r in res])
    f = np.array([r["f"] for r in res])
    conv = np.array([r["exit_reason"] == 0 for r in res])
    evals = int(sum_over_ranks(float(sum(r["gpu_evals"] for r in res))))
    # AUTO schedule (opmm.h): group from 1024 problems per rank, else lock-step
    group = len(res) >= 1024
    return {"metric": "NM-fitted saccades/s", "saccades": S, "n_steps": n_steps,
            "schedule": "group (4 lanes per problem: xr, xe, xc, xcc at once)" if group else
                        "lockstep (one problem per warp, all n + 4 points per iteration)",
            "objective": "propagator fp64, L1", "value": S / (kern_ms * 1e-3),
            "e2e_value": S / e2e_s, "kernel_ms": kern_ms, "mean_iterations": float(its.mean()),
            "converged_frac": float(conv.mean()), "gpu_evaluations": evals,
            "evaluations_per_s": evals / (kern_ms * 1e-3),
            "mean_residual_deg_per_sample": float(np.mean(f / (n_steps + 1))),
            "paper_context": "Table 3: 464.61 saccades/s CUDA (T4), 9.22/s MATLAB; different data"}


def run_gpu(args):
    import torch
    import torch.distributed as dist
    from paper_2007_09884_b200 import opmm

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        idt = torch.zeros(opmm.NCCL_ID_BYTES, dtype=torch.uint8, device="cuda")
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(opmm.opmm_nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        h = opmm.opmm_create_nccl(local, bytes(idt.cpu().numpy()), rank, world)
    else:
        h = opmm.opmm_create(local)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    ctl = W.Control()
    rec = make_trace()
    sp = W.paper_space()
    n_total = args.per_gpu * world
    stream = torch.cuda.ExternalStream(h.stream)
    rec_dev = torch.as_tensor(rec, dtype=torch.float64, device="cuda")
    out_dev = torch.zeros(ctypes.sizeof(opmm.FitResult), dtype=torch.uint8, device="cuda")
    flush = torch.empty(512 * 2**20, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()

    def device_leg(precision, certify=True):
        # fp32 runs with certification: the exact top-K by fp32 error, merged
        # over the ranks and re-scored in fp64
        opts = opmm.fit_options(precision=precision, cpu_check=0,
                                certify=1 if (precision == opmm.FP32 and certify) else 0)
        for _ in range(args.warmup):
            opmm.opmm_fit_async(h, rec_dev, ctl, sp, n_total, out_dev, opts)
        stream.synchronize()
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        barrier()
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            for s in range(args.steps):
                flush.fill_(s & 0xff)                 # evict L2 (outside the events)
                starts[s].record(stream)
                opmm.opmm_fit_async(h, rec_dev, ctl, sp, n_total, out_dev, opts)
                ends[s].record(stream)
        stream.synchronize()
        torch.cuda.synchronize()
        barrier()
        ms = sum(a.elapsed_time(b) for a, b in zip(starts, ends)) / args.steps
        res = opmm.decode_result(bytes(out_dev.cpu().numpy()))
        return max_over_ranks(ms), res

    def kernel_leg(precision, certify=False):
        """The library's own CUDA events around the fit's kernels (kernel
        timing on), for the roofline: the same launches as device_leg, timed
        in a separate pass because the timing events add ~6 us of stream
        time per call that the `value` pass should not carry."""
        opmm.opmm_set_kernel_timing(h, True)
        opts = opmm.fit_options(precision=precision, cpu_check=0, certify=certify)
        for _ in range(args.warmup):
            opmm.opmm_fit_async(h, rec_dev, ctl, sp, n_total, out_dev, opts)
        kms = []
        with torch.cuda.stream(stream):
            for s in range(args.steps):
                flush.fill_(s & 0xff)
                opmm.opmm_fit_async(h, rec_dev, ctl, sp, n_total, out_dev, opts)
                kms.append(opmm.opmm_last_kernel_ms(h))
        opmm.opmm_set_kernel_timing(h, False)
        return max_over_ranks(sum(kms) / len(kms))

    with ClockSampler(local) as clk:
        ms64, res64 = device_leg(opmm.FP64)
    clocks = clk.summary()
    ms32, res32 = device_leg(opmm.FP32)
    ms32_plain, _ = device_leg(opmm.FP32, certify=False)
    # kernel times for the rooflines (library events, separate pass)
    kms64 = kernel_leg(opmm.FP64)
    kms32 = kernel_leg(opmm.FP32, certify=1)
    kms32_plain = kernel_leg(opmm.FP32)   # the fp32 fit kernel alone: its pipes' roofline

    # e2e: synchronous public call, trace in pinned host memory
    rec_host = torch.as_tensor(rec, dtype=torch.float64).pin_memory()
    rec_np = rec_host.numpy()
    opts = opmm.fit_options(precision=opmm.FP64, cpu_check=1)
    # the C-ABI structs are built once, as a caller issuing repeated fits would
    ctl_c, sp_c = opmm.control(ctl), opmm.search_space(sp)
    for _ in range(args.warmup):
        opmm.opmm_fit(h, rec_np, ctl_c, sp_c, n_total, opts)
    barrier()
    torch.cuda.synchronize()
    t_e2e = []
    for s in range(args.steps):
        flush.fill_(s & 0xff)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = opmm.opmm_fit(h, rec_np, ctl_c, sp_c, n_total, opts)
        t_e2e.append(time.perf_counter() - t0)
    barrier()
    e2e_ms = max_over_ranks(1e3 * sum(t_e2e) / len(t_e2e))

    lat = latency_leg(h, opmm, torch, rec, world, max_over_ranks) if not args.no_latency else None
    opmm.opmm_set_kernel_timing(h, True)   # the legs below report kernel times
    score = score_leg(h, opmm, torch, max_over_ranks)
    g4 = g4_leg(h, opmm, torch, max_over_ranks)
    nm = nm_leg(h, opmm, torch, args, max_over_ranks, sum_over_ranks) if not args.no_nm else None
    pop = population_leg(h, opmm, torch, args, max_over_ranks, world) if not args.no_pop else None

    per_cand_flop = FLOP_PER_STEP * N_STEPS + FLOP_SETUP
    achieved = per_cand_flop * args.per_gpu / (kms64 * 1e-3) / 1e12
    line = {
        "metric": "OPC candidate sims/s", "value": n_total / (ms64 * 1e-3),
        "unit": "candidate sims/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms64, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {**workload_config(args.per_gpu, world),
                   "integrator": "rk4-propagator",
                   "l2": "flushed between timed steps (512 MiB write, outside the events)",
                   "parallelism": f"candidates sharded x{world}, 1 ncclAllGather of 32 B/rank"},
        "clocks": clocks,
        "gpu_launches": args.steps * (2 if world > 1 else 1),
        "e2e": {"value": n_total / (e2e_ms * 1e-3), "unit": "candidate sims/s",
                "h2d_bytes_per_step": rec_np.nbytes, "d2h_bytes_per_step": ctypes.sizeof(opmm.FitResult),
                "ms_per_step": e2e_ms, "api": "opmm_fit (sync, host buffers, CPU_check on)"},
        "roofline": {"bound": "alu", "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                     "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS,
                     "traffic": ncu_traffic_bytes(), "traffic_unit": "bytes/launch (ncu, spills)",
                     "kernel": "fit_kernel<double, propagator, L1>", "kernel_ms": kms64,
                     "flop_per_candidate": per_cand_flop,
                     "peak_basis": "148 SM x 64 FP64 lanes x 2 x 1965 MHz (DESIGN.md)",
                     "frac_of_measured_dfma": achieved / FP64_MEASURED_TFLOPS,
                     "measured_dfma_basis": "all-register DFMA microbenchmark, profiles/r02_fma_peak.txt",
                     "fp64_issue_frac": (FP64_INST_PER_STEP * N_STEPS + FP64_INST_SETUP) * args.per_gpu
                     / (kms64 * 1e-3) / (SMS * FP64_LANES * SM_MAX_MHZ * 1e6)},
        "fp32": {"value": n_total / (ms32 * 1e-3), "ms_per_step": ms32, "kernel_ms": kms32,
                 "uncertified_value": n_total / (ms32_plain * 1e-3), "uncertified_ms_per_step": ms32_plain,
                 "roofline": fp32_roofline(args.per_gpu, kms32_plain),
                 "best_index": res32["best_index"], "certified": res32["certified"],
                 "opt_err_fp64": res32["opt_err"],
                 "mode": "fp32 integrate+score, fp64 setup, exact top-8 by fp32 error (merged "
                         "over the ranks) re-scored in fp64 and certified"},
        "result": {"best_index": res64["best_index"], "opt_err": res64["opt_err"],
                   "n_finite": res64["n_finite"], "cpu_check": r["cpu_check"]},
    }
    if nm is not None:
        line["nm"] = nm
    if lat is not None:
        line["latency"] = lat
    line["score_hbm"] = score
    line["g4_grid"] = g4
    if pop is not None:
        line["population"] = pop
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline()
    if rank == 0:
        print(json.dumps(line), flush=True)
    h.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="libopmm", choices=["libopmm", "reference"])
    ap.add_argument("--per-gpu", type=int, default=PER_GPU)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-nm", action="store_true")
    ap.add_argument("--no-latency", action="store_true")
    ap.add_argument("--nm-saccades", type=int, default=16384)
    ap.add_argument("--no-pop", action="store_true")
    ap.add_argument("--pop-saccades", type=int, default=10000)
    ap.add_argument("--pop-candidates", type=int, default=100000)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
