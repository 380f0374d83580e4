"""Thin ctypes binding of libopmm (include/opmm.h): argument marshalling only.

Every function here has the C name of the entry point it wraps and does
nothing but convert Python / numpy / torch arguments into the C ABI and turn a
non-OK status into an exception.  All computation happens in the CUDA kernels
of libopmm.so; if the library is missing this module raises at import time
(there is no CPU fallback).  Device buffers are torch CUDA tensors (PyTorch is
used for device memory and streams only).
"""
from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libopmm.so")

NPARAM = 18
MAX_STEPS = 16384
NCCL_ID_BYTES = 128

OK, ERR_INVALID_ARG, ERR_CUDA, ERR_NCCL, ERR_OOM, ERR_NO_FINITE, ERR_UNSUPPORTED = range(7)
FP64, FP32 = 0, 1
METRIC_L1, METRIC_RMS = 0, 1
INTEG_PROPAGATOR, INTEG_RK4_STAGES = 0, 1
_STATUS = {0: "OK", 1: "INVALID_ARG", 2: "CUDA", 3: "NCCL", 4: "OOM", 5: "NO_FINITE", 6: "UNSUPPORTED"}


class OpmmError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        super().__init__(f"{where}: OPMM_ERR_{_STATUS.get(status, status)}: {msg}")
        self.status = status


class Control(C.Structure):
    _fields_ = [("dt_ms", C.c_double), ("n_steps", C.c_int32), ("substeps", C.c_int32),
                ("amplitude_deg", C.c_double), ("theta0_deg", C.c_double),
                ("pw_default_ms", C.c_double)]


class SearchSpace(C.Structure):
    _fields_ = [("mode", C.c_int32), ("model", C.c_int32), ("seed", C.c_uint64),
                ("lo", C.c_double * NPARAM), ("hi", C.c_double * NPARAM),
                ("log_scale", C.c_uint8 * NPARAM), ("pad2_", C.c_uint8 * 6),
                ("levels", C.c_int32 * NPARAM)]


MAX_TOPK = 32
FIT_FLAG_NO_LANE_SORT, FIT_FLAG_SUPER_SMEM, FIT_FLAG_NO_GRAPH, FIT_FLAG_NO_GRID_TABLES = 1, 2, 4, 8


class FitOptions(C.Structure):
    _fields_ = [("precision", C.c_int32), ("metric", C.c_int32), ("integrator", C.c_int32),
                ("block_size", C.c_int32), ("grid_blocks", C.c_int32), ("cpu_check", C.c_int32),
                ("kernel_variant", C.c_int32), ("certify", C.c_int32), ("top_k", C.c_int32),
                ("flags", C.c_uint32), ("err_out", C.c_void_p)]


class FitResult(C.Structure):
    _fields_ = [("best_index", C.c_int64), ("opt_err", C.c_double), ("cpu_check", C.c_double),
                ("opc", C.c_double * NPARAM), ("n_finite", C.c_int64), ("n_evaluated", C.c_int64),
                ("top_k", C.c_int32), ("certified", C.c_int32), ("topk_index", C.c_int64 * MAX_TOPK),
                ("topk_err", C.c_double * MAX_TOPK)]

    def as_dict(self) -> dict:
        tk = self.top_k
        return {"best_index": self.best_index, "opt_err": self.opt_err, "cpu_check": self.cpu_check,
                "opc": np.frombuffer(self.opc, dtype=np.float64).copy(), "n_finite": self.n_finite,
                "n_evaluated": self.n_evaluated, "top_k": tk, "certified": self.certified,
                "topk_index": self.topk_index[:tk] if tk else [],
                "topk_err": self.topk_err[:tk] if tk else []}


class NmOptions(C.Structure):
    _fields_ = [("precision", C.c_int32), ("objective", C.c_int32), ("metric", C.c_int32),
                ("max_iter", C.c_int32), ("tol_x", C.c_double), ("tol_f", C.c_double),
                ("init_scale", C.c_double), ("cpu_check", C.c_int32), ("schedule", C.c_int32),
                ("time_budget_ms", C.c_double)]


class NmResult(C.Structure):
    _fields_ = [("x", C.c_double * NPARAM), ("f_best", C.c_double), ("cpu_check", C.c_double),
                ("iterations", C.c_int32), ("func_evals", C.c_int32), ("gpu_evals", C.c_int32),
                ("exit_reason", C.c_int32)]

    def as_dict(self, dim: int = NPARAM) -> dict:
        return {"x": np.array(self.x[:dim]), "f": self.f_best, "cpu_check": self.cpu_check,
                "iterations": self.iterations, "func_evals": self.func_evals,
                "gpu_evals": self.gpu_evals, "exit_reason": self.exit_reason}


NM_OBJ_PROPAGATOR, NM_OBJ_RK4_STAGES, NM_OBJ_REFERENCE = 0, 1, 2
NM_SCHEDULE_AUTO, NM_SCHEDULE_LOCKSTEP, NM_SCHEDULE_LANE, NM_SCHEDULE_GROUP = 0, 1, 2, 3
NM_SPHERE, NM_ROSENBROCK, NM_POWELL = 0, 1, 2


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2007_09884_b200.build` "
                          "(libopmm has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, i64, i32, dp = C.c_void_p, C.c_int64, C.c_int32, C.POINTER(C.c_double)
    st = C.c_int
    sig = {
        "opmm_version": ([], C.c_char_p),
        "opmm_last_error": ([], C.c_char_p),
        "opmm_create": ([C.POINTER(vp), C.c_int], st),
        "opmm_nccl_unique_id": ([C.c_char_p], st),
        "opmm_create_nccl": ([C.POINTER(vp), C.c_int, C.c_char_p, C.c_int, C.c_int], st),
        "opmm_destroy": ([vp], st),
        "opmm_get_stream": ([vp, C.POINTER(vp)], st),
        "opmm_last_kernel_ms": ([vp, C.POINTER(C.c_float)], st),
        "opmm_set_kernel_timing": ([vp, C.c_int32], st),
        "opmm_shard_range": ([i64, C.c_int, C.c_int, C.POINTER(i64), C.POINTER(i64)], st),
        "opmm_merge_argmin": ([dp, C.POINTER(i64), C.c_int, dp, C.POINTER(i64)], st),
        "opmm_validate": ([C.POINTER(Control), C.POINTER(SearchSpace), i64], st),
        "opmm_merge_topk": ([dp, C.POINTER(i64), C.c_int, C.c_int, dp, C.POINTER(i64)], st),
        "opmm_certify_topk": ([dp, dp, C.POINTER(i64), C.c_int, C.c_double, C.POINTER(i32),
                               C.POINTER(i64), dp], st),
        "opmm_generate": ([vp, C.POINTER(SearchSpace), C.c_uint32, i64, i64, vp, i64, vp], st),
        "opmm_simulate": ([vp, vp, i64, i64, C.POINTER(Control), i32, i32, vp, i64, vp, vp], st),
        "opmm_simulate_batch": ([vp, vp, i64, i64, C.POINTER(Control), i32, i32, vp, i64, vp, vp], st),
        "opmm_score": ([vp, vp, i64, i64, i32, vp, i32, i32, vp, vp], st),
        "opmm_simulate_score": ([vp, vp, i64, i64, C.POINTER(Control), vp, i32, i32, i32, vp, vp], st),
        "opmm_fit": ([vp, vp, C.POINTER(Control), C.POINTER(SearchSpace), i64,
                      C.POINTER(FitOptions), C.POINTER(FitResult)], st),
        "opmm_fit_async": ([vp, vp, C.POINTER(Control), C.POINTER(SearchSpace), i64,
                            C.POINTER(FitOptions), vp], st),
        "opmm_fit_shard": ([vp, vp, C.POINTER(Control), C.POINTER(SearchSpace), i64, C.c_int, C.c_int,
                            C.POINTER(FitOptions), C.POINTER(FitResult)], st),
        "opmm_fit_batch": ([vp, vp, i64, C.POINTER(Control), C.POINTER(SearchSpace), i64,
                            C.POINTER(FitOptions), C.POINTER(FitResult)], st),
        "opmm_estimate_batch": ([vp, vp, i64, C.POINTER(Control), vp, C.POINTER(NmOptions),
                                 C.POINTER(NmResult)], st),
        "opmm_nm_minimize_test": ([vp, i32, i32, vp, i64, C.POINTER(NmOptions), C.POINTER(NmResult)], st),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    return L


_lib = _load()
EXPORTED = ("opmm_version", "opmm_last_error", "opmm_create", "opmm_nccl_unique_id",
            "opmm_create_nccl", "opmm_destroy", "opmm_get_stream", "opmm_last_kernel_ms", "opmm_set_kernel_timing",
            "opmm_shard_range", "opmm_merge_argmin", "opmm_merge_topk", "opmm_certify_topk",
            "opmm_validate", "opmm_generate",
            "opmm_simulate", "opmm_simulate_batch", "opmm_score", "opmm_simulate_score", "opmm_fit", "opmm_fit_async",
            "opmm_fit_shard", "opmm_fit_batch", "opmm_estimate_batch", "opmm_nm_minimize_test")


def lib():
    return _lib


def _check(status: int, where: str):
    if status != OK:
        raise OpmmError(status, where, _lib.opmm_last_error().decode())


# ---------------------------------------------------------------------- structs
def control(c=None, **kw) -> Control:
    """Control from any object with dt_ms/n_steps/amplitude_deg/theta0_deg/pw_default_ms
    (and optionally substeps)."""
    src = {k: getattr(c, k) for k in ("dt_ms", "n_steps", "amplitude_deg", "theta0_deg", "pw_default_ms")} \
        if c is not None else {}
    if c is not None:
        src["substeps"] = getattr(c, "substeps", 0)
    src.update(kw)
    return Control(float(src.get("dt_ms", 1.0)), int(src.get("n_steps", 100)), int(src.get("substeps", 0)),
                   float(src.get("amplitude_deg", math.nan)), float(src.get("theta0_deg", 0.0)),
                   float(src.get("pw_default_ms", 40.0)))


def search_space(s) -> SearchSpace:
    """SearchSpace from any object with mode/seed/lo/hi/log_scale/levels."""
    out = SearchSpace()
    out.mode = int(s.mode)
    out.model = int(getattr(s, "model", 0))
    out.seed = int(s.seed)
    for d in range(NPARAM):
        out.lo[d] = float(s.lo[d])
        out.hi[d] = float(s.hi[d])
        out.log_scale[d] = int(s.log_scale[d])
        out.levels[d] = int(s.levels[d])
    return out


def fit_options(precision=FP64, metric=METRIC_L1, integrator=INTEG_PROPAGATOR, block_size=0,
                grid_blocks=0, cpu_check=1, err_out=None, kernel_variant=0, certify=0, top_k=0,
                flags=0) -> FitOptions:
    return FitOptions(precision, metric, integrator, block_size, grid_blocks, cpu_check,
                      kernel_variant, certify, top_k, flags,
                      _ptr(err_out) if err_out is not None else None)


def _ptr(x):
    """Raw pointer of a torch tensor / numpy array / int / None."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if isinstance(x, np.ndarray):
        if x.flags.c_contiguous and x.flags.writeable and x.size:
            return C.addressof(C.c_char.from_buffer(x))   # ~1 us cheaper than .ctypes.data
        return x.ctypes.data
    raise TypeError(f"cannot take a pointer of {type(x)}")


CUDA_STREAM_LEGACY = 1   # cudaStreamLegacy: the legacy default ("NULL") stream


def _stream(stream):
    """None -> the handle's own stream (NULL in the C ABI).  A torch stream is
    passed by its cudaStream_t; torch's default stream is the legacy NULL
    stream, which the C ABI would read as "the handle's stream", so it is
    passed as cudaStreamLegacy instead (ordered with torch's work)."""
    if stream is None:
        return None
    s = stream if isinstance(stream, int) else stream.cuda_stream
    return s if s != 0 else CUDA_STREAM_LEGACY


# ---------------------------------------------------------------------- handle
class Handle:
    """Owns an opmm_handle (one GPU, or one rank of an NCCL group)."""

    def __init__(self, device: int = 0, nccl_id: bytes | None = None, rank: int = 0, world: int = 1):
        h = C.c_void_p()
        if nccl_id is None:
            _check(_lib.opmm_create(C.byref(h), device), "opmm_create")
        else:
            _check(_lib.opmm_create_nccl(C.byref(h), device, bytes(nccl_id), rank, world),
                   "opmm_create_nccl")
        self.ptr = h
        self.device, self.rank, self.world = device, rank, world

    def close(self):
        if self.ptr:
            _lib.opmm_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def stream(self) -> int:
        s = C.c_void_p()
        _check(_lib.opmm_get_stream(self.ptr, C.byref(s)), "opmm_get_stream")
        return s.value or 0


def opmm_version() -> str:
    return _lib.opmm_version().decode()


def opmm_create(device: int = 0, kernel_timing: bool = False) -> Handle:
    """kernel_timing: bracket every launch with CUDA events so that
    opmm_last_kernel_ms can report it (costs ~6 us of stream time per call)."""
    h = Handle(device)
    if kernel_timing:
        opmm_set_kernel_timing(h, True)
    return h


def opmm_set_kernel_timing(h, on: bool = True):
    _check(_lib.opmm_set_kernel_timing(h.ptr, 1 if on else 0), "opmm_set_kernel_timing")


def opmm_nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(NCCL_ID_BYTES)
    _check(_lib.opmm_nccl_unique_id(buf), "opmm_nccl_unique_id")
    return buf.raw


def opmm_create_nccl(device: int, nccl_id: bytes, rank: int, world: int) -> Handle:
    return Handle(device, nccl_id, rank, world)


def opmm_destroy(h: Handle):
    h.close()


def opmm_last_kernel_ms(h: Handle) -> float:
    ms = C.c_float()
    _check(_lib.opmm_last_kernel_ms(h.ptr, C.byref(ms)), "opmm_last_kernel_ms")
    return ms.value


# ---------------------------------------------------------------------- host-only
def opmm_shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    b, e = C.c_int64(), C.c_int64()
    _check(_lib.opmm_shard_range(n, rank, world, C.byref(b), C.byref(e)), "opmm_shard_range")
    return b.value, e.value


def opmm_merge_argmin(errs, idxs) -> tuple[float, int]:
    e = np.ascontiguousarray(errs, dtype=np.float64)
    i = np.ascontiguousarray(idxs, dtype=np.int64)
    be, bi = C.c_double(), C.c_int64()
    st = _lib.opmm_merge_argmin(e.ctypes.data_as(C.POINTER(C.c_double)),
                                i.ctypes.data_as(C.POINTER(C.c_int64)), len(e), C.byref(be), C.byref(bi))
    if st not in (OK, ERR_NO_FINITE):
        _check(st, "opmm_merge_argmin")
    return be.value, bi.value


def opmm_merge_topk(errs, idxs, K: int) -> tuple[np.ndarray, np.ndarray]:
    """errs/idxs: [lists, K] sorted lists -> the merged K smallest (err, idx)."""
    e = np.ascontiguousarray(errs, dtype=np.float64).reshape(-1, K)
    i = np.ascontiguousarray(idxs, dtype=np.int64).reshape(-1, K)
    oe, oi = np.zeros(K), np.zeros(K, dtype=np.int64)
    _check(_lib.opmm_merge_topk(e.ctypes.data_as(C.POINTER(C.c_double)),
                                i.ctypes.data_as(C.POINTER(C.c_int64)), e.shape[0], K,
                                oe.ctypes.data_as(C.POINTER(C.c_double)),
                                oi.ctypes.data_as(C.POINTER(C.c_int64))), "opmm_merge_topk")
    return oe, oi


def opmm_certify_topk(e32, e64, idx, scale: float) -> tuple[int, int, float]:
    """(certified, best_index, best_err) of one merged fp32 list."""
    a = np.ascontiguousarray(e32, dtype=np.float64)
    b = np.ascontiguousarray(e64, dtype=np.float64)
    i = np.ascontiguousarray(idx, dtype=np.int64)
    c, bi, be = C.c_int32(), C.c_int64(), C.c_double()
    _check(_lib.opmm_certify_topk(a.ctypes.data_as(C.POINTER(C.c_double)),
                                  b.ctypes.data_as(C.POINTER(C.c_double)),
                                  i.ctypes.data_as(C.POINTER(C.c_int64)), len(a), scale,
                                  C.byref(c), C.byref(bi), C.byref(be)), "opmm_certify_topk")
    return c.value, bi.value, be.value


def opmm_validate(ctl=None, space=None, n_candidates: int = 0) -> None:
    c = control(ctl) if ctl is not None and not isinstance(ctl, Control) else ctl
    s = search_space(space) if space is not None and not isinstance(space, SearchSpace) else space
    _check(_lib.opmm_validate(C.byref(c) if c is not None else None,
                              C.byref(s) if s is not None else None, n_candidates), "opmm_validate")


# ---------------------------------------------------------------------- hot path
def _ctl(c):
    return c if isinstance(c, Control) else control(c)


def _ctl_array(ctls):
    """[S] Control array for the batch entry points, filled column-wise
    (the same conversions as control())."""
    S = len(ctls)
    arr = (Control * S)()
    a = np.frombuffer(arr, dtype=np.dtype(Control))
    if all(isinstance(c, Control) for c in ctls):
        for k in range(S):
            arr[k] = ctls[k]
        return arr
    a["dt_ms"] = [float(c.dt_ms) for c in ctls]
    a["n_steps"] = [int(c.n_steps) for c in ctls]
    a["substeps"] = [int(getattr(c, "substeps", 0)) for c in ctls]
    a["amplitude_deg"] = [float(c.amplitude_deg) for c in ctls]
    a["theta0_deg"] = [float(c.theta0_deg) for c in ctls]
    a["pw_default_ms"] = [float(c.pw_default_ms) for c in ctls]
    return arr


def _fit_results(out, lo: int, hi: int) -> list:
    """[S] FitResult -> list of FitResult.as_dict() for entries [lo, hi), None
    elsewhere (other ranks' saccades), converted column-wise."""
    S = len(out)
    a = np.frombuffer(out, dtype=np.dtype(FitResult))[lo:hi]
    P = np.array(a["opc"])
    TI, TE = a["topk_index"], a["topk_err"]
    cols = zip(a["best_index"].tolist(), a["opt_err"].tolist(), a["cpu_check"].tolist(),
               a["n_finite"].tolist(), a["n_evaluated"].tolist(), a["top_k"].tolist(),
               a["certified"].tolist())
    res = [None] * S
    for k, (bi, oe, cc, nf, ne, tk, ce) in enumerate(cols):
        res[lo + k] = {"best_index": bi, "opt_err": oe, "cpu_check": cc, "opc": P[k], "n_finite": nf,
                       "n_evaluated": ne, "top_k": tk, "certified": ce,
                       "topk_index": TI[k, :tk].tolist() if tk else [],
                       "topk_err": TE[k, :tk].tolist() if tk else []}
    return res


def _nm_results(out, lo: int, hi: int) -> list:
    """[S] NmResult -> list of NmResult.as_dict() for [lo, hi), None elsewhere."""
    S = len(out)
    a = np.frombuffer(out, dtype=np.dtype(NmResult))[lo:hi]
    X = np.array(a["x"])
    cols = zip(a["f_best"].tolist(), a["cpu_check"].tolist(), a["iterations"].tolist(),
               a["func_evals"].tolist(), a["gpu_evals"].tolist(), a["exit_reason"].tolist())
    res = [None] * S
    for k, (f, cc, it, fe, ge, er) in enumerate(cols):
        res[lo + k] = {"x": X[k], "f": f, "cpu_check": cc, "iterations": it, "func_evals": fe,
                       "gpu_evals": ge, "exit_reason": er}
    return res


def _space(s):
    return s if isinstance(s, SearchSpace) else search_space(s)


def opmm_generate(h: Handle, space, begin: int, count: int, opc_out, ld: int | None = None,
                  saccade: int = 0, stream=None):
    _check(_lib.opmm_generate(h.ptr, C.byref(_space(space)), saccade, begin, count, _ptr(opc_out),
                              count if ld is None else ld, _stream(stream)), "opmm_generate")


def opmm_simulate(h: Handle, opc, n: int, ctl, traj, precision=FP64, integrator=INTEG_PROPAGATOR,
                  ld: int | None = None, ld_out: int | None = None, status=None, stream=None):
    c = _ctl(ctl)
    _check(_lib.opmm_simulate(h.ptr, _ptr(opc), n, n if ld is None else ld, C.byref(c), precision,
                              integrator, _ptr(traj), n if ld_out is None else ld_out, _ptr(status),
                              _stream(stream)), "opmm_simulate")


def opmm_score(h: Handle, traj, n: int, n_samples: int, recorded, err, precision=FP64,
               metric=METRIC_L1, ld: int | None = None, stream=None):
    _check(_lib.opmm_score(h.ptr, _ptr(traj), n, n if ld is None else ld, n_samples, _ptr(recorded),
                           precision, metric, _ptr(err), _stream(stream)), "opmm_score")


def opmm_simulate_batch(h: Handle, opc, n: int, ctls, traj, precision=FP64,
                        integrator=INTEG_PROPAGATOR, ld: int | None = None,
                        ld_out: int | None = None, status=None, stream=None):
    """opmm_simulate with one control per candidate (ctls: n controls sharing
    dt_ms and n_steps)."""
    arr = (Control * n)(*[_ctl(c) for c in ctls])
    _check(_lib.opmm_simulate_batch(h.ptr, _ptr(opc), n, n if ld is None else ld, arr, precision,
                                    integrator, _ptr(traj), n if ld_out is None else ld_out,
                                    _ptr(status), _stream(stream)), "opmm_simulate_batch")


def opmm_simulate_score(h: Handle, opc, n: int, ctl, recorded, err, precision=FP64, metric=METRIC_L1,
                        integrator=INTEG_PROPAGATOR, ld: int | None = None, stream=None):
    c = _ctl(ctl)
    _check(_lib.opmm_simulate_score(h.ptr, _ptr(opc), n, n if ld is None else ld, C.byref(c),
                                    _ptr(recorded), precision, metric, integrator, _ptr(err),
                                    _stream(stream)), "opmm_simulate_score")


def opmm_fit(h: Handle, recorded, ctl, space, n_candidates: int, options: FitOptions | None = None,
             raise_no_finite: bool = False) -> dict:
    """Synchronous fit; `recorded` is a host numpy array or a device tensor."""
    rec = recorded
    if isinstance(recorded, np.ndarray):
        rec = np.ascontiguousarray(recorded, dtype=np.float64)
    out = FitResult()
    opts = options if options is not None else fit_options()
    st = _lib.opmm_fit(h.ptr, _ptr(rec), C.byref(_ctl(ctl)), C.byref(_space(space)), n_candidates,
                       C.byref(opts), C.byref(out))
    if st != OK and not (st == ERR_NO_FINITE and not raise_no_finite):
        _check(st, "opmm_fit")
    return out.as_dict()


def opmm_fit_async(h: Handle, recorded_dev, ctl, space, n_candidates: int, out_dev,
                   options: FitOptions | None = None):
    """Enqueue a fit on the handle's stream; out_dev: device buffer of
    ctypes.sizeof(FitResult) bytes (e.g. a uint8 CUDA tensor)."""
    opts = options if options is not None else fit_options(cpu_check=0)
    _check(_lib.opmm_fit_async(h.ptr, _ptr(recorded_dev), C.byref(_ctl(ctl)), C.byref(_space(space)),
                               n_candidates, C.byref(opts), _ptr(out_dev)), "opmm_fit_async")


def decode_result(raw: bytes) -> dict:
    return FitResult.from_buffer_copy(raw).as_dict()


def opmm_fit_shard(h: Handle, recorded, ctl, space, n_candidates: int, rank: int, world: int,
                   options: FitOptions | None = None) -> dict:
    """Rank `rank` of `world`'s share of a fit on a plain handle (opmm.h)."""
    out = FitResult()
    rec = recorded
    if isinstance(recorded, np.ndarray):
        rec = np.ascontiguousarray(recorded, dtype=np.float64)
    opts = options if options is not None else fit_options()
    _check(_lib.opmm_fit_shard(h.ptr, _ptr(rec), C.byref(_ctl(ctl)), C.byref(_space(space)),
                               n_candidates, rank, world, C.byref(opts), C.byref(out)), "opmm_fit_shard")
    return out.as_dict()


def opmm_fit_batch(h: Handle, recorded, ctls, space, n_per: int,
                   options: FitOptions | None = None) -> list[dict]:
    S = len(ctls)
    arr = _ctl_array(ctls)
    out = (FitResult * S)()
    rec = recorded
    if isinstance(recorded, np.ndarray):
        rec = np.ascontiguousarray(recorded, dtype=np.float64)
    opts = options if options is not None else fit_options()
    _check(_lib.opmm_fit_batch(h.ptr, _ptr(rec), S, arr, C.byref(_space(space)), n_per,
                               C.byref(opts), out), "opmm_fit_batch")
    lo, hi = opmm_shard_range(S, h.rank, h.world)
    return _fit_results(out, lo, hi)


# ---------------------------------------------------------------------- Nelder-Mead
def nm_options(precision=FP64, objective=NM_OBJ_PROPAGATOR, metric=METRIC_L1, max_iter=0, tol_x=0.0,
               tol_f=0.0, init_scale=0.0, cpu_check=1, schedule=0, time_budget_ms=0.0) -> NmOptions:
    """schedule: NM_SCHEDULE_AUTO / _LOCKSTEP / _LANE / _GROUP (opmm.h);
    time_budget_ms: the paper's per-problem time boundary (0 = none)."""
    return NmOptions(precision, objective, metric, max_iter, tol_x, tol_f, init_scale, cpu_check,
                     schedule, time_budget_ms)


def opmm_estimate_batch(h: Handle, recorded, ctls, x0=None, options: NmOptions | None = None) -> list:
    """Nelder-Mead OPC estimation of S saccades (recorded [S, n_steps+1])."""
    S = len(ctls)
    arr = _ctl_array(ctls)
    out = (NmResult * S)()
    rec = recorded
    if isinstance(recorded, np.ndarray):
        rec = np.ascontiguousarray(recorded, dtype=np.float64)
    xx = None if x0 is None else np.ascontiguousarray(x0, dtype=np.float64)
    _check(_lib.opmm_estimate_batch(h.ptr, _ptr(rec), S, arr, _ptr(xx),
                                    C.byref(options if options is not None else nm_options()), out),
           "opmm_estimate_batch")
    lo, hi = opmm_shard_range(S, h.rank, h.world)
    return _nm_results(out, lo, hi)


def opmm_nm_minimize_test(h: Handle, fn_id: int, x0, options: NmOptions | None = None) -> list:
    """Nelder-Mead on a SPEC test function for S start points x0 [S, dim]."""
    x = np.ascontiguousarray(np.atleast_2d(x0), dtype=np.float64)
    S, dim = x.shape
    out = (NmResult * S)()
    _check(_lib.opmm_nm_minimize_test(h.ptr, fn_id, dim, _ptr(x), S,
                                      C.byref(options if options is not None else nm_options()), out),
           "opmm_nm_minimize_test")
    return [out[s].as_dict(dim) for s in range(S)]
