"""C-ABI boundary checks that need no GPU (-m "not gpu").

The library must load on a CPU-only box, export every entry point that
include/opmm.h declares, agree with the binding on struct layouts, run its
host-only helpers, and fail loudly (OPMM_ERR_CUDA) instead of falling back to
the CPU when there is no device.
"""
import ctypes
import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "opmm.h")


@pytest.fixture(scope="module")
def opmm():
    from paper_2007_09884_b200 import build
    build.build()
    from paper_2007_09884_b200 import opmm as m
    return m


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(opmm_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for n in ("opmm_simulate", "opmm_score", "opmm_fit", "opmm_simulate_score", "opmm_generate",
              "opmm_fit_batch", "opmm_create", "opmm_destroy", "opmm_create_nccl"):
        assert n in names


def test_library_exports_every_declared_symbol(opmm):
    names = declared_functions()
    lib = ctypes.CDLL(opmm.LIB_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(opmm.EXPORTED)


def test_struct_layouts_match_header(opmm):
    # the C side static_asserts the same sizes (opmm_api.cu)
    assert ctypes.sizeof(opmm.Control) == 40
    assert ctypes.sizeof(opmm.SearchSpace) == 400
    assert ctypes.sizeof(opmm.FitOptions) == 48
    assert ctypes.sizeof(opmm.FitResult) == 704
    assert ctypes.sizeof(opmm.NmOptions) == 56
    assert ctypes.sizeof(opmm.NmResult) == 176
    assert opmm.SearchSpace.levels.offset == 400 - 72
    assert opmm.FitResult.n_finite.offset == 168


def test_version_and_error_string(opmm):
    assert "sm_100a" in opmm.opmm_version()


def test_shard_range_partitions_exactly(opmm):
    for n in (0, 1, 7, 1000, 10**8 + 3, 2**62):
        for R in (1, 2, 3, 8):
            ranges = [opmm.opmm_shard_range(n, r, R) for r in range(R)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            for (b0, e0), (b1, e1) in zip(ranges, ranges[1:]):
                assert e0 == b1
            sizes = [e - b for b, e in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(opmm.OpmmError):
        opmm.opmm_shard_range(10, 3, 3)


def test_merge_argmin_lexicographic(opmm):
    inf = math.inf
    assert opmm.opmm_merge_argmin([3.0, 1.0, 1.0], [5, 9, 7]) == (1.0, 7)
    assert opmm.opmm_merge_argmin([inf, 2.0], [0, 4]) == (2.0, 4)
    assert opmm.opmm_merge_argmin([1.0, 1.0], [-1, 3]) == (1.0, 3)   # -1 = empty shard
    e, i = opmm.opmm_merge_argmin([inf, inf], [1, 2])
    assert i == -1 and e == inf
    assert opmm.opmm_merge_argmin([], []) == (inf, -1)


def test_validation_rejects_bad_arguments(opmm):
    import workloads as W
    sp = W.paper_space()
    opmm.opmm_validate(W.Control(), sp, 10)
    for bad in (dict(dt_ms=0.0), dict(dt_ms=math.nan), dict(n_steps=0), dict(n_steps=16385),
                dict(pw_default_ms=-1.0), dict(amplitude_deg=math.inf)):
        with pytest.raises(opmm.OpmmError) as ei:
            opmm.opmm_validate(opmm.control(W.Control(), **bad), sp, 10)
        assert ei.value.status == opmm.ERR_INVALID_ARG
    bad = W.paper_space()
    bad.lo[3] = -1.0   # log dimension with lo <= 0
    with pytest.raises(opmm.OpmmError):
        opmm.opmm_validate(W.Control(), bad, 10)
    bad = W.paper_space()
    bad.lo[0], bad.hi[0] = 2.0, 1.0
    with pytest.raises(opmm.OpmmError):
        opmm.opmm_validate(W.Control(), bad, 10)
    g = W.g4_space(per_dim=10)
    opmm.opmm_validate(W.Control(), g, 10**4)
    with pytest.raises(opmm.OpmmError):
        opmm.opmm_validate(W.Control(), g, 10**4 + 1)   # grid product != N
    with pytest.raises(opmm.OpmmError):
        opmm.opmm_validate(W.Control(), sp, -1)


def test_no_device_fails_loudly_without_cpu_fallback(opmm):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(opmm.OpmmError) as ei:
        opmm.opmm_create(0)
    assert ei.value.status == opmm.ERR_CUDA


def test_product_does_not_import_the_oracle():
    """The product package never references oracle/ (and vice versa)."""
    pkg = os.path.join(ROOT, "paper_2007_09884_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "opmm_oracle" not in txt and "liboracle" not in txt, f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".c")):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            assert "import paper_2007_09884_b200" not in txt, f
            assert "from paper_2007_09884_b200" not in txt and "libopmm.so" not in txt, f


def test_only_tests_smoke_and_bench_touch_the_oracle():
    """Outside tests/ and oracle/ itself, only __graft_entry__.py (smoke),
    bench.py (its CPU-baseline and reference legs) and scripts/ (the committed
    writers of tests/golden/ fixtures, which call only oracle/) may import
    oracle/; tools/, workloads/, examples/ and the package never do."""
    allowed = {os.path.join(ROOT, "__graft_entry__.py"), os.path.join(ROOT, "bench.py")}
    for dirpath, dirs, files in os.walk(ROOT):
        rel = os.path.relpath(dirpath, ROOT)
        top = rel.split(os.sep)[0]
        if top in ("tests", "oracle", "scripts", ".git", "gpurun_out", "baseline") or "/scratch" in dirpath \
                or "/var" in dirpath:
            dirs[:] = []
            continue
        for f in files:
            path = os.path.join(dirpath, f)
            if f.endswith(".py") and path not in allowed:
                txt = open(path).read()
                assert "import oracle" not in txt and "from oracle" not in txt, path


def test_stream_marshalling():
    """torch's default stream is the legacy NULL stream; the C ABI reads NULL
    as "the handle's own (non-blocking) stream", so the binding must pass
    cudaStreamLegacy for it, and pass None / other streams through."""
    from paper_2007_09884_b200 import opmm

    class S:
        def __init__(self, v):
            self.cuda_stream = v
    assert opmm._stream(None) is None
    assert opmm._stream(S(0)) == opmm.CUDA_STREAM_LEGACY == 1
    assert opmm._stream(0) == 1
    assert opmm._stream(S(0x1234)) == 0x1234
