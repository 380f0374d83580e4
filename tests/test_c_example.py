"""The C ABI used from a plain C program (examples/fit_c_abi.c): compiles
against include/opmm.h + libopmm.so with gcc; without a GPU it must fail
loudly in opmm_create (exit 2); on the GPU box it fits and validates."""
import os
import subprocess

import pytest

from conftest import ROOT


def _build():
    from paper_2007_09884_b200 import build
    build.build()
    os.makedirs(os.path.join(ROOT, "build"), exist_ok=True)
    exe = os.path.join(ROOT, "build", "fit_c_abi")
    subprocess.check_call(["gcc", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "examples", "fit_c_abi.c"),
                           "-L", os.path.join(ROOT, "paper_2007_09884_b200"), "-lopmm",
                           "-Wl,-rpath," + os.path.join(ROOT, "paper_2007_09884_b200"),
                           "-o", exe, "-lm"])
    return exe


def test_c_example_builds_and_fails_loudly_without_gpu():
    import torch
    exe = _build()
    if torch.cuda.is_available():
        pytest.skip("GPU present (covered by the gpu test)")
    p = subprocess.run([exe], capture_output=True, text=True)
    assert p.returncode == 2 and "opmm_create" in p.stderr


@pytest.mark.gpu
def test_c_example_runs_on_gpu():
    exe = _build()
    p = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "fit_c_abi ok" in p.stdout and "invalid dt -> status 1" in p.stdout
