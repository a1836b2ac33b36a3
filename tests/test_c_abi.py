"""The C ABI used from plain C (tests/c_abi/lars_abi_example.c): the header
compiles as C99 with -Wall -Werror, the program links against
liblars_b200.so, and on a B200 one scheduled step matches an fp64 C
restatement of the reference step (on a machine without a GPU the library
reports LARS_ERR_NO_DEVICE through the same entry points)."""

import os
import shutil
import subprocess

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "c_abi", "lars_abi_example.c")
LIBDIR = os.path.join(ROOT, "paper_1709_05011_b200", "_lib")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def _build(tmp_path):
    if shutil.which("gcc") is None or not os.path.exists(os.path.join(CUDA, "include")):
        pytest.skip("gcc or CUDA headers not available")
    from paper_1709_05011_b200 import build
    build.build()
    exe = str(tmp_path / "lars_abi_example")
    cmd = ["gcc", "-std=c99", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(CUDA, "include"), SRC, "-L", LIBDIR, "-llars_b200",
           "-L", os.path.join(CUDA, "lib64"), "-lcudart", "-lm", f"-Wl,-rpath,{LIBDIR}", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_program_builds_and_reports_no_device_without_gpu(tmp_path):
    exe = _build(tmp_path)
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu test")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=60)
    assert out.returncode == 2
    assert "no CUDA device" in out.stderr


@pytest.mark.gpu
def test_c_program_step_matches_fp64_reference(tmp_path, cuda):
    exe = _build(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.strip().endswith("ok")
