"""The C ABI from plain C (examples/c_abi_example.c, no Python): compiles against
include/grpo_async.h and libgrpo_async.so on CPU; runs on a GPU box (-m gpu)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2604_26256_b200")


def _compile(tmp_path):
    exe = os.path.join(str(tmp_path), "c_abi_example")
    cmd = ["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
           "-I", "/usr/local/cuda/include", os.path.join(ROOT, "examples", "c_abi_example.c"),
           "-L", LIBDIR, "-lgrpo_async", "-L", "/usr/local/cuda/lib64", "-lcudart",
           f"-Wl,-rpath,{LIBDIR}", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_example_compiles_against_the_header(tmp_path):
    import paper_2604_26256_b200  # noqa: F401  (builds/loads the library)
    assert os.path.exists(_compile(tmp_path))


@pytest.mark.gpu
def test_c_example_runs(tmp_path):
    exe = _compile(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "J=" in out.stdout and "rows=17" in out.stdout
