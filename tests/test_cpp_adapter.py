"""The C++ adapter include/ompds.hpp compiles against the C ABI and runs the
reference's TeamRuntime unit cases (proj/tests/RuntimeTests.cpp) on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1711_10413_b200", "_build")


def _build(tmp_path):
    exe = str(tmp_path / "runtime_cases")
    subprocess.run(["/usr/bin/g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "runtime_cases.cpp"), "-L", LIBDIR,
                    "-lompds_b200", f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_adapter_compiles_and_links(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_reference_runtime_cases_pass_on_gpu(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
