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


def _build_driver(tmp_path):
    exe = str(tmp_path / "stream_driver")
    cuda = "/usr/local/cuda"
    subprocess.run(["/usr/bin/g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    "-I", f"{cuda}/include", os.path.join(ROOT, "tests", "cpp", "stream_driver.cpp"),
                    "-L", LIBDIR, "-lompds_b200", f"-Wl,-rpath,{LIBDIR}",
                    "-L", f"{cuda}/lib64", "-lcudart", f"-Wl,-rpath,{cuda}/lib64", "-o", exe],
                   check=True)
    return exe


def test_cpp_host_driver_compiles_and_links(tmp_path):
    """C++ host code on the C ABI alone (no Python): the config kernels'
    launchers, host-buffer entry point, team ranges and allocators."""
    assert os.path.exists(_build_driver(tmp_path))


@pytest.mark.gpu
def test_cpp_host_driver_runs_the_configs_on_gpu(tmp_path):
    exe = _build_driver(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "stream driver ok" in r.stdout, r.stdout + r.stderr
