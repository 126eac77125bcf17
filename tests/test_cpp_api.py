"""The ksafem-compatible C++ host API (include/ksafem_b200, libksafem_b200.so) through its C++ tests.

tests/cpp/test_ksafem_b200.cpp restates the reference's own tests (proj/tests/*.cpp) against the B200 API.
CPU: it compiles against the headers and the in-tree libraries, and the host-only mesh case runs.
GPU: every case runs on the device.
"""
import os
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2103_02824_b200" / "_lib"


@pytest.fixture(scope="module")
def binary(tmp_path_factory):
    if not (LIB / "libksafem_b200.so").exists():
        pytest.fail("libksafem_b200.so is not built (run __graft_entry__.build())")
    out = tmp_path_factory.mktemp("cpp") / "test_ksafem_b200"
    cmd = ["g++", "-O1", "-std=c++17", "-Wall", "-Wextra", "-Werror", f"-I{ROOT / 'include'}",
           str(ROOT / "tests" / "cpp" / "test_ksafem_b200.cpp"), "-o", str(out), f"-L{LIB}", "-lksafem_b200", "-lksb",
           f"-Wl,-rpath,{LIB}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]
    return out


def test_cpp_api_builds_and_lists(binary):
    r = subprocess.run([str(binary), "--list"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0
    assert len(r.stdout.split("\n")) >= 9


def test_cpp_mesh_case_on_host(binary):
    r = subprocess.run([str(binary), "box mesh"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS box mesh" in r.stdout


@pytest.mark.gpu
def test_cpp_api_on_device(binary):
    env = dict(os.environ)
    r = subprocess.run([str(binary)], capture_output=True, text=True, timeout=900, env=env)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr[-4000:]
    assert "0 failed" in r.stdout
