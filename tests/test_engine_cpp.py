"""Builds tests/cpp/test_engine.cpp against the drop-in C++ header and libfxg.so
and runs it (host-only cases on CPU, all cases on the GPU)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_engine.cpp")
LIBDIR = os.path.join(ROOT, "paper_2603_12016_b200", "lib")


@pytest.fixture(scope="module")
def binary(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("cpp") / "test_engine")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), SRC,
                    "-L", LIBDIR, "-lfxg", f"-Wl,-rpath,{LIBDIR}", "-o", out], check=True)
    return out


def test_engine_host_cases(binary):
    r = subprocess.run([binary, "--host"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_engine_device_cases(binary):
    r = subprocess.run([binary], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
