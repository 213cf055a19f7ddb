"""The drop-in C++ API (include/sigker/*.hpp -> libsigker.so -> the C-ABI):
tests/cpp/test_api.cpp mirrors the reference's engine unit tests.  The build
check runs on the CPU; the run needs the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2502_20392_b200")
EXE = os.path.join(ROOT, "build", "test_api")


def build():
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_api.cpp"), "-o", EXE, "-L", PKG, "-lsigker",
                    "-lsigker_b200", f"-Wl,-rpath,{PKG}"], check=True)


def test_cpp_api_builds_and_links():
    build()
    assert os.path.exists(EXE)


def test_thread_pool_drop_in():
    """host-only part of the drop-in (no GPU work): runs on the CPU"""
    exe = os.path.join(ROOT, "build", "test_thread_pool")
    os.makedirs(os.path.dirname(exe), exist_ok=True)
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_thread_pool.cpp"), "-o", exe, "-L", PKG, "-lsigker",
                    "-lsigker_b200", f"-Wl,-rpath,{PKG}", "-lpthread"], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr


@pytest.mark.gpu
def test_cpp_api_suite():
    build()
    out = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
