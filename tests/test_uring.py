"""CPU test of the io_uring wrapper used by the O_DIRECT flush / restore
reads (csrc/uring.cpp, raw io_uring_setup / io_uring_enter): compiled with
g++ together with a small driver, no GPU or CUDA needed."""
import os
import shutil
import subprocess

import pytest

from conftest import ROOT


def test_uring_roundtrip(tmp_path):
    if not shutil.which("g++"):
        pytest.skip("no g++")
    csrc = os.path.join(ROOT, "paper_2601_16956_b200", "csrc")
    exe = str(tmp_path / "uring_selftest")
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", csrc, os.path.join(ROOT, "tests", "capi", "uring_selftest.cpp"),
                    os.path.join(csrc, "uring.cpp"), "-o", exe], check=True)
    r = subprocess.run([exe, str(tmp_path / "f.bin")], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    out = r.stdout.split()
    if out[0] == "skip":
        pytest.skip("io_uring not available here")
    assert out[0] == "ok" and int(out[1]) > 0
