"""CPU (and GPU when present): the C++ adapter include/pathtrack_b200.hpp
compiles against the unmodified reference headers, links the C-ABI library,
and behaves (throws without a device, tracks with one)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"


def _build_and_run(tmp_path, use_ref):
    exe = tmp_path / "cpp_api_check"
    inc = ["-I", os.path.join(ROOT, "include"), "-I", os.path.join(ROOT, "oracle")]
    if use_ref:
        inc += ["-I", REF_INC, "-DUSE_REFERENCE_HEADERS", "-include", "vector"]
    lib = os.path.join(ROOT, "paper_1501_06625_b200")
    cmd = ["g++", "-std=c++20", "-O1", "-ffp-contract=off", *inc, os.path.join(ROOT, "tests", "cpp_api_check.cpp"),
           "-L", lib, "-lpathtrack_b200", f"-Wl,-rpath,{lib}", "-o", str(exe)]
    if os.path.exists("/usr/bin/g++"):
        cmd[0] = "/usr/bin/g++"
    subprocess.run(cmd, check=True, capture_output=True)
    return subprocess.run([str(exe)], capture_output=True, text=True)


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers not mounted")
def test_cpp_adapter_on_reference_headers(tmp_path):
    r = _build_and_run(tmp_path, True)
    assert r.returncode == 0, r.stdout + r.stderr


def test_cpp_adapter_on_restated_headers(tmp_path):
    r = _build_and_run(tmp_path, False)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_adapter_tracks_on_device(tmp_path, gpu):
    """The C++ adapter's device path: plan, track_path through the C-ABI,
    end point x = 2 of the SPEC.md:472 homotopy (restated headers: the box
    has no /root/reference)."""
    r = _build_and_run(tmp_path, os.path.isdir(REF_INC))
    assert r.returncode == 0 and "device: success=1" in r.stdout, r.stdout + r.stderr
    assert "batch: 3 paths, all equal to the single path" in r.stdout, r.stdout
