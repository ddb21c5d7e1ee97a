"""The C++ mirror of the reference API (include/sparsefuse_b200.hpp).

tests/cpp/test_api.cpp is compiled against the header, libsfgpu.so and the C
oracle, then run: without a GPU it must refuse to compute (NoDeviceError, no
CPU fallback); on a B200 it drives combos 1-8 through make_state ->
build_g1/g2 -> inter_dag -> joint_dag -> level_info -> make_fused_schedule ->
execute_fused / execute_unfused -> collect_outputs and checks each result bit
for bit against the oracle, plus the FactorizationError / InvalidMatrixError
paths.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    exe = str(tmp_path / "test_api")
    lib = os.path.join(ROOT, "paper_2111_12238_b200")
    orc = os.path.join(ROOT, "oracle")
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", "-Werror", "-I" + os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "test_api.cpp"), "-o", exe, "-L" + lib, "-lsfgpu",
           "-L" + orc, "-loracle", f"-Wl,-rpath,{lib}:{orc}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_cpp_header_compiles_and_refuses_without_device(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe, "--no-device"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().endswith(")") and "OK" in r.stdout


@pytest.mark.gpu
def test_cpp_api_end_to_end(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().splitlines()[-1] == "OK"
    for combo in (1, 2, 3, 4, 5, 6, 7, 8):
        assert f"combo {combo}:" in r.stdout
    assert "breakdown:" in r.stdout
