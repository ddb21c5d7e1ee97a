"""Drop-in check: the reference's own demo program, proj/demos/fuse_demo.cpp,
built against include/sparsefuse_b200.hpp with only its include line changed
(swapped for our header plus `namespace sparsefuse = sparsefuse_b200;`).

* CPU (this container, where /root/reference exists): it compiles with the
  same one-line substitution oracle/Makefile applies, and the binary built by
  `make -C oracle` refuses to compute without a device (no CPU fallback).
* GPU: the prebuilt oracle/_ref/fuse_demo_b200 (it travels with the repo
  snapshot) runs the canonical sequence -- msp, validate_fused_partitioning,
  compile_schedule, execute_fused / execute_unfused / execute_joint_wavefront
  / execute_sequential -- and exits 0.  The same sequence with every result
  checked bit for bit is tests/test_gpu_schedules.py and
  tests/cpp/test_api.cpp.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEMO_SRC = "/root/reference/proj/demos/fuse_demo.cpp"
DEMO_BIN = os.path.join(ROOT, "oracle", "_ref", "fuse_demo_b200")
SUBST = ('s|#include <sparsefuse/sparsefuse.hpp>|#include "sparsefuse_b200.hpp"\\n'
         'namespace sparsefuse = sparsefuse_b200;|')


@pytest.mark.skipif(not os.path.exists(DEMO_SRC), reason="reference tree absent (GPU box)")
def test_reference_demo_compiles_against_the_mirror(tmp_path):
    src = subprocess.run(["sed", SUBST, DEMO_SRC], check=True, capture_output=True, text=True).stdout
    orig = open(DEMO_SRC).read()
    # the only change: the include, replaced by our header + the namespace alias
    inc = "#include <sparsefuse/sparsefuse.hpp>"
    assert orig.count(inc) == 1
    assert src == orig.replace(inc, '#include "sparsefuse_b200.hpp"\nnamespace sparsefuse = sparsefuse_b200;')
    exe = str(tmp_path / "fuse_demo")
    lib = os.path.join(ROOT, "paper_2111_12238_b200")
    r = subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Werror", "-x", "c++", "-",
                        "-I" + os.path.join(ROOT, "include"), "-L" + lib, "-lsfgpu",
                        f"-Wl,-rpath,{lib}", "-o", exe], input=src, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_prebuilt_demo_refuses_without_device():
    from paper_2111_12238_b200 import abi
    if abi.device_available():
        pytest.skip("a CUDA device is present")
    if not os.path.exists(DEMO_BIN):
        pytest.skip("oracle/_ref/fuse_demo_b200 not built (make -C oracle)")
    r = subprocess.run([DEMO_BIN], capture_output=True, text=True, timeout=60)
    assert r.returncode != 0 and "NoDeviceError" in r.stderr


@pytest.mark.gpu
def test_reference_demo_runs_on_the_gpu():
    assert os.path.exists(DEMO_BIN), "oracle/_ref/fuse_demo_b200 is built by __graft_entry__.build()"
    r = subprocess.run([DEMO_BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    out = r.stdout
    assert "n=1024" in out
    for ex in ("sequential", "fused", "unfused", "wavefront"):
        assert any(line.split()[:1] == [ex] for line in out.splitlines()), out
