"""The drop-in adapter (include/lf_gpu.hpp) compiled against the reference's
own headers and library, checked from the reference side.

Host part (no GPU): built and run here when /root/reference exists. The
binary lands in tests/adapter/ (git-ignored, shipped to the GPU box), where
the GPU part compares lf::gpu::interpret / materialize / measure with the
reference's lf::interpret / materialize_tensor in the same process.
"""
import os
import subprocess

import pytest

import oracle_lib as O

HERE = os.path.join(O.ROOT, "tests", "adapter")
BIN = os.path.join(HERE, "adapter_check")
REF_INC = "/root/reference/proj/include"


def build_adapter():
    if not os.path.isdir(REF_INC):
        return os.path.exists(BIN)
    from paper_2210_12415_b200 import build
    build.build()
    cmd = ["g++", "-std=c++20", "-O1", "-I", REF_INC, "-I", os.path.join(O.ROOT, "include"),
           os.path.join(HERE, "adapter_check.cpp"), "-o", BIN,
           os.path.join(O.ROOT, "oracle", "_ref", "libref.so"),
           os.path.join(O.ROOT, "paper_2210_12415_b200", "liblfgpu.so"),
           "-Wl,-rpath,$ORIGIN/../../oracle/_ref:$ORIGIN/../../paper_2210_12415_b200"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return True


@pytest.mark.skipif(not os.path.isdir(REF_INC) or not O.ref_available(),
                    reason="reference headers / build absent")
def test_adapter_host_roundtrips():
    assert build_adapter()
    r = subprocess.run([BIN, "host"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "host: OK" in r.stdout


@pytest.mark.gpu
def test_adapter_gpu_against_reference_interpret():
    if not build_adapter():
        pytest.skip("adapter_check binary not built (needs the reference headers once)")
    r = subprocess.run([BIN, "gpu"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "gpu: OK" in r.stdout
