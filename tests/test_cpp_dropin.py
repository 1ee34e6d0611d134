"""The C++ drop-in rgg::GpuEngine (include/rgg/engine_gpu.hpp) against the reference's
BatchEngine / SequentialEngine, run as a prebuilt binary (oracle/_ref/test_gpu_engine,
built by `make -C oracle dropin` against the reference headers).  Lazy and eager
(host exact resolve) modes, reports, bits, masks, scenario replays."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "test_gpu_engine")


@pytest.mark.gpu
def test_cpp_gpu_engine_matches_reference_engines():
    if not os.path.exists(BIN):
        pytest.skip("drop-in test binary not built (needs /root/reference at build time)")
    r = subprocess.run([BIN, os.path.join(ROOT, "tests", "golden", "scenarios")], capture_output=True, text=True,
                       timeout=600)
    print(r.stdout)
    print(r.stderr[-4000:])
    assert r.returncode == 0, r.stderr[-2000:]
    assert "0 failures" in r.stdout
