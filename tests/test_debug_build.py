"""The debug build (build.py --debug: device-side invariant checks, CGGM_DASSERT) compiles for
sm_100a and exports the same C-ABI (CPU); on a GPU the tiny evaluation runs through it with
CGGM_SYNC_CHECK=1 (every launch synchronised, faults attributed to their kernel) and matches the
oracle -- the in-library stand-in for compute-sanitizer."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEBUG_LIB = os.path.join(ROOT, "paper_1509_04681_b200", "lib", "debug", "libcggm.so")


def _build_debug():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "paper_1509_04681_b200", "build.py"), "--debug"],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    assert os.path.exists(DEBUG_LIB)


def test_debug_build_exports_the_abi():
    import ctypes
    _build_debug()
    from tests.test_abi_symbols import declared_symbols
    lib = ctypes.CDLL(DEBUG_LIB)
    for n in sorted(declared_symbols()):
        assert hasattr(lib, n), n


@pytest.mark.gpu
def test_debug_build_tiny_evaluation_with_sync_check():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(DEBUG_LIB):
        _build_debug()
    env = dict(os.environ, CGGM_LIB=DEBUG_LIB, CGGM_SYNC_CHECK="1")
    code = "import __graft_entry__ as g; g.smoke()"
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "smoke ok" in r.stdout
