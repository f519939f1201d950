"""The C-ABI library loads and exports every symbol include/*.h declares (CPU only: no compute calls)."""
import ctypes
import glob
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"\b(cggm_[a-z0-9_]+)\s*\(", src):
            names.add(m.group(1))
    return names


def test_library_exports_all_declared_symbols():
    from paper_1509_04681_b200 import _abi
    lib = _abi.load()
    names = declared_symbols()
    assert {"cggm_covariances", "cggm_invert_logdet", "cggm_psi_grad", "cggm_active_set",
            "cggm_objective"} <= names
    for n in sorted(names):
        assert hasattr(lib, n), f"{n} declared in include/ but not exported"
    # the binding declares exactly the header's symbols
    assert set(_abi.SIGNATURES) == names


def test_version_string_without_gpu():
    from paper_1509_04681_b200 import _abi
    assert b"sm_100a" in _abi.load().cggm_version()


def test_ctx_create_fails_cleanly_without_gpu():
    import torch
    if torch.cuda.is_available():
        return
    from paper_1509_04681_b200 import _abi
    lib = _abi.load()
    h = ctypes.c_void_p()
    st = lib.cggm_ctx_create(ctypes.byref(h), 0, 0, None)
    assert st != 0 and not h.value
