"""Host-side checks of the C-ABI boundary (no GPU compute)."""
import ast
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "fdfb.h")).read()
    return sorted(set(re.findall(r"\b(fdfb_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2109_02731_b200 import build
    path = build.build()
    lib = ctypes.CDLL(path)
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s


def test_status_strings_and_validation_without_gpu():
    from paper_2109_02731_b200 import build
    lib = ctypes.CDLL(build.build())
    lib.fdfb_status_string.restype = ctypes.c_char_p
    assert lib.fdfb_status_string(0) == b"ok"
    assert b"prime" in lib.fdfb_status_string(-2)
    # NULL params are rejected before touching the device
    h = ctypes.c_void_p()
    assert lib.fdfb_ctx_create(None, 0, ctypes.byref(h)) == -1


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2109_02731_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                tree = ast.parse(open(os.path.join(dp, f)).read())
                for node in ast.walk(tree):
                    if isinstance(node, ast.Import):
                        assert not any(a.name.startswith("oracle") for a in node.names), f
                    if isinstance(node, ast.ImportFrom):
                        assert not (node.module or "").startswith("oracle"), f
    for dp, _, files in os.walk(os.path.join(pkg, "csrc")):
        for f in files:
            assert "oracle" not in open(os.path.join(dp, f)).read().lower().replace("no oracle", ""), f


def test_binding_fails_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    import synth
    from paper_2109_02731_b200 import Context, FdfbError
    with pytest.raises(FdfbError):
        Context(synth.load_config("tiny"))


def test_parameter_validation_before_device_use():
    """fdfb_ctx_create validates every parameter before touching a device (status codes, no throw)."""
    import synth
    from paper_2109_02731_b200 import build
    from paper_2109_02731_b200.fdfb import params_from_config
    lib = ctypes.CDLL(build.build())
    base = synth.load_config("large")

    def rc(**kw):
        cfg = dict(base, **kw)
        h = ctypes.c_void_p()
        return lib.fdfb_ctx_create(ctypes.byref(params_from_config(cfg)), 0, ctypes.byref(h))

    assert rc(N=3000) == -3                                   # N not a power of two in range
    assert rc(Q=base["Q"] + 2) == -2                          # not prime
    assert rc(Q=2**31 - 1) == -2                              # prime, but not 1 mod 2N
    assert rc(Q=72057594037641217) == -2                      # NTT prime, but >= 2^55 (BR CRT headroom)
    assert rc(ell_rgsw=3) == -4                               # ell != ceil(54 / 14)
    assert rc(ell_ks=12) == -4
    assert rc(t=3) == -6                                      # t does not divide 2N
    assert rc(n=0) == -3
