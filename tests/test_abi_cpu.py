"""CPU-side checks of the C-ABI library: it builds for sm_100a, loads, exports every symbol
include/pbe.h declares, and validates arguments synchronously (no GPU needed for that).
Also checks that the product package never imports the oracle."""
import ctypes as C
import math
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2411_00742_b200 import build
    build.build()
    import paper_2411_00742_b200 as pb
    return pb.load_library()


def _header_symbols():
    text = open(os.path.join(ROOT, "include", "pbe.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pbe_[a-z_]+)\s*\(", text)))


def test_header_and_binding_agree():
    import paper_2411_00742_b200 as pb
    assert _header_symbols() == sorted(pb.EXPORTS)


def test_library_exports_every_header_symbol(lib):
    for name in _header_symbols():
        assert hasattr(lib, name), name


def test_library_is_sm100a(lib):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib._name], capture_output=True, text=True)
    assert "sm_100a" in out.stdout, out.stdout + out.stderr


def test_version(lib):
    assert b"sm_100a" in lib.pbe_version()


def _cfg(**kw):
    import paper_2411_00742_b200 as pb
    base = dict(n_bins=100, L_lo=0.0, dL=12.0, limiter=1, courant=0.9, dt_fixed=0.0, dt_max=math.inf,
                max_steps=1000, n_steps=0, rho_c=1.11e-12, k_v=math.pi / 4, n_samples=10, n_tangents=0,
                max_sims=1, kernel=0)
    base.update(kw)
    return pb._Config(**base)


@pytest.mark.parametrize("bad", [dict(n_bins=2), dict(dL=0.0), dict(dL=-1.0), dict(limiter=7), dict(courant=0.0),
                                 dict(courant=1.5), dict(dt_fixed=-1.0), dict(dt_max=0.0), dict(max_steps=0),
                                 dict(n_samples=0), dict(n_tangents=11), dict(max_sims=0), dict(kernel=9),
                                 dict(n_steps=5, n_samples=3), dict(dt_max=math.nan)])
def test_create_rejects_bad_config_synchronously(lib, bad):
    h = C.c_void_p()
    st = lib.pbe_create(C.byref(_cfg(**bad)), 0, C.byref(h))
    assert st == 1 and not h.value
    assert len(lib.pbe_last_error(None)) > 0


def test_create_without_gpu_reports_cuda_error(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    st = lib.pbe_create(C.byref(_cfg()), 0, C.byref(h))
    assert st == 6 and b"CUDA" in lib.pbe_last_error(None)


def test_null_context_calls_fail_cleanly(lib):
    assert lib.pbe_set_kinetics(None, 0, 1, 1, None, 0, 2, None, 1, None, None, 0, None) == 1
    assert lib.pbe_run_batch(None, 1, None, 0, 0, None, None, None, None, None, None) == 1
    assert lib.pbe_moments(None, None, None, None, None, 0) == 1
    lib.pbe_destroy(None)


def test_product_path_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2411_00742_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", text, re.M), f
                assert "liboracle" not in text and "pbe_oracle" not in text, f
