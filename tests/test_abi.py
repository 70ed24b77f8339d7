"""The C-ABI boundary: libssa.so loads and exports every function include/ssa.h declares
(no GPU needed: symbols only, no compute calls); the CUDA code is built for sm_100a."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ssa.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*(ssa_[a-z0-9_]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    from paper_0911_4498_b200 import build
    build.build()
    import paper_0911_4498_b200 as P
    return P.load_library()


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("ssa_plan_create", "ssa_decompose", "ssa_reconstruct", "ssa_spectrum", "ssa_matvec",
                 "ssa_hankelize", "ssa_plan_destroy", "ssa_status_string", "ssa_last_error"):
        assert must in names, must


def test_library_exports_every_declared_symbol(lib):
    import paper_0911_4498_b200 as P
    names = declared_functions()
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert sorted(P.EXPORTS) == names, "binding EXPORTS list out of sync with include/ssa.h"


def test_status_strings_and_defaults(lib):
    import ctypes
    import paper_0911_4498_b200.ssa as S
    for code, name in S.STATUS.items():
        assert lib.ssa_status_string(code).decode() == name
    opt = S.Options()
    assert lib.ssa_options_default(ctypes.byref(opt)) == 0
    assert opt.tol == 1e-12 and opt.seed == 42 and opt.reorth == 3 and opt.check_every == 4
    assert abs(opt.reorth_eta - np.finfo(float).eps ** 0.75) <= 1e-27   # PRO default, R22


def test_validation_happens_before_any_device_work(lib):
    """Argument errors are reported synchronously, before touching the GPU (works on CPU)."""
    import ctypes
    h = ctypes.c_void_p()
    for (N, L, k, B) in [(2, 1, 1, 1), (10, 1, 1, 1), (10, 10, 1, 1), (10, 5, 7, 1), (10, 5, 1, 0), (10, 5, -1, 1)]:
        st = lib.ssa_plan_create(N, L, k, B, None, 0, ctypes.byref(h))
        assert st == 1, (N, L, k, B, st)   # SSA_ERR_INVALID_ARGUMENT
        assert lib.ssa_last_error()
    import paper_0911_4498_b200.ssa as S
    for reorth, eta in [(0, 1e-12), (4, 1e-12), (3, 0.0), (3, 1e-3), (3, -1.0)]:
        opt = S.Options()
        lib.ssa_options_default(ctypes.byref(opt))
        opt.reorth, opt.reorth_eta = reorth, eta
        assert lib.ssa_plan_create(100, 50, 4, 1, ctypes.byref(opt), 0, ctypes.byref(h)) == 1, (reorth, eta)
    assert lib.ssa_plan_fft_size(None) == -1


def test_cubin_is_sm100a():
    so = os.path.join(ROOT, "paper_0911_4498_b200", "libssa.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out, out


def test_product_never_imports_oracle():
    """The product package shares no code with the oracle and never imports it."""
    pkg = os.path.join(ROOT, "paper_0911_4498_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "ssa_oracle" not in txt, f
