"""Host-side checks of the device bidiagonal QR SVD (csrc/bidiag_qr.cuh, the QR option of
ssa_decompose), compiled for the CPU with nvcc through tools/qr_harness.cu.  Pins:
the SPEC.md:227 example alpha = (1, 1), beta_2 = 1 -> sigma = (phi, 1/phi); LAPACK
singular values of random and Lanczos-produced bidiagonals; B = P diag(d) Q^T rebuilt
from the recorded rotations; the tracked last row of P; zero diagonal entries."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HARNESS = os.path.join(ROOT, "tools", "qr_harness.cu")


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("qr") / "qr_harness")
    subprocess.check_call(["nvcc", "-O2", "-std=c++17", "-x", "cu", "-o", out, HARNESS])
    return out


def run(exe, alpha, beta):
    """alpha: alpha_1..alpha_m, beta: beta_2..beta_{m+1}."""
    m = len(alpha)
    inp = f"{m}\n" + " ".join(repr(float(x)) for x in alpha) + "\n" + " ".join(repr(float(x)) for x in beta) + "\n"
    out = subprocess.run([exe], input=inp, capture_output=True, text=True, check=True).stdout.split("\n")
    it = int(out[0].split()[1])
    f = out[1].split()
    stats = dict(recon_rel=float(f[3]), lastrow=float(f[5]), orth=float(f[7]))
    sv = np.array([float(x) for x in out[2:] if x.strip()])
    return it, stats, np.sort(sv)[::-1]


def lower_bidiag(alpha, beta):
    m = len(alpha)
    B = np.zeros((m + 1, m))
    B[np.arange(m), np.arange(m)] = alpha
    B[np.arange(1, m + 1), np.arange(m)] = beta
    return B


def test_spec_golden_ratio(exe):
    it, st, sv = run(exe, [1.0, 1.0], [1.0, 0.0])
    phi = (1 + 5 ** 0.5) / 2
    assert np.allclose(sv, [phi, 1 / phi], rtol=1e-15, atol=0)


@pytest.mark.parametrize("m", [1, 2, 3, 7, 40, 120])
def test_random_bidiagonal(exe, m):
    rng = np.random.default_rng(m)
    a = rng.uniform(0.1, 2, m); b = rng.uniform(0.1, 2, m)
    it, st, sv = run(exe, a, b)
    ref = np.linalg.svd(lower_bidiag(a, b), compute_uv=False)
    assert it >= 0
    assert np.abs(sv - ref).max() <= 1e-14 * ref[0]
    assert st["recon_rel"] <= 1e-13 and st["orth"] <= 1e-13 and st["lastrow"] <= 1e-14


def test_lanczos_bidiagonal_graded(exe):
    """Graded spectrum like the cfg1 series: values spanning 1 .. 1e-3 with tight pairs."""
    rng = np.random.default_rng(5)
    m = 60
    a = np.geomspace(2000, 2, m) * rng.uniform(0.9, 1.1, m)
    b = np.geomspace(500, 0.5, m) * rng.uniform(0.9, 1.1, m)
    it, st, sv = run(exe, a, b)
    ref = np.linalg.svd(lower_bidiag(a, b), compute_uv=False)
    assert np.abs(sv - ref).max() <= 1e-14 * ref[0]
    assert st["recon_rel"] <= 1e-13 and st["orth"] <= 1e-13


def test_zero_diagonal_entries(exe):
    """Lanczos restarts put alpha_j = 0 (or beta = 0) into B: the zero-chasing paths."""
    rng = np.random.default_rng(9)
    for zero_at in ([0], [3], [5, 6], [9]):
        m = 10
        a = rng.uniform(0.5, 1.5, m); b = rng.uniform(0.5, 1.5, m)
        a[zero_at] = 0.0
        it, st, sv = run(exe, a, b)
        ref = np.linalg.svd(lower_bidiag(a, b), compute_uv=False)
        assert np.abs(sv - ref).max() <= 1e-14 * ref[0], zero_at
        assert st["recon_rel"] <= 1e-13 and st["orth"] <= 1e-13
    a = rng.uniform(0.5, 1.5, 8); b = rng.uniform(0.5, 1.5, 8); b[-1] = 0.0; b[2] = 0.0
    it, st, sv = run(exe, a, b)
    ref = np.linalg.svd(lower_bidiag(a, b), compute_uv=False)
    assert np.abs(sv - ref).max() <= 1e-14 * ref[0]
