"""Thin ctypes binding over libssa.so (include/ssa.h) -- argument marshalling only.

Every step of the method runs in the CUDA kernels behind the C-ABI; this module only
checks shapes/dtypes/devices of torch tensors, passes ``data_ptr()`` and the current
CUDA stream, and turns status codes into exceptions.  There is no CPU fallback: if
libssa.so is missing or no CUDA device is present, calls raise.

Names follow the paper: N series length, L window, K = N - L + 1, k triples,
sigma / U / V singular triples, spectrum = rfft of the series
(Alg. 2 lines 1-2).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SSA_LIB", os.path.join(_HERE, "libssa.so"))

SSA_OK = 0
STATUS = {0: "SSA_OK", 1: "SSA_ERR_INVALID_ARGUMENT", 2: "SSA_ERR_NOT_CONVERGED", 3: "SSA_ERR_OUT_OF_MEMORY",
          4: "SSA_ERR_CUDA", 5: "SSA_ERR_INTERNAL", 6: "SSA_ERR_UNSUPPORTED"}

# every symbol include/ssa.h declares
EXPORTS = ["ssa_options_default", "ssa_plan_create", "ssa_plan_destroy", "ssa_plan_fft_size",
           "ssa_plan_max_steps", "ssa_spectrum", "ssa_matvec", "ssa_matvec_multi", "ssa_hankelize", "ssa_decompose",
           "ssa_reconstruct", "ssa_reconstruct_grouped", "ssa_hmatrix", "ssa_hmatrix_plan_create", "ssa_hmatrix_exec",
           "ssa_hmatrix_plan_destroy", "ssa_bootstrap", "ssa_run_host", "ssa_status_string", "ssa_last_error",
           "ssa_plan_launch_count", "ssa_plan_phase_ms", "ssa_plan_profile", "ssa_plan_bidiagonals"]


class SsaError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Options(ctypes.Structure):
    _fields_ = [("tol", ctypes.c_double), ("max_steps", ctypes.c_int32), ("check_every", ctypes.c_int32),
                ("seed", ctypes.c_uint64), ("reorth", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("reorth_eta", ctypes.c_double), ("series_base", ctypes.c_int64), ("restart_dim", ctypes.c_int32),
                ("restart_keep", ctypes.c_int32)]


class SeriesInfo(ctypes.Structure):
    _fields_ = [("steps", ctypes.c_int32), ("converged", ctypes.c_int32), ("breakdown_step", ctypes.c_int32),
                ("reorth_extra", ctypes.c_int32), ("status", ctypes.c_int32), ("restarts", ctypes.c_int32),
                ("max_residual", ctypes.c_double), ("sigma1", ctypes.c_double), ("rows_u", ctypes.c_int32),
                ("rows_v", ctypes.c_int32), ("reorth_steps", ctypes.c_int32), ("reserved", ctypes.c_int32)]


INFO_DTYPE = np.dtype([("steps", "<i4"), ("converged", "<i4"), ("breakdown_step", "<i4"), ("reorth_extra", "<i4"),
                       ("status", "<i4"), ("restarts", "<i4"), ("max_residual", "<f8"), ("sigma1", "<f8"),
                       ("rows_u", "<i4"), ("rows_v", "<i4"), ("reorth_steps", "<i4"), ("reserved", "<i4")])
assert INFO_DTYPE.itemsize == ctypes.sizeof(SeriesInfo) == 56

_lib = None


def load_library():
    """Load libssa.so (built in-tree by paper_0911_4498_b200.build).  Raises if missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not found: run `python -m paper_0911_4498_b200.build` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i64, i32, dp = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
    lib.ssa_options_default.argtypes = [ctypes.POINTER(Options)]
    lib.ssa_plan_create.argtypes = [i64, i64, i32, i64, ctypes.POINTER(Options), ctypes.c_int, ctypes.POINTER(vp)]
    lib.ssa_plan_destroy.argtypes = [vp]
    lib.ssa_plan_destroy.restype = None
    lib.ssa_plan_fft_size.argtypes = [vp]
    lib.ssa_plan_fft_size.restype = i64
    lib.ssa_plan_max_steps.argtypes = [vp]
    lib.ssa_plan_max_steps.restype = i32
    lib.ssa_plan_launch_count.argtypes = [vp]
    lib.ssa_plan_launch_count.restype = i64
    lib.ssa_plan_phase_ms.argtypes = [vp, ctypes.POINTER(ctypes.c_double)]
    lib.ssa_plan_phase_ms.restype = ctypes.c_int
    lib.ssa_plan_profile.argtypes = [vp, ctypes.POINTER(ctypes.c_int64)]
    lib.ssa_plan_profile.restype = ctypes.c_int
    lib.ssa_plan_bidiagonals.argtypes = [vp, vp, vp, vp]
    lib.ssa_plan_bidiagonals.restype = ctypes.c_int
    lib.ssa_spectrum.argtypes = [vp, dp, dp, vp]
    lib.ssa_matvec.argtypes = [vp, dp, dp, dp, ctypes.c_int, vp]
    lib.ssa_matvec_multi.argtypes = [vp, dp, dp, dp, ctypes.c_int32, ctypes.c_int, vp]
    lib.ssa_hankelize.argtypes = [vp, dp, dp, dp, i32, dp, vp]
    lib.ssa_decompose.argtypes = [vp, dp, dp, dp, dp, dp, vp]
    lib.ssa_reconstruct.argtypes = [vp, dp, dp, dp, dp, vp]
    lib.ssa_reconstruct_grouped.argtypes = [vp, dp, dp, dp, vp, i32, dp, vp]
    lib.ssa_bootstrap.argtypes = [vp, dp, dp, ctypes.c_double, dp, dp, dp, dp, dp, vp]
    lib.ssa_hmatrix_plan_create.argtypes = [i64, i64, i64, i64, vp, i32, ctypes.POINTER(Options), ctypes.c_int,
                                            ctypes.POINTER(vp)]
    lib.ssa_hmatrix_exec.argtypes = [vp, dp, dp, dp, vp]
    lib.ssa_hmatrix_plan_destroy.argtypes = [vp]
    lib.ssa_hmatrix_plan_destroy.restype = None
    lib.ssa_hmatrix.argtypes = [dp, i64, i64, i64, i64, vp, i32, ctypes.POINTER(Options), ctypes.c_int, dp, dp, vp]
    lib.ssa_run_host.argtypes = [vp, dp, dp, dp, dp, dp, dp, vp]
    lib.ssa_status_string.argtypes = [ctypes.c_int]
    lib.ssa_status_string.restype = ctypes.c_char_p
    lib.ssa_last_error.argtypes = []
    lib.ssa_last_error.restype = ctypes.c_char_p
    for name in ("ssa_options_default", "ssa_plan_create", "ssa_spectrum", "ssa_matvec", "ssa_matvec_multi", "ssa_hankelize",
                 "ssa_decompose", "ssa_reconstruct", "ssa_run_host"):
        getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


def _check(st: int):
    if st != SSA_OK:
        raise SsaError(st, load_library().ssa_last_error().decode())


def _stream(stream=None, device=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return int(s.cuda_stream)


def _dev_f64(t, shape, name, device=None):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64:
        raise TypeError(f"{name} must be a CUDA float64 tensor")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if device is not None and t.device.index != device:
        raise ValueError(f"{name} is on cuda:{t.device.index}, the plan on cuda:{device}")
    return t


def _dev_info(t, n, name="info", device=None):
    """A device info buffer: uint8 [n][INFO_DTYPE.itemsize], contiguous (ssa_series_info[n])."""
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.uint8:
        raise TypeError(f"{name} must be a CUDA uint8 tensor")
    if tuple(t.shape) != (n, INFO_DTYPE.itemsize) or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous [{n}][{INFO_DTYPE.itemsize}] tensor, got {tuple(t.shape)}")
    if device is not None and t.device.index != device:
        raise ValueError(f"{name} is on cuda:{t.device.index}, the plan on cuda:{device}")
    return t


class Plan:
    """ssa_plan_create / ssa_plan_destroy wrapper.  One plan per (N, L, k, batch)."""

    def __init__(self, N: int, L: int, k: int, batch: int, *, tol: float = 1e-12, max_steps: int = 0,
                 check_every: int = 4, seed: int = 42, reorth: int = 3, reorth_eta: float = 0.0,
                 series_base: int = 0, device: int | None = None, profile: bool = False, svd: str = "tgk",
                 force_long: bool = False, restart_dim: int = 0, restart_keep: int = 0):
        import torch
        lib = load_library()
        if not torch.cuda.is_available():
            raise RuntimeError("no CUDA device: libssa has no CPU fallback")
        self.device = torch.cuda.current_device() if device is None else int(device)
        opt = Options()
        _check(lib.ssa_options_default(ctypes.byref(opt)))
        opt.tol, opt.max_steps, opt.check_every, opt.seed, opt.reorth = tol, max_steps, check_every, seed, reorth
        if reorth_eta > 0.0:
            opt.reorth_eta = reorth_eta
        opt.series_base = int(series_base)
        opt.restart_dim, opt.restart_keep = int(restart_dim), int(restart_keep)
        opt.reserved = (1 if profile else 0) | (2 if svd == "qr" else 0) | (4 if force_long else 0)
        h = ctypes.c_void_p()
        _check(lib.ssa_plan_create(N, L, k, batch, ctypes.byref(opt), self.device, ctypes.byref(h)))
        self._h = h
        self.N, self.L, self.K, self.k, self.batch = N, L, N - L + 1, k, batch
        self.M = int(lib.ssa_plan_fft_size(h))
        self.m_max = int(lib.ssa_plan_max_steps(h))

    def close(self):
        if getattr(self, "_h", None):
            load_library().ssa_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return int(load_library().ssa_plan_launch_count(self._h))

    def phase_ms(self) -> dict:
        """Device ms of the last spectrum / lanczos / hankelize launches (CUDA events)."""
        out = (ctypes.c_double * 5)()
        _check(load_library().ssa_plan_phase_ms(self._h, out))
        return {"spectrum": out[0], "lanczos": out[1], "bidiag_svd": out[2], "ritz": out[3], "hankelize": out[4]}

    def profile(self) -> dict:
        """Per-phase SM cycles of the decompose kernel (plan created with profile=True)."""
        out = (ctypes.c_int64 * 8)()
        _check(load_library().ssa_plan_profile(self._h, out))
        keys = ["fft", "reorth", "check", "n_checks", "check_values", "check_twisted", "svd_fused", "other"]
        return dict(zip(keys, list(out)))

    def bidiagonals(self):
        """(alpha, beta, steps) of the last decompose (test hook): alpha[b][j] = alpha_j,
        beta[b][j] = beta_j (1-based, Alg. 1), steps[b] = m."""
        nb = min(self.batch, self.batch)  # single-chunk plans: all series
        w = self.m_max + 3
        al = np.zeros((nb, w)); be = np.zeros((nb, w)); st = np.zeros(nb, dtype=np.int32)
        _check(load_library().ssa_plan_bidiagonals(self._h, al.ctypes.data, be.ctypes.data, st.ctypes.data))
        return al, be, st

    def _t(self, *shape):
        import torch
        return torch.empty(shape, dtype=torch.float64, device=f"cuda:{self.device}")

    # -- building blocks -------------------------------------------------------------
    def spectrum(self, series, out=None, stream=None):
        """rfft(series, M) per row -> [batch][M/2+1][2] (Alg. 2 l.1-2)."""
        _dev_f64(series, (self.batch, self.N), "series")
        out = self._t(self.batch, self.M // 2 + 1, 2) if out is None else out
        _dev_f64(out, (self.batch, self.M // 2 + 1, 2), "out")
        _check(load_library().ssa_spectrum(self._h, series.data_ptr(), out.data_ptr(), _stream(stream, self.device)))
        return out

    def matvec(self, spec, x, transpose: bool = False, out=None, stream=None):
        """X x (x: [batch][K]) or X^T x (x: [batch][L]) by FFT correlation (Alg. 2/3)."""
        n_in, n_out = (self.L, self.K) if transpose else (self.K, self.L)
        _dev_f64(spec, (self.batch, self.M // 2 + 1, 2), "spec")
        _dev_f64(x, (self.batch, n_in), "x")
        out = self._t(self.batch, n_out) if out is None else out
        _dev_f64(out, (self.batch, n_out), "out")
        _check(load_library().ssa_matvec(self._h, spec.data_ptr(), x.data_ptr(), out.data_ptr(),
                                         1 if transpose else 0, _stream(stream, self.device)))
        return out

    def matvec_multi(self, spec, x, transpose: bool = False, out=None, stream=None):
        """nvec products per series against its spectrum: x [batch][nvec][K] (X x) or
        [batch][nvec][L] (X^T x) -> [batch][nvec][L or K]."""
        n_in, n_out = (self.L, self.K) if transpose else (self.K, self.L)
        if x.dim() != 3:
            raise ValueError("x must be [batch][nvec][n]")
        nvec = x.shape[1]
        _dev_f64(spec, (self.batch, self.M // 2 + 1, 2), "spec")
        _dev_f64(x, (self.batch, nvec, n_in), "x")
        out = self._t(self.batch, nvec, n_out) if out is None else out
        _dev_f64(out, (self.batch, nvec, n_out), "out")
        _check(load_library().ssa_matvec_multi(self._h, spec.data_ptr(), x.data_ptr(), out.data_ptr(), nvec,
                                               1 if transpose else 0, _stream(stream, self.device)))
        return out

    def hankelize(self, sigma, U, V, out=None, stream=None):
        """Diagonal averaging of sigma_i u_i v_i^T (sec 5, Alg. 4 with division by c_t)."""
        nterms = sigma.shape[1]
        _dev_f64(sigma, (self.batch, nterms), "sigma")
        _dev_f64(U, (self.batch, nterms, self.L), "U")
        _dev_f64(V, (self.batch, nterms, self.K), "V")
        out = self._t(self.batch, nterms, self.N) if out is None else out
        _dev_f64(out, (self.batch, nterms, self.N), "out")
        _check(load_library().ssa_hankelize(self._h, sigma.data_ptr(), U.data_ptr(), V.data_ptr(), nterms,
                                            out.data_ptr(), _stream(stream, self.device)))
        return out

    # -- the hot path ---------------------------------------------------------------
    def decompose(self, series, sigma=None, U=None, V=None, info=None, stream=None):
        """k leading singular triples of every trajectory matrix (Alg. 1 + FRO + bidiagonal SVD).
        Returns (sigma [batch][k], U [batch][k][L], V [batch][k][K], info uint8 [batch][56])."""
        import torch
        d = self.device
        _dev_f64(series, (self.batch, self.N), "series", d)
        sigma = self._t(self.batch, self.k) if sigma is None else _dev_f64(sigma, (self.batch, self.k), "sigma", d)
        U = self._t(self.batch, self.k, self.L) if U is None else _dev_f64(U, (self.batch, self.k, self.L), "U", d)
        V = self._t(self.batch, self.k, self.K) if V is None else _dev_f64(V, (self.batch, self.k, self.K), "V", d)
        if info is None:
            info = torch.zeros((self.batch, INFO_DTYPE.itemsize), dtype=torch.uint8, device=f"cuda:{self.device}")
        _dev_info(info, self.batch, device=d)
        _check(load_library().ssa_decompose(self._h, series.data_ptr(), sigma.data_ptr(), U.data_ptr(),
                                            V.data_ptr(), info.data_ptr(), _stream(stream, self.device)))
        return sigma, U, V, info

    def reconstruct(self, sigma, U, V, out=None, stream=None):
        """Elementary reconstructed series [batch][k][N] (grouping I_j = {j} + averaging)."""
        _dev_f64(sigma, (self.batch, self.k), "sigma")
        _dev_f64(U, (self.batch, self.k, self.L), "U")
        _dev_f64(V, (self.batch, self.k, self.K), "V")
        out = self._t(self.batch, self.k, self.N) if out is None else out
        _dev_f64(out, (self.batch, self.k, self.N), "out")
        _check(load_library().ssa_reconstruct(self._h, sigma.data_ptr(), U.data_ptr(), V.data_ptr(),
                                              out.data_ptr(), _stream(stream, self.device)))
        return out

    def reconstruct_grouped(self, sigma, U, V, groups, ngroups=None, out=None, stream=None):
        """Grouped reconstruction [batch][ngroups][N]: groups[i] is the
        group of triple i (0 .. ngroups-1, or -1 to leave it out); ngroups defaults to
        max(groups) + 1."""
        g = np.ascontiguousarray(groups, dtype=np.int32)
        if g.shape != (self.k,):
            raise ValueError(f"groups must have k = {self.k} entries")
        ng = int(ngroups) if ngroups is not None else (int(g.max()) + 1 if g.size else 0)
        _dev_f64(sigma, (self.batch, self.k), "sigma")
        _dev_f64(U, (self.batch, self.k, self.L), "U")
        _dev_f64(V, (self.batch, self.k, self.K), "V")
        out = self._t(self.batch, max(ng, 1), self.N) if out is None else out
        _dev_f64(out, (self.batch, max(ng, 1), self.N), "out")
        _check(load_library().ssa_reconstruct_grouped(self._h, sigma.data_ptr(), U.data_ptr(), V.data_ptr(),
                                                      g.ctypes.data, ng, out.data_ptr(), _stream(stream, self.device)))
        return out

    def bootstrap(self, series, eps, noise_sigma: float, G=None, info=None, stream=None):
        """Bootstrap study of the rank-k reconstruction (ssa_bootstrap):
        series [N] clean F, eps [batch][N] noise.  Returns (mean, var, mse) [N] each."""
        _dev_f64(series, (self.N,), "series")
        _dev_f64(eps, (self.batch, self.N), "eps")
        mean, var, mse = (self._t(self.N) for _ in range(3))
        if G is not None:
            _dev_f64(G, (self.batch, self.N), "G", self.device)
        if info is not None:
            _dev_info(info, self.batch, device=self.device)
        _check(load_library().ssa_bootstrap(self._h, series.data_ptr(), eps.data_ptr(), float(noise_sigma),
                                            mean.data_ptr(), var.data_ptr(), mse.data_ptr(),
                                            G.data_ptr() if G is not None else None,
                                            info.data_ptr() if info is not None else None, _stream(stream, self.device)))
        return mean, var, mse

    def run_host(self, series: np.ndarray, want_vectors: bool = True, stream=None, raise_on_status=True):
        """End-to-end on host arrays (copies inside the C call).  Returns numpy
        (sigma, U, V, recon, info)."""
        series = np.ascontiguousarray(series, dtype=np.float64)
        assert series.shape == (self.batch, self.N)
        sigma = np.empty((self.batch, self.k))
        recon = np.empty((self.batch, self.k, self.N))
        U = np.empty((self.batch, self.k, self.L)) if want_vectors else None
        V = np.empty((self.batch, self.k, self.K)) if want_vectors else None
        info = np.zeros(self.batch, dtype=INFO_DTYPE)
        p = lambda a: a.ctypes.data if a is not None else None
        st = load_library().ssa_run_host(self._h, p(series), p(sigma), p(U), p(V), p(recon), p(info),
                                         _stream(stream, self.device))
        if raise_on_status:
            _check(st)
        return sigma, U, V, recon, info


def hmatrix(series, B: int, T: int, L: int, I, *, tol: float = 1e-12, seed: int = 42, out=None, info=None,
            stream=None):
    """Heterogeneity matrix G[(N-B+1)][(N-T+1)] of a device series [N] (ssa_hmatrix,
    PAPER.md:962-1040): base windows of length B decomposed with window L, the subspace of
    the triples I (1-based), test windows of length T.  Returns (G, info)."""
    import torch
    lib = load_library()
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: libssa has no CPU fallback")
    N = int(series.shape[-1])
    _dev_f64(series, (N,), "series")
    idx = np.ascontiguousarray(I, dtype=np.int32)
    opt = Options()
    _check(lib.ssa_options_default(ctypes.byref(opt)))
    opt.tol, opt.seed = tol, seed
    dev = series.device.index
    nb, nt = N - B + 1, N - T + 1
    if nb < 1 or nt < 1:  # let the C call report the invalid sizes (it validates first)
        _check(lib.ssa_hmatrix(series.data_ptr(), N, B, T, L, idx.ctypes.data, len(idx), ctypes.byref(opt), dev,
                               None, None, _stream(stream, series.device)))
    G = torch.empty((nb, nt), dtype=torch.float64, device=series.device) if out is None else out
    _dev_f64(G, (nb, nt), "out")
    if info is None:
        info = torch.zeros((nb, INFO_DTYPE.itemsize), dtype=torch.uint8, device=series.device)
    _dev_info(info, nb)
    _check(lib.ssa_hmatrix(series.data_ptr(), N, B, T, L, idx.ctypes.data, len(idx), ctypes.byref(opt), dev,
                           G.data_ptr(), info.data_ptr(), _stream(stream, series.device)))
    return G, info


class HMatrix:
    """ssa_hmatrix_plan_create / exec / destroy: the heterogeneity matrix of series of
    length N with base windows B, test windows T, window L and triples I (1-based), the
    sub-plans and workspace allocated once."""

    def __init__(self, N: int, B: int, T: int, L: int, I, *, tol: float = 1e-12, seed: int = 42,
                 device: int | None = None):
        import torch
        lib = load_library()
        if not torch.cuda.is_available():
            raise RuntimeError("no CUDA device: libssa has no CPU fallback")
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.N, self.B, self.T, self.L = N, B, T, L
        idx = np.ascontiguousarray(I, dtype=np.int32)
        opt = Options()
        _check(lib.ssa_options_default(ctypes.byref(opt)))
        opt.tol, opt.seed = tol, seed
        h = ctypes.c_void_p()
        _check(lib.ssa_hmatrix_plan_create(N, B, T, L, idx.ctypes.data, len(idx), ctypes.byref(opt), self.device,
                                           ctypes.byref(h)))
        self._h = h

    def __call__(self, series, out=None, info=None, stream=None):
        import torch
        _dev_f64(series, (self.N,), "series")
        nb, nt = self.N - self.B + 1, self.N - self.T + 1
        G = torch.empty((nb, nt), dtype=torch.float64, device=series.device) if out is None else out
        _dev_f64(G, (nb, nt), "out")
        if info is None:
            info = torch.zeros((nb, INFO_DTYPE.itemsize), dtype=torch.uint8, device=series.device)
        _dev_info(info, nb)
        _check(load_library().ssa_hmatrix_exec(self._h, series.data_ptr(), G.data_ptr(), info.data_ptr(),
                                               _stream(stream, series.device)))
        return G, info

    def close(self):
        if getattr(self, "_h", None):
            load_library().ssa_hmatrix_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def info_to_numpy(info_tensor) -> np.ndarray:
    """Decode the device info buffer returned by Plan.decompose."""
    raw = info_tensor.detach().cpu().numpy().reshape(-1, INFO_DTYPE.itemsize)
    return np.frombuffer(raw.tobytes(), dtype=INFO_DTYPE)
