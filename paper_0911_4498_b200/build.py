"""Compile libssa.so (all CUDA sources of the hot path) in-tree for sm_100a with nvcc."""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libssa.so")
SOURCES = [os.path.join(HERE, "csrc", f) for f in ("ssa_api.cu", "ssa_fft_kernels.cu", "ssa_lanczos.cu", "ssa_svd.cu", "ssa_large_fft.cu",
                                                   "ssa_large_lanczos.cu", "ssa_hmatrix.cu")]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v", "-diag-suppress", "1886,550"]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = glob.glob(os.path.join(HERE, "csrc", "*")) + [os.path.join(ROOT, "include", "ssa.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """nvcc each translation unit in parallel (-c, relocatable objects), then link the
    shared library.  Flags: -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo."""
    if not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    import tempfile
    tmpdir = tempfile.mkdtemp(prefix="ssa_build_")
    compile_flags = [f for f in NVCC_FLAGS if f != "-shared"]

    def cc(src):
        obj = os.path.join(tmpdir, os.path.basename(src) + ".o")
        r = subprocess.run([_nvcc(), *compile_flags, "-c", "-o", obj, src], capture_output=True, text=True)
        return src, obj, r

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        results = list(ex.map(cc, SOURCES))
    logs = []
    for src, obj, r in results:
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n" + r.stdout + r.stderr)
        logs.append(r.stderr)
    tmp = LIB + f".tmp{os.getpid()}"
    r = subprocess.run([_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp,
                        *[o for _, o, _ in results]], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + r.stdout + r.stderr)
    if verbose:
        print("\n".join(logs))
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
