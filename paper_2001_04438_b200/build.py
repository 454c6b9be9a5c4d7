"""Build libtwopass.so in-tree with nvcc for sm_100a (no JIT, no torch extension cache)."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
SO = os.path.join(PKG, "libtwopass.so")
SOURCES = ["tp_kernels.cu", "tp_stream.cu", "tp_rowcl.cu", "tp_rowcl3.cu", "tp_small.cu", "tp_rowph.cu", "tp_rowres.cu", "tp_rowres3.cu", "tp_peer.cu", "tp_api.cu", "tp_debug.cu"]
HEADERS = ["tp_rowres.cuh", "tp_common.cuh", "tp_block.cuh", "tp_sched.cuh", "tp_ops.cuh", "tp_internal.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr", "-fmad=true",
    "-I", os.path.join(ROOT, "include"),
]


def _stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "twopass.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = SO, defines: tuple = ()) -> str:
    """Compile every source to an object in parallel (build/<tag>/), then link the shared library."""
    if not force and out == SO and not _stale():
        return SO
    from concurrent.futures import ThreadPoolExecutor
    tag = "release" if not defines else "_".join(d.replace("=", "-") for d in defines)
    odir = os.path.join(ROOT, "build", tag)
    os.makedirs(odir, exist_ok=True)
    cflags = [f for f in FLAGS if f != "-shared"]
    extra = [*(["-Xptxas", "-v"] if verbose else []), *[f"-D{d}" for d in defines]]

    def compile_one(src):
        obj = os.path.join(odir, src.replace(".cu", ".o"))
        r = subprocess.run([NVCC, *cflags, *extra, "-c", "-o", obj, os.path.join(CSRC, src)],
                           capture_output=True, text=True)
        return src, obj, r

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    for src, _, r in results:
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed compiling {src}")
        if verbose:
            sys.stderr.write(r.stderr)
    r = subprocess.run([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", out,
                        *[obj for _, obj, _ in results]], capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libtwopass.so")
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(SO)
