"""Build libharmony_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2202_01306_b200.build [-j N] [--force]

Every ``csrc/**/*.cpp`` / ``*.cu`` is compiled to an object under
``build/`` (incremental on mtime, headers included) and linked into
``paper_2202_01306_b200/libharmony_b200.so`` with a static CUDA runtime, so
the library loads in processes that already hold torch's runtime and on
boxes without a toolkit.
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libharmony_b200.so")
BUILD = os.path.join(ROOT, "build", "harmony_b200")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3,-Wall,-Wno-unused-function",
          f"-I{os.path.join(ROOT, 'include')}", f"-I{CSRC}"]
CUFLAGS = ARCH + ["--expt-relaxed-constexpr", "-Xptxas", "-v,-warn-spills"] if os.environ.get(
    "HM_PTXAS_VERBOSE") else ARCH + ["--expt-relaxed-constexpr"]


def nvcc() -> str:
    exe = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(exe):
        raise RuntimeError("nvcc not found")
    return exe


def _headers() -> list[str]:
    return (glob.glob(os.path.join(CSRC, "**", "*.h*"), recursive=True)
            + glob.glob(os.path.join(CSRC, "**", "*.cuh"), recursive=True)
            + glob.glob(os.path.join(ROOT, "include", "*.h")))


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "**", "*.cpp"), recursive=True)
                  + glob.glob(os.path.join(CSRC, "**", "*.cu"), recursive=True))


def _obj(src: str) -> str:
    rel = os.path.relpath(src, CSRC).replace(os.sep, "__")
    return os.path.join(BUILD, rel + ".o")


def _compile(src: str, force: bool) -> tuple[str, str]:
    obj = _obj(src)
    newest_dep = max([os.path.getmtime(src)] + [os.path.getmtime(h) for h in _headers()])
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= newest_dep:
        return obj, ""
    # host planner code: no FMA contraction, so double arithmetic rounds like the reference's Python
    flags = COMMON + (CUFLAGS if src.endswith(".cu") else ARCH + ["-x", "cu", "-Xcompiler", "-ffp-contract=off"])
    cmd = [nvcc()] + flags + ["-c", src, "-o", obj]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src}:\n{' '.join(cmd)}\n{p.stdout}\n{p.stderr}")
    return obj, p.stderr


def build(force: bool = False, jobs: int | None = None, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = sources()
    jobs = jobs or min(8, os.cpu_count() or 4)
    with cf.ThreadPoolExecutor(jobs) as ex:
        results = list(ex.map(lambda s: _compile(s, force), srcs))
    objs = [r[0] for r in results]
    if verbose:
        for _, log in results:
            if log:
                sys.stderr.write(log)
    newest = max(os.path.getmtime(o) for o in objs)
    if force or not os.path.exists(OUT) or os.path.getmtime(OUT) < newest:
        # no -lcuda: driver entry points (cuTensorMapEncodeTiled) are fetched
        # with cudaGetDriverEntryPoint so the library also loads on CPU hosts
        cmd = [nvcc()] + ARCH + ["-shared", "-cudart", "static", "-o", OUT] + objs + [
            "-ldl", "-lpthread", "-lrt"]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"link failed:\n{' '.join(cmd)}\n{p.stdout}\n{p.stderr}")
    return OUT


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=None)
    ap.add_argument("-v", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, jobs=a.j, verbose=a.v))


if __name__ == "__main__":
    main()
