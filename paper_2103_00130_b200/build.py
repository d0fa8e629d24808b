"""Builds libabftlp_b200.so in-tree with nvcc for sm_100a.

Every translation unit is compiled with ``-gencode arch=compute_100a,code=sm_100a -lineinfo``;
the shared library links the CUDA runtime statically and resolves the driver's
``cuTensorMapEncodeTiled`` at run time, so loading it needs no ``libcuda`` (the CPU test
suite loads it here to check the exported symbols).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
REPO = PKG.parent
CSRC = PKG / "csrc"
BUILD = REPO / "build" / "abftlp"
LIB = PKG / "libabftlp_b200.so"
CLI = PKG / "abft_cli"
SOURCES = ["gemm.cu", "gemv.cu", "locate.cu", "eb.cu", "lab.cu", "quant.cu", "runtime.cu", "campaign.cu", "hostio.cpp", "capi.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the B200 library cannot be built")


def _flags() -> list[str]:
    return ARCH + [
        "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
        "-Xcompiler", "-fPIC,-fvisibility=hidden", "-Xptxas", "-warn-spills",
        "-I", str(REPO / "include"), "-I", str(CSRC),
    ]


def _compile(src: str) -> Path:
    obj = BUILD / (src + ".o")
    srcp = CSRC / src
    deps = [srcp] + list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + list((REPO / "include").glob("*.h"))
    if obj.exists() and obj.stat().st_mtime >= max(d.stat().st_mtime for d in deps):
        return obj
    cmd = [nvcc()] + _flags()
    if src.endswith(".cpp"):
        cmd += ["-x", "cu"]
    cmd += ["-c", str(srcp), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip():
        sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False, jobs: int | None = None) -> Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    if force:
        for o in BUILD.glob("*.o"):
            o.unlink()
    with cf.ThreadPoolExecutor(max_workers=jobs or min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(_compile, SOURCES))
    if not (LIB.exists() and LIB.stat().st_mtime >= max(o.stat().st_mtime for o in objs)):
        tmp = LIB.with_suffix(".so.tmp")
        cmd = [nvcc()] + ARCH + ["-shared", "-o", str(tmp)] + [str(o) for o in objs] + ["-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, LIB)
    build_cli()
    return LIB


def build_cli() -> Path:
    """abft_cli (csrc/cli.cpp): the command-line front end, linked against the library (rpath $ORIGIN)."""
    src = CSRC / "cli.cpp"
    deps = [src, LIB, REPO / "include" / "abftlp.h"]
    if CLI.exists() and CLI.stat().st_mtime >= max(d.stat().st_mtime for d in deps):
        return CLI
    cxx = shutil.which("g++") or "g++"
    cmd = [cxx, "-std=c++17", "-O2", "-I", str(REPO / "include"), str(src), "-o", str(CLI), "-L", str(PKG),
           "-labftlp_b200", "-Wl,-rpath,$ORIGIN"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"abft_cli build failed:\n{r.stdout}\n{r.stderr}")
    return CLI


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
