"""Builds libgdgpu.so in-tree with nvcc for sm_100a (B200) only."""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
BUILD = PKG / "_build_obj"
LIB = PKG / "libgdgpu.so"
SOURCES = ("gd_build.cu", "gd_count.cu", "gd_parse.cu", "gd_derive.cu", "gd_rank.cu",
           "gd_select.cu", "gd_copy.cu", "gd_api.cu")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "-Xcompiler", "-fopenmp",
    "--expt-relaxed-constexpr",
    f"-I{PKG.parent / 'include'}",
]


def _needs(obj: Path, deps) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False, force: bool = False, defines=(), lib: Path = LIB,
          objdir: Path = BUILD) -> Path:
    """Compile the library; `defines` (-DNAME=V) build an experiment variant
    into `lib` / `objdir` (tools/build_variant.py)."""
    LIB, BUILD = lib, objdir
    BUILD.mkdir(parents=True, exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "gd_api.h"]
    jobs = []
    for src in SOURCES:
        obj = BUILD / (Path(src).stem + ".o")
        if force or _needs(obj, [CSRC / src] + headers):
            jobs.append([NVCC, *FLAGS, *defines, "-Xptxas", "-v" if verbose else "-O3",
                         "-c", str(CSRC / src), "-o", str(obj)])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose:
            sys.stderr.write(r.stderr)

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        list(ex.map(run, jobs))
    objs = [BUILD / (Path(s).stem + ".o") for s in SOURCES]
    if force or jobs or not LIB.exists():
        tmp = LIB.with_suffix(".so.tmp")
        cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a",
               *map(str, objs), "-o", str(tmp), "-lcudart_static", "-lrt", "-ldl", "-lpthread", "-lgomp"]
        run(cmd)
        os.replace(tmp, LIB)
    build_hostpack(force)
    return LIB


def hostpack_path() -> Path:
    import sysconfig
    return PKG / ("_hostpack" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_hostpack(force: bool = False) -> Path:
    """The CPython helper that gathers per-graph array pointers for batches
    (csrc/hostpack.c): plain gcc against this interpreter's headers."""
    import sysconfig
    src, out = CSRC / "hostpack.c", hostpack_path()
    if force or _needs(out, [src]):
        tmp = out.with_suffix(".tmp")
        cmd = [os.environ.get("CC", "gcc"), "-O2", "-shared", "-fPIC", "-fvisibility=hidden",
               f"-I{sysconfig.get_paths()['include']}", str(src), "-o", str(tmp)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"gcc failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
