"""Build the native library in-tree: libpdhg_b200.so for sm_100a.

    python -m paper_2603_03150_b200.build        # rebuild if sources changed

The .so lands next to this file (git-ignored, but it travels to the GPU box
with the gpurun snapshot).  nvcc cross-compiles here without a GPU.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libpdhg_b200.so"
SOURCES = [CSRC / "pdhg_b200.cu", CSRC / "ruiz.cu", CSRC / "stdform.cu", CSRC / "finish.cu",
           CSRC / "sell_build.cu"]
# the experiment build adds the PSR builders (measured slower)
EXPERIMENT_SOURCES = [CSRC / "psr_build.cu"]
EXPERIMENT_LIB = ROOT / "tools" / "_libs" / "libpdhg_b200_exp.so"
CHECKED_LIB = ROOT / "tools" / "_libs" / "libpdhg_b200_checked.so"
HEADERS = [ROOT / "include" / "pdhg_b200.h"] + sorted(CSRC.glob("*.cuh"))

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2",
    "-shared",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; cannot build libpdhg_b200.so")


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in SOURCES + EXPERIMENT_SOURCES + HEADERS)


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stderr[-4000:]}")


def build(force: bool = False, verbose: bool = False, defines: tuple = (), out: Path | None = None) -> Path:
    """Compile every source to an object in parallel (one nvcc per file),
    then link the shared library.  ``defines``/``out``: an experiment variant
    (e.g. ("PDHG_L2_HINT=1",)) linked to another path; the product library
    is always the default build."""
    lib = Path(out) if out is not None else LIB
    if not force and out is None and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    experimental = any(d.startswith("PDHG_EXPERIMENTAL") and not d.endswith("=0") for d in defines)
    sources = SOURCES + (EXPERIMENT_SOURCES if experimental else [])
    objdir = PKG / ("_obj" if not defines else "_obj_" + "_".join(d.replace("=", "") for d in defines))
    objdir.mkdir(exist_ok=True)
    lib.parent.mkdir(parents=True, exist_ok=True)
    flags = [f for f in NVCC_FLAGS if f != "-shared"] + [f"-D{d}" for d in defines]
    objs = [objdir / (src.stem + ".o") for src in sources]
    cmds = [[nvcc(), *flags, "-I", str(ROOT / "include"), "-c", str(src), "-o", str(obj)]
            for src, obj in zip(sources, objs)]
    with ThreadPoolExecutor(max_workers=len(cmds)) as ex:
        list(ex.map(lambda c: _run(c, verbose), cmds))
    _run([nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *map(str, objs),
          "-o", str(lib) + ".tmp"], verbose)
    os.replace(str(lib) + ".tmp", lib)
    return lib


if __name__ == "__main__":
    defs = tuple(a[2:] for a in sys.argv[1:] if a.startswith("-D"))
    outs = [a[len("--out="):] for a in sys.argv[1:] if a.startswith("--out=")]
    if "--experimental" in sys.argv:   # PSR + persistent periods + L2 windows, own .so
        defs = defs + ("PDHG_EXPERIMENTAL=1",)
        outs = outs or [str(EXPERIMENT_LIB)]
    if "--checked" in sys.argv:        # device-side bounds checks on every gather / stream load
        defs = defs + ("PDHG_BOUNDS_CHECK=1",)
        outs = outs or [str(CHECKED_LIB)]
    print(build(force="--force" in sys.argv, verbose=True, defines=defs,
                out=Path(outs[0]) if outs else None))
