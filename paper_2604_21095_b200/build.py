"""Build the in-tree C-ABI library `_lib/libpanelgwas_b200.so` with nvcc.

Every kernel is compiled for sm_100a only (`-gencode arch=compute_100a,code=sm_100a`)
with `-lineinfo` so ncu source pages map back to csrc/. nvcc cross-compiles without
a GPU, so this runs on the CPU build box; the .so travels to the GPU box in-tree.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
REPO = PKG_DIR.parent
CSRC = PKG_DIR / "csrc"
LIB_DIR = PKG_DIR / "_lib"
LIB_NAME = "libpanelgwas_b200.so"
LIB_PATH = LIB_DIR / LIB_NAME
HEADER = REPO / "include" / "panelgwas_b200.h"

ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-lineinfo",
    "-Xcompiler", "-fPIC",
    "-Xcompiler", "-fvisibility=hidden",
    "--expt-relaxed-constexpr",
    "-Xptxas", "-warn-spills",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build panelgwas_b200")


# per-file extra flags: the Student-t code follows numpy's operation order, so no FMA contraction
FILE_FLAGS = {"pstats.cu": ["-fmad=false"]}


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _stale() -> bool:
    if not LIB_PATH.exists():
        return True
    built = LIB_PATH.stat().st_mtime
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + [HEADER, Path(__file__)]
    return any(p.stat().st_mtime > built for p in deps)


def build(force: bool = False, verbose: bool = False, jobs: int | None = None) -> Path:
    """Compile csrc/*.cu into the shared library (object files cached in build/).

    Processes that find the library stale at the same time (the ranks of a torchrun job)
    serialise on a lock file; the later ones see the fresh library and return."""
    if not force and not _stale():
        return LIB_PATH
    import fcntl

    (REPO / "build").mkdir(parents=True, exist_ok=True)
    with open(REPO / "build" / ".lock", "w") as lock:
        fcntl.flock(lock, fcntl.LOCK_EX)
        if not force and not _stale():
            return LIB_PATH
        return _build_locked(force, verbose)


def _build_locked(force: bool, verbose: bool) -> Path:
    nvcc = _nvcc()
    obj_dir = REPO / "build" / "obj"
    obj_dir.mkdir(parents=True, exist_ok=True)
    LIB_DIR.mkdir(parents=True, exist_ok=True)
    include = ["-I", str(REPO / "include"), "-I", str(CSRC)]
    headers = list(CSRC.glob("*.cuh")) + [HEADER]
    newest_header = max(p.stat().st_mtime for p in headers)
    procs = []
    objs = []
    for src in sources():
        obj = obj_dir / (src.stem + ".o")
        objs.append(obj)
        if (not force and obj.exists() and obj.stat().st_mtime > src.stat().st_mtime
                and obj.stat().st_mtime > newest_header):
            continue
        cmd = [nvcc, *ARCH_FLAGS, *NVCC_FLAGS, *FILE_FLAGS.get(src.name, []), *include, "-c", str(src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    failed = []
    for src, p in procs:
        out, _ = p.communicate()
        text = out.decode(errors="replace")
        if p.returncode != 0:
            failed.append((src, text))
        elif verbose and text.strip():
            print(text)
    if failed:
        msg = "\n".join(f"--- {s.name}\n{t}" for s, t in failed)
        raise RuntimeError(f"nvcc failed:\n{msg}")
    tmp = LIB_PATH.with_suffix(".so.tmp")
    link = [nvcc, *ARCH_FLAGS, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs), "-lz", "-lrt",
            "-ldl", "-lpthread"]
    if verbose:
        print(" ".join(link), flush=True)
    res = subprocess.run(link, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


if __name__ == "__main__":
    path = build(force="--force" in sys.argv, verbose=True)
    print(path)
