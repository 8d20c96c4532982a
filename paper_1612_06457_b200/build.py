"""Build the sm_100a CUDA library in-tree (no JIT cache, no torch extension).

    python -m paper_1612_06457_b200.build        # or __graft_entry__.build()

Each ``csrc/*.cu`` is compiled with nvcc for ``sm_100a`` into an object file
(in parallel), then linked into ``paper_1612_06457_b200/lib/libundertext_b200.so``
with the CUDA runtime linked statically, so the library only needs the driver
and shares the caller's streams (plain ``cudaStream_t`` handles) with torch.
The library is stamped with a SHA-256 of its sources (``source_hash()``: every
``csrc/*`` file, ``include/*.h`` and this script, plus the nvcc flags), compiled in
as ``ut_build_hash()``; it is rebuilt whenever the stamp differs from the sources
on disk, and ``_lib`` refuses to load a library whose stamp does not match
(a stale prebuilt ``.so`` can never run against newer sources).
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
OUT_DIR = PKG / "lib"
OBJ_DIR = OUT_DIR / "obj"
LIB = OUT_DIR / "libundertext_b200.so"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the B200 library cannot be built")


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def source_hash() -> str:
    """SHA-256 over the library's sources and build flags (the .so's stamp)."""
    h = hashlib.sha256()
    files = sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + \
        sorted(INCLUDE.glob("*.h")) + [Path(__file__)]
    for f in files:
        h.update(f.name.encode())
        h.update(f.read_bytes())
    h.update(os.environ.get("UT_NVCC_FLAGS", "").encode())
    return h.hexdigest()[:32]


def library_hash(path: Path = LIB) -> str | None:
    """The stamp compiled into a built library (None if absent / unreadable)."""
    if not path.exists():
        return None
    data = path.read_bytes()
    i = data.find(b"UT_SOURCE_HASH=")
    if i < 0:
        return None
    return data[i + 15:i + 47].decode(errors="replace")


def _stale() -> bool:
    return library_hash() != source_hash()


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    nvcc = nvcc_path()
    OBJ_DIR.mkdir(parents=True, exist_ok=True)
    common = [nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-I", str(INCLUDE), "--expt-relaxed-constexpr"]
    if verbose:
        common += ["-Xptxas", "-v"]
    common += os.environ.get("UT_NVCC_FLAGS", "").split()  # e.g. -DUT_PHASES (dev)
    stamp = source_hash()

    def compile_one(src: Path) -> Path:
        obj = OBJ_DIR / (src.stem + ".o")
        cmd = common + ["-c", str(src), "-o", str(obj)]
        if src.stem == "abi":
            cmd.append(f"-DUT_SOURCE_HASH=\"{stamp}\"")
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src.name}:\n{res.stderr}")
        if verbose and res.stderr:
            sys.stderr.write(res.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as pool:
        objs = list(pool.map(compile_one, sources()))
    tmp = LIB.with_suffix(".so.tmp")
    link = [nvcc, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs), "-ldl"]
    res = subprocess.run(link, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    tmp.replace(LIB)
    return LIB


if __name__ == "__main__":
    path = build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(path)
