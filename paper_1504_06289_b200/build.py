"""In-tree build of libtgb.so (CUDA, sm_100a) and of the test-only oracle
libraries.  Invoked by __graft_entry__.build(); every artefact is written
inside the repository so it travels to the GPU box with the snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
PKG = ROOT / "paper_1504_06289_b200"
CSRC = PKG / "csrc"
LIB = PKG / "libtgb.so"
ORACLE_DIR = ROOT / "oracle"
ORACLE_LIB = ORACLE_DIR / "build" / "liboracle.so"
REF_LIB = ORACLE_DIR / "_ref" / "libtengrid_ref.so"
REFERENCE = Path("/root/reference/proj")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale(target: Path, sources: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(s.stat().st_mtime > t for s in sources)


def _run(cmd: list[str]) -> None:
    print("+", " ".join(cmd), file=sys.stderr, flush=True)
    subprocess.run(cmd, check=True)


def build_lib(force: bool = False) -> Path:
    """Each source compiles to its own object (in parallel, only when stale),
    then one link; objects live in build/ (git-ignored)."""
    from concurrent.futures import ThreadPoolExecutor

    srcs = sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))
    hdrs = sorted(CSRC.glob("*.hpp")) + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "tgb.h"]
    hdrs += sorted((ROOT / "include" / "tengrid_b200").glob("*.hpp"))
    objdir = ROOT / "build" / "libtgb"
    objdir.mkdir(parents=True, exist_ok=True)
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
             "-Xptxas", "-v" if os.environ.get("TGB_PTXAS_VERBOSE") else "-O3",
             "-I", str(ROOT / "include"), "-I", str(CSRC)]
    objs = [objdir / (s.name + ".o") for s in srcs]
    todo = [(s, o) for s, o in zip(srcs, objs) if force or _stale(o, [s, *hdrs])]

    def compile_one(so):
        s, o = so
        _run([NVCC, *flags, "-c", str(s), "-o", str(o)])

    if todo:
        with ThreadPoolExecutor(max_workers=min(8, len(todo))) as ex:
            list(ex.map(compile_one, todo))
    if not force and not todo and not _stale(LIB, objs):
        return LIB
    tmp = LIB.with_suffix(".so.tmp")
    _run([NVCC, *ARCH, "-shared", *[str(o) for o in objs], "-o", str(tmp)])
    tmp.replace(LIB)
    return LIB


def build_oracle(force: bool = False) -> Path:
    srcs = [ORACLE_DIR / "tengrid_oracle.cpp", ORACLE_DIR / "oracle_capi.cpp"]
    deps = srcs + [ORACLE_DIR / "tengrid_oracle.hpp"]
    if not force and not _stale(ORACLE_LIB, deps):
        return ORACLE_LIB
    ORACLE_LIB.parent.mkdir(parents=True, exist_ok=True)
    _run(["g++", "-O2", "-std=c++20", "-fPIC", "-shared", "-pthread",
          *[str(s) for s in srcs], "-o", str(ORACLE_LIB)])
    return ORACLE_LIB


REF_TUS = ["fft.cpp", "tensor.cpp", "grid.cpp", "kernel.cpp", "basis.cpp", "lattice.cpp", "parallel.cpp",
           "hf.cpp", "tei.cpp", "reduction.cpp", "mp2.cpp"]


def build_ref(force: bool = False) -> Path | None:
    """Compile the reference's own translation units (read in place from
    /root/reference) against oracle/eigen_shim -> oracle/_ref/; the shim's
    dense decompositions come from the restatement's LA (tengrid_oracle.cpp).  Only
    possible where /root/reference exists (this container); the GPU box uses
    the prebuilt library that travels with the snapshot."""
    if not REFERENCE.exists():
        return REF_LIB if REF_LIB.exists() else None
    srcs = [REFERENCE / "src" / t for t in REF_TUS] + [ORACLE_DIR / "ref_capi.cpp", ORACLE_DIR / "ref_support.cpp",
                                                      ORACLE_DIR / "tengrid_oracle.cpp"]
    deps = srcs + sorted((ORACLE_DIR / "eigen_shim" / "Eigen").glob("*")) + [ORACLE_DIR / "tengrid_oracle.hpp"]
    if not all(s.exists() for s in srcs):
        return None
    if not force and not _stale(REF_LIB, deps):
        return REF_LIB
    REF_LIB.parent.mkdir(parents=True, exist_ok=True)
    _run(["g++", "-O2", "-std=c++20", "-fPIC", "-shared", "-pthread", "-w",
          "-I", str(ORACLE_DIR / "eigen_shim"), "-I", str(REFERENCE / "include"),
          *[str(s) for s in srcs], "-o", str(REF_LIB)])
    return REF_LIB


def build_all(force: bool = False) -> None:
    build_lib(force)
    build_oracle(force)
    if (ORACLE_DIR / "ref_capi.cpp").exists():
        build_ref(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
