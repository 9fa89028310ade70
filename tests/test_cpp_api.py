"""The C++ drop-in header (include/tengrid_b200/tengrid.hpp) compiles against
Eigen-layout containers and links libtgb (CPU); on a GPU it reproduces the
reference semantics (delta identity, weights, scalar product, errors)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
EXE = ROOT / "tests" / "cpp" / "test_cpp_api.bin"


def build_exe():
    src = ROOT / "tests" / "cpp" / "test_cpp_api.cpp"
    if EXE.exists() and EXE.stat().st_mtime > max(src.stat().st_mtime,
                                                   (ROOT / "paper_1504_06289_b200" / "libtgb.so").stat().st_mtime):
        return
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", str(ROOT / "include"), "-I", str(ROOT / "oracle" / "eigen_shim"),
                    str(src), "-L", str(ROOT / "paper_1504_06289_b200"), "-ltgb",
                    f"-Wl,-rpath,{ROOT / 'paper_1504_06289_b200'}", "-o", str(EXE)], check=True)


def test_cpp_header_compiles_and_links():
    build_exe()
    assert EXE.exists()


@pytest.mark.gpu
def test_cpp_header_runs_on_gpu():
    build_exe()
    r = subprocess.run([str(EXE)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
