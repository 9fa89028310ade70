"""The numpy model of the band-limited pair path of k12_pair_kernel (tools/proto_k12_pruned.py:
Zs table -> merged 48-point stage per (t0, k2) -> stage 4) against a plain inverse DFT of the
packed spectrum the reference's conv_central_many inverts (proj/src/fft.cpp:97-122).  Pins the
index scheme and twiddles the CUDA path (csrc/fftconv12k.cu, "band-limited pairs") implements."""
import re

import pytest
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("kband", [128, 144])
def test_pruned_transform_model_matches_inverse_dft(kband):
    out = subprocess.run([sys.executable, str(ROOT / "tools" / "proto_k12_pruned.py"), str(kband)], capture_output=True,
                         text=True, timeout=300, check=True).stdout
    err = float(re.search(r"max err ([0-9.eE+-]+)", out).group(1))
    assert err <= 1e-13, out
