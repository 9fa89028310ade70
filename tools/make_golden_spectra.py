"""Config-1 fixture for TuckerResult::mode_singular_values: the reference's own
rhosvd (oracle/_ref: /root/reference/proj/src/reduction.cpp on the shim LA) of
the unreduced config-1 density Theta (n=2049, rank 12,800), all three modes.
Test infrastructure (tests/test_spectrum_gpu.py); run here, where the reference
exists:  python tools/make_golden_spectra.py"""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
import paper_1504_06289_b200 as tg  # noqa: E402
from paper_1504_06289_b200.inputs import basis_case, occupied_coefficients  # noqa: E402


def main():
    from paper_1504_06289_b200 import build

    build.build_ref()
    assert O.rlib() is not None
    bs, rng = basis_case(1)
    disc = tg.discretize_basis(bs)
    c_occ = occupied_coefficients(rng, len(disc), 8)
    theta = tg.CanonicalTensor3.zero(disc[0].extents())
    for a in range(8):
        phi = tg.orbital_tensor(disc, c_occ[:, a])
        theta = tg.add(theta, tg.scale(tg.hadamard(phi, phi), 2.0))
    rt = O.OCP.from_cp(theta, lib=O.rlib())
    out = {}
    for ax in range(3):
        t0 = time.perf_counter()
        out[f"sigma{ax}"] = O.ref_mode_sigma(rt, ax, eps=1e-6, mode=0)
        print(f"mode {ax}: {len(out[f'sigma{ax}'])} values in {time.perf_counter() - t0:.1f} s", flush=True)
    np.savez_compressed(ROOT / "tests" / "golden" / "reference_cfg1_spectra.npz", rank=np.array(theta.rank()), **out)


if __name__ == "__main__":
    main()
