"""Generate tests/golden/reference_cfg2_vh_samples.npz: config 2's Hartree
potential (n = 16385, R_f = 500, R_N = 41) at the 10^4 seeded sample points,
computed by the REFERENCE's own code (oracle/_ref: proj/src/fft.cpp
conv_central_many + the convolve/hartree_potential weight and h scaling of
tensor.cpp:179-198 / hf.cpp:131-138), without materialising the 8 GB of
factors (ref_hartree_samples in oracle/ref_capi.cpp).

The kernel factors come from the reference's own kernel_tensor
(kernel.cpp:182-203) and are asserted bitwise equal to the inputs the
product path uses (paper_1504_06289_b200.inputs.hartree_case).

Run here (where /root/reference exists):  python tools/make_golden_cfg2.py
The fixture is committed; tests/test_conv_gpu.py and bench.py gate the
benchmarked path against it (1e-10 relative max-norm).
"""
from __future__ import annotations

import ctypes as C
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from paper_1504_06289_b200.inputs import KERNEL_C0, KERNEL_M, hartree_case  # noqa: E402

OUT = ROOT / "tests" / "golden" / "reference_cfg2_vh_samples.npz"


def main(nsamples: int = 10_000):
    from paper_1504_06289_b200 import build

    build.build_ref()
    R = O.rlib()
    assert R is not None, "oracle/_ref not built (needs /root/reference)"
    case = hartree_case(2, nsamples=nsamples)
    n = case.grid.n[0]
    # the reference's own kernel producer
    kt = O.OCP(lib=R)
    b = np.array(case.grid.b_half, dtype=np.float64)
    nn = (C.c_longlong * 3)(*case.grid.n)
    rc = R.ref_kernel_tensor(C.c_void_p(b.ctypes.data), nn, C.c_longlong(KERNEL_M[2]), C.c_double(KERNEL_C0[2]),
                             C.c_int(0), kt.h)
    assert rc == 0, R.ref_last_error().decode()
    for ax in range(3):
        assert np.array_equal(kt.factors()[ax], case.kernel.tensor.factor[ax]), "kernel producer mismatch"
    assert np.array_equal(kt.weight(), case.kernel.tensor.weight)
    th = O.OCP.from_cp(case.theta, lib=R)
    h = np.ascontiguousarray(np.asarray(case.grid.h, dtype=np.float64))
    pts = np.ascontiguousarray(case.samples.astype(np.int64))
    out = np.zeros(pts.shape[0])
    threads = int(os.environ.get("THREADS", os.cpu_count() or 1))
    t0 = time.perf_counter()
    rc = R.ref_hartree_samples(th.h, kt.h, C.c_void_p(h.ctypes.data), C.c_longlong(pts.shape[0]),
                               C.c_void_p(pts.ctypes.data), C.c_int(threads), C.c_void_p(out.ctypes.data))
    assert rc == 0, R.ref_last_error().decode()
    el = time.perf_counter() - t0
    print(f"config 2 V_H at {pts.shape[0]} points: {el:.1f} s on {threads} threads; "
          f"range [{out.min():.6e}, {out.max():.6e}]")
    np.savez_compressed(OUT, samples=pts, vh=out, n=n, ra=case.theta.rank(), rb=case.kernel.rank(),
                        generator="tools/make_golden_cfg2.py (oracle/_ref: reference fft.cpp/tensor.cpp/hf.cpp)")
    print("wrote", OUT)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 10_000)
