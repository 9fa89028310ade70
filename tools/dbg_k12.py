"""Debug: n = 16385 convolution of a few columns through the k12 plan vs the oracle; prints mismatch ranges."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np
import paper_1504_06289_b200 as tg
from paper_1504_06289_b200 import CanonicalTensor3, convolve
from oracle import oracle as O

ra = int(sys.argv[1]) if len(sys.argv) > 1 else 2
rb = int(sys.argv[2]) if len(sys.argv) > 2 else 1
n = 16385
rng = np.random.default_rng(5)
fa = [np.asfortranarray(rng.normal(size=(n, ra))) for _ in range(3)]
x = np.arange(n) - 0.5 * (n - 1)
fb = [np.asfortranarray(np.stack([np.exp(-(x / (300.0 * (j + 1))) ** 2) for j in range(rb)], axis=1)) for _ in range(3)]
ctx = tg.Context(0)
c = convolve(CanonicalTensor3(fa, np.ones(ra)), CanonicalTensor3(fb, np.ones(rb)), (1.0, 1.0, 1.0), ctx)
for ax in range(1):
    for i in range(ra):
        for j in range(rb):
            ref = O.conv_central_many(np.asfortranarray(fa[ax][:, [i]]), np.ascontiguousarray(fb[ax][:, j]))[:, 0]
            got = c.factor[ax][:, i + ra * j]
            bad = np.nonzero(np.abs(got - ref) > 1e-9 * np.abs(ref).max())[0]
            print("col", i, j, "bad", bad.size, "max err", np.abs(got - ref).max() / np.abs(ref).max())
            if bad.size:
                # contiguous ranges
                brk = np.nonzero(np.diff(bad) > 1)[0]
                starts = np.r_[bad[0], bad[brk + 1]]
                ends = np.r_[bad[brk], bad[-1]]
                print("  ranges:", [(int(s), int(e)) for s, e in zip(starts[:24], ends[:24])], "count", starts.size)
                k = bad[0]
                print("  first bad", k, got[k:k+4], ref[k:k+4])
