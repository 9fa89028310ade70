"""tgb_dgemm throughput on the reduction's shapes vs torch (cuBLAS) FP64."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_1504_06289_b200 as tg  # noqa: E402
from paper_1504_06289_b200._lib import check, lib  # noqa: E402

stream = torch.cuda.Stream()
ctx = tg.Context(0, stream=stream.cuda_stream)
shapes = [  # (ta, tb, M, N, K)
    (0, 0, 2049, 96, 12800), (1, 0, 12800, 96, 2049), (1, 0, 96, 96, 2049), (0, 0, 2049, 2950, 12800),
    (1, 0, 53, 12800, 2049), (0, 1, 53, 2950, 12800), (1, 0, 50, 2950, 2049), (0, 0, 4097, 4097, 4097),
    (1, 0, 32768, 820, 2049), (1, 0, 22882, 820, 2049),
]
for ta, tb, M, N, K in shapes:
    A = torch.randn((K, M) if ta else (M, K), dtype=torch.float64, device="cuda").t().contiguous().t()
    B = torch.randn((N, K) if tb else (K, N), dtype=torch.float64, device="cuda").t().contiguous().t()
    C = torch.empty((M, N), dtype=torch.float64, device="cuda").t().contiguous().t()
    lda, ldb = A.stride(1), B.stride(1)
    def run():
        check(lib().tgb_dgemm(ctx.handle, ta, tb, M, N, K, 1.0, A.data_ptr(), lda, B.data_ptr(), ldb, 0.0,
                              C.data_ptr(), M))
    with torch.cuda.stream(stream):
        run()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(5):
            run()
        e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    Am = A.t() if ta else A
    Bm = B.t() if tb else B
    torch.matmul(Am, Bm)
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    for _ in range(5):
        torch.matmul(Am, Bm)
    f1.record()
    torch.cuda.synchronize()
    ms_t = f0.elapsed_time(f1) / 5
    fl = 2.0 * M * N * K
    print(f"ta={ta} tb={tb} M={M} N={N} K={K}: tgb {ms:.3f} ms {fl / ms / 1e9:.1f} TF | cublas {ms_t:.3f} ms {fl / ms_t / 1e9:.1f} TF")
