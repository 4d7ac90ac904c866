"""Time the tcgen05 GEMM against cuBLAS (torch.matmul, comparison only) on the
C2 shapes. CUDA events, median of 30, L2 flushed before each launch."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2010_13887_b200 as P

SHAPES = [(512, 1024, 1024), (512, 3072, 1024), (512, 4096, 1024), (512, 1024, 4096),
          (512, 32000, 1024), (8192, 3072, 1024), (8192, 4096, 1024), (8192, 1024, 4096),
          (8192, 12288, 1024)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def t(fn, n=30):
    ts = []
    for _ in range(n):
        flush.fill_(1)
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    return statistics.median(ts)


for M, N, K in SHAPES:
    a = torch.randn(M, K, device="cuda").half()
    b = torch.randn(N, K, device="cuda").half()
    c = torch.empty(M, N, device="cuda")
    c16 = torch.empty(M, N, device="cuda", dtype=torch.float16)
    ours = t(lambda: P.gemm(a, b, c, transpose_b=True))
    ours16 = t(lambda: P.gemm(a, b, c16, transpose_b=True))
    cub = t(lambda: torch.matmul(a, b.t(), out=c16))
    fl = 2 * M * N * K
    print(f"{M:5d}x{N:5d}x{K:5d}  ours(f32 out) {ours:7.1f} us {fl / ours / 1e6:6.0f} TF | "
          f"ours(fp16 out) {ours16:7.1f} us | cuBLAS(fp16 out) {cub:7.1f} us {fl / cub / 1e6:6.0f} TF",
          flush=True)
