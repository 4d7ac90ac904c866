"""Decode GEMM shapes with the decode step's real epilogues (bias / ReLU /
residual, fp16 or fp32 output), graph-timed, vs the plain GEMM: how much the
fused epilogue costs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2010_13887_b200 as P

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import graph_time  # noqa: E402

for (M, N, K, kind) in [(512, 4096, 1024, "ffn1"), (512, 3072, 1024, "qkv"),
                        (512, 1024, 1024, "out"), (512, 1024, 4096, "ffn2")]:
    a = torch.randn(M, K, device="cuda").half()
    bs = [torch.randn(N, K, device="cuda").half() for _ in range(16)]
    bias = torch.randn(N, device="cuda")
    res = torch.randn(M, N, device="cuda")
    c32 = torch.empty(M, N, device="cuda")
    c16 = torch.empty(M, N, device="cuda", dtype=torch.float16)
    it = [0]

    def plain():
        it[0] += 1
        P.gemm(a, bs[it[0] % 16], c32, transpose_b=True)

    def real():
        it[0] += 1
        b = bs[it[0] % 16]
        if kind == "ffn1":
            P.gemm(a, b, c16, transpose_b=True, bias=bias, activation="relu")
        elif kind == "qkv":
            P.gemm(a, b, c32, transpose_b=True, bias=bias)
        else:
            P.gemm(a, b, c32, transpose_b=True, bias=bias, residual=res)
    print(f"{kind} {M}x{N}x{K}: plain {graph_time(plain) * 1e6:.2f} us, "
          f"real epilogue {graph_time(real) * 1e6:.2f} us", flush=True)
