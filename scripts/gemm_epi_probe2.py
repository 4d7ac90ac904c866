import os, sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2010_13887_b200 as P
from bench import graph_time
M, N, K = 512, 4096, 1024
a = torch.randn(M, K, device="cuda").half()
bs = [torch.randn(N, K, device="cuda").half() for _ in range(16)]
bias = torch.randn(N, device="cuda")
c32 = torch.empty(M, N, device="cuda")
c16 = torch.empty(M, N, device="cuda", dtype=torch.float16)
it = [0]
def mk(out, **kw):
    def f():
        it[0] += 1
        P.gemm(a, bs[it[0] % 16], out, transpose_b=True, **kw)
    return f
for name, f in [("plain fp32", mk(c32)), ("plain fp16", mk(c16)), ("bias fp32", mk(c32, bias=bias)),
                ("bias+relu fp32", mk(c32, bias=bias, activation="relu")),
                ("bias fp16", mk(c16, bias=bias)), ("bias+relu fp16", mk(c16, bias=bias, activation="relu"))]:
    print(f"{name:16s} {graph_time(f) * 1e6:.2f} us", flush=True)
