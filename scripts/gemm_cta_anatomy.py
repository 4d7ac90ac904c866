"""Per-CTA %globaltimer stamps of one persistent tcgen05 GEMM launch (slots:
0 start, 1 setup, 2 first stage landed, 3 first tile's MMAs issued, 4 first
epilogue pass, 5 epilogue done, 6 exit) at the decode's non-split shapes, with
the engine's epilogues (bias, ReLU, fp16 out). Usage: SHAPES=512x3072x1024,..."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2010_13887_b200 as P
from paper_2010_13887_b200 import _abi

lib = _abi.load()
lib.fq_gemm_debug_timestamps.argtypes = [ctypes.c_void_p]
shapes = os.environ.get("SHAPES", "512x3072x1024,512x4096x1024,512x1024x1024")
for sh in shapes.split(","):
    M, N, K = (int(x) for x in sh.split("x"))
    a = torch.randn(M, K, device="cuda").half()
    bs = [torch.randn(N, K, device="cuda").half() for _ in range(4)]
    bias = torch.randn(N, device="cuda")
    c = torch.empty(M, N, device="cuda", dtype=torch.float32 if os.environ.get("F32") else torch.float16)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    clean = torch.ones(64 << 20, dtype=torch.float32, device="cuda")  # read after the fill:
    # evicts the fill's dirty lines, so the GEMM does not pay their write-back
    dbg = torch.zeros(8 * 1024, dtype=torch.int64, device="cuda")
    for i in range(4):
        P.gemm(a, bs[i], c, transpose_b=True, bias=bias, activation="relu")
    for rep in range(3):
        flush.fill_(1)
        if os.environ.get("CLEAN", "1") == "1":
            clean.sum()
        dbg.zero_()
        torch.cuda.synchronize()
        lib.fq_gemm_debug_timestamps(dbg.data_ptr())
        P.gemm(a, bs[rep], c, transpose_b=True, **({} if os.environ.get("PLAIN") else dict(bias=bias, activation="relu")))
        torch.cuda.synchronize()
        lib.fq_gemm_debug_timestamps(None)
        t = dbg.view(-1, 8).cpu()
        t = t[t[:, 0] > 0]
        t0 = int(t[:, 0].min())
        rel = (t - t0).double() / 1e3
        q = lambda i, f: float(rel[:, i][t[:, i] > 0].quantile(f)) if bool((t[:, i] > 0).any()) else -1
        print(f"{sh}: ctas {len(t)} | " + " ".join(
            f"s{i}={q(i, .5):.2f}/{q(i, 1.0):.2f}" for i in range(8)) + "  (median/max us since first CTA)")
