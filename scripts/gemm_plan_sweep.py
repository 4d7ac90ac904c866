"""Empirical (BN, cm, cn) sweep of the tcgen05 GEMM per shape (benchmark aid)."""
import ctypes
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2010_13887_b200 as P
from paper_2010_13887_b200 import _abi

lib = _abi.load()
lib.fq_gemm_force_plan.argtypes = [ctypes.c_int] * 4
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
shapes = [(512, 1024, 1024), (512, 4096, 1024), (512, 1024, 4096), (512, 32000, 1024),
          (8192, 4096, 1024)]
plans = [(bn, 1, 1, 1) for bn in (32, 64, 128, 256)]
plans += [(bn, 1, 1, s) for bn in (64, 128, 256) for s in (2, 3, 4, 6, 8)]
for M, N, K in shapes:
    a = torch.randn(M, K, device="cuda").half()
    b = torch.randn(N, K, device="cuda").half()
    c = torch.empty(M, N, device="cuda")
    res = []
    for bn, cm, cn, sp in plans:
        mt, nt = (M + 127) // 128, (N + bn - 1) // bn
        nkb = (K + 63) // 64
        kbs = -(-nkb // sp)
        if sp > 1 and (mt * nt * sp > 148 or (sp - 1) * kbs >= nkb):
            continue
        lib.fq_gemm_force_plan(bn, cm, cn, sp)
        ts = []
        for _ in range(12):
            flush.fill_(1)
            s, e = torch.cuda.Event(True), torch.cuda.Event(True)
            s.record()
            P.gemm(a, b, c, transpose_b=True)
            e.record()
            e.synchronize()
            ts.append(s.elapsed_time(e) * 1e3)
        res.append((statistics.median(ts), bn, cm, sp))
    lib.fq_gemm_force_plan(0, 0, 0, 1)
    bn_, cm_, cn_, sp_ = (ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int())
    lib.fq_gemm_plan(M, N, K, ctypes.byref(bn_), ctypes.byref(cm_), ctypes.byref(cn_), ctypes.byref(sp_))
    print(f"   auto plan: bn{bn_.value} split{sp_.value}")
    res.sort()
    print(f"{M}x{N}x{K}: " + "  ".join(f"{t:.1f}us(bn{bn},s{cn})" for t, bn, cm, cn in res[:8]),
          flush=True)
    print("      worst: " + "  ".join(f"{t:.1f}us(bn{bn},s{cn})" for t, bn, cm, cn in res[-3:]))
