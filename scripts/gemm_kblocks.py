"""Per-k-block producer-issue / data-arrival timestamps of CTA 0 (benchmark aid)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2010_13887_b200 as P
from paper_2010_13887_b200 import _abi

lib = _abi.load()
lib.fq_gemm_debug_timestamps.argtypes = [ctypes.c_void_p]
lib.fq_gemm_force_plan.argtypes = [ctypes.c_int] * 3
dbg = torch.zeros(600, dtype=torch.int64, device="cuda")
for (M, N, K, plan) in [(512, 1024, 1024, (32, 1, 1)), (512, 4096, 1024, (128, 1, 1)),
                        (512, 4096, 1024, (32, 1, 1)), (128, 128, 64, (128, 1, 1))]:
    a = torch.randn(M, K, device="cuda").half()
    b = torch.randn(N, K, device="cuda").half()
    c = torch.empty(M, N, device="cuda")
    lib.fq_gemm_force_plan(*plan)
    for _ in range(3):
        dbg.zero_()
        lib.fq_gemm_debug_timestamps(dbg.data_ptr())
        P.gemm(a, b, c, transpose_b=True)
        torch.cuda.synchronize()
        lib.fq_gemm_debug_timestamps(None)
    t = dbg.cpu().tolist()
    t0 = t[0]
    nkb = (K + 63) // 64
    tiles = sum(1 for i in range(1, 8, 2) if t[i])
    print(f"== {M}x{N}x{K} plan {plan}: tiles(CTA0)={tiles}")
    for tl in range(tiles):
        print(f"   tile {tl}: acc ready {(t[1 + 2 * tl] - t0) / 1e3:.2f}  epi done {(t[2 + 2 * tl] - t0) / 1e3:.2f} us")
    its = [i for i in range(160) if t[8 + 3 * i]]
    print("   issue : " + " ".join(f"{(t[8 + 3 * i] - t0) / 1e3:.2f}" for i in its[:40]))
    print("   arrive: " + " ".join(f"{(t[9 + 3 * i] - t0) / 1e3:.2f}" for i in its[:40]))
lib.fq_gemm_force_plan(0, 0, 0)
