"""Per-launch time of the tcgen05 GEMM inside a CUDA graph of back-to-back
launches (no Python in the timed region): 'cold' rotates through enough weight
buffers to exceed L2 (each launch streams its weights from HBM, as in a decode
step), 'warm' reuses one. Benchmark aid for the dispatcher's plan table."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2010_13887_b200 as P
from paper_2010_13887_b200 import _abi

lib = _abi.load()
lib.fq_gemm_force_plan.argtypes = [ctypes.c_int] * 4
shapes = [(512, 1024, 1024), (512, 3072, 1024), (512, 4096, 1024), (512, 1024, 4096),
          (512, 32000, 1024), (8192, 4096, 1024)]
plans = [(32, 1, 1, 1), (64, 1, 1, 1), (128, 1, 1, 1), (256, 1, 1, 1), (32, 1, 8, 1), (32, 2, 4, 1), (64, 1, 4, 1)]
plans += [(bn, 1, 1, s) for bn in (64, 128, 256) for s in (2, 4, 8)]
REPS = 24


def run(M, N, K, plan, cold):
    nbuf = max(1, min(REPS, (200 << 20) // (N * K * 2) + 1)) if cold else 1
    a = torch.randn(M, K, device="cuda").half()
    bs = [torch.randn(N, K, device="cuda").half() for _ in range(nbuf)]
    c = torch.empty(M, N, device="cuda")
    lib.fq_gemm_force_plan(*plan)
    P.gemm(a, bs[0], c, transpose_b=True)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(REPS):
            P.gemm(a, bs[i % nbuf], c, transpose_b=True)
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(3):
        g.replay()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) * 1e3 / (3 * REPS)


for M, N, K in shapes:
    line = []
    for plan in plans:
        bn, _, _, sp = plan
        mt, nt, nkb = (M + 127) // 128, (N + bn - 1) // bn, (K + 63) // 64
        if sp > 1 and (mt * nt * sp > 148 or (sp - 1) * (-(-nkb // sp)) >= nkb):
            continue
        if M >= 4096 and bn < 128:
            continue
        line.append((run(M, N, K, plan, True), run(M, N, K, plan, False), plan))
    lib.fq_gemm_force_plan(0, 0, 0, 1)
    line.sort()
    print(f"{M}x{N}x{K}  cold/warm us: " +
          "  ".join(f"{c:.1f}/{w:.1f}(bn{p[0]},s{p[3]})" for c, w, p in line[:6]), flush=True)
