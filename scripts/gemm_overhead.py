"""Per-launch time of the tcgen05 GEMM vs K (graph of back-to-back launches):
separates the fixed per-launch cost from the per-byte cost. Also times a
1-thread kernel (fq_step_advance) in the same way as the launch floor."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2010_13887_b200 as P
from paper_2010_13887_b200 import _abi

lib = _abi.load()
lib.fq_gemm_force_plan.argtypes = [ctypes.c_int] * 4
REPS = 24


def graph_time(fn):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(REPS):
            fn()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(5):
        g.replay()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) * 1e3 / (5 * REPS)


cur = torch.zeros(1, dtype=torch.int32, device="cuda")
print(f"empty kernel: {graph_time(lambda: _abi.call('fq_step_advance', cur.data_ptr(), _abi.stream_handle())):.2f} us")
for M, N in [(512, 1024), (128, 1024), (512, 4096)]:
    for plan in [(32, 1, 1, 1), (128, 1, 1, 1), (128, 1, 1, 2), (128, 1, 1, 4)]:
        row = []
        for K in [64, 128, 256, 512, 1024, 2048, 4096]:
            nkb = K // 64
            bn, _, _, sp = plan
            if sp > 1 and ((M // 128) * (N // bn) * sp > 148 or sp > nkb):
                row.append("   -  ")
                continue
            a = torch.randn(M, K, device="cuda").half()
            b = torch.randn(N, K, device="cuda").half()
            c = torch.empty(M, N, device="cuda")
            lib.fq_gemm_force_plan(*plan)
            t = graph_time(lambda: P.gemm(a, b, c, transpose_b=True))
            row.append(f"{t:6.2f}")
        lib.fq_gemm_force_plan(0, 0, 0, 1)
        print(f"M={M} N={N} bn={plan[0]} split={plan[3]}: K=64..4096 us: " + " ".join(row), flush=True)
