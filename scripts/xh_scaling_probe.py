"""Is the decode-shape exact GEMM bound per SM or chip-wide (L2)? Same per-CTA
work (128 rows x tile x K), different numbers of CTAs: graph-timed us."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2010_13887_b200 as P  # noqa: F401
from paper_2010_13887_b200 import _abi
from paper_2010_13887_b200.model import XHWeight
from paper_2010_13887_b200.tensor import split_pair


def t_gemm(M, N, K, reps=20):
    a = [split_pair(torch.randn(M, K, device="cuda")) for _ in range(2)]
    ws = [XHWeight.from_kn(torch.randn(N, K, device="cuda") * 0.03, transpose=False) for _ in range(4)]
    out = torch.empty(M, N, device="cuda")
    it = [0]

    def run():
        ap, w = a[it[0] % 2], ws[it[0] % 4]
        it[0] += 1
        _abi.call("fq_gemm_x3h", ap[0].data_ptr(), ap[1].data_ptr(), K, w.hi.data_ptr(),
                  w.lo.data_ptr(), K, out.data_ptr(), N, M, N, K, 0, None, None, 0, 0,
                  _abi.stream_handle())
    run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            run()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        g.replay()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e) / reps * 1e3)
    return sorted(ts)[2]


for M, N in ((256, 3072), (512, 3072), (256, 1536), (512, 1536), (256, 768), (512, 768)):
    print(f"M={M} N={N} K=1024: {t_gemm(M, N, 1024):6.1f} us", flush=True)
for M, N in ((256, 1024), (512, 1024)):  # split-K x4 (DSMEM)
    print(f"split M={M} N={N} K=1024: {t_gemm(M, N, 1024):6.1f} us", flush=True)
