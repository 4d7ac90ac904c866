"""Graph-timed exact-mode (3xFP16) GEMM shapes of a C2 request, in isolation:
per-launch us, TFLOP/s against the 3-MMA peak, and the bytes each CTA streams."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2010_13887_b200 as P  # noqa: F401
from paper_2010_13887_b200 import _abi
from paper_2010_13887_b200.model import XHWeight
from paper_2010_13887_b200.tensor import split_pair

peak = json.load(open("MEASURED_PEAKS.json"))["bf16_tflops_sustained"] / 3 if os.path.exists(
    "MEASURED_PEAKS.json") else 474.0
shapes = [("QKV", 512, 3072, 1024, 0), ("FFN1", 512, 4096, 1024, 0), ("cross-q", 512, 1024, 1024, 0),
          ("self-out slab", 512, 1024, 1024, 1), ("FFN2 slab", 512, 1024, 4096, 1),
          ("logits", 512, 32000, 1024, 0), ("enc QKV", 8192, 3072, 1024, 0),
          ("enc out", 8192, 1024, 1024, 0), ("enc FFN1", 8192, 4096, 1024, 0),
          ("enc FFN2", 8192, 1024, 4096, 0), ("cross-KV", 8192, 12288, 1024, 0)]
for name, M, N, K, slab in shapes:
    a = [split_pair(torch.randn(M, K, device="cuda")) for _ in range(2)]
    w = XHWeight.from_kn(torch.randn(N, K, device="cuda") * 0.03, transpose=False)
    out = torch.empty(M, N, device="cuda")
    ws = torch.empty(4 * M * N, device="cuda")
    bias = torch.zeros(N, device="cuda")
    res = torch.zeros(M, N, device="cuda")
    g1 = torch.ones(N, device="cuda")
    it = [0]

    def run():
        ap = a[it[0] % 2]
        it[0] += 1
        if slab:
            _abi.call("fq_gemm_x3h_ln", ap[0].data_ptr(), ap[1].data_ptr(), K, w.hi.data_ptr(),
                      w.lo.data_ptr(), K, bias.data_ptr(), res.data_ptr(), N, g1.data_ptr(),
                      bias.data_ptr(), 1e-5, out.data_ptr(), N, None, None, 0, ws.data_ptr(),
                      ws.numel() * 4, M, N, K, _abi.stream_handle())
        else:
            _abi.call("fq_gemm_x3h", ap[0].data_ptr(), ap[1].data_ptr(), K, w.hi.data_ptr(),
                      w.lo.data_ptr(), K, out.data_ptr(), N, M, N, K, 0, None, None, 0, 0,
                      _abi.stream_handle())
    reps = 20
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
    us = sorted(ts)[2]
    tf = 2 * M * N * K / us / 1e6
    print(f"{name:14s} {M:5d}x{N:5d}x{K:5d} {'slab+LN' if slab else '':8s} {us:8.1f} us "
          f"{tf:7.1f} TF/s  {tf / peak:5.2f} of 3xFP16 peak", flush=True)
