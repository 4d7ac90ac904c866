"""Exact decoder self-attention (C2 layer shape: 512 rows x 16 heads x 64) vs
the history length: graph-timed us per launch at cur = 0 .. 63 (random pair
cache, identity history)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2010_13887_b200 as P  # noqa: F401
from paper_2010_13887_b200 import _abi

R, H, HD, S = 512, 16, 64, 64
d = H * HD
plane = S * R * d
kc = (torch.randn(2 * plane, device="cuda") * 0.1).half()
vc = (torch.randn(2 * plane, device="cuda") * 0.1).half()
hist = torch.arange(R, dtype=torch.int32, device="cuda")[:, None].repeat(1, S).contiguous()
sqkv = torch.randn(R, 3 * d, device="cuda")
oh = torch.empty(R, d, dtype=torch.float16, device="cuda")
ol = torch.empty_like(oh)
for cur in (0, 15, 16, 31, 32, 47, 63):
    dc = torch.full((1,), cur, dtype=torch.int32, device="cuda")

    def run():
        _abi.call("fq_decoder_self_attention_xh", sqkv.data_ptr(), 3 * d, kc.data_ptr(),
                  vc.data_ptr(), plane, hist.data_ptr(), dc.data_ptr(), R, H, HD, S, 0.125, None,
                  oh.data_ptr(), ol.data_ptr(), d, _abi.stream_handle())
    run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(20):
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
        ts.append(s.elapsed_time(e) / 20 * 1e3)
    ts.sort()
    mb = R * (cur + 1) * d * 2 * 4 / 1e6
    print(f"cur {cur:2d}: {ts[2]:6.1f} us  ({mb:6.1f} MB K/V pairs, {mb / ts[2] * 1e-3:5.2f} TB/s)", flush=True)
