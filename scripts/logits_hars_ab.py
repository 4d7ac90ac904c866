"""Graph-timed A/B of the decode step's output layer at C2 (512 rows, V=32000,
d=1024, fp16): materialised logits GEMM + fq_hars_step vs fq_logits_hars
(statistics epilogue) + fq_hars_merge_step, each kernel alone and together."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_2010_13887_b200 as P
from paper_2010_13887_b200 import _abi, decode as D

B, K, V, S, d = 128, 4, 32000, 64, 1024
R = B * K
g = torch.Generator(device="cuda").manual_seed(0)
E = (torch.randn(V, d, device="cuda", generator=g) * 0.05).half()
xs = [torch.randn(R, d, device="cuda", generator=g).half() for _ in range(3)]
logits = torch.empty(R, V, device="cuda")
ldt = (V + 223) // 224
dk = torch.full((R,), 8, dtype=torch.int32, device="cuda")
gmax = torch.full((R, 32), -2139095041, dtype=torch.int32, device="cuda")
tmax = torch.zeros(R, ldt, device="cuda")
tsum = torch.zeros(R, ldt, dtype=torch.float64, device="cuda")
svc = torch.zeros(R, ldt, dtype=torch.int32, device="cuda")
sv = torch.zeros(R, ldt, 128, 2, dtype=torch.int32, device="cuda")
it = [0]


def gemm():
    P.gemm(xs[it[0] % 3], E, logits, transpose_b=True)
    it[0] += 1


def lh():
    _abi.call("fq_logits_hars", xs[it[0] % 3].data_ptr(), d, E.data_ptr(), d, R, V, d,
              dk.data_ptr(), gmax.data_ptr(), tmax.data_ptr(), tsum.data_ptr(), ldt,
              svc.data_ptr(), sv.data_ptr(), 128, _abi.stream_handle())
    it[0] += 1
    gmax.fill_(-2139095041)


def resets():
    gmax.fill_(-2139095041)


t_gemm = bench.graph_time(gemm)
t_lh = bench.graph_time(lh) - bench.graph_time(resets)
lh()
torch.cuda.synchronize()
print(f"logits GEMM {t_gemm * 1e6:.1f} us | fq_logits_hars {t_lh * 1e6:.1f} us | "
      f"survivors per tile-row mean {float(svc.float().mean()):.1f} max {int(svc.max())}")
