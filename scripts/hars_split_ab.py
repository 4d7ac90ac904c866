"""A/B of the two stage-1 layouts (FQ_HARS_SPLIT=0: CTA per row, 1: balanced
split) over the HARS microbench shape range; graph-timed us per call."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
sys.argv = ["x"]
from paper_2010_13887_b200 import decode as D
import bench
res = []
for Vs, beam_s, batch_s in ((32000, 1, 64), (32000, 4, 32), (32000, 4, 64), (50256, 4, 32), (128000, 4, 32), (250000, 4, 16), (250000, 1, 1), (32000, 4, 128)):
    Rs = beam_s * batch_s
    Ls = [torch.randn(Rs, Vs, device="cuda") for _ in range(3)]
    hks = torch.full((Rs,), 2 * beam_s, dtype=torch.int32, device="cuda")
    bufs = (None, None, torch.empty(Rs, dtype=torch.float64, device="cuda"), torch.empty(Rs, Vs, dtype=torch.int32, device="cuda"), torch.empty(Rs, dtype=torch.int64, device="cuda"))
    row = [Vs, beam_s, batch_s]
    for sp in ("0", "1"):
        os.environ["FQ_HARS_SPLIT"] = sp
        js = [0]
        def f():
            D.retrieve_device(Ls[js[0] % 3], 2 * beam_s, d_k=hks, out=bufs); js[0] += 1
        row.append(round(bench.graph_time(f, reps=6) * 1e6, 2))
    print(row, flush=True)
