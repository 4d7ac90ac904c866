"""One stage-1 call at the C2 decode shape (512 x 32000, k = 8 per row) after
warm-up: the target of the HARS ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2010_13887_b200 import decode as D

R, V = 512, 32000
lgs = [torch.randn(R, V, device="cuda") for _ in range(3)]
hk = torch.full((R,), 8, dtype=torch.int32, device="cuda")
for i in range(6):
    D.retrieve_device(lgs[i % 3], 8, d_k=hk)
torch.cuda.synchronize()
