"""One HARS stage-1 launch at the C2 decode shape (512 x 32000 fp32, k = 8 via
d_k) for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2010_13887_b200 import decode as D

R, V = 512, 32000
lg = torch.randn(R, V, device="cuda")
hk = torch.full((R,), 8, dtype=torch.int32, device="cuda")
for _ in range(3):
    D.retrieve_device(lg, 8, d_k=hk)
torch.cuda.synchronize()
