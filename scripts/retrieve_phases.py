"""Per-CTA phase stamps (%globaltimer) of the single-sweep retrieve at the C2
decode shape: start, pilot reduced (R' known), sweep done, sums reduced, end."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2010_13887_b200 import _abi, decode as D

lib = _abi.load()  # stamps need a -DFQ_HARS_STAMPS build: FQ_LIB=build/variants/stamps.so
lib.fq_retrieve_debug_timestamps.argtypes = [ctypes.c_void_p]
R, V = 512, 32000
lgs = [torch.randn(R, V, device="cuda") for _ in range(3)]
hk = torch.full((R,), 8, dtype=torch.int32, device="cuda")
dbg = torch.zeros(R * 8, dtype=torch.int64, device="cuda")
for i in range(4):
    D.retrieve_device(lgs[i % 3], 8, d_k=hk)
torch.cuda.synchronize()
lib.fq_retrieve_debug_timestamps(dbg.data_ptr())
D.retrieve_device(lgs[1], 8, d_k=hk)
torch.cuda.synchronize()
lib.fq_retrieve_debug_timestamps(None)
t = dbg.view(R, 8)[:, :5].cpu().double()
t0 = t[:, 0].min()
st = (t[:, 0] - t0) / 1e3
names = ["pilot", "sweep", "sums", "end"]
print(f"start skew max {st.max():.2f} us, span {(t[:, 4].max() - t0) / 1e3:.2f} us")
for i, n in enumerate(names):
    d = (t[:, i + 1] - t[:, i]) / 1e3
    print(f"  {n:6s} median {d.median():.2f} us  max {d.max():.2f}")
