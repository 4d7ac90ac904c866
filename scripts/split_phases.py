"""Per-CTA phase stamps (%globaltimer) of the balanced-split stage 1 at the C2
decode shape (API fq_retrieve and the fused fq_hars_step): start, first
portion swept, second portion swept, row finalize start/end, CTA end."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2010_13887_b200 import _abi, decode as D

lib = _abi.load()  # stamps need a -DFQ_HARS_STAMPS build: FQ_LIB=build/variants/stamps.so
lib.fq_retrieve_debug_timestamps.argtypes = [ctypes.c_void_p]
B, K, V, S = (int(x) for x in os.environ.get("SHAPE", "128,4,32000,64").split(","))
R = B * K
lgs = [torch.randn(R, V, device="cuda") for _ in range(3)]
hk = torch.full((R,), 8, dtype=torch.int32, device="cuda")
NC = 2048
dbg = torch.zeros(NC * 8, dtype=torch.int64, device="cuda")


def report(tag):
    t = dbg.view(NC, 8)[:, :8].cpu().numpy().astype(np.float64)
    used = t[:, 0] > 0
    t = t[used]
    t0 = t[:, 0].min()
    rel = np.where(t > 0, (t - t0) / 1e3, np.nan)
    print(f"[{tag}] CTAs {used.sum()}: start skew max {np.nanmax(rel[:, 0]):.2f} us, "
          f"end max {np.nanmax(rel[:, 5]):.2f} us")
    for i, n in enumerate(["start", "portion1", "portion2", "final0", "final1", "end", "fin_sums", "fin_surv"]):
        c = rel[:, i]
        c = c[~np.isnan(c)]
        if len(c):
            print(f"  {n:9s} n={len(c):4d} min {c.min():6.2f} median {np.median(c):6.2f} "
                  f"p90 {np.percentile(c, 90):6.2f} max {c.max():6.2f}")


for i in range(4):
    D.retrieve_device(lgs[i % 3], 8, d_k=hk)
torch.cuda.synchronize()
dbg.zero_()
lib.fq_retrieve_debug_timestamps(dbg.data_ptr())
D.retrieve_device(lgs[1], 8, d_k=hk)
torch.cuda.synchronize()
lib.fq_retrieve_debug_timestamps(None)
report("fq_retrieve split")

# fused step
st = D.DeviceBeamState(B, K, S)
st.init()
lse = torch.zeros(R, dtype=torch.float64, device="cuda")
ci = torch.zeros(R, V, dtype=torch.int32, device="cuda")
cc = torch.zeros(R, dtype=torch.int64, device="cuda")
hcnt = torch.zeros(B + 1 + R, dtype=torch.int32, device="cuda")
dcur = torch.full((1,), 5, dtype=torch.int32, device="cuda")
hist = torch.zeros(R, S, dtype=torch.int32, device="cuda")
rt = torch.zeros(R, dtype=torch.int64, device="cuda")
rp = torch.zeros(R, dtype=torch.int64, device="cuda")


def fused(lg):
    st.live.fill_(K)
    st.done.zero_()
    st.step.fill_(5)
    dcur.fill_(5)
    _abi.call("fq_hars_step", lg.data_ptr(), lg.stride(0), st.c, B, K, V, S, 2, None,
              dcur.data_ptr(), 1 << 40, lse.data_ptr(), ci.data_ptr(), ci.stride(0),
              cc.data_ptr(), hcnt.data_ptr(), rt.data_ptr(), rp.data_ptr(), hist.data_ptr(),
              None, 0, 0.0, None, None, None, None, _abi.stream_handle())


for i in range(4):
    fused(lgs[i % 3])
torch.cuda.synchronize()
dbg.zero_()
lib.fq_retrieve_debug_timestamps(dbg.data_ptr())
fused(lgs[2])
torch.cuda.synchronize()
lib.fq_retrieve_debug_timestamps(None)
report("fq_hars_step split")
