"""Per-CTA phase stamps (%globaltimer) of hars_merge_step_kernel at C2: row
work, item arrival, stage 2 (select_item) and the next-step embedding."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2010_13887_b200 import _abi, decode as D

lib = _abi.load()
lib.fq_retrieve_debug_timestamps.argtypes = [ctypes.c_void_p]
B, K, V, S, d = 128, 4, 32000, 64, 1024
R = B * K
g = torch.Generator(device="cuda").manual_seed(0)
E = (torch.randn(V, d, device="cuda", generator=g) * 0.05).half()
x16 = torch.randn(R, d, device="cuda", generator=g).half()
ldt, cap = (V + 223) // 224, 128
dk = torch.zeros(R, dtype=torch.int32, device="cuda")
gmx = torch.full((R, 32), -2139095041, dtype=torch.int32, device="cuda")
tmx = torch.zeros(R, ldt, device="cuda")
tsm = torch.zeros(R, ldt, dtype=torch.float64, device="cuda")
svc = torch.zeros(R, ldt, dtype=torch.int32, device="cuda")
svb = torch.zeros(R, ldt, cap, 2, dtype=torch.int32, device="cuda")
ovf = torch.zeros(1, dtype=torch.int32, device="cuda")
cnt = torch.zeros(B + 1, dtype=torch.int32, device="cuda")
st = D.DeviceBeamState(B, K, S)
lse = torch.empty(R, dtype=torch.float64, device="cuda")
ci = torch.empty(R, V, dtype=torch.int32, device="cuda")
cc = torch.empty(R, dtype=torch.int64, device="cuda")
dcur = torch.full((1,), 5, dtype=torch.int32, device="cuda")
hist = torch.zeros(R, S, dtype=torch.int32, device="cuda")
rt = torch.empty(R, dtype=torch.int64, device="cuda")
rp = torch.empty(R, dtype=torch.int64, device="cuda")
emb = torch.randn(V, d, device="cuda")
pos = torch.randn(S, d, device="cuda")
xn = torch.empty(R, d, device="cuda")
xn16 = torch.empty(R, d, device="cuda", dtype=torch.float16)
dbg = torch.zeros(R * 8, dtype=torch.int64, device="cuda")
st.init()


def one(stamp):
    st.live.fill_(K)
    st.done.zero_()
    st.step.fill_(5)
    dcur.fill_(5)
    _abi.call("fq_hars_groups", st.c, B, K, V, 0, dk.data_ptr(), _abi.stream_handle())
    _abi.call("fq_logits_hars", x16.data_ptr(), d, E.data_ptr(), d, R, V, d, dk.data_ptr(),
              gmx.data_ptr(), tmx.data_ptr(), tsm.data_ptr(), ldt, svc.data_ptr(),
              svb.data_ptr(), cap, _abi.stream_handle())
    torch.cuda.synchronize()
    if stamp:
        lib.fq_retrieve_debug_timestamps(dbg.data_ptr())
    _abi.call("fq_hars_merge_step", st.c, B, K, V, S, 2, None, dcur.data_ptr(), 1 << 40,
              dk.data_ptr(), gmx.data_ptr(), tmx.data_ptr(), tsm.data_ptr(), ldt, ldt,
              svc.data_ptr(), svb.data_ptr(), cap, lse.data_ptr(), ci.data_ptr(), V,
              cc.data_ptr(), cnt.data_ptr(), ovf.data_ptr(), rt.data_ptr(), rp.data_ptr(),
              hist.data_ptr(), emb.data_ptr(), d, 32.0, pos.data_ptr(), xn.data_ptr(),
              xn16.data_ptr(), None, _abi.stream_handle())
    torch.cuda.synchronize()
    if stamp:
        lib.fq_retrieve_debug_timestamps(None)


for _ in range(3):
    one(False)
dbg.zero_()
one(True)
t = dbg.view(R, 8).cpu().numpy().astype(np.float64)
t0 = t[:, 0][t[:, 0] > 0].min()
rel = np.where(t > 0, (t - t0) / 1e3, np.nan)
for i, n in enumerate(["start", "row_done", "sel_start", "select_done", "end", "sel_pre",
                       "sel_ranked", "sel_walked"]):
    c = rel[:, i]
    c = c[~np.isnan(c)]
    print(f"{n:12s} n={len(c):4d} min {c.min():6.2f} median {np.median(c):6.2f} max {c.max():6.2f}")
