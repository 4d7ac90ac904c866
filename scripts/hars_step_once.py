"""fq_hars_step (the HARS step on materialised fp32 logits, BASELINE metric 2)
at the C2 shape, a few launches after warm-up: the target of the HARS ncu
capture (the engine's own output layer is fq_logits_hars + fq_hars_merge_step)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2010_13887_b200 import _abi, decode as D

B, K, V, S = 128, 4, 32000, 64
R = B * K
lgs = [torch.randn(R, V, device="cuda") for _ in range(3)]
st = D.DeviceBeamState(B, K, S)
lse = torch.empty(R, dtype=torch.float64, device="cuda")
ci = torch.empty(R, V, dtype=torch.int32, device="cuda")
cc = torch.empty(R, dtype=torch.int64, device="cuda")
cnt = torch.zeros(B + 1 + R, dtype=torch.int32, device="cuda")
dcur = torch.full((1,), 5, dtype=torch.int32, device="cuda")
hist = torch.zeros(R, S, dtype=torch.int32, device="cuda")
rt = torch.empty(R, dtype=torch.int64, device="cuda")
rp = torch.empty(R, dtype=torch.int64, device="cuda")
st.init()
for i in range(6):
    st.live.fill_(K)
    st.done.zero_()
    st.step.fill_(5)
    dcur.fill_(5)
    lg = lgs[i % 3]
    _abi.call("fq_hars_step", lg.data_ptr(), V, st.c, B, K, V, S, 2, None, dcur.data_ptr(),
              1 << 40, lse.data_ptr(), ci.data_ptr(), V, cc.data_ptr(), cnt.data_ptr(),
              rt.data_ptr(), rp.data_ptr(), hist.data_ptr(), None, 0, 0.0, None, None, None,
              None, _abi.stream_handle())
torch.cuda.synchronize()
