"""Per-CTA phase stamps (%globaltimer) of the fused row-per-CTA HARS step at the
C2 shape: stage 1 (start, pilot, sweep, sums, end) and, for the CTA that ran its
item's stage 2, inputs loaded / ranked / walk done / select done / embedding done."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2010_13887_b200 import _abi, decode as D

lib = _abi.load()  # stamps need a -DFQ_HARS_STAMPS build: FQ_LIB=build/variants/stamps.so
lib.fq_retrieve_debug_timestamps.argtypes = [ctypes.c_void_p]
B, K, V, S = 128, 4, 32000, 64
R = B * K
lgs = [torch.randn(R, V, device="cuda") for _ in range(3)]
dbg = torch.zeros(2048 * 8, dtype=torch.int64, device="cuda")
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
emb = torch.randn(V, 1024, device="cuda")
pos = torch.randn(S, 1024, device="cuda")
xn = torch.empty(R, 1024, device="cuda")


def fused(lg):
    st.live.fill_(K)
    st.done.zero_()
    st.step.fill_(5)
    dcur.fill_(5)
    _abi.call("fq_hars_step", lg.data_ptr(), lg.stride(0), st.c, B, K, V, S, 2, None,
              dcur.data_ptr(), 1 << 40, lse.data_ptr(), ci.data_ptr(), ci.stride(0),
              cc.data_ptr(), hcnt.data_ptr(), rt.data_ptr(), rp.data_ptr(), hist.data_ptr(),
              emb.data_ptr(), 1024, 32.0, pos.data_ptr(), xn.data_ptr(), None, None,
              _abi.stream_handle())


for i in range(4):
    fused(lgs[i % 3])
torch.cuda.synchronize()
for rep in range(2):
    dbg.zero_()
    torch.cuda.synchronize()
    lib.fq_retrieve_debug_timestamps(dbg.data_ptr())
    fused(lgs[rep])
    torch.cuda.synchronize()
    lib.fq_retrieve_debug_timestamps(None)
    t = dbg.view(2048, 8).cpu().numpy().astype(np.float64)
    t0 = t[:R, 0][t[:R, 0] > 0].min()
    rel = np.where(t > 0, (t - t0) / 1e3, np.nan)

    def q(name, c):
        c = c[~np.isnan(c)]
        if len(c):
            print(f"  {name:14s} n={len(c):4d} min {c.min():6.2f} med {np.median(c):6.2f} "
                  f"p90 {np.percentile(c, 90):6.2f} max {c.max():6.2f}")
    print(f"rep {rep}")
    for i, n in enumerate(["start", "pilot", "sweep", "sums", "s1 end", "s2 inputs", "s2 ranked",
                           "s2 walked"]):
        q(n, rel[:R, i])
    q("s2 selected", rel[1024:1024 + R, 0])
    q("s2 embedded", rel[1024:1024 + R, 1])
    sm = t[1536:1536 + R, 0].astype(int)
    per = np.bincount(sm, minlength=148)
    nrow = per[sm]
    for c in sorted(set(nrow)):
        sel = nrow == c
        print(f"  SMs with {c} rows: {np.sum(per == c)} SMs; sweep end med "
              f"{np.nanmedian(rel[:R, 2][sel]):.2f} max {np.nanmax(rel[:R, 2][sel]):.2f}; "
              f"pilot med {np.nanmedian(rel[:R, 1][sel]):.2f}")
    # by die: SM id halves
    for lo, hi in ((0, 74), (74, 148)):
        sel = (sm >= lo) & (sm < hi)
        print(f"  smid [{lo},{hi}): rows {sel.sum()} sweep end med {np.nanmedian(rel[:R, 2][sel]):.2f}")
    # per stage-2 CTA: phase deltas after its own stage-1 end
    has = ~np.isnan(rel[:R, 5])
    ch = [rel[:R, 4], rel[:R, 5], rel[:R, 6], rel[:R, 7], rel[1024:1024 + R, 0], rel[1024:1024 + R, 1]]
    names = ["arrive+inputs", "ranked", "walked", "selected", "embedded"]
    for j, n in enumerate(names):
        d = (ch[j + 1] - ch[j])[has]
        print(f"  d {n:14s} med {np.nanmedian(d):5.2f} p90 {np.nanpercentile(d, 90):5.2f} max {np.nanmax(d):5.2f}")
    last = np.nanargmax(rel[1024:1024 + R, 1])
    print(f"  last item's CTA: s1 end {rel[last, 4]:.2f} -> embedded {rel[1024 + last, 1]:.2f}")
