"""Per-CTA start/end (%globaltimer) of one tcgen05 GEMM launch: launch skew and
CTA runtime spread (benchmark aid)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2010_13887_b200 as P
from paper_2010_13887_b200 import _abi

lib = _abi.load()
lib.fq_gemm_debug_timestamps.argtypes = [ctypes.c_void_p]
lib.fq_gemm_force_plan.argtypes = [ctypes.c_int] * 4
dbg = torch.zeros(2048, dtype=torch.int64, device="cuda")
for (M, N, K, plan) in [(512, 1024, 1024, (32, 1, 1, 1)), (512, 1024, 1024, (128, 1, 1, 4)),
                        (512, 4096, 1024, (128, 1, 1, 1))]:
    a = torch.randn(M, K, device="cuda").half()
    b = torch.randn(N, K, device="cuda").half()
    c = torch.empty(M, N, device="cuda")
    lib.fq_gemm_force_plan(*plan)
    x = torch.randn(512, 1024, device="cuda").half()
    y = torch.empty(512, 1024, device="cuda")
    w_prev = torch.randn(1024, 1024, device="cuda").half()
    for _ in range(3):
        dbg.zero_()
        P.gemm(x, w_prev, y, transpose_b=True)   # a preceding kernel
        lib.fq_gemm_debug_timestamps(dbg.data_ptr())
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        P.gemm(a, b, c, transpose_b=True)
        e.record()
        torch.cuda.synchronize()
        lib.fq_gemm_debug_timestamps(None)
    t = dbg.cpu().view(-1, 2)
    t = t[t[:, 0] > 0]
    st, en = t[:, 0].double(), t[:, 1].double()
    t0 = st.min()
    print(f"{M}x{N}x{K} {plan}: ctas={len(t)} event={s.elapsed_time(e) * 1e3:.1f}us "
          f"start spread={(st.max() - t0) / 1e3:.2f}us  run min/med/max="
          f"{(en - st).min() / 1e3:.2f}/{(en - st).median() / 1e3:.2f}/{(en - st).max() / 1e3:.2f}us "
          f"span={(en.max() - t0) / 1e3:.2f}us")
lib.fq_gemm_force_plan(0, 0, 0, 1)
