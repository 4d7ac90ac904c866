"""Per-CTA start/end (%globaltimer) of one tcgen05 GEMM launch at the decode
shapes: launch skew, per-CTA duration distribution, kernel span."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2010_13887_b200 as P
from paper_2010_13887_b200 import _abi

lib = _abi.load()
lib.fq_gemm_debug_timestamps.argtypes = [ctypes.c_void_p]
for M, N, K in [(512, 1024, 1024), (512, 1024, 4096)]:
    a = torch.randn(M, K, device="cuda").half()
    nb = int(os.environ.get("NBUF", "4"))
    bs = [torch.randn(N, K, device="cuda").half() for _ in range(nb)]
    c = torch.empty(M, N, device="cuda")
    dbg = torch.zeros(8 * 1024, dtype=torch.int64, device="cuda")
    for i in range(nb):
        P.gemm(a, bs[i], c, transpose_b=True)
    torch.cuda.synchronize()
    lib.fq_gemm_debug_timestamps(dbg.data_ptr())
    P.gemm(a, bs[0], c, transpose_b=True)
    torch.cuda.synchronize()
    lib.fq_gemm_debug_timestamps(None)
    t = dbg.view(-1, 8).cpu()
    t = t[t[:, 0] > 0]
    t0 = int(t[:, 0].min())
    rel = (t - t[:, :1]).double() / 1e3
    st = (t[:, 0] - t0).double() / 1e3
    en = (t[:, 6] - t0).double() / 1e3
    names = ["prologue", "acc_ready", "staged+pushed", "recv_done", "reduced", "exit"]
    med = [float(rel[:, i].median()) for i in range(1, 7)]
    print(f"{M}x{N}x{K}: ctas {len(t)} skew {st.max():.2f} span {en.max():.2f} us | median since CTA start: " +
          " ".join(f"{n}={v:.2f}" for n, v in zip(names, med)))
