"""Per-CTA %globaltimer stamps of the logits GEMM with the HARS statistics
epilogue (fq_logits_hars) at C2: when the last tile's MMAs were issued (s7)
vs when the statistics epilogue finished (s5) — the epilogue tail the
persistent double-buffered TMEM does not hide."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2010_13887_b200 import _abi

lib = _abi.load()
lib.fq_gemm_debug_timestamps.argtypes = [ctypes.c_void_p]
R, V, d, cap = 512, 32000, 1024, 128
ldt = (V + 223) // 224
x = (torch.randn(R, d, device="cuda") * 0.5).half()
E = (torch.randn(V, d, device="cuda") / 32).half()
dk = torch.full((R,), 8, dtype=torch.int32, device="cuda")
gmax = torch.empty(R, 32, dtype=torch.int32, device="cuda")
tmax = torch.empty(R, ldt, device="cuda")
tsum = torch.empty(R, ldt, dtype=torch.float64, device="cuda")
cnt = torch.empty(R, ldt, dtype=torch.int32, device="cuda")
sv = torch.empty(R, ldt, cap, 2, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
dbg = torch.zeros(8 * 1024, dtype=torch.int64, device="cuda")


def run():
    gmax.fill_(-2139095041)
    _abi.call("fq_logits_hars", x.data_ptr(), d, E.data_ptr(), d, R, V, d, dk.data_ptr(),
              gmax.data_ptr(), tmax.data_ptr(), tsum.data_ptr(), ldt, cnt.data_ptr(),
              sv.data_ptr(), cap, _abi.stream_handle())


for _ in range(3):
    run()
for rep in range(3):
    flush.fill_(1)
    dbg.zero_()
    torch.cuda.synchronize()
    lib.fq_gemm_debug_timestamps(dbg.data_ptr())
    run()
    torch.cuda.synchronize()
    lib.fq_gemm_debug_timestamps(None)
    t = dbg.view(-1, 8).cpu()
    t = t[t[:, 0] > 0]
    t0 = int(t[:, 0].min())
    rel = (t - t0).double() / 1e3
    q = lambda i, f: float(rel[:, i][t[:, i] > 0].quantile(f)) if bool((t[:, i] > 0).any()) else -1
    print(f"logits_hars: ctas {len(t)} | " + " ".join(
        f"s{i}={q(i, .5):.2f}/{q(i, 1.0):.2f}" for i in range(8)) + "  (median/max us)")
