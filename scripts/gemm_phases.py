"""Phase timestamps (%globaltimer, CTA 0) of one tcgen05 GEMM launch: kernel
start, prologue done, first/last TMA issue, first stage landed, last commit,
accumulator ready, epilogue done, exit barrier."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2010_13887_b200 as P
from paper_2010_13887_b200 import _abi

lib = _abi.load()
lib.fq_gemm_debug_timestamps.argtypes = [ctypes.c_void_p]
dbg = torch.zeros(16, dtype=torch.int64, device="cuda")
names = ["start", "prologue", "tma0", "tma_last", "full0", "commit_last", "tfull", "epi_done",
         "exit_bar"]
for M, N, K in [(512, 1024, 1024), (512, 1024, 4096), (512, 4096, 1024), (128, 1024, 1024),
                (512, 1024, 256)]:
    a = torch.randn(M, K, device="cuda").half()
    b = torch.randn(N, K, device="cuda").half()
    c = torch.empty(M, N, device="cuda")
    for i in range(3):
        lib.fq_gemm_debug_timestamps(dbg.data_ptr())
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        P.gemm(a, b, c, transpose_b=True)
        e.record()
        e.synchronize()
        lib.fq_gemm_debug_timestamps(None)
    t = dbg.cpu().tolist()
    print(f"{M}x{N}x{K}: event {s.elapsed_time(e) * 1e3:.1f} us | " +
          " ".join(f"{n}={(t[i] - t[0]) / 1e3:.2f}" for i, n in enumerate(names)))
