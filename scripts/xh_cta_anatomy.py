"""Per-CTA %globaltimer stamps of one exact-mode (3xFP16) GEMM launch (slots: 0
start, 1 setup, 2 first stage landed, 4 first tile accumulated (all chunks
added), 5 epilogue done, 6 exit, 7 all MMAs issued), cold L2 (256 MiB flush)
or warm (WARM=1). Usage: SHAPES=512x3072x1024,..."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2010_13887_b200 as P  # noqa: F401
from paper_2010_13887_b200 import _abi
from paper_2010_13887_b200.model import XHWeight
from paper_2010_13887_b200.tensor import split_pair

lib = _abi.load()  # stamps need a -DFQ_GEMM_STAMPS build: FQ_LIB=build/variants/<name>.so
lib.fq_gemm_debug_timestamps.argtypes = [ctypes.c_void_p]
shapes = os.environ.get("SHAPES", "512x3072x1024,512x4096x1024,512x32000x1024")
for sh in shapes.split(","):
    M, N, K = (int(x) for x in sh.split("x"))
    a = split_pair(torch.randn(M, K, device="cuda"))
    ws = [XHWeight.from_kn(torch.randn(N, K, device="cuda") * 0.03, transpose=False)
          for _ in range(3)]
    bias = torch.randn(N, device="cuda")
    c = torch.empty(M, N, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    dbg = torch.zeros(8 * 4096, dtype=torch.int64, device="cuda")

    slab_ws = torch.empty(8 * M * N, device="cuda")
    nsl = ctypes.c_int32(0)

    def run(w):
        if os.environ.get("SLABS"):  # the decode N = 1024 GEMMs: split-K slabs, no reduction
            _abi.call("fq_gemm_x3h_slabs", a[0].data_ptr(), a[1].data_ptr(), K, w.hi.data_ptr(),
                      w.lo.data_ptr(), K, slab_ws.data_ptr(), slab_ws.numel() * 4, M, N, K,
                      ctypes.addressof(nsl), _abi.stream_handle())
            return
        _abi.call("fq_gemm_x3h", a[0].data_ptr(), a[1].data_ptr(), K, w.hi.data_ptr(),
                  w.lo.data_ptr(), K, c.data_ptr(), N, M, N, K, 0, bias.data_ptr(), None, 0, 1,
                  _abi.stream_handle())
    for w in ws:
        run(w)
    for rep in range(3):
        if not os.environ.get("WARM"):
            flush.fill_(1)
        dbg.zero_()
        torch.cuda.synchronize()
        lib.fq_gemm_debug_timestamps(dbg.data_ptr())
        run(ws[rep])
        torch.cuda.synchronize()
        lib.fq_gemm_debug_timestamps(None)
        t = dbg.view(-1, 8).cpu()
        t = t[t[:, 0] > 0]
        t0 = int(t[:, 0].min())
        rel = (t - t0).double() / 1e3
        q = lambda i, f: float(rel[:, i][t[:, i] > 0].quantile(f)) if bool((t[:, i] > 0).any()) else -1
        print(f"{sh}: ctas {len(t)} | " + " ".join(
            f"s{i}={q(i, .5):.2f}/{q(i, 1.0):.2f}" for i in (0, 1, 2, 4, 5, 6, 7))
            + "  (median/max us since first CTA)", flush=True)
