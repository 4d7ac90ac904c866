import ctypes, os, statistics, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch
import paper_2010_13887_b200 as P
from paper_2010_13887_b200 import _abi
lib = _abi.load()
lib.fq_gemm_force_plan.argtypes = [ctypes.c_int] * 4
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for M, N, K in [(512, 3072, 1024), (512, 4096, 1024), (512, 32000, 1024)]:
    a = torch.randn(M, K, device="cuda").half()
    b = torch.randn(N, K, device="cuda").half()
    c = torch.empty(M, N, device="cuda", dtype=torch.float16)
    bias = torch.randn(N, device="cuda")
    out = []
    for plan in [(0, 0, 0, 1), (128, 1, 1, 1), (96, 1, 1, 1), (128, 1, 2, 1), (128, 1, 4, 1), (96, 1, 2, 1), (96, 1, 4, 1), (128, 2, 1, 1), (128, 4, 1, 1), (256, 1, 2, 1), (224, 1, 1, 1), (224, 1, 2, 1)]:
        lib.fq_gemm_force_plan(*plan)
        ts = []
        for _ in range(10):
            flush.fill_(1)
            s, e = torch.cuda.Event(True), torch.cuda.Event(True)
            s.record(); P.gemm(a, b, c, transpose_b=True, bias=bias, activation="relu"); e.record(); e.synchronize()
            ts.append(s.elapsed_time(e) * 1e3)
        out.append(f"{plan}:{statistics.median(ts[2:]):.1f}")
    lib.fq_gemm_force_plan(0, 0, 0, 1)
    print(M, N, K, " ".join(out))
