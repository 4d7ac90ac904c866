"""C2 exact-mode generate with ragged source lengths (padding mask on):
ms per request for the current library vs FQ_LIB (run twice, alternating)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2010_13887_b200 as P

cfg = P.ModelConfig(6, 6, 1024, 4096, 16, 32000, 128, 64, 4)
sess = P.Session(cfg, P.make_random_weights(cfg, 0), precision="fp32")
rng = np.random.default_rng(0)
src = torch.from_numpy(rng.integers(3, 32000, size=(128, 64))).cuda()
lens = rng.integers(24, 65, size=128)
dc = P.DecodeConfig(beam_size=4, max_steps=64)
for _ in range(2):
    sess.generate(src, dc, src_lengths=lens, return_device_state=True)
ts = []
for _ in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sess.generate(src, dc, src_lengths=lens, return_device_state=True)
    torch.cuda.synchronize()
    ts.append((time.perf_counter() - t0) * 1e3)
print(f"{os.environ.get('FQ_LIB', 'current') or 'current'}: {np.median(ts):.2f} ms / masked request")
