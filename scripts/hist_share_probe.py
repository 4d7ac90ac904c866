"""How much of the self-attention K/V history do the beams of one item share?
Runs the C2 beam search for s steps and counts, over the history table, the
distinct (position, physical row) slots per item vs beam x positions."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2010_13887_b200 as P

cfg = P.ModelConfig(6, 6, 1024, 4096, 16, 32000, 128, 64, 4)
sess = P.Session(cfg, P.make_random_weights(cfg, 0), precision="fp32")
src = np.random.default_rng(0).integers(3, 32000, size=(128, 64))
src_dev = torch.from_numpy(src).cuda()
for s in (8, 16, 32, 48, 63):
    dc = P.DecodeConfig(beam_size=4, max_steps=s)
    sess.generate(src_dev, dc)
    torch.cuda.synchronize()
    hist = sess._buffers.get("dec.cache.hist", (512, 64), torch.int32).cpu().numpy()
    cur = int(sess._buffers.get("dec.cache.cur", (1,), torch.int32).item())
    h = hist[:, :cur].reshape(128, 4, cur)
    tot = 0
    for i in range(128):
        tot += sum(len(set(h[i, :, t].tolist())) for t in range(cur))
    print(f"steps {s} cur {cur}: distinct slots / (beam x pos) = {tot / (128 * 4 * cur):.3f}",
          flush=True)
