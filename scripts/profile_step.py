"""One Transformer-big (C2) beam-4 generate between cudaProfilerStart/Stop, for
`ncu --profile-from-start off` launch lists and captures (see profiles/README.md)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2010_13887_b200 as P

ap = argparse.ArgumentParser()
ap.add_argument("--precision", default="fp16")
ap.add_argument("--batch", type=int, default=128)
ap.add_argument("--steps", type=int, default=64)
ap.add_argument("--graphs", type=int, default=1)
a = ap.parse_args()
cfg = P.ModelConfig(6, 6, 1024, 4096, 16, 32000, a.batch, 64, 4)
sess = P.Session(cfg, P.make_random_weights(cfg, 0), precision=a.precision,
                 use_graphs=bool(a.graphs))
src = torch.from_numpy(np.random.default_rng(0).integers(3, 32000, size=(a.batch, 64))).cuda()
dc = P.DecodeConfig(beam_size=4, max_steps=a.steps)
sess.generate(src, dc, return_device_state=True)   # warm-up + graph capture
torch.cuda.synchronize()
torch.cuda.profiler.start()
sess.generate(src, dc, return_device_state=True)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled one generate")
