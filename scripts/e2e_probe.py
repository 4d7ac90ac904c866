"""Where the end-to-end (host tokens in, host hypotheses out) time goes beyond
the device-resident generate: H2D + encode setup, host_items, finalize."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2010_13887_b200 as P

cfg = P.ModelConfig(6, 6, 1024, 4096, 16, 32000, 128, 64, 4)
sess = P.Session(cfg, P.make_random_weights(cfg, 0), precision=os.environ.get("PREC", "fp32"))
src = np.random.default_rng(0).integers(3, 32000, size=(128, 64))
src_dev = torch.from_numpy(src).cuda()
src_pin = torch.from_numpy(src).pin_memory()
dc = P.DecodeConfig(beam_size=4, max_steps=64)
for _ in range(3):
    sess.generate(src_dev, dc)
torch.cuda.synchronize()


def t(fn, n=5):
    ts = []
    for _ in range(n):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return np.median(ts) * 1e3, r


a, st = t(lambda: sess.generate(src_dev, dc, return_device_state=True))
b, _ = t(lambda: sess.generate(src_pin, dc))
c, _ = t(lambda: sess.generate(src_dev, dc))
d, items = t(lambda: st.host_items())
e, _ = t(lambda: [s.finalize(dc) for s in items])
f_, _ = t(lambda: st.finalize_batch(dc))
import paper_2010_13887_b200.decode as D
g_, _ = t(lambda: st._to_host())
h_, _ = t(lambda: D.check_error_flags(st.error_flags))
print(f"finalize_batch {f_:.2f} ms | _to_host {g_:.2f} | error flags {h_:.2f}")
print(f"device-state generate {a:.2f} ms | host-in generate {b:.2f} | device-in host-out {c:.2f} "
      f"| host_items {d:.2f} | finalize {e:.2f}")
