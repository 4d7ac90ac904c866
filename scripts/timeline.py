"""CUPTI kernel timeline of one C2 generate (torch.profiler; nsys is not in the
image): busy time per kernel family vs. wall span, i.e. how much of a decode
step is kernel execution and how much is launch/dependency gaps."""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2010_13887_b200 as P

prec = sys.argv[1] if len(sys.argv) > 1 else "fp16"
cfg = P.ModelConfig(6, 6, 1024, 4096, 16, 32000, 128, 64, 4)
sess = P.Session(cfg, P.make_random_weights(cfg, 0), precision=prec)
src = torch.from_numpy(np.random.default_rng(0).integers(3, 32000, size=(128, 64))).cuda()
dc = P.DecodeConfig(beam_size=4, max_steps=64)
sess.generate(src, dc, return_device_state=True)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    sess.generate(src, dc, return_device_state=True)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0, t1 = ev[0].time_range.start, ev[-1].time_range.end
busy = sum(e.time_range.end - e.time_range.start for e in ev)
# decode steps: delimited by step_advance
adv = [e for e in ev if "step_advance" in e.name]
print(f"kernels {len(ev)}, wall {(t1 - t0) / 1e3:.2f} ms, busy {busy / 1e3:.2f} ms "
      f"({100 * busy / (t1 - t0):.0f}%)")
if len(adv) > 3:
    s0, s1 = adv[10].time_range.end, adv[11].time_range.end
    st = [e for e in ev if s0 <= e.time_range.start < s1]
    b = sum(e.time_range.end - e.time_range.start for e in st)
    print(f"one decode step: wall {(s1 - s0):.1f} us, busy {b:.1f} us, {len(st)} kernels, "
          f"mean gap {((s1 - s0) - b) / len(st):.2f} us")
    agg = collections.defaultdict(float)
    for e in st:
        agg[e.name[:70]] += e.time_range.end - e.time_range.start
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:14]:
        print(f"   {v:8.1f} us  {k}")
tot = collections.defaultdict(lambda: [0, 0.0])
for e in ev:
    tot[e.name[:70]][0] += 1
    tot[e.name[:70]][1] += e.time_range.end - e.time_range.start
print("whole generate, per kernel (n, total us, avg us):")
for k, (n, v) in sorted(tot.items(), key=lambda kv: -kv[1][1])[:16]:
    print(f"   {n:5d} {v:10.1f} {v / n:8.2f}  {k}")
enc = [e for e in ev if e.time_range.end <= adv[0].time_range.start] if adv else []
if enc:
    print(f"prefix (encoder + setup + step 0): {(adv[0].time_range.end - t0) / 1e3:.2f} ms")
