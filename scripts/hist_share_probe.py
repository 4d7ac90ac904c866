import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2010_13887_b200 as P
from paper_2010_13887_b200 import model as M
cfg = P.ModelConfig(6, 6, 1024, 4096, 16, 32000, 128, 64, 4)
sess = P.Session(cfg, P.make_random_weights(cfg, 0), precision="fp16")
src = np.random.default_rng(0).integers(3, 32000, size=(128, 64))
dc = P.DecodeConfig(beam_size=4, max_steps=64)
# capture hist at several steps by running generate with max_steps = s
for steps in (8, 16, 32, 48, 64):
    dc = P.DecodeConfig(beam_size=4, max_steps=steps)
    st = sess.generate(torch.from_numpy(src).cuda(), dc, return_device_state=True)
    torch.cuda.synchronize()
    # find the cache hist buffer in the arena
    hist = sess._buffers.get("dec.cache.hist", (512, 64), torch.int32).cpu().numpy()
    cur = steps - 1
    h = hist[:, :cur].reshape(128, 4, cur)
    same_pos = (h == h[:, :1, :]).all(axis=1)           # [item, pos] all 4 beams same physical row
    chunks = (cur + 15) // 16
    full = 0; tot = 0
    for c in range(chunks):
        seg = same_pos[:, 16 * c: min(16 * c + 16, cur)]
        full += seg.all(axis=1).sum(); tot += 128
    distinct = np.array([[len(set(h[b, :, t])) for t in range(cur)] for b in range(128)])
    print(f"step {steps}: positions shared by all 4 beams {same_pos.mean():.2f}; chunks fully shared {full / max(tot,1):.2f}; mean distinct rows per position {distinct.mean():.2f}")
