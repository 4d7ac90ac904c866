"""Per-CTA phase stamps (%globaltimer) of the fp16 mode's output-layer merge
(hars_merge_step_kernel) in a C2 generate: the last decode step's launch.
Row CTAs: 0 start (after the grid-dependency wait), 1 candidates merged and
ranked, 2 the item's last row past its arrival, 4 stage 2 + embedding done;
item rows 1024 + b: 0 selection done, 1 next-step embedding done.
Needs a -DFQ_HARS_STAMPS build: FQ_LIB=build/variants/stamps.so."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2010_13887_b200 as P
from paper_2010_13887_b200 import _abi

lib = _abi.load()
lib.fq_retrieve_debug_timestamps.argtypes = [ctypes.c_void_p]
cfg = P.ModelConfig(6, 6, 1024, 4096, 16, 32000, 128, 64, 4)
sess = P.Session(cfg, P.make_random_weights(cfg, 0), precision="fp16")
src = torch.from_numpy(np.random.default_rng(0).integers(3, 32000, size=(128, 64))).cuda()
steps = int(os.environ.get("STEPS", "20"))
dc = P.DecodeConfig(beam_size=4, max_steps=steps)
for _ in range(2):
    sess.generate(src, dc, return_device_state=True)
dbg = torch.zeros(2048 * 8, dtype=torch.int64, device="cuda")
for rep in range(3):
    dbg.zero_()
    torch.cuda.synchronize()
    lib.fq_retrieve_debug_timestamps(dbg.data_ptr())
    sess.generate(src, dc, return_device_state=True)
    torch.cuda.synchronize()
    lib.fq_retrieve_debug_timestamps(None)
    t = dbg.view(2048, 8).cpu().numpy().astype(np.float64)
    R = 512
    t0 = t[:R, 0][t[:R, 0] > 0].min()
    rel = np.where(t > 0, (t - t0) / 1e3, np.nan)

    def q(a):
        a = a[~np.isnan(a)]
        return f"{np.median(a):6.2f}/{a.max():6.2f}" if a.size else "   -   "
    print(f"rep {rep}: rows start {q(rel[:R, 0])} merged {q(rel[:R, 1])} last-row {q(rel[:R, 2])} "
          f"stage2 {q(rel[:R, 4])} | items select {q(rel[1024:1024 + 128, 0])} "
          f"embed {q(rel[1024:1024 + 128, 1])}  (median/max us)", flush=True)
