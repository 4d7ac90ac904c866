"""HARS step / stage-1 A/B at the C2 shape (bench.py's hars_micro) for the
library FQ_LIB points at: one compact line per run."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2010_13887_b200 as P
from paper_2010_13887_b200 import _abi, decode as D

cfg = P.ModelConfig(6, 6, 1024, 4096, 16, 32000, 128, 64, 4)
r = bench.hars_micro(P, D, _abi, cfg, 128, torch.device("cuda", 0), 6454.0)[0]
print(os.environ.get("FQ_LIB", "default"), json.dumps(
    {"step_us": round(r["value"], 2), "frac": round(r["frac"], 3),
     "stage1_us": round(r["stage1_us"], 2),
     "sweep": [(s["vocab"], s["beam"], s["batch"], round(s["us"], 1), round(s["frac_hbm"], 3))
               for s in r["stage1_sweep"]]}), flush=True)
