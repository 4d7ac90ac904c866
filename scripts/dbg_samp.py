import json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2010_13887_b200 as P
golden_path = lambda n: os.path.join("tests", "golden", n)
g = np.load(golden_path("sampling_golden.npz"))
kw = json.loads(str(g["cfgs"]))[0]
cfg = P.ModelConfig(**kw)
print(cfg)
w = P.make_random_weights(cfg, seed=10)
for graphs in (False, True):
    sess = P.Session(cfg, w, precision="fp32", use_graphs=graphs)
    src, lens = g["m0_src"], g["m0_len"]
    for run in json.loads(str(g["runs"])):
        if run["model"] != 0: continue
        dc = P.DecodeConfig(method=run["method"], sample_k=run["sample_k"], sample_p=run["sample_p"], seed=run["seed"], max_steps=12, eos_token=run["eos"])
        try:
            hyps = sess.generate(src, dc, src_lengths=lens if run["lengths"] else None)
            p = run["key"]
            ok = all(h.tokens == g[p + "tok"][b, i][:g[p + "len"][b, i]].tolist() for b, hs in enumerate(hyps) for i, h in enumerate(hs))
            print(graphs, run["method"], run["sample_k"], run["lengths"], "ok" if ok else "MISMATCH")
        except Exception as e:
            print(graphs, run["method"], run["sample_k"], run["lengths"], "ERR", type(e).__name__, e)
