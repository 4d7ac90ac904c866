import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2010_13887_b200 as P
cfg = P.ModelConfig(num_encoder_layers=2, num_decoder_layers=2, d_model=128, d_ff=256,
                    num_heads=4, vocab_size=3000, max_batch=16, max_seq_len=24, max_beam_size=4)
w = P.make_random_weights(cfg, seed=21)
sess = P.Session(cfg, w, precision="fp32")
src = np.random.default_rng(3).integers(3, cfg.vocab_size, size=(13, 9))
lens = np.random.default_rng(4).integers(3, 10, size=13)
for k in (1, 7, 40):
    dc = P.DecodeConfig(method="top_k", sample_k=k, seed=0, max_steps=20, eos_token=2)
    for L in (None, lens):
        got = sess._generate_sampling_device(src, L, dc, 1)
        b = sess._sample_buffers[(13, 20)]
        print(k, L is not None, "err", int(b["err"].item()), "cc", b["cc"].cpu().numpy()[:13], "draw", int(b["draw"].item()))
