"""LSQR golden logits from the REFERENCE converter (pkg/converter, torch):
seeded toy torch models exported to LSQW (export.py:131-169) with their
teacher-forced torch logits (export.py:203-227), the end-to-end fixture of
SURVEY §8(f)4 / converter/tests/test_parity.py:26-58.

    cp -r /root/reference/pkg /tmp/refcopy
    FUSEQ_REF=/tmp/refcopy python tests/golden/make_lsqr_golden.py

Writes tests/golden/lsqr/<name>.lsqw (the exported weights, read by
weights_io.load_weights on the device side) and <name>.npz (src, tgt, the
torch logits) — the LSQR reader is the reference's, run here, so the GPU box
needs neither the reference nor torch's converter.
"""

import os
import sys

import numpy as np

REF = os.environ.get("FUSEQ_REF", "/tmp/refcopy")
sys.path.insert(0, os.path.join(REF, "converter", "src"))
sys.path.insert(0, os.path.join(REF, "src"))

from lsqw_converter import ConvConfig, make_toy_model, read_reference_logits  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lsqr")

CASES = {  # converter/tests/test_parity.py's configurations
    "seed0": (ConvConfig(num_encoder_layers=2, num_decoder_layers=2, d_model=32, d_ff=64,
                         num_heads=4, vocab_size=101, max_seq_len=24), 0),
    "seed1": (ConvConfig(num_encoder_layers=2, num_decoder_layers=2, d_model=32, d_ff=64,
                         num_heads=4, vocab_size=101, max_seq_len=24), 1),
    "seed2": (ConvConfig(num_encoder_layers=2, num_decoder_layers=2, d_model=32, d_ff=64,
                         num_heads=4, vocab_size=101, max_seq_len=24), 2),
    "gelu": (ConvConfig(num_encoder_layers=1, num_decoder_layers=1, d_model=16, d_ff=48,
                        num_heads=2, vocab_size=67, max_seq_len=16, activation="gelu"), 11),
    "untied": (ConvConfig(num_encoder_layers=1, num_decoder_layers=1, d_model=16, d_ff=32,
                          num_heads=2, vocab_size=53, max_seq_len=16, tie_output=False), 12),
    # head_dim 16: the exact mode's 3xFP16 attention path
    "hd16": (ConvConfig(num_encoder_layers=2, num_decoder_layers=2, d_model=64, d_ff=128,
                        num_heads=4, vocab_size=211, max_seq_len=24), 5),
}


def main():
    os.makedirs(OUT, exist_ok=True)
    for name, (cfg, seed) in CASES.items():
        path = os.path.join(OUT, f"{name}.lsqw")
        make_toy_model(cfg, seed=seed, out_path=path, n_inputs=4)
        src, tgt, ref = read_reference_logits(path + ".ref.lsqr")
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), src=src, tgt=tgt, logits=ref)
        for ext in (".ref.lsqr", ".ckpt.pt", ".manifest.json"):
            if os.path.exists(path + ext):
                os.remove(path + ext)
        print(name, src.shape, tgt.shape, ref.shape, os.path.getsize(path))


if __name__ == "__main__":
    main()
