"""Generate golden fixtures by running the REAL reference (`fuseq`, CPU).

This script is the only place that imports the reference. It needs a
writable copy of `/root/reference/pkg` (numba's ``cache=True`` writes next
to the sources), e.g.::

    cp -r /root/reference/pkg /tmp/refcopy
    FUSEQ_REF=/tmp/refcopy python tests/golden/make_golden.py [--big]

Outputs small ``.npz`` fixtures next to this file. The fixtures travel to
the GPU box; the reference does not. ``--big`` adds the Transformer-big
(C2) batch-128 generate fixture (~80 s on 8 cores).

Fixture inventory (all seeds fixed):

* ``ops_golden.npz``      fused op inputs/outputs (ops.py:81-218)
* ``retrieve_golden.npz`` retrieve over random + tie-heavy rows (decode.py:58-92)
* ``beam_golden.npz``     pure-logit-stream beam search incl. EOS (decode.py:217-240)
* ``tiny_golden.npz``     tiny seq2seq models: generate / forced_logits / encode
* ``c1_golden.npz``       Transformer-base C1 generate (BASELINE config 1)
* ``c2_golden.npz``       Transformer-big C2 generate (BASELINE config 2), --big only
* ``sampling_golden.npz`` tiny models: top-k / top-p sampling generate (engine.py:175-195,
                          decode.py:378-430), seeded PCG64 draws
* ``classify_golden.npz`` encoder-only models: classify labels + probabilities
                          (engine.py:198-224, decode.py:485-492)
* ``diverse_golden.npz``  tiny models: diverse beam search generate, hierarchical and
                          exhaustive (decode.py:274-371)
"""

from __future__ import annotations

import json
import math
import os
import sys
import time

import numpy as np

REF = os.environ.get("FUSEQ_REF", "/tmp/refcopy")
sys.path.insert(0, os.path.join(REF, "src"))

from fuseq import decode as D  # noqa: E402
from fuseq import model as M  # noqa: E402
from fuseq import ops  # noqa: E402
from fuseq.bench import synthetic_tokens  # noqa: E402
from fuseq.engine import Session  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
F32 = np.float32


def weight_checksums(cfg, w):
    return np.array([float(np.asarray(a, np.float64).sum()) for _, a in w.named_tensors(cfg)])


def pack_hyps(hyps, beam, max_len):
    """hypotheses -> tokens [B, beam, max_len] (-1 pad), lens [B, beam], scores [B, beam], n [B]."""
    B = len(hyps)
    toks = np.full((B, beam, max_len), -1, np.int32)
    lens = np.zeros((B, beam), np.int32)
    scores = np.zeros((B, beam), np.float64)
    n = np.zeros(B, np.int32)
    for b, hs in enumerate(hyps):
        n[b] = len(hs)
        for i, h in enumerate(hs):
            toks[b, i, :len(h.tokens)] = h.tokens
            lens[b, i] = len(h.tokens)
            scores[b, i] = h.score
    return toks, lens, scores, n


def cfg_dict(cfg):
    return json.dumps(cfg.to_dict(), sort_keys=True)


# ---------------------------------------------------------------------------
def make_ops():
    rng = np.random.default_rng(1234)
    out = {}

    def r(*s):
        return rng.normal(size=s).astype(F32)

    for i, (n, d) in enumerate([(7, 33), (64, 512), (5, 1024)]):
        x, g, b = r(n, d), r(d), r(d)
        out[f"ln{i}_x"], out[f"ln{i}_g"], out[f"ln{i}_b"] = x, g, b
        out[f"ln{i}_out"] = ops.fused_layer_norm(x, g, b, 1e-5).data.copy()
        bias, res = r(d), r(n, d)
        out[f"brln{i}_x"], out[f"brln{i}_bias"], out[f"brln{i}_res"] = x, bias, res
        out[f"brln{i}_out"] = ops.fused_bias_residual_layer_norm(x, bias, res, g, b, 1e-5).data.copy()
        for act in ("none", "relu", "gelu"):
            out[f"act{i}_{act}_nores"] = ops.fused_bias_residual_activation(x, bias, None, act).data.copy()
            out[f"act{i}_{act}_res"] = ops.fused_bias_residual_activation(x, bias, res, act).data.copy()
    # attention softmax, with and without mask
    s = (r(3, 4, 5, 11) * 3).astype(F32)
    mask = np.zeros((3, 11), F32)
    mask[0, 7:] = -np.inf
    mask[2, 3:] = -np.inf
    out["sm_scores"], out["sm_mask"] = s, mask
    out["sm_scale"] = np.array([0.125], F32)
    out["sm_out_mask"] = ops.fused_attention_softmax(s, 0.125, mask).data.copy()
    out["sm_out_nomask"] = ops.fused_attention_softmax(s, 0.125, None).data.copy()
    # qkv reshape / heads
    batch, seq, heads, d = 2, 5, 4, 32
    qkv, qb = r(batch * seq, 3 * d), r(3 * d)
    q, k, v = ops.fused_qkv_bias_reshape(qkv, qb, batch, seq, heads)
    out["qkv_in"], out["qkv_bias"] = qkv, qb
    out["qkv_q"], out["qkv_k"], out["qkv_v"] = q.data.copy(), k.data.copy(), v.data.copy()
    xh, hb = r(batch * seq, d), r(d)
    out["heads_in"], out["heads_bias"] = xh, hb
    out["heads_out"] = ops.fused_bias_reshape_heads(xh, hb, batch, seq, heads).data.copy()
    # embed
    emb, pos = r(50, 16), r(9, 16)
    toks = rng.integers(0, 50, size=12).astype(np.int64)
    out["emb_tab"], out["emb_pos"], out["emb_tok"] = emb, pos, toks
    out["emb_out"] = ops.fused_embed(toks, emb, 4.0, pos, 2, 6).data.copy()
    np.savez_compressed(os.path.join(HERE, "ops_golden.npz"), **out)


def make_retrieve():
    rng = np.random.default_rng(77)
    rows, ks, offs = [], [], [0]
    gm_all, th, lse, ctok, clog, coff = [], [], [], [], [], [0]
    vocab_list = []
    for i in range(310):
        vocab = int(rng.integers(1, 300)) if i < 300 else int(rng.choice([32000, 50257]))
        if i % 3 == 0:
            pool = rng.normal(size=max(vocab // 4, 1))
            row = rng.choice(pool, size=vocab).astype(F32)
        else:
            row = rng.normal(scale=3, size=vocab).astype(F32)
        k = int(rng.integers(1, min(vocab, 20) + 1))
        rr = D.retrieve(row[None, :], k)
        rows.append(row)
        offs.append(offs[-1] + vocab)
        vocab_list.append(vocab)
        ks.append(k)
        gm_all.append(rr.group_maxima[0].copy())
        th.append(float(rr.threshold[0]))
        lse.append(float(rr.logsumexp_full[0]))
        ctok.append(rr.candidate_tokens[0].astype(np.int32))
        clog.append(rr.candidate_logits[0].astype(F32))
        coff.append(coff[-1] + len(rr.candidate_tokens[0]))
    np.savez_compressed(
        os.path.join(HERE, "retrieve_golden.npz"),
        logits=np.concatenate(rows), row_off=np.array(offs, np.int64),
        vocab=np.array(vocab_list, np.int64), k=np.array(ks, np.int64),
        group_max=np.concatenate(gm_all).astype(F32), threshold=np.array(th, F32),
        lse=np.array(lse, np.float64), cand_tok=np.concatenate(ctok),
        cand_logit=np.concatenate(clog), cand_off=np.array(coff, np.int64))


def make_beam():
    """Pure logit-stream beam search (no model), EOS forced at some steps."""
    rng = np.random.default_rng(5)
    out = {}
    cases = []
    for ci in range(24):
        vocab = int(rng.choice([16, 40, 300]))
        beam = int(rng.integers(1, 9))
        steps = int(rng.integers(3, 12))
        alpha = float(rng.choice([0.0, 0.0, 0.6, 1.0]))
        eos = 2
        cfg = D.DecodeConfig(method="beam", beam_size=beam, max_steps=steps, eos_token=eos,
                             length_penalty=alpha)
        st = D.BeamState()
        stream = np.zeros((steps, beam, vocab), F32)
        live_hist = np.zeros(steps, np.int32)
        parents = np.zeros((steps, beam), np.int32)
        tokens = np.zeros((steps, beam), np.int32)
        n_steps = 0
        for t in range(steps):
            lg = rng.normal(scale=2.0, size=(beam, vocab)).astype(F32)
            if ci % 2 == 0 and t >= 1 and rng.random() < 0.5:
                lg[:, eos] += 3.0  # make EOS competitive
            if ci % 5 == 0:
                lg = np.round(lg)  # tie-heavy
            stream[t] = lg
            live_hist[t] = st.live
            st = D.beam_search_step(st, lg[:st.live], cfg)
            parents[t, :st.live] = st.parents
            tokens[t, :st.live] = st.last_tokens
            n_steps = t + 1
            if st.should_stop(cfg) or not st.prefixes:
                break
        fin = st.finalize(cfg)
        ft = np.full((beam, steps + 1), -1, np.int32)
        fs = np.zeros(beam, np.float64)
        fl = np.zeros(beam, np.int32)
        for i, (seq, sc) in enumerate(fin):
            ft[i, :len(seq)] = seq
            fl[i] = len(seq)
            fs[i] = sc
        p = f"c{ci}_"
        out[p + "stream"] = stream[:n_steps]
        out[p + "live"] = live_hist[:n_steps]
        out[p + "parents"] = parents[:n_steps]
        out[p + "tokens"] = tokens[:n_steps]
        out[p + "final_tok"], out[p + "final_len"], out[p + "final_score"] = ft, fl, fs
        out[p + "n_final"] = np.array([len(fin)], np.int32)
        cases.append(dict(vocab=vocab, beam=beam, steps=steps, alpha=alpha, eos=eos,
                          n_steps=n_steps))
    out["cases"] = np.array(json.dumps(cases))
    np.savez_compressed(os.path.join(HERE, "beam_golden.npz"), **out)


TINY_CFGS = [
    dict(num_encoder_layers=2, num_decoder_layers=2, d_model=64, d_ff=128, num_heads=4,
         vocab_size=1000, max_batch=4, max_seq_len=24, max_beam_size=4),
    dict(num_encoder_layers=1, num_decoder_layers=2, d_model=32, d_ff=96, num_heads=2,
         vocab_size=300, max_batch=3, max_seq_len=16, max_beam_size=8, activation="gelu"),
    dict(num_encoder_layers=2, num_decoder_layers=1, d_model=48, d_ff=64, num_heads=3,
         vocab_size=77, max_batch=2, max_seq_len=12, max_beam_size=2, tie_output=False),
]


def make_tiny():
    out = {}
    runs = []
    rng = np.random.default_rng(99)
    for ci, kw in enumerate(TINY_CFGS):
        cfg = M.ModelConfig(**kw)
        w = M.make_random_weights(cfg, seed=10 + ci)
        out[f"m{ci}_wsum"] = weight_checksums(cfg, w)
        sess = Session(cfg, w, engine="fused")
        batch = cfg.max_batch
        seq = int(min(cfg.max_seq_len, 7))
        src = rng.integers(3, cfg.vocab_size, size=(batch, seq)).astype(np.int64)
        lengths = np.array([seq - (b % 3) for b in range(batch)], np.int64)
        out[f"m{ci}_src"], out[f"m{ci}_len"] = src, lengths
        out[f"m{ci}_enc"] = sess.encode(src).copy()
        out[f"m{ci}_enc_masked"] = sess.encode(src, lengths).copy()
        tgt = rng.integers(3, cfg.vocab_size, size=(batch, 5)).astype(np.int64)
        out[f"m{ci}_tgt"] = tgt
        out[f"m{ci}_forced"] = sess.forced_logits(src, tgt, lengths).copy()
        for mi, (method, beam) in enumerate([("beam", cfg.max_beam_size), ("greedy", 1),
                                             ("beam", 2)]):
            for use_len in (False, True):
                dc = D.DecodeConfig(method=method, beam_size=beam, max_steps=10, eos_token=2)
                hyps = sess.generate(src, dc, src_lengths=lengths if use_len else None)
                K = dc.effective_beam_size
                t, l, s, n = pack_hyps(hyps, K, cfg.max_seq_len + 1)
                p = f"m{ci}_g{mi}{int(use_len)}_"
                out[p + "tok"], out[p + "len"], out[p + "score"], out[p + "n"] = t, l, s, n
                runs.append(dict(model=ci, key=p, method=method, beam=beam, lengths=use_len))
    out["cfgs"] = np.array(json.dumps(TINY_CFGS))
    out["runs"] = np.array(json.dumps(runs))
    np.savez_compressed(os.path.join(HERE, "tiny_golden.npz"), **out)


def make_sampling():
    """Sampling generate on the tiny models (only_sampling: python make_golden.py --sampling)."""
    out = {}
    runs = []
    rng = np.random.default_rng(5)
    for ci, kw in enumerate(TINY_CFGS[:2]):
        cfg = M.ModelConfig(**kw)
        w = M.make_random_weights(cfg, seed=10 + ci)
        sess = Session(cfg, w, engine="fused")
        batch = cfg.max_batch
        seq = int(min(cfg.max_seq_len, 6))
        src = rng.integers(3, cfg.vocab_size, size=(batch, seq)).astype(np.int64)
        lengths = np.array([seq - (b % 2) for b in range(batch)], np.int64)
        out[f"m{ci}_src"], out[f"m{ci}_len"] = src, lengths
        for si, (method, kk, pp, seed, eos) in enumerate(
                [("top_k", 5, 1.0, 7, 2), ("top_k", 1, 1.0, 3, 2), ("top_p", 1, 0.9, 11, 2),
                 ("top_p", 1, 0.5, 13, 5), ("top_k", 40, 1.0, 17, 7), ("top_k", 5, 1.0, 7, -1),
                 ("top_p", 1, 0.9, 11, -1)]):
            if eos < 0:  # EOS = a token the eos=2 run samples early for item 1: finished path
                probe = sess.generate(src, D.DecodeConfig(method=method, sample_k=kk,
                                                          sample_p=pp, seed=seed, max_steps=12,
                                                          eos_token=2))
                eos = int(probe[1][0].tokens[3])
            for use_len in (False, True):
                dc = D.DecodeConfig(method=method, sample_k=kk, sample_p=pp, seed=seed,
                                    max_steps=12, eos_token=eos)
                hyps = sess.generate(src, dc, src_lengths=lengths if use_len else None)
                t, l, s, n = pack_hyps(hyps, 1, cfg.max_seq_len + 1)
                p = f"m{ci}_s{si}{int(use_len)}_"
                out[p + "tok"], out[p + "len"], out[p + "score"], out[p + "n"] = t, l, s, n
                runs.append(dict(model=ci, key=p, method=method, sample_k=kk, sample_p=pp,
                                 seed=seed, eos=eos, lengths=use_len))
    out["cfgs"] = np.array(json.dumps(TINY_CFGS[:2]))
    out["runs"] = np.array(json.dumps(runs))
    np.savez_compressed(os.path.join(HERE, "sampling_golden.npz"), **out)


def make_diverse():
    out = {}
    runs = []
    rng = np.random.default_rng(8)
    for ci, kw in enumerate(TINY_CFGS[:2]):
        cfg = M.ModelConfig(**kw)
        w = M.make_random_weights(cfg, seed=10 + ci)
        sess = Session(cfg, w, engine="fused")
        batch = cfg.max_batch
        seq = int(min(cfg.max_seq_len, 6))
        src = rng.integers(3, cfg.vocab_size, size=(batch, seq)).astype(np.int64)
        lengths = np.array([seq - (b % 2) for b in range(batch)], np.int64)
        out[f"m{ci}_src"], out[f"m{ci}_len"] = src, lengths
        variants = [(4, 2, 0.5, 0.0, "hierarchical", False), (4, 4, 1.5, 0.6, "hierarchical", True),
                    (2, 2, 0.0, 0.0, "hierarchical", False), (4, 2, 0.5, 0.0, "exhaustive", True)]
        for vi, (beam, G, lam, alpha, search, use_len) in enumerate(variants):
            beam = min(beam, cfg.max_beam_size)
            dc = D.DecodeConfig(method="diverse_beam", beam_size=beam, diversity_groups=G,
                                diversity_penalty=lam, length_penalty=alpha, max_steps=10,
                                eos_token=2)
            hyps = sess.generate(src, dc, src_lengths=lengths if use_len else None, search=search)
            t, l, sc, n = pack_hyps(hyps, beam, cfg.max_seq_len + 1)
            p = f"m{ci}_d{vi}_"
            out[p + "tok"], out[p + "len"], out[p + "score"], out[p + "n"] = t, l, sc, n
            runs.append(dict(model=ci, key=p, beam=beam, groups=G, penalty=lam, alpha=alpha,
                             search=search, lengths=use_len))
    out["cfgs"] = np.array(json.dumps(TINY_CFGS[:2]))
    out["runs"] = np.array(json.dumps(runs))
    np.savez_compressed(os.path.join(HERE, "diverse_golden.npz"), **out)


CLS_CFGS = [
    dict(num_encoder_layers=2, num_decoder_layers=0, d_model=64, d_ff=128, num_heads=4,
         vocab_size=500, max_batch=6, max_seq_len=16, max_beam_size=1, activation="gelu"),
    dict(num_encoder_layers=1, num_decoder_layers=0, d_model=32, d_ff=64, num_heads=2,
         vocab_size=50, max_batch=5, max_seq_len=9, max_beam_size=1, activation="gelu",
         tie_output=False),
]


def make_classify():
    out = {}
    rng = np.random.default_rng(21)
    for ci, kw in enumerate(CLS_CFGS):
        cfg = M.ModelConfig(**kw)
        w = M.make_random_weights(cfg, seed=30 + ci)
        sess = Session(cfg, w, engine="fused")
        batch, seq = cfg.max_batch, cfg.max_seq_len
        tok = rng.integers(3, cfg.vocab_size, size=(batch, seq)).astype(np.int64)
        lengths = np.array([seq - (b % 4) for b in range(batch)], np.int64)
        out[f"m{ci}_tok"], out[f"m{ci}_len"] = tok, lengths
        for use_len in (False, True):
            lab, prob = sess.classify(tok, lengths if use_len else None)
            out[f"m{ci}_labels{int(use_len)}"] = np.asarray(lab, np.int64)
            out[f"m{ci}_probs{int(use_len)}"] = np.asarray(prob, np.float64)
    out["cfgs"] = np.array(json.dumps(CLS_CFGS))
    np.savez_compressed(os.path.join(HERE, "classify_golden.npz"), **out)


BASE = dict(num_encoder_layers=6, num_decoder_layers=6, d_model=512, d_ff=2048, num_heads=8,
            vocab_size=32000, max_batch=8, max_seq_len=64, max_beam_size=4)
BIG = dict(num_encoder_layers=6, num_decoder_layers=6, d_model=1024, d_ff=4096, num_heads=16,
           vocab_size=32000, max_batch=128, max_seq_len=64, max_beam_size=4)


def make_generate(name, kw, batch, seq, steps):
    cfg = M.ModelConfig(**kw)
    w = M.make_random_weights(cfg, seed=0)
    sess = Session(cfg, w, engine="fused")
    src = synthetic_tokens(batch, seq, cfg.vocab_size, seed=0)
    dc = D.DecodeConfig(method="beam", beam_size=4, max_steps=steps, eos_token=2)
    t0 = time.perf_counter()
    hyps = sess.generate(src, dc)
    el = time.perf_counter() - t0
    t, l, s, n = pack_hyps(hyps, 4, cfg.max_seq_len + 1)
    # encoder memory summary (first item, full) for layer-level parity
    mem = sess.encode(src)
    out = dict(cfg=np.array(cfg_dict(cfg)), src=src, tok=t, len=l, score=s, n=n,
               wsum=weight_checksums(cfg, w), mem_row_sums=mem.astype(np.float64).sum(1),
               mem_item0=mem[:seq].copy(), seconds=np.array([el]))
    # step-0 logits of batch item 0 (one row), via forced_logits with bos
    fl = sess.forced_logits(src[:1], np.ones((1, 1), np.int64))
    out["step0_logits_item0"] = fl[0, 0].copy()
    np.savez_compressed(os.path.join(HERE, f"{name}_golden.npz"), **out)
    print(f"{name}: generate {el:.1f}s")


if __name__ == "__main__":
    if "--sampling" in sys.argv:
        make_sampling()
        make_classify()
        make_diverse()
        print("done")
        sys.exit(0)
    make_sampling()
    make_classify()
    make_diverse()
    make_ops()
    make_retrieve()
    make_beam()
    make_tiny()
    make_generate("c1", BASE, 8, 32, 32)
    if "--big" in sys.argv:
        make_generate("c2", BIG, 128, 64, 64)
    print("done")
