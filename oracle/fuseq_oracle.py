"""CPU oracle for the LightSeq (`fuseq`) inference hot path — TEST INFRASTRUCTURE.

This module is a numpy restatement of the reference algorithm. It is the
checker for the B200 product, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it. Nothing in
``paper_2010_13887_b200/`` imports it.

Parity of this oracle is PINNED: ``tests/test_oracle_golden.py`` checks it
against fixtures produced by running the real reference
(``tests/golden/make_golden.py``) — op outputs, retrieve results, logit
stream beam searches, tiny-model generate/forced-logits, and the
Transformer-base (C1) / Transformer-big (C2) generate hypotheses.

Numerics follow SURVEY.md Appendix A (numba-inferred types of
``pkg/src/fuseq/kernels.py``): float64 statistics in layer norm and softmax,
fp32 ``expf`` with a float64 sum in retrieve, fp32 two-rounding affine
epilogues. GEMMs are numpy ``matmul`` (OpenBLAS SGEMM) exactly as in
``pkg/src/fuseq/tensor.py:179-227``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
from scipy.special import erf as _erf

F32 = np.float32
F64 = np.float64
I64 = np.int64


# ---------------------------------------------------------------------------
# config + weights  (model.py:44-94, :139-164, :214-260, :263-278)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class OracleConfig:
    num_encoder_layers: int
    num_decoder_layers: int
    d_model: int
    d_ff: int
    num_heads: int
    vocab_size: int
    max_batch: int
    max_seq_len: int
    max_beam_size: int
    activation: str = "relu"
    tie_output: bool = True
    ln_eps: float = 1e-5

    @property
    def head_dim(self) -> int:
        return self.d_model // self.num_heads


ENC_FIELDS = ["w_qkv", "b_qkv", "w_out", "b_out", "ln1_gamma", "ln1_beta",
              "w_ff1", "b_ff1", "w_ff2", "b_ff2", "ln2_gamma", "ln2_beta"]
DEC_FIELDS = ["w_qkv", "b_qkv", "w_self_out", "b_self_out", "ln1_gamma", "ln1_beta",
              "w_cross_q", "b_cross_q", "w_cross_k", "b_cross_k", "w_cross_v", "b_cross_v",
              "w_cross_out", "b_cross_out", "ln2_gamma", "ln2_beta",
              "w_ff1", "b_ff1", "w_ff2", "b_ff2", "ln3_gamma", "ln3_beta"]


def make_random_weights(cfg: OracleConfig, seed: int = 0) -> dict:
    """Same generator draws, same order as model.py:214-260: embedding,
    (untied output projection), encoder layers, decoder layers; within a
    layer the dataclass keyword order; layer-norm params are not drawn."""
    rng = np.random.default_rng(seed)
    d, ff = cfg.d_model, cfg.d_ff

    def mat(m, n):
        return rng.normal(0.0, math.sqrt(2.0 / (m + n)), size=(m, n)).astype(F32)

    def vec(n):
        return rng.normal(0.0, 0.02, size=n).astype(F32)

    w = {"token_embedding": rng.normal(0.0, 1.0 / math.sqrt(d),
                                       size=(cfg.vocab_size, d)).astype(F32)}
    if not cfg.tie_output:
        w["output_projection"] = rng.normal(0.0, 1.0 / math.sqrt(d),
                                            size=(cfg.vocab_size, d)).astype(F32)
    ones, zeros = (lambda: np.ones(d, F32)), (lambda: np.zeros(d, F32))
    for i in range(cfg.num_encoder_layers):
        p = f"encoder.{i}."
        w[p + "w_qkv"], w[p + "b_qkv"] = mat(d, 3 * d), vec(3 * d)
        w[p + "w_out"], w[p + "b_out"] = mat(d, d), vec(d)
        w[p + "ln1_gamma"], w[p + "ln1_beta"] = ones(), zeros()
        w[p + "w_ff1"], w[p + "b_ff1"] = mat(d, ff), vec(ff)
        w[p + "w_ff2"], w[p + "b_ff2"] = mat(ff, d), vec(d)
        w[p + "ln2_gamma"], w[p + "ln2_beta"] = ones(), zeros()
    for i in range(cfg.num_decoder_layers):
        p = f"decoder.{i}."
        w[p + "w_qkv"], w[p + "b_qkv"] = mat(d, 3 * d), vec(3 * d)
        w[p + "w_self_out"], w[p + "b_self_out"] = mat(d, d), vec(d)
        w[p + "ln1_gamma"], w[p + "ln1_beta"] = ones(), zeros()
        for nm in ("cross_q", "cross_k", "cross_v", "cross_out"):
            w[p + "w_" + nm], w[p + "b_" + nm] = mat(d, d), vec(d)
        w[p + "ln2_gamma"], w[p + "ln2_beta"] = ones(), zeros()
        w[p + "w_ff1"], w[p + "b_ff1"] = mat(d, ff), vec(ff)
        w[p + "w_ff2"], w[p + "b_ff2"] = mat(ff, d), vec(d)
        w[p + "ln3_gamma"], w[p + "ln3_beta"] = ones(), zeros()
    return w


def canonical_names(cfg: OracleConfig) -> list[str]:
    """model.py:154-164 order."""
    names = ["token_embedding"] + ([] if cfg.tie_output else ["output_projection"])
    names += [f"encoder.{i}.{f}" for i in range(cfg.num_encoder_layers) for f in ENC_FIELDS]
    names += [f"decoder.{i}.{f}" for i in range(cfg.num_decoder_layers) for f in DEC_FIELDS]
    return names


def sinusoidal_positions(max_len: int, d: int) -> np.ndarray:
    """model.py:263-270."""
    pos = np.arange(max_len, dtype=F64)[:, None]
    ang = pos / np.power(10000.0, np.arange(0, d, 2, dtype=F64)[None, :] / d)
    pe = np.zeros((max_len, d), F64)
    pe[:, 0::2] = np.sin(ang)
    pe[:, 1::2] = np.cos(ang[:, : d // 2])
    return pe.astype(F32)


def lengths_mask(lengths, seq: int) -> np.ndarray:
    """model.py:273-278: 0 valid / -inf padding."""
    lengths = np.asarray(lengths, I64)
    m = np.zeros((lengths.shape[0], seq), F32)
    m[np.arange(seq)[None, :] >= lengths[:, None]] = -np.inf
    return m


# ---------------------------------------------------------------------------
# fused kernels  (kernels.py; numerics per SURVEY Appendix A)
# ---------------------------------------------------------------------------

def layer_norm(x, gamma, beta, eps):
    """kernels.py:22-35 (E7): f64 mean/var, F32((x-mean)*inv)*g + b in fp32."""
    x64 = np.asarray(x, F64)
    d = x64.shape[1]
    mean = x64.sum(axis=1, keepdims=True) / d
    t = x64 - mean
    inv = 1.0 / np.sqrt((t * t).sum(axis=1, keepdims=True) / d + eps)
    return (t * inv).astype(F32) * gamma + beta


def bias_residual_act(x, bias, residual, act):
    """kernels.py:39-53 (E9): fp32 x+b, ReLU / f64 erf-GELU, residual added
    after activation as an f64 sum rounded to fp32."""
    t = np.asarray(x, F32) + bias
    if act == "relu":
        t = np.where(t < 0.0, F32(0.0), t)
    elif act == "gelu":
        t64 = t.astype(F64)
        t = (0.5 * t64 * (1.0 + _erf(t64 * (1.0 / math.sqrt(2.0))))).astype(F32)
    if residual is not None:
        t = (t.astype(F64) + np.asarray(residual, F64)).astype(F32)
    return t


def bias_residual_layer_norm(x, bias, residual, gamma, beta, eps):
    """kernels.py:57-73: summand (x+b)+r in two fp32 adds, then E7 norm."""
    u = (np.asarray(x, F32) + bias) + residual
    return layer_norm(u, gamma, beta, eps)


def qkv_bias_reshape(qkv, bias, batch, seq, heads):
    """kernels.py:77-89: [n,3d]+bias -> three [batch, heads, seq, hd]."""
    t = np.asarray(qkv, F32) + bias
    d = t.shape[1] // 3
    hd = d // heads
    return tuple(np.ascontiguousarray(t[:, i * d:(i + 1) * d].reshape(batch, seq, heads, hd)
                                      .transpose(0, 2, 1, 3)) for i in range(3))


def bias_reshape_heads(x, bias, batch, seq, heads):
    """kernels.py:93-102."""
    t = np.asarray(x, F32) + bias
    hd = t.shape[1] // heads
    return np.ascontiguousarray(t.reshape(batch, seq, heads, hd).transpose(0, 2, 1, 3))


def scale_mask_softmax(scores, scale, mask=None):
    """kernels.py:106-139 (E8): fp32 scale (+mask), f64 exp and sum,
    F32(exp * (1/sum)); masked -> 0. Returns (probs, n_fully_masked_rows)."""
    t = np.asarray(scores, F32) * F32(scale)
    if mask is not None:
        m2 = np.asarray(mask, F32).reshape(t.shape[0], t.shape[-1])
        t = t + m2[:, None, None, :]
    m = t.max(axis=-1, keepdims=True).astype(F64)
    bad = int(np.isneginf(m).sum())
    with np.errstate(invalid="ignore"):
        e = np.exp(t.astype(F64) - m)
    e = np.where(np.isneginf(t), 0.0, e)
    inv = 1.0 / e.sum(axis=-1, keepdims=True)
    out = (e * inv).astype(F32)
    return out, bad


def embed_scale_pos(tokens, emb, scale, pos, pos_offset, seq):
    """kernels.py:143-151 (E10): emb*scale then +pos, both fp32."""
    tokens = np.asarray(tokens, I64)
    p = np.arange(tokens.shape[0]) % seq + pos_offset
    return emb[tokens] * F32(scale) + pos[p]


@dataclass
class RetrieveOut:
    group_maxima: np.ndarray
    threshold: np.ndarray
    candidate_tokens: list
    candidate_logits: list
    logsumexp_full: np.ndarray


def retrieve(logits, k):
    """kernels.py:155-185 / decode.py:58-92 (E1): strided group maxima
    (token j -> group j % k), R = min, candidates x >= R ascending,
    lse = f64(row_max) + log(sum_j f64(expf(x_j - row_max)))."""
    L = np.asarray(logits, F32)
    rows, V = L.shape
    if not 1 <= k <= V:
        raise ValueError(f"group count {k} outside [1, {V}]")
    pad = (-V) % k
    Lp = np.concatenate([L, np.full((rows, pad), -np.inf, F32)], axis=1) if pad else L
    gm = Lp.reshape(rows, -1, k).max(axis=1)
    th = gm.min(axis=1)
    rmax = gm.max(axis=1)
    e = np.exp(L - rmax[:, None])           # fp32 subtraction, fp32 exp
    lse = rmax.astype(F64) + np.log(e.astype(F64).sum(axis=1))
    toks, lgs = [], []
    for b in range(rows):
        idx = np.nonzero(L[b] >= th[b])[0].astype(np.int32)
        toks.append(idx)
        lgs.append(L[b, idx])
    return RetrieveOut(gm.astype(F32), th.astype(F32), toks, lgs, lse)


# ---------------------------------------------------------------------------
# sampling output layer  (decode.py:378-430)
# ---------------------------------------------------------------------------

def draw(tokens, probs, rng):
    """decode.py:378-386: r = U * sum(probs) (numpy sum), first prefix with
    cumulative mass >= r (sequential Python float sum)."""
    r = rng.random() * probs.sum()
    c = 0.0
    for t, p in zip(tokens, probs):
        c += p
        if r <= c:
            return int(t)
    return int(tokens[-1])


def _sorted_survivors(rr, b=0):
    toks, lgs = rr.candidate_tokens[b], rr.candidate_logits[b]
    order = np.lexsort((toks, -lgs.astype(F64)))   # (-logit, token)
    return toks[order], lgs[order]


def sample_top_k(row, k, rng):
    """decode.py:399-409: the true top-k from one retrieve with k groups."""
    rr = retrieve(np.atleast_2d(row), min(k, np.shape(row)[-1]))
    toks, lgs = _sorted_survivors(rr)
    toks, lgs = toks[:k], lgs[:k]
    return draw(toks, np.exp(lgs.astype(F64) - rr.logsumexp_full[0]), rng)


def sample_top_p(row, p, rng):
    """decode.py:412-430: survivors of min(32, V) groups, escalated x8 until
    their cumulative mass reaches p; nucleus = shortest sorted prefix >= p."""
    row = np.atleast_2d(row)
    V = row.shape[1]
    groups = min(32, V)
    while True:
        rr = retrieve(row, groups)
        toks, lgs = _sorted_survivors(rr)
        probs = np.exp(lgs.astype(F64) - rr.logsumexp_full[0])
        cum = np.cumsum(probs)
        if cum.size and (cum[-1] >= p or groups == V):
            cut = min(int(np.searchsorted(cum, p, side="left")), cum.size - 1)
            return draw(toks[:cut + 1], probs[:cut + 1], rng)
        groups = min(groups * 8, V)


# ---------------------------------------------------------------------------
# beam state + HARS selection  (decode.py:99-240)
# ---------------------------------------------------------------------------

@dataclass
class OBeamState:
    prefixes: list = field(default_factory=lambda: [[]])
    cum_log_prob: list = field(default_factory=lambda: [0.0])
    finished: list = field(default_factory=list)
    step: int = 0
    parents: list = field(default_factory=lambda: [0])
    last_tokens: list = field(default_factory=list)

    @property
    def live(self):
        return len(self.prefixes)

    def should_stop(self, k, alpha):
        """decode.py:160-171."""
        if not self.prefixes:
            return True
        if len(self.finished) < k:
            return False
        best = max(self.cum_log_prob)
        if alpha:
            best = best / max(self.step, 1) ** alpha
        return best <= self.finished[k - 1][1]

    def finalize(self, k, alpha):
        """decode.py:173-183."""
        out = list(self.finished)
        have = {tuple(s) for s, _ in out}
        for p, c in zip(self.prefixes, self.cum_log_prob):
            if p and tuple(p) not in have:
                out.append((p, c / (len(p) ** alpha) if alpha else c))
        out.sort(key=lambda h: (-h[1], h[0]))
        return out[:k]


def apply_selection(state, picks, eos, alpha, k):
    """decode.py:186-214 (E4)."""
    new = OBeamState(prefixes=[], cum_log_prob=[], finished=list(state.finished),
                     step=state.step + 1, parents=[], last_tokens=[])
    length = state.step + 1
    for cum, tok, parent in picks:
        if tok == eos:
            seq = state.prefixes[parent] + [tok]
            new.finished.append((seq, cum / (length ** alpha) if alpha else cum))
            new.finished.sort(key=lambda h: (-h[1], h[0]))
            del new.finished[k:]
        elif len(new.prefixes) < k:
            new.prefixes.append(state.prefixes[parent] + [tok])
            new.cum_log_prob.append(cum)
            new.parents.append(parent)
            new.last_tokens.append(tok)
        if len(new.prefixes) >= k:
            break
    return new


def beam_search_step(state, logits, k, eos, alpha):
    """decode.py:217-240: groups = min(k+live, V); score = cum + (logit - lse)
    in f64; order (-score, token, beam)."""
    L = np.asarray(logits, F32)
    groups = min(k + state.live, L.shape[1])
    rr = retrieve(L, groups)
    cands = []
    for b in range(state.live):
        base = state.cum_log_prob[b]
        lse = float(rr.logsumexp_full[b])
        for tok, lg in zip(rr.candidate_tokens[b].tolist(), rr.candidate_logits[b].tolist()):
            cands.append((base + (lg - lse), tok, b))
    cands.sort(key=lambda c: (-c[0], c[1], c[2]))
    return apply_selection(state, cands, eos, alpha, k)


def exhaustive_beam_search_step(state, logits, k, eos, alpha):
    """decode.py:243-267: full f64 softmax + stable sort, token-major."""
    L = np.asarray(logits, F32).astype(F64)
    m = L.max(axis=1, keepdims=True)
    lp = L - (m + np.log(np.exp(L - m).sum(axis=1, keepdims=True)))
    scores = np.asarray(state.cum_log_prob, F64)[:, None] + lp
    flat = scores.T.ravel()
    order = np.argsort(-flat, kind="stable")
    live = state.live
    picks = [(float(flat[i]), int(i // live), int(i % live)) for i in order[:k + live]]
    return apply_selection(state, picks, eos, alpha, k)


# ---------------------------------------------------------------------------
# model  (model.py:306-360, :407-445, :452-631)
# ---------------------------------------------------------------------------

class OracleModel:
    def __init__(self, cfg: OracleConfig, weights: dict):
        self.cfg = cfg
        self.w = weights
        self.pos = sinusoidal_positions(cfg.max_seq_len, cfg.d_model)

    def out_matrix(self):
        return self.w["token_embedding" if self.cfg.tie_output else "output_projection"]

    # -- encoder ---------------------------------------------------------
    def encoder_layer(self, x, i, mask, batch):
        """model.py:306-360: 6 GEMM + 6 fused."""
        c, w, p = self.cfg, self.w, f"encoder.{i}."
        n, d = x.shape
        seq, h, hd = n // batch, c.num_heads, c.head_dim
        qkv = x @ w[p + "w_qkv"]
        q4, k4, v4 = qkv_bias_reshape(qkv, w[p + "b_qkv"], batch, seq, h)
        scores = np.matmul(q4, k4.swapaxes(-1, -2))
        probs, bad = scale_mask_softmax(scores, 1.0 / math.sqrt(hd), mask)
        if bad:
            raise ValueError(f"{bad} attention row(s) fully masked")
        ctx = np.matmul(probs, v4).transpose(0, 2, 1, 3).reshape(n, d)
        attn = ctx @ w[p + "w_out"]
        res1 = bias_residual_act(attn, w[p + "b_out"], x, "none")
        norm1 = layer_norm(res1, w[p + "ln1_gamma"], w[p + "ln1_beta"], c.ln_eps)
        ffn_h = bias_residual_act(norm1 @ w[p + "w_ff1"], w[p + "b_ff1"], None, c.activation)
        return bias_residual_layer_norm(ffn_h @ w[p + "w_ff2"], w[p + "b_ff2"], norm1,
                                        w[p + "ln2_gamma"], w[p + "ln2_beta"], c.ln_eps)

    def encode(self, tokens, lengths=None):
        """model.py:407-445."""
        T = np.asarray(tokens, I64)
        batch, seq = T.shape
        mask = lengths_mask(lengths, seq) if lengths is not None else None
        x = embed_scale_pos(T.reshape(-1), self.w["token_embedding"],
                            math.sqrt(self.cfg.d_model), self.pos, 0, seq)
        for i in range(self.cfg.num_encoder_layers):
            x = self.encoder_layer(x, i, mask, batch)
        return x

    def build_cross_kv(self, memory, batch, seq):
        """model.py:515-534."""
        out = []
        for i in range(self.cfg.num_decoder_layers):
            p = f"decoder.{i}."
            ck = bias_reshape_heads(memory @ self.w[p + "w_cross_k"], self.w[p + "b_cross_k"],
                                    batch, seq, self.cfg.num_heads)
            cv = bias_reshape_heads(memory @ self.w[p + "w_cross_v"], self.w[p + "b_cross_v"],
                                    batch, seq, self.cfg.num_heads)
            out.append((ck, cv))
        return out

    # -- decoder ---------------------------------------------------------
    def new_cache(self, rows):
        c = self.cfg
        shape = (rows, c.num_heads, c.max_seq_len, c.head_dim)
        return {"k": [np.zeros(shape, F32) for _ in range(c.num_decoder_layers)],
                "v": [np.zeros(shape, F32) for _ in range(c.num_decoder_layers)],
                "len": 0}

    def decode_step(self, last_tokens, cache, cross, enc_mask, batch, beam, parents=None):
        """model.py:537-631 with KVCache semantics of model.py:452-512:
        the history is gathered by ``parents`` (only when not identity)."""
        c, w = self.cfg, self.w
        T = np.asarray(last_tokens, I64)
        rows = T.shape[0]
        h, hd, d = c.num_heads, c.head_dim, c.d_model
        cur0 = cache["len"]
        if cur0 >= c.max_seq_len:
            raise ValueError("KV cache full")
        if parents is not None:
            p = np.asarray(parents, I64)
            if not np.array_equal(p, np.arange(rows)):
                for i in range(c.num_decoder_layers):
                    cache["k"][i][:, :, :cur0] = cache["k"][i][p, :, :cur0]
                    cache["v"][i][:, :, :cur0] = cache["v"][i][p, :, :cur0]
        x = embed_scale_pos(T, w["token_embedding"], math.sqrt(d), self.pos, cur0, 1)
        cur = cur0 + 1
        scale = 1.0 / math.sqrt(hd)
        for i in range(c.num_decoder_layers):
            p = f"decoder.{i}."
            q4, kn, vn = qkv_bias_reshape(x @ w[p + "w_qkv"], w[p + "b_qkv"], rows, 1, h)
            cache["k"][i][:, :, cur0] = kn[:, :, 0]
            cache["v"][i][:, :, cur0] = vn[:, :, 0]
            kc, vc = cache["k"][i][:, :, :cur], cache["v"][i][:, :, :cur]
            ss, _ = scale_mask_softmax(np.matmul(q4, kc.swapaxes(-1, -2)), scale, None)
            sctx = np.matmul(ss, vc).transpose(0, 2, 1, 3).reshape(rows, d)
            sres = bias_residual_act(sctx @ w[p + "w_self_out"], w[p + "b_self_out"], x, "none")
            snorm = layer_norm(sres, w[p + "ln1_gamma"], w[p + "ln1_beta"], c.ln_eps)
            cq4 = bias_reshape_heads(snorm @ w[p + "w_cross_q"], w[p + "b_cross_q"],
                                     batch, beam, h)
            cs, bad = scale_mask_softmax(np.matmul(cq4, cross[i][0].swapaxes(-1, -2)), scale,
                                         enc_mask)
            if bad:
                raise ValueError("fully masked cross-attention row")
            cctx = np.matmul(cs, cross[i][1]).transpose(0, 2, 1, 3).reshape(rows, d)
            cres = bias_residual_act(cctx @ w[p + "w_cross_out"], w[p + "b_cross_out"], snorm,
                                     "none")
            cnorm = layer_norm(cres, w[p + "ln2_gamma"], w[p + "ln2_beta"], c.ln_eps)
            ffn_h = bias_residual_act(cnorm @ w[p + "w_ff1"], w[p + "b_ff1"], None, c.activation)
            x = bias_residual_layer_norm(ffn_h @ w[p + "w_ff2"], w[p + "b_ff2"], cnorm,
                                         w[p + "ln3_gamma"], w[p + "ln3_beta"], c.ln_eps)
        cache["len"] = cur
        return x @ self.out_matrix().T

    # -- sessions --------------------------------------------------------
    def forced_logits(self, src, tgt, lengths=None):
        """engine.py:227-263."""
        src, tgt = np.asarray(src, I64), np.asarray(tgt, I64)
        batch, seq = src.shape
        mem = self.encode(src, lengths)
        mask = lengths_mask(lengths, seq) if lengths is not None else None
        cross = self.build_cross_kv(mem, batch, seq)
        cache = self.new_cache(batch)
        out = np.empty((batch, tgt.shape[1], self.cfg.vocab_size), F32)
        for t in range(tgt.shape[1]):
            out[:, t] = self.decode_step(tgt[:, t], cache, cross, mask, batch, 1)
        return out

    def generate(self, src, beam_size=4, max_steps=32, eos=2, alpha=0.0, lengths=None,
                 bos=1, method="beam", exhaustive=False, sample_k=1, sample_p=1.0, seed=0):
        """engine.py:81-173 (beam / greedy; top_k / top_p through
        _sampling_step, engine.py:197-216, one PCG64 stream seeded with
        ``seed`` consumed item by item): returns per item a list of
        (tokens, score), best first."""
        src = np.asarray(src, I64)
        batch, seq = src.shape
        sampling = method in ("top_k", "top_p")
        K = 1 if method in ("greedy", "top_k", "top_p") else beam_size
        rng = np.random.default_rng(seed)
        rows = batch * K
        mem = self.encode(src, lengths)
        mask = lengths_mask(lengths, seq) if lengths is not None else None
        cross = self.build_cross_kv(mem, batch, seq)
        cache = self.new_cache(rows)
        step_fn = exhaustive_beam_search_step if exhaustive else beam_search_step
        states = [OBeamState() for _ in range(batch)]
        done = [False] * batch
        tokens = np.full(rows, bos, I64)
        parents = None
        steps = min(max_steps, self.cfg.max_seq_len)
        for t in range(steps):
            logits = self.decode_step(tokens, cache, cross, mask, batch, K, parents)
            parents = np.empty(rows, I64)
            tokens = np.zeros(rows, I64)
            last = t == steps - 1
            for b in range(batch):
                r0 = b * K
                parents[r0:r0 + K] = r0
                if done[b]:
                    continue
                if sampling:
                    old = states[b]
                    tok = (sample_top_k(logits[r0], sample_k, rng) if method == "top_k"
                           else sample_top_p(logits[r0], sample_p, rng))
                    st = OBeamState(prefixes=[old.prefixes[0] + [tok]], cum_log_prob=[0.0],
                                    finished=list(old.finished), step=old.step + 1,
                                    parents=[0], last_tokens=[tok])
                    if tok == eos:
                        st.finished.append((st.prefixes[0], 0.0))
                        st.prefixes = []
                else:
                    st = step_fn(states[b], logits[r0:r0 + states[b].live], K, eos, alpha)
                states[b] = st
                if st.should_stop(K, alpha) or last or not st.prefixes:
                    done[b] = True
                    continue
                for i in range(st.live):
                    parents[r0 + i] = r0 + st.parents[i]
                    tokens[r0 + i] = st.last_tokens[i]
            if all(done):
                break
        return [st.finalize(K, alpha) for st in states]


# ---------------------------------------------------------------------------
# memory plan  (memory_plan.py:78-127) — host algorithm, used by tests
# ---------------------------------------------------------------------------

def build_plan(specs):
    """Greedy first-fit over (name, bytes, first, last), 64-B aligned."""
    def al(n):
        return (n + 63) // 64 * 64
    no_share = sum(s[1] for s in specs)
    order = sorted(range(len(specs)), key=lambda i: (specs[i][2], i))
    assign, placed, arena = {}, [], 0
    for i in order:
        name, nb, f, l = specs[i]
        busy = sorted(assign[p[0]] for p in placed if p[2] <= l and f <= p[3])
        off = 0
        for bo, bs in busy:
            if off + nb <= bo:
                break
            off = max(off, al(bo + bs))
        assign[name] = (off, nb)
        placed.append(specs[i])
        arena = max(arena, off + nb)
    if arena > no_share:
        assign, off = {}, 0
        for name, nb, _, _ in specs:
            assign[name] = (off, nb)
            off += nb
        arena = off
    return assign, arena, no_share
