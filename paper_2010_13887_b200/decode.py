"""HARS output layer on the B200 (reference: pkg/src/fuseq/decode.py).

Stage 1 (``retrieve``) and stage 2 (rerank + beam selection) run on the device
(csrc/fq_hars.cu). The host-facing functions keep the reference's signatures
and return types so callers and tests are unchanged:

* ``retrieve(logits, k)`` -> ``RetrieveResult`` (group maxima, threshold,
  candidates ascending, f64 full-vocabulary logsumexp), decode.py:58-92;
* ``beam_search_step(state, logits, config)`` -> next ``BeamState``,
  decode.py:217-240 (device stage 1 + device stage 2 on one item);
* ``argmax_output``, ``sample_top_k``, ``sample_top_p`` use the device
  retrieve and the reference's host-side draw (decode.py:378-492);
* ``DeviceBeamState`` is the engine's batched, device-resident beam state.

Tie-breaking everywhere: higher score first, then lower token id, then lower
beam index (decode.py:19-20).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _abi
from .errors import DimensionError, EngineError, FullMaskError, ParameterError
from .tensor import OpCounters, as_device, global_counters

F32 = np.float32
BIG_STEPS = 1 << 40  # "no last step" for the standalone beam step


def _ctr(counters) -> OpCounters:
    return counters if counters is not None else global_counters()


def logsumexp(row) -> float:
    """log(sum(exp(row))) via max shift (decode.py:40-44), host f64."""
    r = np.asarray(row, dtype=np.float64)
    m = r.max()
    return float(m + np.log(np.exp(r - m).sum()))


@dataclass
class RetrieveResult:
    """Survivors of the grouped-maximum threshold pass, one set per beam."""

    group_maxima: np.ndarray            # [beams, k]
    threshold: np.ndarray               # [beams]
    candidate_tokens: list              # per beam, int32 token ids (ascending)
    candidate_logits: list              # per beam, float32 logits
    logsumexp_full: np.ndarray          # [beams], float64


def retrieve_device(L: torch.Tensor, k: int, *, d_k=None, out=None, with_group_max=True):
    """Launch stage 1 on a device fp32 [rows, V] view; returns device outputs
    (group_max, threshold, lse, cand_idx, cand_count)."""
    rows, V = L.shape
    dev = L.device
    if out is None:
        gm = torch.empty((rows, max(k, 1)), dtype=torch.float32, device=dev) if with_group_max else None
        th = torch.empty(rows, dtype=torch.float32, device=dev)
        lse = torch.empty(rows, dtype=torch.float64, device=dev)
        ci = torch.empty((rows, V), dtype=torch.int32, device=dev)
        cc = torch.empty(rows, dtype=torch.int64, device=dev)
    else:
        gm, th, lse, ci, cc = out
    _abi.call("fq_retrieve", L.data_ptr(), L.stride(0), rows, V, k, _abi.ptr(d_k), _abi.ptr(gm),
              gm.stride(0) if gm is not None else 0, _abi.ptr(th), lse.data_ptr(), ci.data_ptr(),
              ci.stride(0), cc.data_ptr(), _abi.stream_handle())
    return gm, th, lse, ci, cc


def retrieve(logits, k: int, *, counters: OpCounters | None = None,
             bufs: dict | None = None) -> RetrieveResult:
    """One kernel call: group maxima, threshold, full-vocabulary logsumexp and
    candidate selection, with no vocabulary-sized intermediate (decode.py:58)."""
    L = as_device(logits, torch.float32)
    if L.dim() != 2:
        raise DimensionError(f"logits must be [beams, vocab], got {tuple(L.shape)}")
    beams, vocab = L.shape
    if not 1 <= k <= vocab:
        raise ParameterError(f"group count {k} outside [1, vocab={vocab}]")
    if L.stride(1) != 1:
        L = L.contiguous()
    out = None
    if bufs is not None:
        # reference-style bufs (decode.py _retrieve_bufs: numpy group_max /
        # threshold / lse / cand_idx) are accepted: host arrays are replaced by
        # device ones and a missing cand_count is allocated
        dev = {}
        for name, shape, dt in (("group_max", (beams, k), torch.float32),
                                ("threshold", (beams,), torch.float32),
                                ("lse", (beams,), torch.float64),
                                ("cand_idx", (beams, vocab), torch.int32),
                                ("cand_count", (beams,), torch.int64)):
            b = bufs.get(name)
            if isinstance(b, torch.Tensor) and b.is_cuda and b.dtype == dt:
                dev[name] = b
            else:
                dev[name] = torch.empty(shape, dtype=dt, device=L.device)
        out = (dev["group_max"][:beams, :k], dev["threshold"][:beams], dev["lse"][:beams],
               dev["cand_idx"][:beams, :vocab], dev["cand_count"][:beams])
    gm, th, lse, ci, cc = retrieve_device(L, k, out=out)
    _ctr(counters).count_fused("retrieve", beams * vocab * 4)
    counts = cc.cpu().numpy()
    cmax = int(counts.max()) if beams else 0
    idx = ci[:, :max(cmax, 1)].cpu().numpy()
    Lh = None
    toks, lgs = [], []
    for b in range(beams):
        t = idx[b, :counts[b]].astype(np.int32).copy()
        toks.append(t)
        lgs.append(L[b, torch.from_numpy(t.astype(np.int64)).to(L.device)].cpu().numpy()
                   if t.size else np.zeros(0, F32))
    del Lh
    return RetrieveResult(group_maxima=gm.cpu().numpy(), threshold=th.cpu().numpy(),
                          candidate_tokens=toks, candidate_logits=lgs,
                          logsumexp_full=lse.cpu().numpy())


# ---------------------------------------------------------------------------
# decoding configuration and beam state  (decode.py:99-183)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class DecodeConfig:
    method: str = "beam"              # beam | diverse_beam | top_k | top_p | greedy
    beam_size: int = 4
    diversity_groups: int = 1
    diversity_penalty: float = 0.0
    sample_k: int = 1
    sample_p: float = 1.0
    length_penalty: float = 0.0
    max_steps: int = 32
    eos_token: int = 2
    seed: int = 0

    def validate(self, vocab_size: int, max_beam_size: int):
        if self.method not in ("beam", "diverse_beam", "top_k", "top_p", "greedy"):
            raise ParameterError(f"unknown decode method {self.method!r}")
        k = self.effective_beam_size
        if not 1 <= k <= max_beam_size:
            raise ParameterError(f"beam size {k} outside [1, {max_beam_size}]")
        if not 1 <= self.sample_k <= vocab_size:
            raise ParameterError(f"sample_k {self.sample_k} outside [1, {vocab_size}]")
        if not 0.0 < self.sample_p <= 1.0:
            raise ParameterError(f"sample_p {self.sample_p} outside (0, 1]")
        if self.diversity_penalty < 0:
            raise ParameterError("diversity penalty must be >= 0")
        if self.length_penalty < 0:
            raise ParameterError("length penalty must be >= 0")
        if self.method == "diverse_beam":
            if self.diversity_groups < 1 or k % self.diversity_groups:
                raise ParameterError(
                    f"beam size {k} not divisible by {self.diversity_groups} groups")
        if not 0 <= self.eos_token < vocab_size:
            raise ParameterError(f"eos token {self.eos_token} outside vocabulary")
        if self.max_steps < 1:
            raise ParameterError("max_steps must be >= 1")

    @property
    def effective_beam_size(self) -> int:
        return 1 if self.method in ("greedy", "top_k", "top_p") else self.beam_size


@dataclass
class BeamState:
    """Live beams (score-sorted), finished hypotheses and reorder bookkeeping."""

    prefixes: list = field(default_factory=lambda: [[]])
    cum_log_prob: list = field(default_factory=lambda: [0.0])
    finished: list = field(default_factory=list)
    step: int = 0
    parents: list = field(default_factory=lambda: [0])
    last_tokens: list = field(default_factory=list)
    chosen_tokens: list = field(default_factory=list)

    @property
    def live(self) -> int:
        return len(self.prefixes)

    def next_input_tokens(self, bos: int) -> list:
        return [p[-1] if p else bos for p in self.prefixes]

    def should_stop(self, config: DecodeConfig) -> bool:
        """decode.py:160-171."""
        if not self.prefixes:
            return True
        k = config.effective_beam_size
        if len(self.finished) < k:
            return False
        alpha = config.length_penalty
        best_live = max(self.cum_log_prob)
        if alpha:
            best_live = best_live / max(self.step, 1) ** alpha
        return best_live <= self.finished[k - 1][1]

    def finalize(self, config: DecodeConfig) -> list:
        """Best-first hypotheses; unfinished live beams scored as-is (decode.py:173-183)."""
        out = list(self.finished)
        have = {tuple(seq) for seq, _ in out}
        alpha = config.length_penalty
        for p, c in zip(self.prefixes, self.cum_log_prob):
            if p and tuple(p) not in have:
                out.append((p, c / (len(p) ** alpha) if alpha else c))
        out.sort(key=lambda h: (-h[1], h[0]))
        return out[:config.effective_beam_size]


_PINNED: dict = {}  # pinned host staging buffers for DeviceBeamState.host_items, by size


def check_error_flags(flags: dict | None):
    """Raise the reference's errors for one generate's device flags (read when
    the host reads the state): a fully masked cross-attention row
    (FullMaskError) or a fused logits/HARS survivor overflow (EngineError)."""
    if not flags:
        return
    if any(int(b.item()) for b in flags.get("bad", [])):
        raise FullMaskError("fully masked cross-attention row")
    if any(int(o.item()) for o in flags.get("ovf", [])):
        raise EngineError("more than 2048 candidates in a row (tie-heavy logits) on the fused "
                          "logits/HARS path; set FQ_LOGITS_HARS=0")


class DeviceBeamState:
    """Batched beam state in device memory (fq_beam_state, fq_abi.h)."""

    FIELDS = (("live", torch.int32, "B"), ("step", torch.int32, "B"), ("done", torch.int32, "B"),
              ("prefix", torch.int32, "BKS"), ("cum", torch.float64, "BK"),
              ("fin_count", torch.int32, "B"), ("fin_tok", torch.int32, "BKS"),
              ("fin_len", torch.int32, "BK"), ("fin_score", torch.float64, "BK"),
              ("last_tok", torch.int32, "BK"), ("parent", torch.int32, "BK"),
              ("n_done", torch.int32, "1"))

    def __init__(self, batch: int, beam: int, max_len: int, buffers=None):
        self.batch, self.beam, self.max_len = batch, beam, max_len
        dims = {"B": batch, "K": beam, "S": max_len, "1": 1}
        for name, dt, shape in self.FIELDS:
            shp = tuple(dims[c] for c in shape)
            t = (buffers.get(f"beam.{name}", shp, dt) if buffers is not None
                 else torch.zeros(shp, dtype=dt, device=torch.device("cuda")))
            setattr(self, name, t)
        self.c = _abi.BeamStateC(*[getattr(self, n).data_ptr() for n, _, _ in self.FIELDS])

    def init(self):
        _abi.call("fq_beam_state_init", self.c, self.batch, self.beam, self.max_len,
                  _abi.stream_handle())

    @classmethod
    def from_host(cls, state: BeamState, beam: int, max_len: int) -> "DeviceBeamState":
        ds = cls(1, beam, max_len)
        live = state.live
        pre = np.zeros((1, beam, max_len), np.int32)
        for i, p in enumerate(state.prefixes):
            pre[0, i, :len(p)] = p
        ds.prefix.copy_(torch.from_numpy(pre))
        cum = np.zeros((1, beam)); cum[0, :live] = state.cum_log_prob
        ds.cum.copy_(torch.from_numpy(cum))
        ft = np.zeros((1, beam, max_len), np.int32)
        fl = np.zeros((1, beam), np.int32)
        fs = np.zeros((1, beam))
        for i, (seq, sc) in enumerate(state.finished[:beam]):
            ft[0, i, :len(seq)] = seq
            fl[0, i] = len(seq)
            fs[0, i] = sc
        ds.fin_tok.copy_(torch.from_numpy(ft))
        ds.fin_len.copy_(torch.from_numpy(fl))
        ds.fin_score.copy_(torch.from_numpy(fs))
        ds.fin_count.fill_(min(len(state.finished), beam))
        ds.live.fill_(live)
        ds.step.fill_(state.step)
        ds.done.zero_()
        ds.n_done.zero_()
        return ds

    def to_host(self, b: int) -> BeamState:
        """Item b as a reference BeamState (prefixes, cum, finished, bookkeeping)."""
        return self.host_items()[b]

    def _to_host(self) -> dict:
        """Every field in one pinned staging buffer: async copies, one sync."""
        sizes = [getattr(self, n).numel() * getattr(self, n).element_size()
                 for n, _, _ in self.FIELDS]
        total = sum((z + 63) // 64 * 64 for z in sizes)
        buf = _PINNED.get(total)
        if buf is None:
            buf = _PINNED[total] = torch.empty(total, dtype=torch.uint8, pin_memory=True)
        out, off = {}, 0
        for (n, dt, _), z in zip(self.FIELDS, sizes):
            t = getattr(self, n)
            view = buf[off:off + z].view(dt).view(t.shape)
            view.copy_(t, non_blocking=True)
            out[n] = view
            off += (z + 63) // 64 * 64
        torch.cuda.current_stream().synchronize()
        return {n: v.numpy() for n, v in out.items()}

    error_flags = None  # set by Session.generate: checked when the host reads the state

    def finalize_batch(self, config: DecodeConfig) -> list:
        """[state.finalize(config) for state in host_items()] in one native pass
        over the host copy (fq_finalize_beams): (tokens, score) lists per item."""
        from . import _abi
        check_error_flags(self.error_flags)
        h = self._to_host()
        B, K, S = self.batch, self.beam, self.max_len
        keep = config.effective_beam_size
        ot = np.zeros((B, keep, S), np.int32)
        ol = np.zeros((B, keep), np.int32)
        osc = np.zeros((B, keep), np.float64)
        on = np.zeros(B, np.int32)
        arrs = [np.ascontiguousarray(h[n]) for n in ("live", "step", "prefix", "cum", "fin_count",
                                                      "fin_tok", "fin_len", "fin_score")]
        _abi.call("fq_finalize_beams", *[_np_ptr(a) for a in arrs], B, K, S,
                  float(config.length_penalty), keep, _np_ptr(ot), _np_ptr(ol), _np_ptr(osc),
                  _np_ptr(on))
        # only the used tokens to Python, in one call: ragged (b, i) order
        flat = ot[np.arange(S)[None, None, :] < ol[:, :, None]].tolist()
        offs = np.concatenate([[0], np.cumsum(ol.ravel())]).tolist()
        ll, sl, nl = ol.tolist(), osc.tolist(), on.tolist()
        out = []
        for b in range(B):
            base = b * keep
            out.append([(flat[offs[base + i]:offs[base + i + 1]], sl[b][i]) for i in range(nl[b])])
        return out

    def host_items(self) -> list:
        check_error_flags(self.error_flags)
        h = self._to_host()
        live, step, pre, cum = h["live"], h["step"], h["prefix"], h["cum"]
        fc, ft, fl, fs = h["fin_count"], h["fin_tok"], h["fin_len"], h["fin_score"]
        lt, par = h["last_tok"], h["parent"]
        out = []
        live_l, step_l, fc_l = live.tolist(), step.tolist(), fc.tolist()
        for b in range(self.batch):
            nl, st, nf = live_l[b], step_l[b], fc_l[b]
            lens = fl[b, :nf].tolist()
            toks = ft[b, :nf].tolist()
            fin = [(toks[i][:lens[i]], sc) for i, sc in enumerate(fs[b, :nf].tolist())]
            last = lt[b, :nl].tolist()
            out.append(BeamState(prefixes=pre[b, :nl, :st].tolist(),
                                 cum_log_prob=cum[b, :nl].tolist(), finished=fin, step=st,
                                 parents=par[b, :nl].tolist(), last_tokens=last,
                                 chosen_tokens=list(last)))
        return out


def _np_ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def length_penalty_table(alpha: float, max_len: int, device, out=None):
    """[l ** alpha for l in 0..max_len] from the host's libm (None when alpha == 0),
    so device scores divide by the same doubles as decode.py:170/:203."""
    if not alpha:
        return None
    vals = torch.tensor([float(l) ** alpha for l in range(max_len + 1)], dtype=torch.float64)
    if out is None:
        return vals.to(device)
    out[:max_len + 1].copy_(vals)
    return out


def _device_beam_step(state: BeamState, L: torch.Tensor, config: DecodeConfig, exhaustive: bool,
                      counters=None) -> BeamState:
    k = config.effective_beam_size
    if L.shape[0] != state.live:
        raise DimensionError(f"logits rows {L.shape[0]} != live beams {state.live}")
    if state.live > k:
        raise DimensionError(f"{state.live} live beams exceed beam size {k}")
    V = L.shape[1]
    max_len = state.step + 1
    ds = DeviceBeamState.from_host(state, k, max_len)
    rows = torch.zeros((k, V), dtype=torch.float32, device=L.device)
    rows[:state.live] = L
    dk = torch.empty(k, dtype=torch.int32, device=L.device)
    _abi.call("fq_hars_groups", ds.c, 1, k, V, int(exhaustive), dk.data_ptr(), _abi.stream_handle())
    _, _, lse, ci, cc = retrieve_device(rows, V if exhaustive else k + state.live, d_k=dk,
                                        with_group_max=False)
    _ctr(counters).count_fused("retrieve", state.live * V * 4)
    rt = torch.empty(k, dtype=torch.int64, device=L.device)
    rp = torch.empty(k, dtype=torch.int64, device=L.device)
    lp = length_penalty_table(config.length_penalty, max_len, L.device)
    _abi.call("fq_hars_select", rows.data_ptr(), rows.stride(0), lse.data_ptr(), ci.data_ptr(),
              ci.stride(0), cc.data_ptr(), ds.c, 1, k, V, max_len, config.eos_token,
              _abi.ptr(lp), None, BIG_STEPS, rt.data_ptr(), rp.data_ptr(), None,
              None, 0, _abi.stream_handle())
    return ds.to_host(0)


def beam_search_step(state: BeamState, logits, config: DecodeConfig, *,
                     counters: OpCounters | None = None, bufs: dict | None = None) -> BeamState:
    """One hierarchical beam step (decode.py:217-240): device retrieve with
    groups = min(k + live, V), device rerank/selection. Identical to
    :func:`exhaustive_beam_search_step` on the same logits."""
    return _device_beam_step(state, as_device(logits, torch.float32), config, False, counters)


def exhaustive_beam_search_step(state: BeamState, logits, config: DecodeConfig, *,
                                counters: OpCounters | None = None) -> BeamState:
    """Exhaustive twin (decode.py:243-267): every token is a candidate (groups = V)."""
    return _device_beam_step(state, as_device(logits, torch.float32), config, True, counters)


# ---------------------------------------------------------------------------
# sampling and argmax  (decode.py:378-513): device retrieve + reference draw
# ---------------------------------------------------------------------------

def _draw(tokens, probs, rng) -> int:
    """Inverse-CDF draw over a small renormalised candidate set (decode.py:378-386)."""
    r = rng.random() * probs.sum()
    c = 0.0
    for t, p in zip(tokens, probs):
        c += p
        if r <= c:
            return int(t)
    return int(tokens[-1])


def _sorted_prefix(rr: RetrieveResult, beam: int = 0):
    toks = rr.candidate_tokens[beam]
    lgs = rr.candidate_logits[beam]
    order = np.lexsort((toks, -lgs.astype(np.float64)))
    return toks[order], lgs[order]


def sample_top_k(logits_row, k: int, rng, *, counters=None, bufs=None) -> int:
    """Draw from the renormalised true top-k set (decode.py:399-409)."""
    row = as_device(logits_row, torch.float32).reshape(1, -1)
    vocab = row.shape[1]
    if not 1 <= k <= vocab:
        raise ParameterError(f"top-k {k} outside [1, {vocab}]")
    rr = retrieve(row, min(k, vocab), counters=counters)
    toks, lgs = _sorted_prefix(rr)
    toks, lgs = toks[:k], lgs[:k]
    probs = np.exp(lgs.astype(np.float64) - rr.logsumexp_full[0])
    return _draw(toks, probs, rng)


def sample_top_p(logits_row, p: float, rng, *, counters=None, bufs=None) -> int:
    """Nucleus draw with group-count escalation (decode.py:412-430)."""
    if not 0.0 < p <= 1.0:
        raise ParameterError(f"top-p {p} outside (0, 1]")
    row = as_device(logits_row, torch.float32).reshape(1, -1)
    vocab = row.shape[1]
    groups = min(32, vocab)
    while True:
        rr = retrieve(row, groups, counters=counters)
        toks, lgs = _sorted_prefix(rr)
        probs = np.exp(lgs.astype(np.float64) - rr.logsumexp_full[0])
        cum = np.cumsum(probs)
        if cum.size and (cum[-1] >= p or groups == vocab):
            cut = min(int(np.searchsorted(cum, p, side="left")), cum.size - 1)
            return _draw(toks[:cut + 1], probs[:cut + 1], rng)
        groups = min(groups * 8, vocab)


def argmax_output(logits_row, *, counters=None, bufs=None) -> tuple:
    """Highest-logit label and its exact probability from one retrieve pass (decode.py:485-492)."""
    row = as_device(logits_row, torch.float32).reshape(1, -1)
    rr = retrieve(row, 1, counters=counters)
    label = int(rr.candidate_tokens[0].min())
    prob = float(np.exp(float(rr.group_maxima[0, 0]) - rr.logsumexp_full[0]))
    return label, prob


def perplexity(per_step_logits, target_tokens) -> float:
    """exp of the mean negative log-probability of the targets (decode.py:503-513);
    the logsumexp comes from the device retrieve pass."""
    L = as_device(per_step_logits, torch.float32)
    T = np.asarray(target_tokens, dtype=np.int64).reshape(-1)
    if L.dim() != 2 or L.shape[0] != T.shape[0]:
        raise DimensionError(f"{L.shape[0] if L.dim() == 2 else tuple(L.shape)} logit rows "
                             f"for {T.shape[0]} targets")
    rr = retrieve(L, 1)
    tgt = L[torch.arange(T.shape[0], device=L.device), torch.from_numpy(T).to(L.device)]
    ll = tgt.double().cpu().numpy() - rr.logsumexp_full
    return float(np.exp(-ll.mean()))


# ---------------------------------------------------------------------------
# diverse beam search  (decode.py:274-371): device penalty + device retrieve,
# host group walk over the few survivors
# ---------------------------------------------------------------------------

def _finished_insert(finished: list, seq: list, score: float, cap: int):
    """decode.py:186-189."""
    finished.append((seq, score))
    finished.sort(key=lambda h: (-h[1], h[0]))
    del finished[cap:]


def apply_selection(state: BeamState, picks: list, eos: int, alpha: float, k: int) -> BeamState:
    """decode.py:192-214: score-ordered (cum, token, parent) picks -> next
    state; EOS picks become finished (cum / len^alpha), the rest live until k."""
    new = BeamState(prefixes=[], cum_log_prob=[], finished=list(state.finished),
                    step=state.step + 1, parents=[], last_tokens=[], chosen_tokens=[])
    length = state.step + 1
    for cum, tok, parent in picks:
        if tok == eos:
            seq = state.prefixes[parent] + [tok]
            score = cum / (length ** alpha) if alpha else cum
            _finished_insert(new.finished, seq, score, k)
            new.chosen_tokens.append(tok)
        elif len(new.prefixes) < k:
            new.prefixes.append(state.prefixes[parent] + [tok])
            new.cum_log_prob.append(cum)
            new.parents.append(parent)
            new.last_tokens.append(tok)
            new.chosen_tokens.append(tok)
        if len(new.prefixes) >= k:
            break
    return new


def _walk_group(cands, kg, eos):
    """decode.py:341-353: score-ordered candidates until kg non-EOS picks."""
    picks = []
    non_eos = 0
    for cum, tok, parent in cands:
        picks.append((cum, tok, parent))
        if tok != eos:
            non_eos += 1
            if non_eos >= kg:
                break
    return picks


def _diverse_step(state: BeamState, logits, config: DecodeConfig, exhaustive: bool,
                  counters=None) -> BeamState:
    """decode.py:274-303 (hierarchical :306-320, exhaustive :323-338): groups
    pick in sequence from all live beams' candidates; group g sees the logits
    penalised by lambda * count(token chosen by earlier groups this step)
    (fq_penalize_counts) and skips beam-token pairs already taken. The
    exhaustive twin is the same walk with every token a candidate (groups = V)."""
    L = as_device(logits, torch.float32)
    if L.dim() != 2 or L.shape[0] != state.live:
        raise DimensionError(f"logits rows {L.shape[0]} != live beams {state.live}")
    if L.stride(1) != 1:
        L = L.contiguous()
    k = config.effective_beam_size
    G = config.diversity_groups
    kg = k // G
    lam = config.diversity_penalty
    vocab = L.shape[1]
    counts = np.zeros(vocab, np.int32)
    dcounts = torch.zeros(vocab, dtype=torch.int32, device=L.device)
    pen_buf = torch.empty_like(L)
    taken: set = set()
    all_picks: list = []
    for _ in range(G):
        if lam and counts.any():
            dcounts.copy_(torch.from_numpy(counts))
            _abi.call("fq_penalize_counts", L.data_ptr(), L.stride(0), L.shape[0], vocab,
                      dcounts.data_ptr(), float(np.float32(lam)), pen_buf.data_ptr(),
                      pen_buf.stride(0), _abi.stream_handle())
            _ctr(counters).count_fused("diversity_penalty", L.numel() * 4)
            pen = pen_buf
        else:
            pen = L
        # every beam's top-(taken + kg + live) must survive (decode.py:307-309)
        groups = vocab if exhaustive else min(len(taken) + kg + state.live, vocab)
        rr = retrieve(pen, groups, counters=counters)
        cands = []
        for b in range(state.live):
            base = state.cum_log_prob[b]
            lse = float(rr.logsumexp_full[b])
            for tok, lg in zip(rr.candidate_tokens[b], rr.candidate_logits[b]):
                if (b, int(tok)) not in taken:
                    cands.append((base + (float(lg) - lse), int(tok), b))
        cands.sort(key=lambda c: (-c[0], c[1], c[2]))
        if exhaustive:
            cands = cands[:kg + state.live]
        picks = _walk_group(cands, kg, config.eos_token)
        for cum, tok, parent in picks:
            taken.add((parent, tok))
            counts[tok] += 1
            all_picks.append((cum, tok, parent))
    return apply_selection(state, all_picks, config.eos_token, config.length_penalty, k)


def diverse_beam_search_step(state: BeamState, logits, config: DecodeConfig, *,
                             counters=None, bufs=None) -> BeamState:
    """decode.py:356-359."""
    return _diverse_step(state, logits, config, False, counters)


def exhaustive_diverse_beam_search_step(state: BeamState, logits, config: DecodeConfig, *,
                                        counters=None) -> BeamState:
    """decode.py:362-365."""
    return _diverse_step(state, logits, config, True, counters)


def top_k_set(logits_row, k: int) -> set:
    row = np.asarray(logits_row, np.float64).reshape(-1)
    order = np.lexsort((np.arange(row.size), -row))
    return {int(t) for t in order[:k]}
