"""Inference sessions on the B200 (reference: pkg/src/fuseq/engine.py).

A :class:`Session` owns one HBM arena, one counter set and one timer set
(engine.py:36-59). ``generate`` keeps the reference's semantics
(engine.py:81-173) but runs the whole decode loop on the device:

* encoder + the one-GEMM cross-K/V setup run eagerly (a few dozen launches);
* each decode step — embed, L decoder layers, logits GEMM, HARS stage 1 and
  stage 2 (rerank, beam selection, finished list, stop rule, next-step tokens
  and parents, copy-free KV history update) and the position advance — is
  captured once into a CUDA graph and replayed; nothing in it touches the host;
* the host only polls the "all items done" counter one step behind, through
  pinned memory, to stop early (engine.py:170-171).

``precision="fp32"`` is the exact mode (FFMA GEMMs, f64 softmax/LN
statistics): token ids match the reference CPU implementation.
``precision="fp16"`` is the throughput mode (tcgen05 GEMMs, fp16 weights,
KV cache and GEMM operands, fp32 accumulation and residual stream).
"""

from __future__ import annotations

import dataclasses
import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _abi
from . import decode as D
from . import model as M
from .errors import EngineError, FullMaskError, InputError
from .memory_plan import Arena, batch_buckets, bucket_of, build_plan
from .tensor import OpCounters, Timers, gemm

I64 = np.int64


@dataclass(frozen=True)
class Hypothesis:
    tokens: list
    score: float


class _GroupedBeamState:
    """The device beam states of the item groups of one generate, in item order."""

    def __init__(self, states):
        self.states = states
        self.error_flags = None

    def host_items(self) -> list:
        D.check_error_flags(self.error_flags)
        out = []
        for st in self.states:
            out.extend(st.host_items())
        return out


_ORD_NEG_INF = -2139095041  # -inf as the ordered int of fq_logits_hars' running maxima


class Session:
    def __init__(self, config: M.ModelConfig, weights: M.ModelWeights, engine: str = "fused",
                 share_plan: bool = True, precision: str = "fp32", use_graphs: bool = True,
                 streams: int = 1):
        if engine != "fused":
            raise InputError(f"unknown engine {engine!r} (the B200 product is the fused engine; "
                             "the naive twin is the CPU baseline)")
        if precision not in M.PRECISIONS:
            raise InputError(f"unknown precision {precision!r}")
        if not torch.cuda.is_available():
            raise EngineError("a CUDA device is required (no CPU fallback)")
        _abi.call("fq_prepare")
        weights.validate(config)
        self.config, self.weights, self.engine, self.precision = config, weights, engine, precision
        self.use_graphs = use_graphs
        if streams not in (1, 2):
            raise InputError("streams must be 1 or 2")
        self.streams = streams
        self.counters = OpCounters()
        self.timers = Timers()
        self.dw = M.DeviceWeights.get(config, weights, precision)
        # one plan per batch bucket (shape-bucketed arena), ONE HBM allocation
        # sized for the largest; every request is served from its bucket's plan
        self._buckets = batch_buckets(config.max_batch)
        self._plans = {}
        for b in self._buckets:
            specs = M.plan_intermediates(config, precision, batch=b)
            if not share_plan:
                specs = [dataclasses.replace(s, first_use=0, last_use=1) for s in specs]
            self._plans[b] = build_plan(specs, bucket=(b,))
        self.plan = self._plans[self._buckets[-1]]
        self.arena = Arena(list(self._plans.values()))
        self._buffers = M.ArenaBuffers(self.arena)
        self._graphs: dict = {}
        self._sample_buffers: dict = {}
        self._pinned_done = torch.zeros((max(config.max_seq_len, 1), 2), dtype=torch.int32,
                                        pin_memory=True)
        self._side_stream = torch.cuda.Stream()
        self._buffers2 = None

    def _group_buffers(self):
        """Decode buffers of the second item group (its own arena, same plans)."""
        if self._buffers2 is None:
            self._arena2 = Arena(list(self._plans.values()))
            self._buffers2 = M.ArenaBuffers(self._arena2)
        self._arena2.use(self.arena.plan)
        return self._buffers2

    @staticmethod
    def _next16(step) -> tuple:
        """The fused HARS launch's half outputs for the next step's input:
        fp16 mode its fp16 copy, exact mode its fp16 pair (hi, lo)."""
        if isinstance(step.x16, tuple):
            return step.x16[0].data_ptr(), step.x16[1].data_ptr()
        return _abi.ptr(step.x16), None

    def _use_bucket(self, batch: int):
        """Serve this request's buffers from its batch bucket's plan."""
        if batch > self.config.max_batch:
            raise M.CapacityError(f"batch {batch} exceeds max_batch {self.config.max_batch}")
        self.arena.use(self._plans[bucket_of(max(int(batch), 1), self._buckets)])

    # ------------------------------------------------------------------
    def _encode_dev(self, src: np.ndarray, lengths=None):
        self._use_bucket(src.shape[0])
        return M.encode(src, self.dw, self.config, lengths, buffers=self._buffers,
                        counters=self.counters, timers=self.timers, precision=self.precision,
                        return_half=True)

    def encode(self, tokens, lengths=None) -> np.ndarray:
        """Encoder memory [batch*seq, d_model] (engine.py:62-66), copied to the host."""
        x, _ = self._encode_dev(np.asarray(tokens, dtype=I64), lengths)
        return x.cpu().numpy()

    def _setup_decoder(self, src: np.ndarray, lengths, rows: int):
        batch, seq = src.shape
        memory, memory16 = self._encode_dev(src, lengths)
        packed = M.build_cross_kv(memory, self.dw, self.config, batch, seq, buffers=self._buffers,
                                  counters=self.counters, timers=self.timers,
                                  precision=self.precision, memory16=memory16)
        mask = self._buffers.get("enc.mask", (batch, seq)) if lengths is not None else None
        cache = M.KVCache(self.config, rows, self._buffers, precision=self.precision)
        return packed, mask, cache

    # ------------------------------------------------------------------
    def generate(self, src_tokens, decode_config: D.DecodeConfig, src_lengths=None,
                 bos_token: int = 1, search: str | None = None, *,
                 return_device_state: bool = False, _materialise: bool = False):
        """Encode, then auto-regressively decode every batch item on the device.

        ``src_tokens`` is host [batch, seq] (copied in) or an int64 device
        tensor already resident in HBM (used as is, not range-checked). With
        ``return_device_state`` the final ``DeviceBeamState`` is returned
        instead of host hypotheses (no device->host traffic)."""
        cfg = decode_config
        cfg.validate(self.config.vocab_size, self.config.max_beam_size)
        if isinstance(src_tokens, torch.Tensor) and src_tokens.is_cuda:
            src = src_tokens
        else:
            src = np.asarray(src_tokens, dtype=I64)
        if src.ndim != 2:
            raise InputError(f"source tokens must be [batch, seq], got {tuple(src.shape)}")
        if self.config.num_decoder_layers < 1:
            raise InputError("generation requires a decoder")
        if cfg.method in ("top_k", "top_p"):
            if return_device_state:
                raise EngineError("sampling returns host hypotheses only")
            return self._generate_sampling(src, src_lengths, cfg, bos_token)
        if cfg.method == "diverse_beam":
            if return_device_state:
                raise EngineError("diverse beam search returns host hypotheses only")
            if search not in (None, "hierarchical", "exhaustive"):
                raise InputError(f"unknown search {search!r}")
            return self._generate_diverse(src, src_lengths, cfg, bos_token,
                                          search == "exhaustive")
        if cfg.method not in ("beam", "greedy"):
            raise EngineError(f"decode method {cfg.method!r} is not on the B200 device path yet "
                              "(SURVEY §8(f))")
        if search is None:
            search = "hierarchical"
        if search not in ("hierarchical", "exhaustive"):
            raise InputError(f"unknown search {search!r}")
        if not 0 <= bos_token < self.config.vocab_size:
            raise InputError("bos token outside vocabulary")
        batch, seq = src.shape
        K = cfg.effective_beam_size
        rows = batch * K
        max_steps = min(cfg.max_steps, self.config.max_seq_len)

        packed, mask, cache0 = self._setup_decoder(src, src_lengths, rows)
        V = self.config.vocab_size
        exhaustive = int(search == "exhaustive")
        fused = (not exhaustive and 2 * K <= 32 and V % 4 == 0
                 and self.config.d_model % 4 == 0)
        # Two-group overlap (streams=2, opt-in): the items are split in two
        # halves decoded by two independent chains on two streams inside the
        # step graph (every op is per row / per item, so results are
        # unchanged). Measured on C2: no gain over one chain (the halves'
        # GEMMs keep the same per-SM ingest and double the launches), so the
        # default is one chain.
        ngroups = 2 if (self.streams == 2 and fused and self.use_graphs and batch >= 2) else 1
        # output layer (fp16): the logits GEMM with the HARS stage-1 statistics
        # epilogue + fq_hars_merge_step, the [rows, V] logits never written
        # (C2: 49.5 us GEMM + merge vs 40.7 us GEMM + 39 us HARS).
        # FQ_LOGITS_HARS=0: materialised logits + fq_hars_step
        # exact mode (opt-in, FQ_LOGITS_HARS_X3H=1): the 3xFP16 logits GEMM
        # (128-column tiles) with the same statistics epilogue
        # (fq_logits_hars_x3h); measured slower at C2 than the materialised
        # logits + fq_hars_step (191 vs 130 us: the per-thread statistics on the
        # 128-float row accumulator spill), so off by default
        lh = (fused and os.environ.get("FQ_LOGITS_HARS", "1") != "0" and not _materialise
              and (self.dw.half or os.environ.get("FQ_LOGITS_HARS_X3H") == "1")
              and M.logits_hars_tiles(self.config, self.precision) > 0)
        bounds = [0, batch] if ngroups == 1 else [0, (batch + 1) // 2, batch]
        groups = []
        for g in range(ngroups):
            i0, i1 = bounds[g], bounds[g + 1]
            nb, nr = i1 - i0, (i1 - i0) * K
            bufs = self._buffers if g == 0 else self._group_buffers()
            cache = cache0 if ngroups == 1 else M.KVCache(self.config, nr, bufs,
                                                          precision=self.precision)
            # (exact mode: packed is the [2, n, 2*L*d] fp16 pair planes)
            gp = packed[:, i0 * seq:i1 * seq] if packed.dim() == 3 else packed[i0 * seq:i1 * seq]
            gm = mask[i0:i1] if mask is not None else None
            # the fused LN's row-block exchange needs every CTA of its launch resident:
            # one step chain at a time (not with the two-stream overlap)
            step = M.DecoderStep(self.dw, self.config, nb, K, seq, cache, gp, gm, bufs,
                                 self.counters, self.timers,
                                 fuse_ln=ngroups == 1 or os.environ.get("FQ_FUSE_LN", "slab") ==
                                 "slab")
            st = D.DeviceBeamState(nb, K, self.config.max_seq_len, bufs)
            st.init()
            step.tokens.fill_(bos_token)
            step.bad.zero_()
            if fused:
                step.embed()  # step 0's input; later steps' come from fq_hars_step
            grp = dict(batch=nb, rows=nr, cache=cache, step=step, st=st,
                       hk=bufs.get("hars.k", (nr,), torch.int32),
                       lse=bufs.get("hars.lse", (nr,), torch.float64),
                       ci=bufs.get("hars.cand_idx", (nr, V), torch.int32),
                       cc=bufs.get("hars.cand_count", (nr,), torch.int64),
                       parents=bufs.get("dec.parents", (nr,), torch.int64),
                       lp=D.length_penalty_table(
                           cfg.length_penalty, self.config.max_seq_len, None,
                           out=bufs.get("hars.len_pow", (self.config.max_seq_len + 1,),
                                        torch.float64)))
            if fused:
                grp["hcnt"] = bufs.get("hars.counters", (nb + 1 + nr,), torch.int32)
                grp["hcnt"].zero_()
            if fused and lh:  # fused logits + HARS stage 1 (the logits never materialised)
                ldt = M.logits_hars_tiles(self.config, self.precision)
                grp["ldt"] = ldt
                grp["gmax"] = bufs.get("hars.gmax", (nr, 32), torch.int32)
                grp["gmax"].fill_(_ORD_NEG_INF)
                grp["tmax"] = bufs.get("hars.tmax", (nr, ldt), torch.float32)
                grp["tsum"] = bufs.get("hars.tsum", (nr, ldt), torch.float64)
                grp["svcnt"] = bufs.get("hars.svcnt", (nr, ldt), torch.int32)
                grp["sv"] = bufs.get("hars.sv", (nr, ldt, M.LH_SV_CAP, 2), torch.int32)
                grp["ovf"] = bufs.get("hars.ovf", (1,), torch.int32)
                grp["ovf"].zero_()
                _abi.call("fq_hars_groups", st.c, nb, K, V, 0, grp["hk"].data_ptr(),
                          _abi.stream_handle())
            groups.append(grp)

        def body(gr):
            step, st, cache = gr["step"], gr["st"], gr["cache"]
            nb, nr = gr["batch"], gr["rows"]
            lse, ci, cc, hk, parents, lp = (gr[k] for k in ("lse", "ci", "cc", "hk", "parents",
                                                           "lp"))
            stream = _abi.stream_handle()
            if fused and lh:
                # layers, then the logits GEMM whose epilogue emits HARS stage-1
                # statistics, then the per-row merge + stage 2 + next embedding
                step.run(embed=False, logits=False)
                d = self.config.d_model
                if self.dw.half:
                    _abi.call("fq_logits_hars", step.x16.data_ptr(), d,
                              self.dw.out_proj.data_ptr(), self.dw.out_proj.stride(0), nr, V, d,
                              hk.data_ptr(), gr["gmax"].data_ptr(), gr["tmax"].data_ptr(),
                              gr["tsum"].data_ptr(), gr["ldt"], gr["svcnt"].data_ptr(),
                              gr["sv"].data_ptr(), M.LH_SV_CAP, stream)
                else:  # exact mode: the step's fp16 pair x16 (written by the last LN)
                    xh, xl = step.x16
                    E = self.dw.out_xh
                    _abi.call("fq_logits_hars_x3h", xh.data_ptr(), xl.data_ptr(), xh.stride(0),
                              E.hi.data_ptr(), E.lo.data_ptr(), E.hi.stride(0), nr, V, d,
                              hk.data_ptr(), gr["gmax"].data_ptr(), gr["tmax"].data_ptr(),
                              gr["tsum"].data_ptr(), gr["ldt"], gr["svcnt"].data_ptr(),
                              gr["sv"].data_ptr(), M.LH_SV_CAP, stream)
                _abi.call("fq_hars_merge_step", st.c, nb, K, V, self.config.max_seq_len,
                          cfg.eos_token, _abi.ptr(lp), cache.d_cur.data_ptr(), max_steps,
                          hk.data_ptr(), gr["gmax"].data_ptr(), gr["tmax"].data_ptr(),
                          gr["tsum"].data_ptr(), gr["ldt"], gr["ldt"], gr["svcnt"].data_ptr(),
                          gr["sv"].data_ptr(), M.LH_SV_CAP, lse.data_ptr(), ci.data_ptr(),
                          ci.stride(0),
                          cc.data_ptr(), gr["hcnt"].data_ptr(), gr["ovf"].data_ptr(),
                          step.tokens.data_ptr(), parents.data_ptr(), cache.hist.data_ptr(),
                          self.dw.embedding.data_ptr(), d,
                          float(np.float32(math.sqrt(d))), self.dw.positions.data_ptr(),
                          step.x.data_ptr(), *self._next16(step), stream)
                self.counters.count_fused("logits_hars", nr * gr["ldt"] * 12)
                return
            logits = step.run(embed=not fused)
            if fused:  # groups + stage 1 + stage 2 + position advance + next embedding
                _abi.call("fq_hars_step", logits.data_ptr(), logits.stride(0), st.c, nb, K, V,
                          self.config.max_seq_len, cfg.eos_token, _abi.ptr(lp),
                          cache.d_cur.data_ptr(), max_steps, lse.data_ptr(), ci.data_ptr(),
                          ci.stride(0), cc.data_ptr(), gr["hcnt"].data_ptr(),
                          step.tokens.data_ptr(), parents.data_ptr(), cache.hist.data_ptr(),
                          self.dw.embedding.data_ptr(), self.config.d_model,
                          float(np.float32(math.sqrt(self.config.d_model))),
                          self.dw.positions.data_ptr(), step.x.data_ptr(),
                          *self._next16(step), stream)
                self.counters.count_fused("retrieve", nr * V * 4)
                return
            _abi.call("fq_hars_groups", st.c, nb, K, V, exhaustive, hk.data_ptr(), stream)
            # k bound for the per-row group counts min(K + live, V) (exhaustive: V)
            D.retrieve_device(logits, V if exhaustive else min(2 * K, V), d_k=hk,
                              out=(None, None, lse, ci, cc))
            self.counters.count_fused("retrieve", nr * V * 4)
            _abi.call("fq_hars_select", logits.data_ptr(), logits.stride(0), lse.data_ptr(),
                      ci.data_ptr(), ci.stride(0), cc.data_ptr(), st.c, nb, K, V,
                      self.config.max_seq_len, cfg.eos_token, _abi.ptr(lp),
                      cache.d_cur.data_ptr(), max_steps, step.tokens.data_ptr(),
                      parents.data_ptr(), cache.hist.data_ptr(), None, 0, stream)
            _abi.call("fq_step_advance", cache.d_cur.data_ptr(), stream)

        def body_all():
            if ngroups == 1:
                body(groups[0])
                return
            main = torch.cuda.current_stream()
            side = self._side_stream
            side.wait_stream(main)
            body(groups[0])
            with torch.cuda.stream(side):
                body(groups[1])
            main.wait_stream(side)

        # every path choice the captured graph bakes in is part of the key
        key = (batch, seq, K, max_steps, mask is not None, exhaustive, cfg.eos_token,
               float(cfg.length_penalty), ngroups, lh, fused,
               groups[0]["step"].ln_ws is not None, groups[0]["step"].q_slabs)
        graph = None
        if self.use_graphs:
            entry = self._graphs.get(key)
            if entry is None:
                graph = torch.cuda.CUDAGraph()
                n0 = _abi.launch_count()
                with torch.cuda.graph(graph):
                    body_all()
                entry = (graph, _abi.launch_count() - n0)
                _abi.add_launches(-entry[1])  # captured, not launched
                self._graphs[key] = entry
            graph, per_step = entry
        pinned = self._pinned_done
        events = []
        for t in range(max_steps):
            if graph is not None:
                graph.replay()
                _abi.add_launches(per_step)
            else:
                body_all()
            for g, gr in enumerate(groups):
                pinned[t, g:g + 1].copy_(gr["st"].n_done, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            events.append(ev)
            if t >= 1:
                events[t - 1].synchronize()
                if int(pinned[t - 1, :ngroups].sum()) >= batch:
                    break
        if lh and any(int(g["ovf"].item()) for g in groups):
            # a tie-heavy row overflowed the fused output layer's survivor slots
            # (e.g. all-equal logits make every token a candidate, reference
            # tests/test_decode.py:53-59): decode the request again on the
            # materialised logits + fq_hars_step path, which has no cap
            return self.generate(src_tokens, decode_config, src_lengths, bos_token, search,
                                 return_device_state=return_device_state, _materialise=True)
        result = groups[0]["st"] if ngroups == 1 else _GroupedBeamState([g["st"] for g in groups])
        # the device error flags travel with the state: checked when the host
        # reads it (host_items), or here for host hypotheses
        result.error_flags = {"bad": [g["step"].bad for g in groups],
                              "ovf": [g["ovf"] for g in groups if "ovf" in g]}
        if return_device_state:
            return result
        if isinstance(result, D.DeviceBeamState):  # finalize natively from the host copy
            return [[Hypothesis(tokens=s, score=sc) for s, sc in item]
                    for item in result.finalize_batch(cfg)]
        states = result.host_items()
        return [[Hypothesis(tokens=s, score=sc) for s, sc in state.finalize(cfg)]
                for state in states]

    # ------------------------------------------------------------------
    def _sample_bufs(self, batch: int, max_steps: int, V: int) -> dict:
        """Persistent device buffers of the device-resident sampling loop (one
        set per (batch, max_steps) shape, allocated on first use)."""
        key = (batch, max_steps)
        b = self._sample_buffers.get(key)
        if b is None and len(self._sample_buffers) >= 4:  # bounded: drop the oldest shape
            old = next(iter(self._sample_buffers))
            del self._sample_buffers[old]
            for gk in [gk for gk in self._graphs if gk[0] == "sample" and gk[1] == old[0]
                       and gk[3] == old[1]]:
                del self._graphs[gk]  # its graph points at the dropped buffers
        if b is None:
            dev = torch.device("cuda", torch.cuda.current_device())
            i32 = dict(dtype=torch.int32, device=dev)
            b = {"uniforms": torch.empty(batch * max_steps, dtype=torch.float64, device=dev),
                 "draw": torch.zeros(1, dtype=torch.int64, device=dev),
                 "done": torch.zeros(2, batch, **i32), "dk": torch.zeros(batch, **i32),
                 "out_tok": torch.zeros(batch, max_steps, **i32),
                 "out_len": torch.zeros(batch, **i32), "fin": torch.zeros(batch, **i32),
                 "counters": torch.zeros(2, **i32), "err": torch.zeros(1, **i32),
                 "lse": torch.empty(batch, dtype=torch.float64, device=dev),
                 "ci": torch.empty(batch, V, **i32),
                 "cc": torch.empty(batch, dtype=torch.int64, device=dev),
                 "pinned": torch.zeros(max_steps, dtype=torch.int32).pin_memory()}
            self._sample_buffers[key] = b
        return b

    def _generate_sampling_device(self, src, src_lengths, cfg: D.DecodeConfig, bos_token: int):
        """Top-k / top-p sampling with the whole step on the device (SURVEY
        §8(f)2): decoder step -> batched retrieve (per-row group counts, 0 for
        done rows) -> fq_sample_step, captured as one CUDA graph per step and
        replayed with the host polling the live-row count one step behind. The
        draws are the reference's: its seeded PCG64 stream is generated on the
        host up front (numpy's random(n) equals n successive random() calls)
        and consumed on the device in its order. Returns None when a row
        overflowed the device's survivor cap or a top-p row's survivors miss
        the nucleus (the reference escalates the group count x8): the caller
        re-runs the request on the host-driven path."""
        batch, seq = src.shape
        V = self.config.vocab_size
        max_steps = min(cfg.max_steps, self.config.max_seq_len)
        top_p = cfg.method == "top_p"
        k = 0 if top_p else min(cfg.sample_k, V)
        g0 = min(32, V) if top_p else k  # retrieve group count of a live row
        packed, mask, cache = self._setup_decoder(src, src_lengths, batch)
        step = M.DecoderStep(self.dw, self.config, batch, 1, seq, cache, packed, mask,
                             self._buffers, self.counters, self.timers)
        step.bad.zero_()
        b = self._sample_bufs(batch, max_steps, V)
        rng = np.random.default_rng(cfg.seed)
        b["uniforms"].copy_(torch.from_numpy(rng.random(batch * max_steps)))
        for n in ("draw", "done", "out_len", "fin", "counters", "err"):
            b[n].zero_()
        b["dk"].fill_(g0)
        step.tokens.fill_(bos_token)

        def body():  # (stream handle read inside: graph capture runs on a side stream)
            logits = step.run()
            D.retrieve_device(logits, g0, d_k=b["dk"], out=(None, None, b["lse"], b["ci"], b["cc"]))
            self.counters.count_fused("retrieve", batch * V * 4)
            _abi.call("fq_sample_step", logits.data_ptr(), logits.stride(0),
                      b["lse"].data_ptr(), b["ci"].data_ptr(), b["ci"].stride(0),
                      b["cc"].data_ptr(), batch, k, float(cfg.sample_p), g0, V, cfg.eos_token,
                      b["uniforms"].data_ptr(),
                      b["uniforms"].numel(), b["draw"].data_ptr(), b["done"].data_ptr(),
                      cache.d_cur.data_ptr(), max_steps, max_steps, b["dk"].data_ptr(),
                      step.tokens.data_ptr(), b["out_tok"].data_ptr(), b["out_len"].data_ptr(),
                      b["fin"].data_ptr(), b["counters"].data_ptr(), b["err"].data_ptr(),
                      _abi.stream_handle())

        graph = None
        if self.use_graphs:
            key = ("sample", batch, seq, max_steps, k, float(cfg.sample_p) if top_p else None,
                   cfg.eos_token, mask is not None)
            entry = self._graphs.get(key)
            if entry is None:
                graph = torch.cuda.CUDAGraph()
                n0 = _abi.launch_count()
                with torch.cuda.graph(graph):
                    body()
                entry = (graph, _abi.launch_count() - n0)
                _abi.add_launches(-entry[1])
                self._graphs[key] = entry
            graph, per_step = entry
        pinned = b["pinned"]
        events = []
        for t in range(max_steps):
            if graph is not None:
                graph.replay()
                _abi.add_launches(per_step)
            else:
                body()
            pinned[t:t + 1].copy_(b["counters"][1:2], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            events.append(ev)
            if t >= 1:
                events[t - 1].synchronize()
                if int(pinned[t - 1]) == 0:
                    break
        torch.cuda.synchronize()
        if int(step.bad.item()):
            raise FullMaskError("fully masked cross-attention row")
        self.last_sampling_err = int(b["err"].item())  # 1 cap, 2 uniforms, 3 nucleus
        if self.last_sampling_err:
            return None
        toks = b["out_tok"].cpu().numpy()
        lens = b["out_len"].cpu().numpy()
        out = []
        for i in range(batch):
            seq_i = [int(x) for x in toks[i, :lens[i]]]
            out.append([Hypothesis(tokens=seq_i, score=0.0)] if seq_i else [])
        return out

    def _generate_sampling(self, src, src_lengths, cfg: D.DecodeConfig, bos_token: int):
        """Top-k / top-p sampling generate (engine.py:175-195 + _sampling_step
        :197-216, decode.py:378-430). Every step: the device decoder step over
        all rows, ONE batched device retrieve (per-row group counts: done rows
        0), the candidates (a few per row) copied to the host, and the
        reference's own draw there: one seeded PCG64 stream consumed item by
        item in order, sorted prefix (-logit, token), probs exp(logit - lse)
        in f64, inverse-CDF walk. Top-p rows whose survivors miss the nucleus
        escalate their group count x8 with a per-row retrieve (:420-430)."""
        if isinstance(src, torch.Tensor):
            src = src.cpu().numpy()
        self.last_sampling_path = "host"
        if os.environ.get("FQ_SAMPLE_HOST") != "1":
            got = self._generate_sampling_device(src, src_lengths, cfg, bos_token)
            if got is not None:
                self.last_sampling_path = "device"
                return got
        batch, seq = src.shape
        V = self.config.vocab_size
        max_steps = min(cfg.max_steps, self.config.max_seq_len)
        packed, mask, cache = self._setup_decoder(src, src_lengths, batch)
        step = M.DecoderStep(self.dw, self.config, batch, 1, seq, cache, packed, mask,
                             self._buffers, self.counters, self.timers)
        step.bad.zero_()
        rng = np.random.default_rng(cfg.seed)
        states = [D.BeamState() for _ in range(batch)]
        done = [False] * batch
        tokens = np.full(batch, bos_token, dtype=I64)
        dk = torch.empty(batch, dtype=torch.int32, device="cuda")
        stream = _abi.stream_handle()
        for t in range(max_steps):
            step.tokens.copy_(torch.from_numpy(tokens))
            logits = step.run()
            live = [b for b in range(batch) if not done[b]]
            g0 = min(cfg.sample_k, V) if cfg.method == "top_k" else min(32, V)
            kv = np.zeros(batch, np.int32)
            kv[live] = g0
            dk.copy_(torch.from_numpy(kv))
            _, _, lse, ci, cc = D.retrieve_device(logits, g0, d_k=dk, with_group_max=False)
            self.counters.count_fused("retrieve", batch * V * 4)
            cnt = cc.cpu().numpy()
            w = int(min(cnt.max(initial=0), V))
            toks_h = ci[:, :max(w, 1)].cpu().numpy()
            lg_h = logits.gather(1, ci[:, :max(w, 1)].long().clamp(0, V - 1)).cpu().numpy()
            lse_h = lse.cpu().numpy()
            _abi.call("fq_step_advance", cache.d_cur.data_ptr(), stream)
            last = t == max_steps - 1
            tokens = np.zeros(batch, dtype=I64)
            for b in live:
                n = int(cnt[b])
                toks, lgs = toks_h[b, :n].astype(np.int64), lg_h[b, :n]
                if cfg.method == "top_k":
                    order = np.lexsort((toks, -lgs.astype(np.float64)))
                    toks, lgs = toks[order][:cfg.sample_k], lgs[order][:cfg.sample_k]
                    probs = np.exp(lgs.astype(np.float64) - lse_h[b])
                    tok = D._draw(toks, probs, rng)
                else:
                    tok = self._top_p_row(logits[b:b + 1], toks, lgs, float(lse_h[b]), g0, cfg,
                                          rng)
                st = states[b]
                new = D.BeamState(prefixes=[st.prefixes[0] + [tok]], cum_log_prob=[0.0],
                                  finished=list(st.finished), step=st.step + 1, parents=[0],
                                  last_tokens=[tok], chosen_tokens=[tok])
                if tok == cfg.eos_token:
                    new.finished.append((new.prefixes[0], 0.0))
                    new.prefixes = []
                states[b] = new
                if new.should_stop(cfg) or last or not new.prefixes:
                    done[b] = True
                    continue
                tokens[b] = tok
            if all(done):
                break
        torch.cuda.synchronize()
        if int(step.bad.item()):
            raise FullMaskError("fully masked cross-attention row")
        return [[Hypothesis(tokens=s_, score=sc) for s_, sc in st.finalize(cfg)]
                for st in states]

    def _generate_diverse(self, src, src_lengths, cfg: D.DecodeConfig, bos_token: int,
                          exhaustive: bool):
        """Diverse beam search generate (engine.py:81-173 with
        diverse_beam_search_step, decode.py:274-371): the device decoder step
        over all rows with the copy-free KV history reordered by the parents;
        per item and group the device penalty (fq_penalize_counts) and the
        device retrieve, the group walk over the survivors on the host."""
        if isinstance(src, torch.Tensor):
            src = src.cpu().numpy()
        batch, seq = src.shape
        K = cfg.effective_beam_size
        rows = batch * K
        max_steps = min(cfg.max_steps, self.config.max_seq_len)
        packed, mask, cache = self._setup_decoder(src, src_lengths, rows)
        step = M.DecoderStep(self.dw, self.config, batch, K, seq, cache, packed, mask,
                             self._buffers, self.counters, self.timers)
        step.bad.zero_()
        states = [D.BeamState() for _ in range(batch)]
        done = [False] * batch
        tokens = np.full(rows, bos_token, dtype=I64)
        parents = None
        fn = D.exhaustive_diverse_beam_search_step if exhaustive else D.diverse_beam_search_step
        for t in range(max_steps):
            cache.begin_step(parents)
            step.tokens.copy_(torch.from_numpy(tokens))
            logits = step.run()
            cache.end_step()
            parents = np.empty(rows, dtype=I64)
            tokens = np.zeros(rows, dtype=I64)
            last = t == max_steps - 1
            for b in range(batch):
                row0 = b * K
                parents[row0:row0 + K] = row0
                if done[b]:
                    continue
                st = fn(states[b], logits[row0:row0 + states[b].live], cfg,
                        counters=self.counters)
                states[b] = st
                if st.should_stop(cfg) or last or not st.prefixes:
                    done[b] = True
                    continue
                for i in range(st.live):
                    parents[row0 + i] = row0 + st.parents[i]
                    tokens[row0 + i] = st.last_tokens[i]
            if all(done):
                break
        torch.cuda.synchronize()
        if int(step.bad.item()):
            raise FullMaskError("fully masked cross-attention row")
        return [[Hypothesis(tokens=s_, score=sc) for s_, sc in st.finalize(cfg)]
                for st in states]

    def _top_p_row(self, row, toks, lgs, lse, groups, cfg, rng) -> int:
        """decode.py:412-430 on one row: survivors of `groups` groups sorted by
        (-logit, token); escalate x8 until they hold the nucleus mass."""
        V = self.config.vocab_size
        while True:
            order = np.lexsort((toks, -lgs.astype(np.float64)))
            toks, lgs = toks[order], lgs[order]
            probs = np.exp(lgs.astype(np.float64) - lse)
            cum = np.cumsum(probs)
            if cum.size and (cum[-1] >= cfg.sample_p or groups == V):
                cut = min(int(np.searchsorted(cum, cfg.sample_p, side="left")), cum.size - 1)
                return D._draw(toks[:cut + 1], probs[:cut + 1], rng)
            groups = min(groups * 8, V)
            rr = D.retrieve(row, groups, counters=self.counters)
            toks = rr.candidate_tokens[0].astype(np.int64)
            lgs = rr.candidate_logits[0]
            lse = float(rr.logsumexp_full[0])

    # ------------------------------------------------------------------
    def forced_logits(self, src_tokens, tgt_tokens, src_lengths=None) -> np.ndarray:
        """Teacher-forced per-position decoder logits [batch, tgt_len, vocab]
        (engine.py:227-263)."""
        src = np.asarray(src_tokens, dtype=I64)
        tgt = np.asarray(tgt_tokens, dtype=I64)
        batch, seq = src.shape
        if tgt.ndim != 2 or tgt.shape[0] != batch:
            raise InputError(f"target tokens must be [batch, steps], got {tgt.shape}")
        M._check_tokens(tgt, self.config)
        packed, mask, cache = self._setup_decoder(src, src_lengths, batch)
        step = M.DecoderStep(self.dw, self.config, batch, 1, seq, cache, packed, mask,
                             self._buffers, self.counters, self.timers)
        step.bad.zero_()
        out = np.empty((batch, tgt.shape[1], self.config.vocab_size), np.float32)
        for t in range(tgt.shape[1]):
            if cache.current_len >= cache.max_seq_len:
                raise M.CapacityError(f"KV cache full at {cache.current_len} positions")
            step.tokens.copy_(torch.from_numpy(tgt[:, t]))
            logits = step.run()
            out[:, t] = logits.cpu().numpy()
            cache.end_step()
        if int(step.bad.item()):
            raise FullMaskError("fully masked cross-attention row")
        return out

    # ------------------------------------------------------------------
    def classify(self, tokens, lengths=None) -> tuple:
        """Encoder-only classification: first-position pooling, output
        projection, argmax via the retrieve pass (engine.py:198-224)."""
        T = np.asarray(tokens, dtype=I64)
        batch, seq = T.shape
        memory, memory16 = self._encode_dev(T, lengths)
        d, V = self.config.d_model, self.config.vocab_size
        pooled = memory.view(batch, seq, d)[:, 0, :].contiguous()
        logits = torch.empty((batch, V), dtype=torch.float32, device=memory.device)
        if self.dw.half:
            gemm(pooled.to(torch.float16), self.dw.out_proj, logits, transpose_b=True,
                 counters=self.counters)
        else:
            gemm(pooled, self.dw.out_proj, logits, transpose_b=True, counters=self.counters)
        gm, _, lse, ci, cc = D.retrieve_device(logits, 1)
        labels = ci[:, 0].long().cpu().numpy().astype(I64)   # lowest index among ties
        probs = np.exp(gm[:, 0].double().cpu().numpy() - lse.cpu().numpy())
        return labels, probs

    def plan_report(self) -> dict | None:
        return self.plan.report()
