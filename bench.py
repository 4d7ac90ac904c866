#!/usr/bin/env python
"""Benchmark: decoded tokens/s for Transformer-big beam-4 translation (BASELINE.json
config 2: 6+6 layers, d=1024, 16 heads, ff=4096, V=32000, batch 128, src 64,
64 decode steps) through the B200 device engine, plus the HARS step microbench.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--precision fp32|fp16] [--batch B] [--scaling strong|weak]

One "step" = one full request: encoder + cross-K/V + 64 decode steps with HARS
beam search over the batch (seeded random-init weights of the architecture,
synthetic_tokens-style source ids, reference bench.py:62-66).

Headline (`value`, `e2e`): the exact fp32 mode (`precision="fp32"`: 3xFP16
tcgen05 GEMMs on fp16 operand pairs with 22-bit precision, the reference's
fp32/f64 elementwise numerics), the precision whose tokens
are pinned bit-exact to the reference at this very config
(tests/test_gpu_c2.py). The half-precision throughput mode is reported beside
it under `half_mode` with its own roofline.

Multi-GPU (torchrun, one process per GPU): `--scaling strong` (default) splits
the 128-item batch into contiguous shards (replicas.batch_shard);
`weak` gives every rank its own 128 items. No collective on the data path;
value = all tokens / max-over-ranks time.

Timing: W untimed warm-up requests, then exactly K, each bracketed by CUDA
events on the launching stream, with a >L2 (256 MiB) buffer written before
every request (outside the events); barrier + synchronize around the timed
region. Kernel-family shares and the roofline come from one extra request
profiled with CUPTI (torch.profiler) with programmatic dependent launch off,
so kernel durations do not overlap.

`--impl reference` times the reference itself (`fuseq`, installed into
baseline/_ref from /root/reference; pure Python + numba + OpenBLAS) on the host
cores, rank 0 only: each timed step decodes 16 of the 128 C2 items (the steps
rotate through the batch), all 64 steps, beam 4.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
REF_PATH = os.path.join(ROOT, "baseline", "_ref")

C2 = dict(num_encoder_layers=6, num_decoder_layers=6, d_model=1024, d_ff=4096, num_heads=16,
          vocab_size=32000, max_batch=128, max_seq_len=64, max_beam_size=4)
GLOBAL_BATCH, SRC_LEN, BEAM, MAX_STEPS = 128, 64, 4, 64
METRIC = "decoded tokens/sec (Transformer-big, beam=4)"
REF_SAMPLE_ITEMS = 16  # reference arm: items per timed step (a slice of the C2 batch)

REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
           0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
           0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
           0x100: "display_clock_setting"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp16"])
    ap.add_argument("--half", default="fp16", choices=["fp16", "none"],
                    help="throughput mode reported beside the headline")
    ap.add_argument("--batch", type=int, default=GLOBAL_BATCH, help="global batch (items)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-micro", action="store_true")
    return ap.parse_args()


def synthetic_tokens(batch, seq, vocab, seed):
    """bench.py:62-66 of the reference: uniform ids in [3, vocab)."""
    import numpy as np
    return np.random.default_rng(seed).integers(min(3, vocab - 1), vocab, size=(batch, seq),
                                                dtype=np.int64)


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, device_index: int):
        self.idx = device_index
        self.proc = None
        self.lines = []
        self.t = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.active", "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], [], set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 3:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                bits = int(parts[2], 16)
            except ValueError:
                continue
            for b, name in REASONS.items():
                if bits & b and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------------ reference
def _import_reference():
    """The reference package `fuseq` from baseline/_ref (pip-installed from
    /root/reference/pkg), or None when it was not installed."""
    if not os.path.isdir(os.path.join(REF_PATH, "fuseq")):
        return None
    if REF_PATH not in sys.path:
        sys.path.insert(0, REF_PATH)
    import fuseq  # noqa: F401
    from fuseq import decode as rd, engine as re_, model as rm
    return rm, re_, rd


def reference_generate_timer(items: int):
    """(kind, description, fn(src) -> (seconds, tokens)) for the reference's own
    CPU path on the C2 model: fuseq Session.generate (engine.py:81-173) when
    installed, else the oracle port (oracle/, numpy + OpenBLAS)."""
    ref = _import_reference()
    if ref is not None:
        rm, re_, rd = ref
        cfg = rm.ModelConfig(**dict(C2, max_batch=items))
        sess = re_.Session(cfg, rm.make_random_weights(cfg, 0), engine="fused")
        dc = rd.DecodeConfig(method="beam", beam_size=BEAM, max_steps=MAX_STEPS, eos_token=2)

        def run(src, steps=MAX_STEPS):
            d = dc if steps == MAX_STEPS else rd.DecodeConfig(method="beam", beam_size=BEAM,
                                                              max_steps=steps, eos_token=2)
            t0 = time.perf_counter()
            hyps = sess.generate(src, d)
            dt = time.perf_counter() - t0
            return dt, sum(len(h[0].tokens) for h in hyps if h)
        return "reference", "fuseq (baseline/_ref, the unmodified reference package)", run
    from oracle import fuseq_oracle as O
    ocfg = O.OracleConfig(**C2)
    model = O.OracleModel(ocfg, O.make_random_weights(ocfg, 0))

    def run(src, steps=MAX_STEPS):
        t0 = time.perf_counter()
        hyps = model.generate(src, beam_size=BEAM, max_steps=steps, eos=2)
        dt = time.perf_counter() - t0
        return dt, sum(len(h[0][0]) for h in hyps)
    return "port", "oracle port (numpy/OpenBLAS; baseline/_ref not installed)", run


def run_reference(args, rank):
    if rank != 0:
        return
    cores = host_cores()
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(cores))
    kind, what, run = reference_generate_timer(REF_SAMPLE_ITEMS)
    src_all = synthetic_tokens(args.batch, SRC_LEN, C2["vocab_size"], 0)
    for _ in range(args.warmup):  # JIT / caches: one item, two decode steps
        run(src_all[:1], steps=2)
    times, toks = [], 0
    nslice = max(args.batch // REF_SAMPLE_ITEMS, 1)
    for i in range(args.steps):
        j = (i % nslice) * REF_SAMPLE_ITEMS
        dt, n = run(src_all[j:j + REF_SAMPLE_ITEMS])
        times.append(dt)
        toks += n
    sec = sum(times)
    value = toks / sec
    sample = (f"C2 model (seed-0 weights), {REF_SAMPLE_ITEMS} of the {args.batch} seed-0 items "
              f"per step (steps rotate through the batch), beam {BEAM}, {MAX_STEPS} steps; "
              f"{what}; {cpu_model()}, OpenBLAS threads {os.environ['OPENBLAS_NUM_THREADS']}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sec / len(times) * 1e3, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "Transformer-big beam4 translate (BASELINE config 2), "
                               f"{REF_SAMPLE_ITEMS}-item sample per step",
                   "batch": REF_SAMPLE_ITEMS, "global_batch": args.batch, "src_len": SRC_LEN,
                   "beam": BEAM, "max_steps": MAX_STEPS},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- ours
def gemm_flops(cfg, batch, seq, beam, steps) -> dict:
    """Algorithmic GEMM flops (2MNK) of one generate (SURVEY §2.3 shapes)."""
    d, ff, V = cfg.d_model, cfg.d_ff, cfg.vocab_size
    n, R = batch * seq, batch * beam
    enc = cfg.num_encoder_layers * 2 * n * (3 * d * d + d * d + 2 * d * ff)
    cross = 2 * n * d * 2 * cfg.num_decoder_layers * d
    dec = steps * cfg.num_decoder_layers * 2 * R * (3 * d * d + 3 * d * d + 2 * d * ff)
    logits = steps * 2 * R * d * V
    return {"encoder": enc, "cross_kv": cross, "decoder": dec, "logits": logits,
            "total": enc + cross + dec + logits}


FAMILIES = (("gemm", ("_gemm", "sgemm")), ("layer_norm", ("layer_norm",)),
            ("self_attention", ("self_attention",)), ("cross_attention", ("cross_attention",)),
            ("encoder_attention", ("encoder_attention",)),
            ("hars", ("hars", "retrieve")), ("embed", ("embed",)))


def family(name: str) -> str:
    for fam, keys in FAMILIES:
        if any(k in name for k in keys):
            return fam
    return "other"


def cupti_profile(sess, src_dev, dc) -> dict:
    """One generate under CUPTI (torch.profiler) with programmatic dependent
    launch off (re-captured step graph), kernel durations per family."""
    import torch
    from torch.profiler import ProfilerActivity, profile

    from paper_2010_13887_b200 import _abi
    saved = dict(sess._graphs)
    _abi.call("fq_set_pdl", 0)
    sess._graphs.clear()
    try:
        sess.generate(src_dev, dc, return_device_state=True)  # capture without PDL
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            sess.generate(src_dev, dc, return_device_state=True)
            torch.cuda.synchronize()
    finally:
        _abi.call("fq_set_pdl", -1)
        sess._graphs.clear()
        sess._graphs.update(saved)
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA
          and "Memcpy" not in e.name and "Memset" not in e.name]
    t0 = min(e.time_range.start for e in ev)
    t1 = max(e.time_range.end for e in ev)
    fams, kern = {}, {}
    for e in ev:
        dur = e.time_range.end - e.time_range.start
        f = fams.setdefault(family(e.name), [0, 0.0])
        f[0] += 1
        f[1] += dur
        k = kern.setdefault(e.name.split("(")[0][:90], [0, 0.0])
        k[0] += 1
        k[1] += dur
    top = sorted(kern.items(), key=lambda kv: -kv[1][1])[:8]
    return {"wall_us": t1 - t0, "busy_us": sum(v[1] for v in fams.values()),
            "launches": len(ev),
            "families": {k: {"n": v[0], "us": round(v[1], 1)} for k, v in
                         sorted(fams.items(), key=lambda kv: -kv[1][1])},
            "top_kernels": [{"kernel": k, "n": v[0], "us_total": round(v[1], 1),
                             "us_avg": round(v[1] / v[0], 2)} for k, v in top]}


def graph_time(fn, reps=12, rounds=3):
    """Per-call device time (s) of `fn` replayed as a CUDA graph of `reps`
    back-to-back calls (how the kernels run inside the decode-step graph);
    CUDA events on the launching stream, median over `rounds` replays."""
    import torch
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    times = []
    for _ in range(rounds):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        g.replay()
        e.record()
        e.synchronize()
        times.append(s.elapsed_time(e) / 1e3 / reps)
    return statistics.median(times)


def time_mode(P, cfg, host_w, precision, src_host, args, world, dev, flush, barrier,
              clock=None):
    """Build a session, warm it, time K device-resident requests and the e2e
    path. Returns (session, result dict)."""
    import torch

    from paper_2010_13887_b200 import _abi, decode as D, replicas
    sess = P.Session(cfg, host_w, precision=precision)
    dc = P.DecodeConfig(method="beam", beam_size=BEAM, max_steps=MAX_STEPS, eos_token=2)
    src_dev = torch.from_numpy(src_host).to(dev)
    src_pinned = torch.from_numpy(src_host).pin_memory()
    for _ in range(args.warmup):
        st = sess.generate(src_dev, dc, return_device_state=True)
    torch.cuda.synchronize()
    l0 = _abi.launch_count()
    barrier()
    step_times = []
    ctx = ClockSampler(torch.cuda.current_device()) if clock else None
    if ctx:
        ctx.__enter__()
    try:
        for _ in range(args.steps):
            flush()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            st = sess.generate(src_dev, dc, return_device_state=True)
            e.record()
            e.synchronize()
            step_times.append(s.elapsed_time(e) / 1e3)
        barrier()
    finally:
        if ctx:
            ctx.__exit__(None, None, None)
    launches = (_abi.launch_count() - l0) // args.steps
    sec = sum(step_times) / len(step_times)
    states = st.host_items()
    tokens = sum(len(s_.finalize(dc)[0][0]) if s_.finalize(dc) else 0 for s_ in states)
    steps_run = max(int(x.step) for x in states) if states else MAX_STEPS
    sec_max, tok_total = replicas.reduce_step_stats(sec, float(tokens), dev)
    # end to end through the public API: host tokens in (pinned), host hypotheses out
    e2e_times = []
    h2d = src_host.nbytes
    dims = {"B": len(src_host), "K": BEAM, "S": cfg.max_seq_len, "1": 1}
    d2h = 0
    for _, dt, shape in D.DeviceBeamState.FIELDS:
        n = 1
        for c in shape:
            n *= dims[c]
        d2h += n * torch.empty((), dtype=dt).element_size()
    for i in range(max(1, min(args.steps, 3)) + 1):
        flush()
        barrier()
        t0 = time.perf_counter()
        sess.generate(src_pinned, dc)
        dt = time.perf_counter() - t0
        if i:
            e2e_times.append(dt)
    e2e_sec, _ = replicas.reduce_step_stats(sum(e2e_times) / len(e2e_times), 0.0, dev)
    res = {"value": tok_total / sec_max, "ms_per_step": sec_max * 1e3, "tokens": tok_total,
           "local_tokens": tokens, "steps_run": steps_run, "gpu_launches": launches,
           "clocks": ctx.summary() if ctx else None,
           "e2e": {"value": tok_total / e2e_sec, "unit": "tokens/s",
                   "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}}
    return sess, src_dev, dc, res


def gemm_traffic(precision: str):
    """Mean DRAM bytes (read + write) per tc_gemm launch of one decode step,
    from the committed ncu capture of this precision (profiles/r2b/), or None."""
    path = os.path.join(ROOT, "profiles", "r2b", f"ncu_gemm_traffic_{precision}.json")
    if os.path.exists(path):
        return json.load(open(path)).get("bytes_per_launch_mean")
    return None


def roofline_gemm(sess, src_dev, dc, cfg, batch, steps_run, peak, peak_source, dtype_note):
    prof = cupti_profile(sess, src_dev, dc)
    fl = gemm_flops(cfg, batch, SRC_LEN, BEAM, steps_run)
    g = prof["families"].get("gemm", {"n": 1, "us": 1e-9})
    achieved = fl["total"] / (g["us"] * 1e-6) / 1e12
    return {
        "kernel": f"tc_gemm family ({dtype_note}): every GEMM launch of one request "
                  "(encoder, cross-K/V, 6 per decoder layer per step, logits)",
        "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
        "frac": achieved / peak, "traffic": gemm_traffic(sess.precision),
        "traffic_source": "profiles/r2b/ncu_gemm_traffic_<precision>.json (ncu, one decode "
                          "step's GEMM launches, mean dram bytes read + written per launch)",
        "launches": g["n"], "us_per_launch_mean": g["us"] / max(g["n"], 1),
        "flops_per_launch_mean": fl["total"] / max(g["n"], 1),
        "algorithmic_flops": fl, "share_of_request_time": g["us"] / prof["wall_us"],
        "peak_source": peak_source,
        "timing": "CUPTI kernel durations (torch.profiler) of one request after the timed "
                  "region, step graph re-captured with programmatic dependent launch off "
                  "(no overlapped durations); share = family busy / request span",
        "profile": prof}


def hars_micro(P, D, _abi, cfg, batch, dev, hbm_peak):
    import torch
    R, V = batch * BEAM, cfg.vocab_size
    lgs = [torch.randn(R, V, device=dev) for _ in range(3)]
    hst = D.DeviceBeamState(batch, BEAM, cfg.max_seq_len)
    hk = torch.full((R,), 2 * BEAM, dtype=torch.int32, device=dev)
    lse = torch.empty(R, dtype=torch.float64, device=dev)
    ci = torch.empty(R, V, dtype=torch.int32, device=dev)
    cc = torch.empty(R, dtype=torch.int64, device=dev)
    rt = torch.empty(R, dtype=torch.int64, device=dev)
    rp = torch.empty(R, dtype=torch.int64, device=dev)
    it = [0]

    def stage1():
        lg = lgs[it[0] % 3]
        it[0] += 1
        D.retrieve_device(lg, 2 * BEAM, d_k=hk, out=(None, None, lse, ci, cc))
        return lg

    def hars_step():
        hst.live.fill_(BEAM)
        hst.done.zero_()
        hst.step.fill_(5)
        lg = stage1()
        _abi.call("fq_hars_select", lg.data_ptr(), lg.stride(0), lse.data_ptr(),
                  ci.data_ptr(), ci.stride(0), cc.data_ptr(), hst.c, batch, BEAM, V,
                  cfg.max_seq_len, 2, None, None, 1 << 40, rt.data_ptr(), rp.data_ptr(),
                  None, None, 0, _abi.stream_handle())
    hcnt = torch.zeros(batch + 1 + R, dtype=torch.int32, device=dev)
    dcur = torch.full((1,), 5, dtype=torch.int32, device=dev)
    hist = torch.zeros(R, cfg.max_seq_len, dtype=torch.int32, device=dev)

    def resets():  # the per-step state reset alone (not HARS work)
        hst.live.fill_(BEAM)
        hst.done.zero_()
        hst.step.fill_(5)
        dcur.fill_(5)

    def hars_fused():  # the product path: groups + stage 1 + stage 2 in one launch
        resets()
        lg = lgs[it[0] % 3]
        it[0] += 1
        _abi.call("fq_hars_step", lg.data_ptr(), lg.stride(0), hst.c, batch, BEAM, V,
                  cfg.max_seq_len, 2, None, dcur.data_ptr(), 1 << 40, lse.data_ptr(),
                  ci.data_ptr(), ci.stride(0), cc.data_ptr(), hcnt.data_ptr(),
                  rt.data_ptr(), rp.data_ptr(), hist.data_ptr(), None, 0, 0.0, None, None,
                  None, None, _abi.stream_handle())

    hst.init()
    t_s1 = graph_time(stage1)
    t_sep = graph_time(hars_step)
    hst.init()
    t_hars_raw = graph_time(hars_fused)
    t_reset = graph_time(resets)
    t_hars = max(t_hars_raw - t_reset, 1e-9)
    hars_bytes = R * V * 4
    sweep = []
    for Vs, beam_s, batch_s in ((32000, 1, 64), (32000, 8, 512), (50257, 4, 128),
                                (128000, 4, 32), (250000, 4, 16), (250000, 1, 1)):
        Rs = beam_s * batch_s
        Ls = [torch.randn(Rs, Vs, device=dev) for _ in range(2 if Rs * Vs * 4 > 64 << 20 else 3)]
        hks = torch.full((Rs,), 2 * beam_s, dtype=torch.int32, device=dev)
        bufs_s = (None, None, torch.empty(Rs, dtype=torch.float64, device=dev),
                  torch.empty(Rs, Vs, dtype=torch.int32, device=dev),
                  torch.empty(Rs, dtype=torch.int64, device=dev))
        js = [0]

        def st1s():
            D.retrieve_device(Ls[js[0] % len(Ls)], 2 * beam_s, d_k=hks, out=bufs_s)
            js[0] += 1
        ts = graph_time(st1s, reps=6)
        bs = Rs * Vs * 4
        sweep.append({"vocab": Vs, "beam": beam_s, "batch": batch_s, "us": ts * 1e6,
                      "gbs": bs / ts / 1e9, "frac_hbm": bs / ts / 1e9 / hbm_peak})
        del Ls, bufs_s
    out = {
        "metric": "HARS step us (stage 1 retrieve + stage 2 rerank/select), fp32 logits",
        "value": t_hars * 1e6, "unit": "us", "rows": R, "vocab": V, "beam": BEAM,
        "batch": batch, "algorithmic_bytes": hars_bytes,
        "achieved_gbs": hars_bytes / t_hars / 1e9, "peak_gbs": hbm_peak,
        "frac": hars_bytes / t_hars / 1e9 / hbm_peak,
        "stage1_us": t_s1 * 1e6, "stage1_frac": hars_bytes / t_s1 / 1e9 / hbm_peak,
        "separate_launches_us": t_sep * 1e6,
        "with_state_reset_us": t_hars_raw * 1e6, "state_reset_us": t_reset * 1e6,
        "path": "fq_hars_step (one launch: groups + stage 1 + stage 2 + next embedding); "
                "value = graph time minus the 4-fill state reset timed alone",
        "timing": "CUDA graph of 12 back-to-back steps, 3 logit buffers rotated (196 MB > L2)",
        "stage1_sweep": sweep,
        "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)"}
    return out, (hst, hk, lse, ci, cc, rt, rp, hcnt, dcur, hist, resets, t_reset, it)


def output_layer_micro(P, _abi, sess16, cfg, batch, dev, ctx):
    """The half mode's output layer at C2: fq_logits_hars + merge (logits never
    written) vs the materialised logits GEMM + fq_hars_step."""
    import torch
    hst, hk, lse, ci, cc, rt, rp, hcnt, dcur, hist, resets, t_reset, it = ctx
    R, V, d_m = batch * BEAM, cfg.vocab_size, cfg.d_model
    E16 = sess16.dw.out_proj
    x16s = [torch.randn(R, d_m, device=dev).to(E16.dtype) for _ in range(3)]
    ldt = (V + 223) // 224
    cap = 128
    dk = torch.zeros(R, dtype=torch.int32, device=dev)
    gmx = torch.full((R, 32), -2139095041, dtype=torch.int32, device=dev)
    tmx = torch.zeros(R, ldt, device=dev)
    tsm = torch.zeros(R, ldt, dtype=torch.float64, device=dev)
    svc = torch.zeros(R, ldt, dtype=torch.int32, device=dev)
    svb = torch.zeros(R, ldt, cap, 2, dtype=torch.int32, device=dev)
    ovf = torch.zeros(1, dtype=torch.int32, device=dev)
    mcnt = torch.zeros(batch + 1, dtype=torch.int32, device=dev)
    lg1 = torch.empty(R, V, device=dev)

    def out_fused():
        resets()
        x = x16s[it[0] % 3]
        it[0] += 1
        _abi.call("fq_logits_hars", x.data_ptr(), d_m, E16.data_ptr(), d_m, R, V, d_m,
                  dk.data_ptr(), gmx.data_ptr(), tmx.data_ptr(), tsm.data_ptr(), ldt,
                  svc.data_ptr(), svb.data_ptr(), cap, _abi.stream_handle())
        _abi.call("fq_hars_merge_step", hst.c, batch, BEAM, V, cfg.max_seq_len, 2, None,
                  dcur.data_ptr(), 1 << 40, dk.data_ptr(), gmx.data_ptr(), tmx.data_ptr(),
                  tsm.data_ptr(), ldt, ldt, svc.data_ptr(), svb.data_ptr(), cap,
                  lse.data_ptr(), ci.data_ptr(), ci.stride(0), cc.data_ptr(), mcnt.data_ptr(),
                  ovf.data_ptr(), rt.data_ptr(), rp.data_ptr(), hist.data_ptr(), None, 0, 0.0,
                  None, None, None, None, _abi.stream_handle())

    def out_mat():
        resets()
        x = x16s[it[0] % 3]
        it[0] += 1
        P.gemm(x, E16, lg1, transpose_b=True)
        _abi.call("fq_hars_step", lg1.data_ptr(), V, hst.c, batch, BEAM, V,
                  cfg.max_seq_len, 2, None, dcur.data_ptr(), 1 << 40, lse.data_ptr(),
                  ci.data_ptr(), ci.stride(0), cc.data_ptr(), hcnt.data_ptr(),
                  rt.data_ptr(), rp.data_ptr(), hist.data_ptr(), None, 0, 0.0, None, None,
                  None, None, _abi.stream_handle())
    hst.init()
    _abi.call("fq_hars_groups", hst.c, batch, BEAM, V, 0, dk.data_ptr(), _abi.stream_handle())
    t_of = graph_time(out_fused) - t_reset
    hst.init()
    t_om = graph_time(out_mat) - t_reset
    return {"what": "the half mode's decode-step output layer at C2 (512 x 1024 -> 32000 "
                    "logits, HARS stages 1+2): graph-timed us, state-reset fills subtracted",
            "fused_us": t_of * 1e6, "materialised_us": t_om * 1e6,
            "fused": "fq_logits_hars (tcgen05 logits GEMM, epilogue emits per-tile group "
                     "maxima, sum exp and survivors; [rows, V] never written) + "
                     "fq_hars_merge_step",
            "materialised": "fq_gemm (65.5 MB fp32 logits) + fq_hars_step",
            "hbm_bytes_avoided_per_step": 2 * R * V * 4}


def extra_workloads(P, dev, args) -> dict:
    """BASELINE configs 4 and 5 on the same engine, exact mode
    and fp16, end to end through the public API (host tokens in, host results
    out; wall clock after warm-up, synchronized):
    * BERT-base-like encoder + classification head (12 layers, d = 768, GELU,
      V = 30522, seq 128, batch 64): Session.classify sequences/s (the
      reference measured 6.7 seq/s on 8 CPU cores);
    * top-k sampling generate (k = 8) on the C2 model, batch 64, 64 steps:
      decoded tokens/s, device-resident (decoder step + retrieve +
      fq_sample_step in one step graph, the reference's PCG64 stream
      consumed on the device in its order), and the host-driven draw
      (FQ_SAMPLE_HOST=1) beside it; a decoder-only GPT-2 is not expressible in
      the reference."""
    import numpy as np
    import torch
    res = {}
    bert = P.ModelConfig(num_encoder_layers=12, num_decoder_layers=0, d_model=768, d_ff=3072,
                         num_heads=12, vocab_size=30522, max_batch=64, max_seq_len=128,
                         max_beam_size=1, activation="gelu")
    wb = P.make_random_weights(bert, seed=0)
    toks = np.random.default_rng(0).integers(3, bert.vocab_size, size=(64, 128))
    for prec in ("fp32", "fp16"):
        sess = P.Session(bert, wb, precision=prec)
        for _ in range(2):
            sess.classify(toks)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        n = 5
        for _ in range(n):
            sess.classify(toks)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / n
        res[f"classify_bert_base_{prec}"] = {"value": 64 / dt, "unit": "sequences/s",
                                             "ms_per_batch": dt * 1e3, "batch": 64, "seq": 128}
        del sess
    cfg = P.ModelConfig(**dict(C2, max_batch=64))
    w = P.make_random_weights(cfg, seed=0)
    src = synthetic_tokens(64, SRC_LEN, cfg.vocab_size, 0)
    dc = P.DecodeConfig(method="top_k", sample_k=8, max_steps=MAX_STEPS, eos_token=2, seed=0)
    for prec in ("fp32", "fp16"):
        sess = P.Session(cfg, w, precision=prec)
        for path in ("device", "host"):
            if path == "host":
                os.environ["FQ_SAMPLE_HOST"] = "1"
            try:
                sess.generate(src, dc)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                hyps = sess.generate(src, dc)
                dt = time.perf_counter() - t0
            finally:
                os.environ.pop("FQ_SAMPLE_HOST", None)
            ntok = sum(len(h[0].tokens) for h in hyps if h)
            name = f"sampling_top_k_{prec}" + ("" if path == "device" else "_host_draw")
            res[name] = {"value": ntok / dt, "unit": "tokens/s", "ms_per_request": dt * 1e3,
                         "batch": 64, "max_steps": MAX_STEPS}
        del sess
    return res


def cpu_baseline_sample():
    """The reference's own CPU path on the box's host cores, bounded sample
    (one 16-item C2 request, ~10 s)."""
    cores = host_cores()
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(cores))
    kind, what, run = reference_generate_timer(REF_SAMPLE_ITEMS)
    src = synthetic_tokens(GLOBAL_BATCH, SRC_LEN, C2["vocab_size"], 0)[:REF_SAMPLE_ITEMS]
    run(src[:1], steps=2)  # JIT warm-up
    dt, toks = run(src)
    return {"value": toks / dt, "unit": "tokens/s", "cores": cores, "kind": kind,
            "sample": f"C2 model, the first {REF_SAMPLE_ITEMS} seed-0 items x {MAX_STEPS} "
                      f"steps, beam {BEAM}: {dt:.1f} s ({what}; {cpu_model()})"}


def run_ours(args, rank, world):
    import torch

    import paper_2010_13887_b200 as P
    from paper_2010_13887_b200 import _abi, decode as D, replicas

    dev = torch.device("cuda", torch.cuda.current_device())
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    f16_peak = peaks.get("bf16_tflops_sustained", 1400.0)
    if args.scaling == "strong":
        sl = replicas.batch_shard(args.batch, rank, world)
        src_host = synthetic_tokens(args.batch, SRC_LEN, C2["vocab_size"], 0)[sl].copy()
    else:
        src_host = synthetic_tokens(args.batch, SRC_LEN, C2["vocab_size"], rank)
    local = len(src_host)
    cfg = P.ModelConfig(**dict(C2, max_batch=max(local, 1)))
    host_w = P.make_random_weights(cfg, seed=0)
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def flush():
        flush_buf.fill_(1)

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    sess, src_dev, dc, res = time_mode(P, cfg, host_w, args.precision, src_host, args, world,
                                       dev, flush, barrier, clock=True)
    dtype = {"fp32": "f32", "fp16": "f16"}[args.precision]
    out = None
    if rank == 0:
        out = {
            "metric": METRIC, "value": res["value"], "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_per_step"],
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": dtype, "data": "synthetic (seeded random-init weights, uniform source ids)",
            "config": {"workload": "Transformer-big beam4 translate (BASELINE config 2)",
                       "layers": "6+6", "d_model": 1024, "heads": 16, "d_ff": 4096,
                       "vocab": 32000, "global_batch": args.batch if args.scaling == "strong"
                       else args.batch * world, "batch_per_gpu": local, "src_len": SRC_LEN,
                       "beam": BEAM, "max_steps": MAX_STEPS, "steps_run": res["steps_run"],
                       "parallelism": f"replicas x{world} ({args.scaling}: batch-sharded)",
                       "precision": f"{args.precision} ("
                       + ("exact mode: 3xFP16 tcgen05 GEMMs, fp32/f64 elementwise, tokens "
                          "bit-exact vs the reference at this config)" if args.precision ==
                          "fp32" else "fp16 throughput mode") + ")",
                       "tokens_per_step": res["tokens"],
                       "l2": "256 MiB buffer written before every timed request; working set "
                             ">> 126 MB L2"},
            "clocks": res["clocks"], "gpu_launches": res["gpu_launches"], "e2e": res["e2e"],
        }
    half = None
    if args.half != "none" and args.precision == "fp32":
        half, hsrc, hdc, hres = time_mode(P, cfg, host_w, args.half, src_host, args, world, dev,
                                          flush, barrier)
        if rank == 0:
            out["half_mode"] = {"precision": args.half, "value": hres["value"],
                                "unit": "tokens/s", "ms_per_step": hres["ms_per_step"],
                                "e2e": hres["e2e"], "gpu_launches": hres["gpu_launches"],
                                "steps_run": hres["steps_run"]}

    if rank == 0 and not args.no_micro:
        if args.precision == "fp32":
            out["roofline"] = roofline_gemm(
                sess, src_dev, dc, cfg, local, res["steps_run"], f16_peak / 3,
                "MEASURED_PEAKS.json bf16_tflops_sustained (measured; fp16 kind::f16 runs at the "
                "same rate) / 3: the exact mode issues three kind::f16 MMAs (a_hi.b_hi, "
                "a_hi.b_lo, a_lo.b_hi) per algorithmic product", "3xFP16 exact mode")
            out["roofline"]["frac_of_f16_peak"] = out["roofline"]["achieved"] / f16_peak
        else:
            out["roofline"] = roofline_gemm(sess, src_dev, dc, cfg, local, res["steps_run"],
                                            f16_peak, "MEASURED_PEAKS.json bf16_tflops_"
                                            "sustained (measured; same rate for fp16)", "fp16")
        if half is not None:
            out["half_mode"]["roofline"] = roofline_gemm(
                half, hsrc, hdc, cfg, local, hres["steps_run"], f16_peak,
                "MEASURED_PEAKS.json bf16_tflops_sustained (measured)", args.half)
    # the single-GPU micro-benchmarks (HARS step + stage-1 sweep, output layer,
    # BASELINE configs 4/5) belong to the N = 1 line only
    if rank == 0 and world == 1 and not args.no_micro:
        out["hars"], ctx = hars_micro(P, D, _abi, cfg, local, dev, hbm_peak)
        sess16 = half if half is not None else (sess if args.precision != "fp32" else None)
        if sess16 is not None:
            out["output_layer"] = output_layer_micro(P, _abi, sess16, cfg, local, dev, ctx)
        out["extras"] = extra_workloads(P, dev, args)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline_sample()
    if rank == 0:
        print(json.dumps(out), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    import torch
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # FQ_BENCH_ONE_GPU=1: every rank on cuda:0 with gloo (plumbing checks of the
    # multi-rank path on a 1-GPU box; NCCL needs one GPU per rank)
    one_gpu = os.environ.get("FQ_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if one_gpu:
            torch.distributed.init_process_group("gloo")
        else:
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
    try:
        run_ours(args, rank, world)
    finally:
        if world > 1:
            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
