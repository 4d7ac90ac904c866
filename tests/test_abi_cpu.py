"""CPU-only checks: the C-ABI library loads and exports every declared symbol,
and the host-side logic (plan, configs, beam-state bookkeeping, LSQW I/O,
seeded init) matches the reference. No compute calls (no GPU here)."""

import json
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden_path
import paper_2010_13887_b200 as P
from paper_2010_13887_b200 import _abi


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "fq_abi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fq_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = _abi.load()
    syms = _header_symbols()
    assert len(syms) >= 24
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/fq_abi.h but not exported"
        assert s in _abi.SIGNATURES, f"{s} has no ctypes signature"
    assert lib.fq_abi_version() == 1


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _abi.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_weights_match_reference_seeded_init():
    g = np.load(golden_path("tiny_golden.npz"))
    for ci, kw in enumerate(json.loads(str(g["cfgs"]))):
        cfg = P.ModelConfig(**kw)
        w = P.make_random_weights(cfg, seed=10 + ci)
        sums = np.array([float(np.asarray(a, np.float64).sum()) for _, a in w.named_tensors(cfg)])
        assert np.array_equal(sums, g[f"m{ci}_wsum"])


def test_lsqw_round_trip_byte_stable(tmp_path):
    cfg = P.ModelConfig(1, 1, 16, 32, 2, 50, 2, 8, 2, tie_output=False)
    w = P.make_random_weights(cfg, 3)
    p1, p2 = tmp_path / "a.lsqw", tmp_path / "b.lsqw"
    P.save_weights(p1, cfg, w)
    cfg2, w2 = P.load_weights(p1)
    assert cfg2 == cfg
    P.save_weights(p2, cfg2, w2)
    assert p1.read_bytes() == p2.read_bytes()
    P.save_weights(p2, cfg, w, fp16=True)
    _, w3 = P.load_weights(p2)
    assert w3.token_embedding.dtype == np.float32
    with pytest.raises(P.FormatError):
        p2.write_bytes(b"XXXX" + p1.read_bytes()[4:])
        P.load_weights(p2)


def test_config_and_decode_validation():
    with pytest.raises(P.ConsistencyError):
        P.ModelConfig(1, 1, 10, 8, 3, 50, 1, 8, 1)
    dc = P.DecodeConfig(beam_size=5)
    with pytest.raises(P.ParameterError):
        dc.validate(100, 4)
    with pytest.raises(P.ParameterError):
        P.DecodeConfig(eos_token=100).validate(100, 4)
    assert P.DecodeConfig(method="greedy", beam_size=4).effective_beam_size == 1


def test_beam_state_host_semantics():
    # decode.py:160-183: should_stop / finalize
    cfg = P.DecodeConfig(beam_size=2)
    st = P.BeamState(prefixes=[[5, 6], [5, 7]], cum_log_prob=[-1.0, -2.0],
                     finished=[([5, 2], -0.5), ([4, 2], -1.5)], step=2)
    assert st.should_stop(cfg) is False  # best live -1.0 > -1.5
    st2 = P.BeamState(prefixes=[[5, 6]], cum_log_prob=[-3.0],
                      finished=[([5, 2], -0.5), ([4, 2], -1.5)], step=2)
    assert st2.should_stop(cfg) is True
    fin = st.finalize(cfg)
    assert fin == [([5, 2], -0.5), ([5, 6], -1.0)]


def test_device_plan_shares_and_never_overlaps():
    cfg = P.ModelConfig(6, 6, 1024, 4096, 16, 32000, 128, 64, 4)
    for prec in ("fp32", "fp16"):
        specs = P.plan_intermediates(cfg, prec)
        plan = P.build_plan(specs)
        assert plan.arena_bytes < plan.no_share_bytes
        by = {s.name: s for s in specs}
        items = sorted(plan.assignments.items(), key=lambda kv: kv[1][0])
        for i, (na, (oa, sa)) in enumerate(items):
            assert oa % 64 == 0
            for nb, (ob, sb) in items[i + 1:]:
                if ob >= oa + sa:
                    break
                a, b = by[na], by[nb]
                assert not (a.first_use <= b.last_use and b.first_use <= a.last_use), (na, nb)
    # C2 fp16 arena well under the reference's 3.9 GB fp32 plan
    assert P.build_plan(P.plan_intermediates(cfg, "fp16")).arena_bytes < 2e9


def test_plan_alignment_buckets_and_best_fit():
    """B200 planner: 1024-B TMA alignment for every buffer, per-batch-bucket
    plans no larger than the max-batch plan, and random interval sets never
    share bytes between lifetime-overlapping buffers."""
    import numpy as np
    from paper_2010_13887_b200 import memory_plan as MP
    cfg = P.ModelConfig(6, 6, 1024, 4096, 16, 32000, 128, 64, 4)
    assert MP.batch_buckets(128) == [1, 2, 4, 8, 16, 32, 64, 128]
    assert MP.batch_buckets(6) == [1, 2, 4, 6]
    assert MP.bucket_of(5, MP.batch_buckets(6)) == 6
    for prec in ("fp32", "fp16"):
        sizes = []
        for b in MP.batch_buckets(128):
            plan = P.build_plan(P.plan_intermediates(cfg, prec, batch=b))
            assert all(off % 1024 == 0 for off, _ in plan.assignments.values())
            sizes.append(plan.arena_bytes)
        assert sizes == sorted(sizes) and sizes[0] < sizes[-1] / 50
    rng = np.random.default_rng(7)
    for _ in range(200):
        specs = []
        for i in range(int(rng.integers(1, 40))):
            f = int(rng.integers(0, 30))
            specs.append(P.IntermediateSpec(f"b{i}", int(rng.integers(1, 1 << 20)), f,
                                            f + int(rng.integers(0, 8)),
                                            int(rng.choice([64, 256, 1024]))))
        plan = P.build_plan(specs)
        assert plan.arena_bytes <= plan.no_share_bytes
        for a in specs:
            oa, sa = plan.assignments[a.name]
            assert oa % a.align == 0
            for b in specs:
                if a.name < b.name and a.first_use <= b.last_use and b.first_use <= a.last_use:
                    ob, sb = plan.assignments[b.name]
                    assert oa + sa <= ob or ob + sb <= oa, (a, b)


def test_plan_errors():
    with pytest.raises(P.PlanError):
        P.build_plan([])
    with pytest.raises(P.PlanError):
        P.build_plan([P.IntermediateSpec("a", 10, 3, 1)])


def test_finalize_beams_host_helper_equals_beamstate_finalize():
    """fq_finalize_beams (host helper, no GPU) == BeamState.finalize
    (decode.py:173-183) over random batched states: finished lists with score
    ties (sequence order decides), live prefixes duplicating a finished one,
    length penalties, empty prefixes and partially finished items."""
    import paper_2010_13887_b200 as P
    from paper_2010_13887_b200 import _abi
    rng = np.random.default_rng(7)
    for trial in range(200):
        B, K, S = int(rng.integers(1, 6)), int(rng.integers(1, 6)), int(rng.integers(2, 9))
        alpha = float(rng.choice([0.0, 0.6, 1.0]))
        live = rng.integers(0, K + 1, B).astype(np.int32)
        step = rng.integers(0, S, B).astype(np.int32)
        prefix = rng.integers(0, 4, (B, K, S)).astype(np.int32)
        cum = np.round(rng.normal(size=(B, K)), 1)
        fc = rng.integers(0, K + 1, B).astype(np.int32)
        ft = rng.integers(0, 4, (B, K, S)).astype(np.int32)
        fl = rng.integers(1, S + 1, (B, K)).astype(np.int32)
        fs = np.round(rng.normal(size=(B, K)), 1)
        states = []
        for b in range(B):
            fin = [(ft[b, i, :fl[b, i]].tolist(), float(fs[b, i])) for i in range(fc[b])]
            if fc[b] and live[b] and step[b]:  # a live prefix equal to a finished sequence
                ft[b, 0, :step[b]] = prefix[b, 0, :step[b]]
                fl[b, 0] = step[b]
                fin[0] = (prefix[b, 0, :step[b]].tolist(), fin[0][1])
            fin.sort(key=lambda h: (-h[1], h[0]))  # the device keeps it sorted
            for i, (sq, sc) in enumerate(fin):
                ft[b, i, :len(sq)] = sq
                fl[b, i] = len(sq)
                fs[b, i] = sc
            states.append(P.BeamState(prefixes=[prefix[b, i, :step[b]].tolist()
                                                for i in range(live[b])],
                                      cum_log_prob=cum[b, :live[b]].tolist(), finished=fin,
                                      step=int(step[b])))
        cfg = P.DecodeConfig(beam_size=K, length_penalty=alpha)
        ot = np.zeros((B, K, S), np.int32)
        ol = np.zeros((B, K), np.int32)
        osc = np.zeros((B, K))
        on = np.zeros(B, np.int32)
        arrs = [np.ascontiguousarray(a) for a in (live, step, prefix, cum, fc, ft, fl, fs)]
        assert _abi.call("fq_finalize_beams", *[a.ctypes.data for a in arrs], B, K, S, alpha, K,
                         ot.ctypes.data, ol.ctypes.data, osc.ctypes.data, on.ctypes.data) == 0
        for b in range(B):
            want = states[b].finalize(cfg)
            got = [(ot[b, i, :ol[b, i]].tolist(), float(osc[b, i])) for i in range(on[b])]
            assert got == want, (trial, b, got, want)
