"""Engine-level contracts on the device, ported from the reference's acceptance
suite (pkg/tests/test_acceptance.py) and SURVEY §8(e):

* zero allocation after warm-up (test_acceptance.py:208-247; north_star: "no
  allocation happens at runtime"): neither the engine's tracked arena count
  nor torch's CUDA allocator counters move across repeated generates;
* HARS exactness over 1000 seeded tiny configurations (:48-80): hierarchical
  search token-identical to the exhaustive oracle, scores within 1e-5;
* KV-cache equivalence on 50 seeded tiny models (:254-272): the device's
  cached greedy decode equals a recompute-from-scratch greedy decode;
* the per-layer counter contract (:180-201): 6 GEMMs + one pass of each
  FusedPassKind, run here as 7 launches;
* batch sharding (§8(e), engine.py:151-169): two processes each decoding a
  shard of the batch on the device reproduce the single-process hypotheses
  bit for bit (exact mode's numerics do not depend on M).
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P(gpu):
    import paper_2010_13887_b200 as pkg
    return pkg


@pytest.mark.parametrize("prec", ["fp32", "fp16"])
def test_generate_allocates_nothing_after_warmup(P, prec):
    import torch
    cfg = P.ModelConfig(2, 2, 128, 256, 4, 2000, 8, 24, 4)
    sess = P.Session(cfg, P.make_random_weights(cfg, 3), precision=prec)
    rng = np.random.default_rng(0)
    srcs = [rng.integers(3, 2000, size=(b, 9)) for b in (8, 3)]
    dc = P.DecodeConfig(beam_size=4, max_steps=16)
    devs = [torch.from_numpy(s).cuda() for s in srcs]

    def requests():
        for s, dv in zip(srcs, devs):
            sess.generate(s, dc)                                  # host in, host out
            sess.generate(dv, dc, return_device_state=True)       # device-resident
        sess.forced_logits(srcs[1], rng.integers(3, 2000, size=(3, 5)))
    requests()  # warm-up: graph capture, pinned staging
    requests()
    torch.cuda.synchronize()
    n0 = P.allocation_count()
    s0 = torch.cuda.memory_stats()
    for _ in range(3):
        requests()
    torch.cuda.synchronize()
    s1 = torch.cuda.memory_stats()
    assert P.allocation_count() == n0
    for k in ("allocation.all.allocated", "segment.all.allocated"):
        assert s1[k] == s0[k], (k, s0[k], s1[k])


def test_hars_exactness_1000_configs(P):
    """test_acceptance.py:48-80 on the device (fp32 exact mode)."""
    rng = np.random.default_rng(20240)
    for i in range(1000):
        d = int(rng.choice([16, 32]))
        heads = int(rng.choice([2, 4]))
        vocab = int(rng.integers(32, 513))
        batch = int(rng.integers(1, 5))
        beam = int(rng.integers(1, 9))
        steps = int(rng.integers(2, 17))
        src_len = int(rng.integers(2, 7))
        cfg = P.ModelConfig(num_encoder_layers=1, num_decoder_layers=1, d_model=d,
                            d_ff=2 * d, num_heads=heads, vocab_size=vocab,
                            max_batch=4, max_seq_len=24, max_beam_size=8)
        sess = P.Session(cfg, P.make_random_weights(cfg, seed=i), precision="fp32",
                         use_graphs=False)
        src = rng.integers(3, vocab, size=(batch, src_len))
        dc = P.DecodeConfig(method="beam", beam_size=beam, max_steps=steps, eos_token=2)
        hars = sess.generate(src, dc, search="hierarchical")
        exact = sess.generate(src, dc, search="exhaustive")
        for b in range(batch):
            assert [h.tokens for h in hars[b]] == [h.tokens for h in exact[b]], (i, b)
            for ha, he in zip(hars[b], exact[b]):
                assert abs(ha.score - he.score) <= 1e-5, (i, b)


def _greedy_no_cache(O, om, src, steps, bos=1, eos=2):
    """Greedy chain recomputed from scratch every step (reference
    tests/reference.py:173-198) on the CPU oracle: a fresh cache re-runs the
    whole prefix for each new token."""
    batch = src.shape[0]
    mem = om.encode(src)
    cross = om.build_cross_kv(mem, batch, src.shape[1])
    out, fed, done = [[] for _ in range(batch)], [[] for _ in range(batch)], [False] * batch
    for _ in range(steps):
        cache = om.new_cache(batch)
        for t in range(len(fed[0]) + 1):
            toks = np.array([([bos] + fed[b])[t] for b in range(batch)])
            logits = om.decode_step(toks, cache, cross, None, batch, 1)
        for b in range(batch):
            if done[b]:
                fed[b].append(eos)
                continue
            tok = int(np.argmax(logits[b]))
            out[b].append(tok)
            fed[b].append(tok)
            done[b] = tok == eos
        if all(done):
            break
    return out


def test_kv_cache_equivalence_50_models(P):
    """test_acceptance.py:254-272: the device's cached greedy decode (fp32
    exact mode, copy-free KV cache, captured step graph) token-identical to a
    recompute-from-scratch greedy decode."""
    from oracle import fuseq_oracle as O
    rng = np.random.default_rng(31337)
    for i in range(50):
        d = int(rng.choice([16, 32]))
        vocab = int(rng.integers(32, 129))
        cfg = P.ModelConfig(num_encoder_layers=1, num_decoder_layers=1, d_model=d,
                            d_ff=2 * d, num_heads=2, vocab_size=vocab, max_batch=2,
                            max_seq_len=16, max_beam_size=2)
        sess = P.Session(cfg, P.make_random_weights(cfg, seed=1000 + i), precision="fp32")
        batch = int(rng.integers(1, 3))
        src = rng.integers(3, vocab, size=(batch, int(rng.integers(3, 7))))
        steps = int(rng.integers(3, 8))
        dc = P.DecodeConfig(method="greedy", max_steps=steps, eos_token=2)
        cached = [h[0].tokens for h in sess.generate(src, dc)]
        ocfg = O.OracleConfig(**cfg.to_dict())
        om = O.OracleModel(ocfg, O.make_random_weights(ocfg, 1000 + i))
        assert cached == _greedy_no_cache(O, om, src, steps), i


@pytest.mark.parametrize("prec", ["fp32", "fp16"])
def test_encoder_layer_counter_contract(P, prec):
    """test_acceptance.py:180-201: one encoder layer = 6 GEMMs + one pass of
    each of the 6 FusedPassKinds (ops.py:45-58), on the device as 7 kernel
    launches (the fp32 mode adds the attention output's pair split)."""
    from paper_2010_13887_b200 import _abi
    from paper_2010_13887_b200 import model as M
    cfg = P.ModelConfig(num_encoder_layers=1, num_decoder_layers=0, d_model=64, d_ff=128,
                        num_heads=4, vocab_size=100, max_batch=2, max_seq_len=12,
                        max_beam_size=1)
    w = P.make_random_weights(cfg, seed=0)
    dw = M.DeviceWeights(cfg, w, prec)
    x = np.random.default_rng(0).normal(size=(2 * 6, 64)).astype(np.float32)
    import torch
    X = torch.from_numpy(x).cuda()
    x16 = X.half() if prec == "fp16" else M.split_pair(X)
    mask = torch.from_numpy(M.lengths_mask([6, 5], 6)).cuda()
    torch.cuda.synchronize()
    cf = P.OpCounters()
    l0 = _abi.launch_count()
    M.encoder_layer_forward(X, dw.enc[0], cfg, mask, batch=2, counters=cf, x16=x16)
    launches = _abi.launch_count() - l0
    assert cf.gemm_calls == 6
    assert cf.fused_passes == 6
    assert cf.fused_kind_counts == {k.value: 1 for k in P.FusedPassKind}
    assert launches == (7 if prec == "fp16" else 8), launches


def _shard_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2010_13887_b200 as P
        from paper_2010_13887_b200 import replicas
        torch.cuda.set_device(0)
        cfg = P.ModelConfig(2, 2, 128, 256, 4, 1000, 8, 20, 4)
        src = np.random.default_rng(5).integers(3, 1000, size=(7, 8))
        sl = replicas.batch_shard(len(src), rank, world)
        sess = P.Session(cfg, P.make_random_weights(cfg, 4), precision="fp32")
        hyps = sess.generate(src[sl], P.DecodeConfig(beam_size=4, max_steps=12))
        local = [[(h.tokens, h.score) for h in hs] for hs in hyps]
        allh = replicas.gather_hypotheses(local, world)
        if rank == 0:
            q.put(allh)
    finally:
        torch.distributed.destroy_process_group()


def test_batch_sharded_generate_bit_identical(P):
    """Two processes (gloo for the host gather), each decoding its contiguous
    shard of a 7-item batch on the device in fp32 mode: the gathered
    hypotheses equal the single-process run's tokens AND score bits."""
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    cfg = P.ModelConfig(2, 2, 128, 256, 4, 1000, 8, 20, 4)
    src = np.random.default_rng(5).integers(3, 1000, size=(7, 8))
    sess = P.Session(cfg, P.make_random_weights(cfg, 4), precision="fp32")
    want = [[(h.tokens, h.score) for h in hs]
            for hs in sess.generate(src, P.DecodeConfig(beam_size=4, max_steps=12))]
    assert got == want
