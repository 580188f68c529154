"""Batched heterogeneous-precision decode on the tensor-core path (BASELINE config 5).

B >= 16 rows of a llama model step through batched.cu + one tcgen05 GEMM per (linear, precision
copy present in the batch), each launch writing only its rows.  Every row must equal its own
single-sequence oracle run (oracle/llama.py with that sequence's precision table -- the
per-sequence set_precision state of src/model.cpp:268-278): logits within 1e-2 relative,
entropy within 1e-4 + 3x the oracle's fp32-vs-fp64 envelope (tests/test_c3_shape_gpu.py).
"""
import numpy as np
import pytest

import oracle
import oracle.llama

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2506_12024_b200 import capi  # noqa: E402

TINY = dict(vocab_size=8192, d_model=512, n_heads=8, head_dim=64, n_layers=4, ffn_dim=1376, max_seq_len=64)
HD128 = dict(vocab_size=4096, d_model=256, n_heads=2, head_dim=128, n_layers=2, ffn_dim=768, max_seq_len=64)


@pytest.mark.parametrize("cfg,B", [(TINY, 24), (HD128, 16), (TINY, 32)], ids=["tiny-B24", "hd128-B16", "tiny-B32"])
def test_batched_heterogeneous_rows_match_oracle(ctx, cfg, B):
    m = capi.Model(ctx, arch=capi.ARCH_LLAMA, act_dtype=capi.DT_BF16, max_batch=B, group_size=128, **cfg)
    orc = oracle.llama.LlamaOracle(dict(cfg, group_size=128), seed=3)
    orc.upload(m, capi)
    o32 = orc.variant(acc="f32")
    rng = np.random.default_rng(B)
    n_lin = len(orc.ids)
    tables = []
    for s in range(B):
        # a different table per sequence: all W8, all W4, and random mixes
        r = [8] * n_lin if s == 0 else [4] * n_lin if s == 1 else [int(x) for x in rng.choice([8, 4], n_lin)]
        tables.append(r)
        for i, b in enumerate(r):
            m.set_rung(s, i, capi.RUNG_INT8 if b == 8 else capi.RUNG_INT4)
    V = cfg["vocab_size"]
    plen = [1 + (s % 5) for s in range(B)]  # ragged histories: prefill 1..5 tokens per slot
    caches = [orc.new_cache() for _ in range(B)]
    caches32 = [o32.new_cache() for _ in range(B)]
    for s in range(B):
        p = oracle.random_tokens(plen[s], V, 500 + s)
        m.prefill(s, p)
        orc.forward(p, caches[s], tables[s])
        o32.forward(p, caches32[s], tables[s])
    out = torch.zeros((B, V), dtype=torch.float32, device="cuda")
    worst_rel, worst_dh, worst_env = 0.0, 0.0, 0.0
    for step in range(3):
        toks = oracle.random_tokens(B, V, 900 + step)
        st = m.decode(list(range(B)), toks, out)
        ctx.synchronize()
        got = out.cpu().numpy()
        for s in range(B):
            want = orc.forward([int(toks[s])], caches[s], tables[s])[0]
            alt = o32.forward([int(toks[s])], caches32[s], tables[s])[0]
            rel = np.max(np.abs(got[s] - want)) / np.max(np.abs(want))
            h = oracle.row_stats(want)["entropy"]
            env = abs(oracle.row_stats(alt)["entropy"] - h)
            dh = abs(float(st["entropy"][s]) - h)
            worst_rel, worst_dh, worst_env = max(worst_rel, rel), max(worst_dh, dh), max(worst_env, env)
            assert rel <= 1e-2, (step, s, rel)
            assert dh <= 1e-4 + 3 * max(env, worst_env), (step, s, dh, env)
    print(f"B={B}: max rel logit err {worst_rel:.3e}, max |dH| {worst_dh:.3e}, envelope {worst_env:.3e}")
    for s in range(B):
        assert m.slot_length(s) == plen[s] + 3
    m.close()


def test_batched_path_agrees_with_step_program(ctx):
    """The same rows through the tensor-core batched path (B = 16) and through the persistent step
    program one row at a time: identical greedy choices where the margin allows, entropy close."""
    cfg = TINY
    B = 16
    m = capi.Model(ctx, arch=capi.ARCH_LLAMA, act_dtype=capi.DT_BF16, max_batch=B, group_size=128, **cfg)
    m.init_random(11, 0.02)
    m1 = capi.Model(ctx, arch=capi.ARCH_LLAMA, act_dtype=capi.DT_BF16, max_batch=1, group_size=128, **cfg)
    m1.init_random(11, 0.02)
    toks = oracle.random_tokens(B * 4, cfg["vocab_size"], 1).reshape(B, 4)
    for s in range(B):
        m.set_all_rungs(s, capi.RUNG_INT4 if s % 2 else capi.RUNG_INT8)
    rows = [m.decode(list(range(B)), toks[:, t]) for t in range(4)]
    for s in range(B):
        m1.reset_slot(0)
        m1.set_all_rungs(0, capi.RUNG_INT4 if s % 2 else capi.RUNG_INT8)
        for t in range(4):
            r1 = m1.decode([0], [int(toks[s, t])])[0]
            assert abs(r1["entropy"] - rows[t]["entropy"][s]) <= 5e-4
    m.close()
    m1.close()


def test_batched_graphs_survive_a_larger_prefill(ctx, monkeypatch):
    """The batched step's CUDA graphs run on the prefill workspace; a longer prompt reallocates that
    workspace, so the graphs must be rebuilt (replaying them read freed buffers before).  Steps
    after the regrow equal the same steps of a model that never captured a graph."""
    cfg = dict(TINY, max_seq_len=128)
    B = 16
    outs = []
    for graphs in (True, False):
        if not graphs:
            monkeypatch.setenv("FQ_NO_GRAPHS", "1")  # read when the model is created
        m = capi.Model(ctx, arch=capi.ARCH_LLAMA, act_dtype=capi.DT_BF16, max_batch=B, group_size=128, **cfg)
        orc = oracle.llama.LlamaOracle(dict(cfg, group_size=128), seed=4)
        orc.upload(m, capi)
        V = cfg["vocab_size"]
        rng = np.random.default_rng(9)
        for s in range(B):
            m.reset_slot(s)
            m.prefill(s, oracle.random_tokens(16, V, 50 + s))
        toks = [int(t) for t in rng.integers(0, V, B)]
        out = torch.zeros((B, V), dtype=torch.float32, device="cuda")
        got = []
        for step in range(6):
            if step == 3:  # a 100-token prompt regrows the prefill workspace under live graphs
                m.reset_slot(B - 1)
                m.prefill(B - 1, oracle.random_tokens(100, V, 77))
            st = m.decode(list(range(B)), toks, out)
            ctx.synchronize()
            got.append(out.cpu().numpy().copy())
            toks = [int(r["argmax"]) for r in st]
        outs.append(got)
        m.close()
    for a, b in zip(outs[0], outs[1]):
        assert np.all(np.isfinite(a))
        assert np.array_equal(a, b)
