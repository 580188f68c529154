"""Tensor-parallel variant, host side (no GPU): shard layout, quantized slicing, statistics merge,
and the torch.distributed exchange on gloo at world size 2.

The reference has no distribution (its block: src/model.cpp:201-233); these pin the pieces the
sharded step is built from against the unsplit reference semantics:
* slicing a g128 QuantizedTensor is bit-identical to quantizing the sliced fp32 weights
  (quantize_impl is per group, src/quantizer.cpp:111-189);
* merging the ranks' softmax partials reproduces softmax_double / ppl_entropy / fault_tolerance /
  argmax_token of the whole row (src/scheduler.cpp:13-49, src/engine.cpp:144-155), ties included;
* the row-split partials summed by the all-reduce equal the unsplit linear.
"""
import os
import socket

import numpy as np
import pytest

import oracle
from paper_2506_12024_b200 import capi, tp

C3 = dict(vocab_size=32000, d_model=4096, n_heads=32, head_dim=128, n_layers=32, ffn_dim=11008, max_seq_len=512)
C1 = dict(vocab_size=8192, d_model=512, n_heads=8, head_dim=64, n_layers=4, ffn_dim=1376, max_seq_len=128)


def _cfg(d):
    return capi.model_config(arch=capi.ARCH_LLAMA, group_size=128, **d)


@pytest.mark.parametrize("dims,sizes", [(C3, (1, 2, 4, 8)), (C1, (1, 2, 4))])
def test_shard_spec_partitions_the_model(dims, sizes):
    cfg = _cfg(dims)
    for size in sizes:
        sh = [capi.tp_shard_spec(cfg, r, size) for r in range(size)]
        assert [s.head0 for s in sh] == [r * dims["n_heads"] // size for r in range(size)]
        assert sum(s.heads for s in sh) == dims["n_heads"]
        assert sum(s.ffn for s in sh) == dims["ffn_dim"] and sum(s.vocab for s in sh) == dims["vocab_size"]
        for a, b in zip(sh, sh[1:]):
            assert a.ffn0 + a.ffn == b.ffn0 and a.vocab0 + a.vocab == b.vocab0
        assert all(s.ffn0 % 128 == 0 for s in sh)  # no quantization group straddles two ranks
        assert all(s.n_segments == 2 * dims["n_layers"] + 1 for s in sh)
    # C1 ffn 1376 = 10 groups + a 96 tail: the tail stays with the last rank
    s = capi.tp_shard_spec(_cfg(C1), 1, 2)
    assert (s.ffn0, s.ffn) == (640, 736)


def test_shard_spec_rejects_bad_splits():
    with pytest.raises(capi.ConfigError):
        capi.tp_shard_spec(_cfg(C1), 0, 8)  # 1 head x 64 = half a group per rank
    with pytest.raises(capi.ConfigError):
        capi.tp_shard_spec(_cfg(C1), 0, 3)  # 8 heads over 3 ranks
    with pytest.raises(capi.ConfigError):
        capi.tp_shard_spec(_cfg(C1), 2, 2)


@pytest.mark.parametrize("bits", [8, 4])
@pytest.mark.parametrize("N,K,rows,cols", [
    (48, 1376, (16, 40), (0, 1376)),     # column split of gate/up: rows
    (40, 1376, (0, 40), (640, 1376)),    # row split of down: input columns incl. the ragged tail
    (40, 1376, (0, 40), (128, 512)),
    (64, 512, (8, 56), (256, 512)),
])
def test_shard_quantized_equals_quantizing_the_slice(bits, N, K, rows, cols):
    w = oracle.normal(N * K, 3, 1, 0.02).reshape(N, K)
    w[5, 128:256] = 0.25  # a constant group (exact path of quantize_impl)
    p, s, z = oracle.quantize(w, 128, bits)
    got = capi.shard_quantized(bits, N, K, 128, p, s, z, rows, cols)
    want = oracle.quantize(np.ascontiguousarray(w[rows[0]:rows[1], cols[0]:cols[1]]), 128, bits)
    assert np.array_equal(got[0], want[0])
    assert np.array_equal(got[1], want[1].ravel()) and np.array_equal(got[2], want[2].ravel())


def test_shard_quantized_rejects_straddling_groups():
    w = oracle.normal(16 * 512, 3, 2, 0.02).reshape(16, 512)
    p, s, z = oracle.quantize(w, 128, 8)
    with pytest.raises(capi.DimensionError):
        capi.shard_quantized(8, 16, 512, 128, p, s, z, (0, 16), (64, 512))


def _part(l: np.ndarray) -> np.ndarray:
    """The mergeable softmax partial of one slice (what the head segment's STATS phase emits)."""
    out = np.zeros(1, capi.STAT_PART_DTYPE)
    m = float(np.max(l))
    e = np.exp(l.astype(np.float64) - m)
    out["S"], out["T"] = e.sum(), (e * (l.astype(np.float64) - m)).sum()
    srt = np.sort(l)
    out["m"], out["v1"] = m, srt[-1]
    out["v2"] = srt[-2] if l.size > 1 else -np.inf
    out["arg"] = int(np.argmax(l))  # lowest index of the max
    return out[0]


@pytest.mark.parametrize("size", [2, 3, 4, 8])
def test_merge_stats_equals_whole_row(size):
    V, B = 8192, 3
    rng = np.random.default_rng(size)
    logits = rng.normal(0, 2.0, (B, V)).astype(np.float32)
    logits[1, 100] = logits[1, 5000] = logits[1].max() + 1.0  # tie across ranks: lowest index wins
    logits[2, :] = 0.5  # flat row: p1 == p2
    cfg = _cfg(dict(C1, vocab_size=V))
    sh = [capi.tp_shard_spec(cfg, r, size) if size in (2, 4) else None for r in range(size)]
    bounds = [V * r // size for r in range(size + 1)]
    if size in (2, 4):
        assert [s.vocab0 for s in sh] == bounds[:-1]
    parts = np.zeros((size, B), capi.STAT_PART_DTYPE)
    for r in range(size):
        for b in range(B):
            parts[r, b] = _part(logits[b, bounds[r]:bounds[r + 1]])
    got = capi.tp_merge_stats(parts, bounds[:-1])
    for b in range(B):
        want = oracle.row_stats(logits[b])
        assert got["argmax"][b] == want["argmax"]
        for k in ("entropy", "ppl_entropy", "p1", "p2", "fault_tolerance"):
            assert abs(got[k][b] - want[k]) <= 1e-12 * max(1.0, abs(want[k])), (b, k)
    assert got["argmax"][1] == 100


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = _cfg(C1)
        sh = capi.tp_shard_spec(cfg, rank, world)
        ex = tp.DistExchange()
        # row-split down projection: this rank's input columns of the ffn activation
        d, f = C1["d_model"], C1["ffn_dim"]
        w = oracle.normal(d * f, 5, 0, 0.02).reshape(d, f)
        x = oracle.normal(2 * f, 5, 1, 1.0).reshape(2, f)
        (r0, r1), (c0, c1) = tp.linear_ranges("blocks.0.ffn.w_down", cfg, sh)
        part = torch.from_numpy((x[:, c0:c1].astype(np.float64) @ w[r0:r1, c0:c1].T.astype(np.float64))
                                .astype(np.float32))
        ex.allreduce([part])
        # vocab-split head statistics: all-gather of the 32-byte partials, host merge
        V = C1["vocab_size"]
        logits = np.random.default_rng(9).normal(0, 3.0, (2, V)).astype(np.float32)
        mine = np.stack([_part(logits[b, sh.vocab0:sh.vocab0 + sh.vocab]) for b in range(2)])
        gathered = ex.allgather([torch.from_numpy(mine.view(np.uint8).copy())])
        parts = np.stack([g.numpy().view(capi.STAT_PART_DTYPE) for g in gathered])
        v0 = [capi.tp_shard_spec(cfg, r, world).vocab0 for r in range(world)]
        st = capi.tp_merge_stats(parts, v0)
        q.put((rank, part.numpy(), (x.astype(np.float64) @ w.T.astype(np.float64)), st, logits))
    finally:
        dist.destroy_process_group()


def test_exchange_gloo_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, summed, want, st, logits in res:
        assert np.max(np.abs(summed - want)) <= 1e-5 * np.max(np.abs(want))  # fp32 sum of 2 partials
        for b in range(2):
            o = oracle.row_stats(logits[b])
            assert st["argmax"][b] == o["argmax"] and abs(st["entropy"][b] - o["entropy"]) <= 1e-12
    assert np.array_equal(res[0][1], res[1][1])  # every rank holds the same reduced partial
