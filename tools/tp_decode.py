"""Tensor-parallel decode (north_star's TP variant): one rank per GPU under torchrun, NCCL all-reduce
of the row-split partials between step segments (paper_2506_12024_b200/tp.py), vocab-split head
with the softmax partials all-gathered and merged on the host.

Each rank builds the full model on its GPU from the deterministic device generator (identical on
every rank), downloads each linear's W8/W4 copies, keeps its slice (fq_shard_quantized) in a TP
rank model and frees the full model.  Timed: `--steps` decode steps after a `--prompt`-token prompt
fed through the same segments, CUDA events on the engine stream, max over ranks.  Prints one JSON
line (rank 0).

  python tools/tp_decode.py --shape 7b                      # TP 1 (one GPU; NCCL with one rank)
  torchrun --nproc-per-node 8 --master-addr 127.0.0.1 tools/tp_decode.py --shape 13b
  python tools/tp_decode.py --local 2 --layers 2            # 2 ranks in one process (functional)
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12024_b200 import capi, tp  # noqa: E402

SHAPES = {
    "7b": dict(vocab_size=32000, d_model=4096, n_heads=32, head_dim=128, n_layers=32, ffn_dim=11008),
    "13b": dict(vocab_size=32000, d_model=5120, n_heads=40, head_dim=128, n_layers=40, ffn_dim=13824),
}


def build_rank(ctx, cfg, rank, size, seed):
    full = capi.Model(ctx, arch=capi.ARCH_LLAMA, act_dtype=capi.DT_BF16, max_batch=1, group_size=128, **cfg)
    full.init_random(seed, 0.02)
    m = capi.Model(ctx, tp=(rank, size), arch=capi.ARCH_LLAMA, act_dtype=capi.DT_BF16, max_batch=1,
                   group_size=128, **cfg)
    emb = full.get_param("tok_emb", cfg["vocab_size"] * cfg["d_model"])
    for idx, lid in enumerate(full.ids):
        q = {}
        L = full.linear(idx)
        for bits, rung in ((8, capi.RUNG_INT8), (4, capi.RUNG_INT4)):
            p, s, z = L.download_quantized(rung)
            q[bits] = (p, s, z)
        tp.upload_shard_one(m, idx, lid, q)
    m.set_param("tok_emb", emb)
    full.close()
    return m


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="7b", choices=list(SHAPES))
    ap.add_argument("--layers", type=int, default=0, help="override n_layers (0 = the shape's)")
    ap.add_argument("--prompt", type=int, default=16)
    ap.add_argument("--steps", type=int, default=32)
    ap.add_argument("--local", type=int, default=0, help="run this many ranks in one process (functional)")
    ap.add_argument("--w4-frac", type=float, default=0.5)
    ap.add_argument("--no-graphs", action="store_true", help="enqueue the segments from the host every step")
    a = ap.parse_args()
    cfg = dict(SHAPES[a.shape], max_seq_len=a.prompt + a.steps + 8)
    if a.layers:
        cfg["n_layers"] = a.layers
    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    import torch.distributed as dist
    if a.local:
        size, ranks = a.local, list(range(a.local))
        ex = tp.LocalExchange(size)
    else:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=rank, world_size=world)
        size, ranks = world, [rank]
        ex = tp.DistExchange()
    ctx = capi.Context(local)
    t0 = time.time()
    models = [build_rank(ctx, cfg, r, size, 1234) for r in ranks]
    build_s = time.time() - t0
    rng = np.random.default_rng(5)
    table = [capi.RUNG_INT4 if rng.random() < a.w4_frac else capi.RUNG_INT8 for _ in range(models[0].n_linears)]
    for m in models:
        for i, r in enumerate(table):
            m.set_rung(0, i, r)
    dec = tp.TpDecoder(models, ex, graphs=not a.no_graphs)
    toks = np.random.default_rng(7).integers(0, cfg["vocab_size"], a.prompt + a.steps)
    tok = int(toks[0])
    for i in range(a.prompt):  # the prompt through the same segments
        dec.step([0], [int(toks[i])])
    st = dec.stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if not a.local:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record(st)
    argmaxes = []
    for i in range(a.steps):
        stats = dec.step([0], [tok])
        tok = int(stats["argmax"][0])
        argmaxes.append(tok)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if not a.local and world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    if rank == 0:
        sh = models[0].tp_shard()
        print(json.dumps({
            "tool": "tp_decode", "shape": a.shape, "n_layers": cfg["n_layers"], "tp": size,
            "in_process_ranks": len(models), "prompt": a.prompt, "steps": a.steps,
            "ms_per_token": ms / a.steps, "tokens_per_s": 1000.0 * a.steps / ms,
            "segments_per_token": sh.n_segments, "allreduces_per_token": sh.n_segments - 1,
            "exchange": "local (one process, sum on device)" if a.local else f"nccl x{world}",
            "w4_frac": a.w4_frac, "graphs": not a.no_graphs, "build_s": build_s, "argmax_tail": argmaxes[-4:],
            "note": "timing includes the host-side segment loop and the host merge of the head statistics",
        }))
    for m in models:
        m.close()
    if not a.local:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
