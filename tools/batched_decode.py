"""BASELINE config 5: batched heterogeneous-precision decode, B sequences per GPU.  Every sequence
has its own per-linear precision table (a random W8/W4 mix per slot, so a batch mixes both weight
copies), its own KV cache slot and position.  B < 16 rows step through the persistent step
program; B >= 16 through the tensor-core batched path (one tcgen05 GEMM per linear and copy
present, each copy streamed once per step).  Prints one JSON line per batch size: aggregate
tokens/s from device events on the engine stream around the timed steps, algorithmic bytes per
step (both weight copies where the batch mixes them + KV) and the HBM fraction.

Rank-aware (BASELINE C5 is 32 sequences per GPU on 8 GPUs): under torchrun every rank decodes its
own B sequences on its own GPU (no collective on the decode path); the time is the max over
ranks and tokens/s the whole-job aggregate.

  python tools/batched_decode.py --shape 13b --batches 1,8,32 --prompt 128 --steps 16
  torchrun --nproc-per-node 8 --master-addr 127.0.0.1 tools/batched_decode.py --batches 32
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12024_b200 import capi  # noqa: E402

SHAPES = {
    "7b": dict(vocab_size=32000, d_model=4096, n_heads=32, head_dim=128, n_layers=32, ffn_dim=11008),
    "13b": dict(vocab_size=32000, d_model=5120, n_heads=40, head_dim=128, n_layers=40, ffn_dim=13824),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="13b", choices=list(SHAPES))
    ap.add_argument("--batches", default="1,8,32")
    ap.add_argument("--prompt", type=int, default=128)
    ap.add_argument("--steps", type=int, default=16)
    ap.add_argument("--w4-frac", type=float, default=0.5, help="fraction of linears at W4 per slot")
    a = ap.parse_args()
    batches = [int(b) for b in a.batches.split(",")]
    maxb = max(batches)
    hbm = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                      "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) else 6650.0
    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    ctx = capi.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream_handle())
    m = capi.Model(ctx, arch=capi.ARCH_LLAMA, act_dtype=capi.DT_BF16, max_batch=maxb, group_size=128,
                   max_seq_len=a.prompt + a.steps + 8, **SHAPES[a.shape])
    m.init_random(1234, 0.02)
    rng = np.random.default_rng(1000 + rank)
    for s in range(maxb):
        for li in range(m.n_linears):
            m.set_rung(s, li, capi.RUNG_INT4 if rng.random() < a.w4_frac else capi.RUNG_INT8)
    for B in batches:
        slots = list(range(B))
        for s in slots:
            m.reset_slot(s)
            m.prefill(s, rng.integers(0, SHAPES[a.shape]["vocab_size"], a.prompt).astype(np.int32))
        toks = [int(t) for t in rng.integers(0, SHAPES[a.shape]["vocab_size"], B)]
        for _ in range(2):  # warm-up (builds and captures the B-row step program)
            st = m.decode(slots, toks)
            toks = [int(r["argmax"]) for r in st]
        torch.cuda.synchronize()
        wb, kb = m.step_bytes(slots)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        e0.record(stream)
        for _ in range(a.steps):
            st = m.decode(slots, toks)
            toks = [int(r["argmax"]) for r in st]
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        per = ms / a.steps
        if rank == 0:
            print(json.dumps({"shape": a.shape, "batch_per_gpu": B, "n_gpus": world, "w4_frac": a.w4_frac,
                              "context": a.prompt, "path": "tensor-core batched" if B >= 16 else "step program",
                              "ms_per_step": round(per, 4), "tokens_per_s": round(world * B / (per / 1e3), 1),
                              "weight_bytes_per_step": wb, "kv_bytes_per_step": kb,
                              "step_GBps": round((wb + kb) / (per / 1e3) / 1e9, 1),
                              "hbm_frac": round((wb + kb) / (per / 1e3) / 1e9 / hbm, 3), "steps": a.steps}), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
