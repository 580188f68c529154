"""BASELINE config 5 on one GPU: batched heterogeneous-precision decode.  B sequences decode
together in one step program per token; every sequence has its own per-linear precision table
(a random W8/W4 mix per slot, so a batch mixes both weight copies inside each GEMV phase), its own
KV cache slot and position.  Prints one JSON line per batch size: aggregate tokens/s from device
events around the step launches, algorithmic bytes per step (both weight copies where the batch
mixes them + KV) and the HBM fraction.

  python tools/batched_decode.py --shape 13b --batches 1,8,32 --prompt 128 --steps 16
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
    ctx = capi.Context(0)
    m = capi.Model(ctx, arch=capi.ARCH_LLAMA, act_dtype=capi.DT_BF16, max_batch=maxb, group_size=128,
                   max_seq_len=a.prompt + a.steps + 8, **SHAPES[a.shape])
    m.init_random(1234, 0.02)
    rng = np.random.default_rng(0)
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
        m.step_kernel_time(reset=True)
        wb, kb = m.step_bytes(slots)
        for _ in range(a.steps):
            st = m.decode(slots, toks)
            toks = [int(r["argmax"]) for r in st]
        torch.cuda.synchronize()
        ms, n = m.step_kernel_time(reset=True)
        per = ms / max(n, 1)
        print(json.dumps({"shape": a.shape, "batch": B, "w4_frac": a.w4_frac, "context": a.prompt,
                          "ms_per_step": round(per, 4), "tokens_per_s": round(B / (per / 1e3), 1),
                          "weight_bytes_per_step": wb, "kv_bytes_per_step": kb,
                          "step_GBps": round((wb + kb) / (per / 1e3) / 1e9, 1),
                          "hbm_frac": round((wb + kb) / (per / 1e3) / 1e9 / hbm, 3), "steps": n}), flush=True)


if __name__ == "__main__":
    main()
