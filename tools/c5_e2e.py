"""BASELINE config 5 end to end on one GPU: the 13B shape (40 blocks, d 5120, 40 heads, ffn 13824,
V 32000), 32 sequences per GPU, 128-token random prompts, 512 decode tokens, every sequence with
its own SchedulerState and precision table, through the reference-facing C++ API
(flexquant::generate_batch, libflexquant_b200.so): the prompts' tcgen05 prefills, then the
batched decode steps (tensor-core path at B >= 16, one CUDA graph per (B, copies present)
signature; the signature changes as the schedulers switch blocks from W8 to W4).

Plan: 8 -> 4 block by block, the last block first (the shape of C4's ranking on random weights,
profiles/r02c_calibration_c4_full.json), head last.  Scheduler: Prefill threshold mode (theta x
the mean PPLE of the last W prompt rows), W = 20, 7 linears (one block) per switch.

  python tools/c5_e2e.py [--seqs 32 --prompt 128 --decode 512 --theta 1.05]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12024_b200 import _flexquant as fq  # noqa: E402

C13B = dict(vocab_size=32000, d_model=5120, n_heads=40, head_dim=128, n_layers=40, ffn_dim=13824)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seqs", type=int, default=32)
    ap.add_argument("--prompt", type=int, default=128)
    ap.add_argument("--decode", type=int, default=512)
    ap.add_argument("--theta", type=float, default=1.05)
    ap.add_argument("--window", type=int, default=20)
    a = ap.parse_args()
    fc = fq.ModelConfig()
    fc.arch = fq.Arch.Llama
    for k, v in C13B.items():
        setattr(fc, k, v)
    fc.max_seq_len, fc.group_size, fc.max_batch = a.prompt + a.decode + 8, 128, a.seqs
    model = fq.Model(fc)
    model.init_random(1234, 0.02)
    ids = list(model.linear_ids())
    per = 7
    blocks = [ids[b * per:(b + 1) * per] for b in range(C13B["n_layers"])]
    plan = fq.SwitchPlan()
    ents = []
    for blk in reversed(blocks):
        for lid in blk:
            e = fq.SwitchEntry()
            e.layer_id, e.from_, e.to, e.kl = lid, fq.Rung.Int8, fq.Rung.Int4, 0.0
            ents.append(e)
    plan.entries = ents
    cfg = fq.GenerationConfig()
    cfg.max_new_tokens = a.decode
    cfg.start_rung = fq.Rung.Int8
    cfg.scheduler.threshold_mode = fq.ThresholdMode.Prefill
    cfg.scheduler.theta = a.theta
    cfg.scheduler.window_len = a.window
    cfg.scheduler.layers_per_switch = per
    rng = np.random.default_rng(55)
    prompts = [rng.integers(0, C13B["vocab_size"], a.prompt).astype(np.int32).tolist() for _ in range(a.seqs)]
    stream = torch.cuda.ExternalStream(fq.runtime_stream())
    warm = fq.GenerationConfig()
    warm.max_new_tokens = 4
    warm.start_rung = fq.Rung.Int8
    fq.generate_batch([p[:32] for p in prompts], model, plan, warm)  # program builds / first captures
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    res = fq.generate_batch(prompts, model, plan, cfg)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    toks = sum(len(r.sequence) for r in res)
    switches = [sum(len(rec.switch_events) for rec in r.trace.records) for r in res]
    final_bits = [r.trace.records[-1].effective_bits for r in res]
    print(json.dumps({"config": "C5 (13B shape), one GPU", "sequences": a.seqs, "prompt": a.prompt, "decode": a.decode,
                      "seconds": round(ms / 1e3, 3), "decode_tokens": toks,
                      "tokens_per_s": round(toks / (ms / 1e3), 1),
                      "ms_per_step": round(ms / a.decode, 3),
                      "switch_events_per_sequence": {"min": min(switches), "max": max(switches),
                                                     "mean": float(np.mean(switches))},
                      "final_effective_bits": {"min": min(final_bits), "max": max(final_bits)},
                      "theta": a.theta, "window": a.window, "api": "flexquant::generate_batch"}), flush=True)


if __name__ == "__main__":
    main()
