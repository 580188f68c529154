"""Times fq_model_prefill on the 7B shape for a few prompt lengths (wall clock around the
synchronous call; the threshold env FQ_GEMM_PREFILL_MIN picks the tensor-core or the 8-row
program path) and checks that both paths agree on the last row's statistics."""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12024_b200 import capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--lens", default="64,256,512")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--w4", action="store_true")
a = ap.parse_args()
ctx = capi.Context(0)
m = capi.Model(ctx, arch=capi.ARCH_LLAMA, act_dtype=capi.DT_BF16, max_batch=1, group_size=128, max_seq_len=1024,
               vocab_size=32000, d_model=4096, n_heads=32, head_dim=128, n_layers=32, ffn_dim=11008)
m.init_random(1234, 0.02)
if a.w4:
    m.set_all_rungs(0, capi.RUNG_INT4)
for n in [int(x) for x in a.lens.split(",")]:
    toks = (np.arange(n, dtype=np.int64) * 7919 % 32000).astype(np.int32)
    times = []
    for _ in range(a.reps + 1):
        m.reset_slot(0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = m.prefill(0, toks)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    t = sorted(times[1:])[len(times[1:]) // 2]
    print(json.dumps({"prompt": n, "ms": round(t * 1e3, 3), "tok_per_s": round(n / t, 1),
                      "path": "gemm" if int(os.environ.get("FQ_GEMM_PREFILL_MIN", "16") or 0) and
                      n >= int(os.environ.get("FQ_GEMM_PREFILL_MIN", "16")) else "program",
                      "last_entropy": float(st["entropy"][-1]), "last_argmax": int(st["argmax"][-1]),
                      "mean_entropy": float(np.mean(st["entropy"]))}))
