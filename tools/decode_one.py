"""Builds the 7B-shape model, prefills a short prompt and runs a few decode steps (target for
ncu launch lists and captures of the decode step)."""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12024_b200 import capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--prompt", type=int, default=8)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--w4", action="store_true")
ap.add_argument("--layers", type=int, default=32)
ap.add_argument("--fixed-token", type=int, default=-1)
a = ap.parse_args()
ctx = capi.Context(0)
m = capi.Model(ctx, arch=capi.ARCH_LLAMA, act_dtype=capi.DT_BF16, max_batch=1, group_size=128, max_seq_len=512,
               vocab_size=32000, d_model=4096, n_heads=32, head_dim=128, n_layers=a.layers, ffn_dim=11008)
m.init_random(1234, 0.02)
if a.w4:
    m.set_all_rungs(0, capi.RUNG_INT4)
toks = np.arange(a.prompt, dtype=np.int32) * 37 % 32000
st = m.prefill(0, toks)
row = st[-1]
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(a.steps):
    row = m.decode([0], [int(row["argmax"]) if a.fixed_token < 0 else a.fixed_token])[0]
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / a.steps
ms, n, b = m.profile_gemvs(0, 10)
print(f"step {dt*1e3:.3f} ms  gemv {ms*1e3:.2f} us x {n} launches = {ms*n:.3f} ms  bytes/pass {b/1e9:.3f} GB")
