"""Runs one GEMV shape a few times (target for ncu captures)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12024_b200 import capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--K", type=int, default=4096)
ap.add_argument("--N", type=int, default=11008)
ap.add_argument("--bits", type=int, default=8)
ap.add_argument("--B", type=int, default=1)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
ctx = capi.Context(0)
w = torch.empty(a.N * a.K, dtype=torch.float32, device="cuda")
ctx.fill_normal(w, a.N * a.K, 0, 1, 0.02)
L = capi.Layer(ctx, a.N, a.K, 128)
rung = capi.RUNG_INT8 if a.bits == 8 else capi.RUNG_INT4
L.quantize_device(rung, w)
x = torch.randn(a.B, a.K, device="cuda").half()
y = torch.empty(a.B, a.N, device="cuda")
for _ in range(a.reps):
    ctx.gemv(L, rung, a.B, x, capi.DT_F16, y, capi.DT_F32)
ctx.synchronize()
print("ok", float(y.abs().sum()))
