"""One chained-GEMV program launch (R independent 4096x32000 layers, one rung) for ncu captures of
the GEMV loop without the decode step's barriers: python tools/gemv_chain_one.py --bits 4"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12024_b200 import capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--bits", type=int, default=4)
ap.add_argument("--K", type=int, default=4096)
ap.add_argument("--N", type=int, default=32000)
ap.add_argument("--R", type=int, default=4)
a = ap.parse_args()
ctx = capi.Context(0)
w = torch.empty(a.N * a.K, dtype=torch.float32, device="cuda")
ctx.fill_normal(w, a.N * a.K, 0, 7, 0.02)
rung = capi.RUNG_INT8 if a.bits == 8 else capi.RUNG_INT4
layers = []
for r in range(a.R):
    L = capi.Layer(ctx, a.N, a.K, 128)
    L.quantize_device(rung, w)
    layers.append(L)
x = torch.randn(1, a.K, device="cuda").half()
ys = [torch.empty(1, a.N, device="cuda", dtype=torch.float32) for _ in layers]
ms = ctx.gemv_chain_time(layers, rung, 1, x, capi.DT_F16, ys, capi.DT_F32, 2)
print(f"{a.K}x{a.N} W{a.bits} x{a.R}: {ms * 1e3 / a.R:.2f} us per GEMV")
