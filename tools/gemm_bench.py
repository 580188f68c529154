"""tcgen05 dequant-GEMM throughput at Llama-7B linear shapes (prefill / calibration, BASELINE
config 4): TFLOP/s of y[T,N] = x[T,K] . dequant(W)^T with CUDA events on the launch stream."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12024_b200 import capi  # noqa: E402

SHAPES = [(4096, 4096), (4096, 11008), (11008, 4096), (4096, 32000)]  # (K, N)

ap = argparse.ArgumentParser()
ap.add_argument("--T", default="512,2048")
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--bits", default="8,4")
ap.add_argument("--shapes", default="all")
ap.add_argument("--graph", action="store_true", help="time a CUDA graph of the launches (no host launch gaps)")
a = ap.parse_args()
peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
ctx = capi.Context(0)
stream = torch.cuda.Stream()
ctx.set_stream(stream)
shapes = SHAPES if a.shapes == "all" else [SHAPES[int(i)] for i in a.shapes.split(",")]
for K, N in shapes:
    w = torch.empty(N * K, dtype=torch.float32, device="cuda")
    ctx.fill_normal(w, N * K, 0, 7, 0.02)
    L = capi.Layer(ctx, N, K, 128)
    for bits in [int(b) for b in a.bits.split(",")]:
        rung = capi.RUNG_INT8 if bits == 8 else capi.RUNG_INT4
        L.quantize_device(rung, w)
        for T in [int(t) for t in a.T.split(",")]:
            x = torch.randn(T, K, device="cuda").to(torch.bfloat16)
            y = torch.empty(T, N, device="cuda")
            # the prefill's own operand format: activations pre-tiled once (fq_tile_activations)
            xt = torch.zeros(ctx.tiled_activation_bytes(T, K), dtype=torch.uint8, device="cuda")
            with torch.cuda.stream(stream):
                ctx.tile_activations(x, capi.DT_BF16, T, K, capi.DT_F16, xt)
                for _ in range(2):
                    ctx.gemm_tiled(L, rung, T, xt, capi.DT_F16, y)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                if a.graph:
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=stream):
                        for _ in range(a.iters):
                            ctx.gemm_tiled(L, rung, T, xt, capi.DT_F16, y)
                    g.replay()
                    e0.record(stream)
                    g.replay()
                    e1.record(stream)
                else:
                    e0.record(stream)
                    for _ in range(a.iters):
                        ctx.gemm_tiled(L, rung, T, xt, capi.DT_F16, y)
                    e1.record(stream)
                e1.synchronize()
            ms = e0.elapsed_time(e1) / a.iters
            tf = 2.0 * T * N * K / (ms * 1e-3) / 1e12
            print(json.dumps({"K": K, "N": N, "T": T, "bits": bits, "ms": round(ms, 4), "tflops": round(tf, 1),
                              "frac_of_bf16_peak": round(tf / peaks["bf16_tflops"], 3)}), flush=True)
    L.close()
