"""BASELINE config 2: quantized-GEMV sweep at Llama-7B linear shapes.

For every (K x N) shape, bit-width and batch: device-generated N(0,0.02) weights quantized
per-group-128 on the device (K9), fp16 N(0,1) activations.  Two timings, both with CUDA events
on the launching stream:

* ``cold``  — one launch after a 256 MiB L2 flush (median of --iters);
* ``chain`` — R distinct copies of the layer (> 2x L2 in total, so every launch streams from
  HBM) launched back to back inside one CUDA graph; per-launch time = graph time / R (each
  launch pays the persistent program's start-up, ~10 us);
* ``program`` — the same R layers as R independent phases of ONE step-program launch (no grid
  barrier between them), as the decode step streams its linears; per-GEMV time = launch / R.

Prints one JSON line per case: algorithmic bytes / time and the fraction of measured HBM peak.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12024_b200 import capi  # noqa: E402

SHAPES = [(4096, 4096), (4096, 11008), (11008, 4096), (4096, 32000)]  # (K, N)


def peak():
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        return json.load(open(p))["hbm_gbs"], "measured"
    except Exception:
        return 6650.0, "fallback"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--batches", default="1,4,16")
    ap.add_argument("--bits", default="8,4")
    ap.add_argument("--shapes", default="all")
    args = ap.parse_args()
    hbm, kind = peak()
    ctx = capi.Context(0)
    stream = torch.cuda.Stream()
    ctx.set_stream(stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    shapes = SHAPES if args.shapes == "all" else [SHAPES[int(i)] for i in args.shapes.split(",")]
    for K, N in shapes:
        w = torch.empty(N * K, dtype=torch.float32, device="cuda")
        ctx.fill_normal(w, N * K, 0, K * 100000 + N, 0.02)
        per = N * K * 1.5
        R = max(4, int(400e6 // per) + 1)
        layers = []
        for r in range(R):
            L = capi.Layer(ctx, N, K, 128)
            L.quantize_device(capi.RUNG_INT8, w)
            L.quantize_device(capi.RUNG_INT4, w)
            layers.append(L)
        del w
        for bits in [int(b) for b in args.bits.split(",")]:
            rung = capi.RUNG_INT8 if bits == 8 else capi.RUNG_INT4
            for B in [int(b) for b in args.batches.split(",")]:
                x = torch.randn(B, K, device="cuda").half()
                y = torch.empty(B, N, device="cuda", dtype=torch.float32)
                L0 = layers[0]
                with torch.cuda.stream(stream):
                    for _ in range(3):
                        ctx.gemv(L0, rung, B, x, capi.DT_F16, y, capi.DT_F32)
                    times = []
                    for _ in range(args.iters):
                        flush.fill_(1)
                        e0 = torch.cuda.Event(enable_timing=True)
                        e1 = torch.cuda.Event(enable_timing=True)
                        e0.record(stream)
                        ctx.gemv(L0, rung, B, x, capi.DT_F16, y, capi.DT_F32)
                        e1.record(stream)
                        e1.synchronize()
                        times.append(e0.elapsed_time(e1) * 1e-3)
                    times.sort()
                    t_cold = times[len(times) // 2]
                    # chain of distinct layers inside one graph
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=stream):
                        for L in layers:
                            ctx.gemv(L, rung, B, x, capi.DT_F16, y, capi.DT_F32)
                    for _ in range(3):
                        g.replay()
                    ch = []
                    for _ in range(max(3, args.iters // 4)):
                        e0 = torch.cuda.Event(enable_timing=True)
                        e1 = torch.cuda.Event(enable_timing=True)
                        e0.record(stream)
                        g.replay()
                        e1.record(stream)
                        e1.synchronize()
                        ch.append(e0.elapsed_time(e1) * 1e-3 / len(layers))
                    ch.sort()
                    t_chain = ch[len(ch) // 2]
                    # the same layers as ONE step-program launch (independent phases, no barrier):
                    # the TMA weight stream runs across layer boundaries as inside a decode step
                    ys = [torch.empty(B, N, device="cuda", dtype=torch.float32) for _ in layers]
                    t_prog = ctx.gemv_chain_time(layers, rung, B, x, capi.DT_F16, ys, capi.DT_F32,
                                                 max(3, args.iters // 4)) * 1e-3 / len(layers)
                    # the program's outputs are the stand-alone GEMV's
                    ctx.gemv(layers[-1], rung, B, x, capi.DT_F16, y, capi.DT_F32)
                    torch.cuda.synchronize()
                    prog_err = float((ys[-1] - y).abs().max() / y.abs().max().clamp_min(1e-30))
                byts = L0.algorithmic_bytes(rung, B)
                print(json.dumps({"K": K, "N": N, "bits": bits, "B": B, "bytes": byts,
                                  "cold_us": round(t_cold * 1e6, 2), "cold_GBps": round(byts / t_cold / 1e9, 1),
                                  "chain_us": round(t_chain * 1e6, 2), "chain_GBps": round(byts / t_chain / 1e9, 1),
                                  "chain_frac": round(byts / t_chain / 1e9 / hbm, 3),
                                  "program_us": round(t_prog * 1e6, 2), "program_GBps": round(byts / t_prog / 1e9, 1),
                                  "program_frac": round(byts / t_prog / 1e9 / hbm, 3), "program_vs_gemv_maxrel": prog_err,
                                  "layers": len(layers), "peak": hbm,
                                  "peak_kind": kind}), flush=True)
        for L in layers:
            L.close()


if __name__ == "__main__":
    main()
