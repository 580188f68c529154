"""BASELINE config 2: quantized-GEMV sweep at Llama-7B linear shapes.

For every (K x N) shape, bit-width and batch: device-generated N(0,0.02) weights quantized
per-group-128 on the device (K9), fp16 N(0,1) activations, one GEMV timed with CUDA events
on the launching stream; L2 is flushed (256 MiB write) before every timed launch.  Prints one
JSON line per case with algorithmic bytes / time and the fraction of measured HBM peak.
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
    args = ap.parse_args()
    hbm, kind = peak()
    ctx = capi.Context(0)
    stream = torch.cuda.Stream()
    ctx.set_stream(stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for K, N in SHAPES:
        w = torch.empty(N * K, dtype=torch.float32, device="cuda")
        ctx.fill_normal(w, N * K, 0, K * 100000 + N, 0.02)
        L = capi.Layer(ctx, N, K, 128)
        L.quantize_device(capi.RUNG_INT8, w)
        L.quantize_device(capi.RUNG_INT4, w)
        del w
        for bits in [int(b) for b in args.bits.split(",")]:
            rung = capi.RUNG_INT8 if bits == 8 else capi.RUNG_INT4
            for B in [int(b) for b in args.batches.split(",")]:
                x = torch.randn(B, K, device="cuda").half()
                y = torch.empty(B, N, device="cuda", dtype=torch.float32)
                with torch.cuda.stream(stream):
                    for _ in range(3):
                        ctx.gemv(L, rung, B, x, capi.DT_F16, y, capi.DT_F32)
                    times = []
                    for _ in range(args.iters):
                        flush.fill_(1)
                        e0 = torch.cuda.Event(enable_timing=True)
                        e1 = torch.cuda.Event(enable_timing=True)
                        e0.record(stream)
                        ctx.gemv(L, rung, B, x, capi.DT_F16, y, capi.DT_F32)
                        e1.record(stream)
                        e1.synchronize()
                        times.append(e0.elapsed_time(e1) * 1e-3)
                times.sort()
                t = times[len(times) // 2]
                byts = L.algorithmic_bytes(rung, B)
                gbs = byts / t / 1e9
                print(json.dumps({"K": K, "N": N, "bits": bits, "B": B, "us": round(t * 1e6, 2),
                                  "bytes": byts, "GBps": round(gbs, 1), "frac": round(gbs / hbm, 3),
                                  "peak": hbm, "peak_kind": kind}), flush=True)
        L.close()


if __name__ == "__main__":
    main()
