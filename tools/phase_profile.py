"""Per-phase timing of one 7B-shape decode step (the persistent step program): for every phase,
the slowest CTA's work time and the grid-barrier wait that follows, aggregated by phase kind."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12024_b200 import capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--prompt", type=int, default=256)
ap.add_argument("--w4", action="store_true")
ap.add_argument("--layers", type=int, default=32)
ap.add_argument("--reps", type=int, default=9)
a = ap.parse_args()
ctx = capi.Context(0)
m = capi.Model(ctx, arch=capi.ARCH_LLAMA, act_dtype=capi.DT_BF16, max_batch=1, group_size=128, max_seq_len=512,
               vocab_size=32000, d_model=4096, n_heads=32, head_dim=128, n_layers=a.layers, ffn_dim=11008)
m.init_random(1234, 0.02)
if a.w4:
    m.set_all_rungs(0, capi.RUNG_INT4)
toks = (np.arange(a.prompt, dtype=np.int32) * 37) % 32000
m.prefill(0, toks)
names = {0: "gemv", 1: "embed", 2: "attn", 3: "stats", 4: "append"}
totals = []
for rep in range(a.reps):
    types, end, after, start = m.profile_step(0, 5)
    t0 = start.min()
    prev = np.full(end.shape[1], t0)
    work = []  # per phase: max over CTAs of (end - previous release)
    for i in range(len(types)):
        w = end[i] - prev
        work.append((types[i], w.max(), w.mean(), after[i].max() - end[i].max()))
        prev = after[i]
    total = after[-1].max() - t0
    totals.append(total / 1e3)
    if rep == a.reps - 1:
        print("step totals (us):", " ".join(f"{x:.0f}" for x in totals), " median", f"{np.median(totals):.0f}")
        agg = {}
        for ty, wmax, wmean, bar in work:
            k = names[int(ty)]
            s = agg.setdefault(k, [0, 0.0, 0.0, 0.0])
            s[0] += 1
            s[1] += wmax
            s[2] += wmean
            s[3] += bar
        print(f"step {total/1e3:.1f} us, {len(types)} phases ({'W4' if a.w4 else 'W8'}, ctx {a.prompt})")
        for k, (n, wmax, wmean, bar) in agg.items():
            print(f"  {k:6s} x{n:4d}: slowest-CTA work {wmax/1e3:8.1f} us  mean-CTA work {wmean/1e3:8.1f} us  "
                  f"barrier tail {bar/1e3:7.1f} us")
        roles = {}
        for i, (ty, wmax, wmean, bar) in enumerate(work):
            if names[int(ty)] != "gemv":
                continue
            r = "head" if i == len(work) - 2 else ["qkv", "attn", "o", "gate_up", "down"][(i - 1) % 5]
            e = roles.setdefault(r, [0, 0.0])
            e[0] += 1
            e[1] += wmax
        for r, (n, t) in roles.items():
            print(f"  gemv[{r:7s}] x{n:3d}: {t/1e3:8.1f} us  ({t/n/1e3:6.2f} us each)")
        for i in range(min(12, len(types))):
            ty, wmax, wmean, bar = work[i]
            print(f"    phase {i:3d} {names[int(ty)]:5s} max {wmax/1e3:7.2f} mean {wmean/1e3:7.2f} bar {bar/1e3:6.2f} us")
# ring trace of CTA 0 over the last profiled step, per weight stage: producer got the slot (issue),
# consumer warp 0 started waiting for it, data ready
tr = m.last_ring_trace
tr = tr[tr[:, 0] > 0]
if len(tr) and not tr[:, 1].any():
    print(f"ring trace CTA0: {len(tr)} producer stamps; consumer stamps off (build program.cu with -DFQ_RING_TRACE=1, "
          "e.g. tools/ab_build.sh trace -DFQ_RING_TRACE=1 and FQ_CUDA_LIB=...)")
elif len(tr):
    t0 = tr[0, 0]
    lat = tr[:, 2] - tr[:, 0]
    waited = np.maximum(tr[:, 2] - tr[:, 1], 0)
    print(f"ring trace CTA0: {len(tr)} stages; issue->ready median {np.median(lat)/1e3:.2f} us; consumer wait total "
          f"{waited.sum()/1e3:.1f} us (stages waited >0.2us: {(waited > 200).sum()})")
    proc = tr[1:, 1] - tr[:-1, 2]
    print(f"  warp-0 time per stage between ready and the next want: median {np.median(proc)/1e3:.2f} us, "
          f"p90 {np.percentile(proc, 90)/1e3:.2f} us")
    for i in list(range(0, min(len(tr), 24))) + list(range(min(len(tr), 200), min(len(tr), 240))):
        print(f"   stage {i:3d} issue {(tr[i,0]-t0)/1e3:8.2f} want {(tr[i,1]-t0)/1e3:8.2f} ready {(tr[i,2]-t0)/1e3:8.2f}")
# GEMV phase detail: per role, sums over phases of the per-phase max over CTAs of each interval
det = m.last_gemv_detail
labels = ["setup(w1)", "rstd(w0)", "bar1", "stage", "loop", "red.sync", "red.rest", "tail"]
segs = {}
for i in range(len(types)):
    if names[int(types[i])] != "gemv":
        continue
    st = after[i - 1] if i > 0 else start
    d = det[i].astype(np.float64)
    r = "head" if i == len(types) - 2 else ["qkv", "attn", "o", "gate_up", "down"][(i - 1) % 5]
    e = segs.setdefault(r, np.zeros(8))
    e += [np.max(d[:, 0] - st), np.max(d[:, 1] - st), np.max(d[:, 2] - st), np.max(d[:, 3] - d[:, 2]),
          np.max(d[:, 4] - d[:, 3]), np.max(d[:, 7] - d[:, 4]), np.max(d[:, 5] - d[:, 7]), np.max(d[:, 6] - d[:, 5])]
for r, v in segs.items():
    print(f"  detail {r:8s}: " + "  ".join(f"{l} {x/1e3:7.1f}" for l, x in zip(labels, v)) + " us")
# raw stamps of phase 3 (O-proj of layer 0) for a few CTAs, relative to the previous release
i = 3
st = after[i - 1]
for c in (0, 5, 77, 147):
    d = det[i, c]
    print(f"  phase {i} cta {c:3d}: " + " ".join(f"{l}={(d[k] - st[c]) / 1e3:6.2f}" for k, l in
          [(0, "setup"), (1, "rstd"), (2, "bar1"), (3, "staged"), (4, "loop"), (7, "redsync"), (5, "red"), (6, "end")]))
# attention work distribution over CTAs (layer 0 and the median layer)
att = [i for i in range(len(types)) if names[int(types[i])] == "attn"]
for i in att[:1] + att[len(att) // 2: len(att) // 2 + 1]:
    w = (end[i] - after[i - 1]) / 1e3
    print(f"  attn phase {i}: work us p0 {np.min(w):.2f} p50 {np.median(w):.2f} p90 {np.percentile(w, 90):.2f} "
          f"max {np.max(w):.2f} (argmax cta {int(np.argmax(w))})")
for i in att[:4]:
    w = (end[i] - after[i - 1]) / 1e3
    top = np.argsort(-w)[:4]
    print(f"  attn phase {i}: slowest ctas " + ", ".join(f"{int(c)}:{w[c]:.2f}" for c in top))
for i in [1, 3, 4, 5]:
    w = (end[i] - (after[i - 1] if i > 0 else start)) / 1e3
    top = np.argsort(-w)[:4]
    print(f"  {names[int(types[i])]} phase {i}: slowest ctas " + ", ".join(f"{int(c)}:{w[c]:.2f}" for c in top) + f"  median {np.median(w):.2f}")
