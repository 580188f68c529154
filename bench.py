#!/usr/bin/env python
"""Headline benchmark: entropy-switched W8/W4 decode of the Llama-2-7B-shaped config (BASELINE
config 3) on the B200 engine, plus the kernel roofline of the dominant kernel (the GEMV) and the
reference CPU path timed on the same box.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c3|c1]

One step = one greedy decode token of every sequence, driven by the engine loop: fused step graph
(prefetching GEMVs, RoPE/attention, head, softmax statistics) -> D2H of the row statistics ->
host scheduler (SchedulerState::observe semantics) -> precision-table writes for the switches.
Multi-GPU: one process per GPU, independent sequences per rank (data-parallel, no collective on
the decode path); the timed region is bracketed by barriers and the time is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c3": dict(vocab_size=32000, d_model=4096, n_heads=32, head_dim=128, n_layers=32, ffn_dim=11008, prompt=256,
               decode=256, name="llama2-7b-shape"),
    "c1": dict(vocab_size=8192, d_model=512, n_heads=8, head_dim=64, n_layers=4, ffn_dim=1376, prompt=32, decode=64,
               name="tiny-4L-d512"),
}
METRIC = "decode tokens/s (7B-shape, entropy-switched W8/W4)"
CAL_SEQS, CAL_LEN = 4, 128  # logit-KL calibration sample that orders the switch plan


def peaks():
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clock / throttle-reason sampling during the timed region: NVML polled every 2 ms from a
    thread (the timed region of the default run is ~45 ms, shorter than nvidia-smi's start-up);
    nvidia-smi -lms 100 when NVML is unavailable."""

    # nvmlClocksEventReason bits (nvml.h)
    REASONS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, device: int):
        self.device = device
        self.samples = []  # (sm_mhz, max_mhz, reasons set)
        self.proc = None
        self.stop = threading.Event()
        self.thread = None
        self.nvml = None

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        self.nvml = pynvml
        # NVML numbers all GPUs; CUDA device d is the d-th of CUDA_VISIBLE_DEVICES when it lists indices
        index = self.device
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        ids = [v.strip() for v in vis.split(",") if v.strip()]
        if ids and all(v.isdigit() for v in ids) and self.device < len(ids):
            index = int(ids[self.device])
        return pynvml.nvmlDeviceGetHandleByIndex(index)

    def _poll_nvml(self, h):
        nv = self.nvml
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self.stop.is_set():
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            try:
                bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            except Exception:
                bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
            self.samples.append((float(sm), float(mx), {n for n, m in self.REASONS.items() if bits & m}))
            time.sleep(0.002)

    def __enter__(self):
        try:
            h = self._nvml_handle()
            self.thread = threading.Thread(target=self._poll_nvml, args=(h,), daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7 and parts[0].replace(".", "").isdigit():
                self.samples.append((float(parts[0]), float(parts[1]) if parts[1].replace(".", "").isdigit() else 0.0,
                                     {n for n, v in zip(names, parts[3:7]) if v.lower() == "active"}))

    def __exit__(self, *exc):
        self.stop.set()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=5)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        reasons = set()
        for _, _, r in self.samples:
            reasons |= r
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples), "reasons": sorted(reasons),
                "samples": len(self.samples), "source": "nvml" if self.nvml is not None else "nvidia-smi"}


def build_plan(ids, kl4):
    """build_switch_plan (src/analyzer.cpp:124-139) for 8 -> 4: sort by (kl, layer_id)."""
    order = sorted(range(len(ids)), key=lambda i: (kl4[i], ids[i]))
    return [(ids[i], i) for i in order]


class Scheduler:
    """SchedulerState::observe (src/scheduler.cpp:85-104); the C++ host library carries the
    product implementation, this mirror drives the C-ABI-level timing loop."""

    def __init__(self, W, thre, plan_len, lps):
        self.W, self.thre, self.plan_len, self.lps = W, thre, plan_len, lps
        self.win, self.cool, self.cursor = [], 0, 0

    def observe(self, v):
        self.win.append(v)
        if len(self.win) > self.W:
            self.win.pop(0)
        if self.cool > 0:
            self.cool -= 1
        if len(self.win) < self.W:
            return None, 0, 0
        avg = sum(self.win) / len(self.win)
        if self.cool > 0 or not (avg < self.thre) or self.cursor >= self.plan_len:
            return avg, 0, 0
        first, cnt = self.cursor, min(self.lps, self.plan_len - self.cursor)
        self.cursor += cnt
        self.win = []
        self.cool = self.W
        return avg, first, cnt

    def safe_observes(self):
        """How many of the next observe() calls cannot fire whatever the values: observe j (from
        1) can fire only once the window is full (len + j >= W) and the cooldown has run out
        (cool - j <= 0), or never once the plan is exhausted."""
        if self.cursor >= self.plan_len:
            return 1 << 30
        return max(self.W - len(self.win), self.cool, 1) - 1


def cpu_decode_sample(cfg, blocks: int = 1, steps: int = 2):
    """The reference's decode on ONE host core (oracle/_ref, built from its sources): a
    reference-architecture model at the 7B block dimensions with `blocks` blocks and the full
    head, a 16-token prompt, then `steps` real forward_decode + statistics + argmax tokens;
    tokens/s scaled to a full 7B-shape token by linear parameter count."""
    import ctypes as C
    R = _ref_decoder_lib()
    if R is None:
        return None
    prompt = np.random.default_rng(7).integers(0, cfg["vocab_size"], 16).astype(np.int32)
    t0 = time.perf_counter()
    h = R.ref_decoder_create(cfg["vocab_size"], cfg["d_model"], cfg["n_heads"], cfg["head_dim"], blocks, cfg["ffn_dim"],
                             16 + steps + 1, 7, prompt, 16, 0.5)
    if not h:
        return None
    build_s = time.perf_counter() - t0
    secs = []
    for _ in range(steps):
        s_, p_ = C.c_double(), C.c_double()
        R.ref_decoder_step(h, C.byref(s_), C.byref(p_))
        secs.append(s_.value)
    scale = params_per_token(cfg) / R.ref_decoder_params(h)
    R.ref_decoder_destroy(h)
    per_tok = statistics.mean(secs) * scale
    return {"value": 1.0 / per_tok, "unit": "tokens/s", "cores": 1, "kind": "reference",
            "sample": f"{steps} real decode tokens (forward_decode + ppl_entropy + fault_tolerance + argmax, 50/50 "
                      f"W8/W4) of a {blocks}-block reference model at the 7B block dimensions after a 16-token "
                      f"prompt, one core, scaled x{scale:.2f} by parameters to a 7B-shape token "
                      f"({build_s:.0f} s to build the model, not timed)"}


def params_per_token(cfg):
    d, f, V, L = cfg["d_model"], cfg["ffn_dim"], cfg["vocab_size"], cfg["n_layers"]
    return L * (4 * d * d + 3 * d * f) + V * d


def _ref_decoder_lib():
    import ctypes as C
    import oracle  # noqa: E402  (reference arm only)
    R = oracle.ref()
    if R is None:
        return None
    i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
    R.ref_decoder_create.restype = C.c_void_p
    R.ref_decoder_create.argtypes = [C.c_int64] * 7 + [C.c_uint64, i32p, C.c_int64, C.c_double]
    R.ref_decoder_step.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    R.ref_decoder_params.argtypes = [C.c_void_p]
    R.ref_decoder_params.restype = C.c_int64
    R.ref_decoder_destroy.argtypes = [C.c_void_p]
    return R


def run_reference(args, cfg, rank, world):
    """--impl reference: the reference's own decode loop (forward_decode + ppl_entropy +
    fault_tolerance + argmax_token, src/engine.cpp:89-136; library built from its sources into
    oracle/_ref) on every host core, one independent sequence per thread (rank 0 only).

    Each thread holds a reference-architecture model with the 7B block dimensions (d 4096, 32
    heads x 128, ffn 11008, vocab 32000) but REF_BLOCKS of the 32 blocks -- a full 7B reference
    model is 36 GB of fp32 master + rungs per sequence and ~50 s per token -- at the switched
    schedule's 50/50 W8/W4 mix, prefilled with a 16-token prompt.  One step = one real greedy
    decode token on every thread; tokens/s is scaled to the full 7B-shape token by linear
    parameter count (the reference's decode time is dequantize + linear per parameter:
    BASELINE.md)."""
    if rank != 0:
        return
    import ctypes as C
    R = _ref_decoder_lib()
    if R is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libfqref.so not built (reference sources absent at build time)"}))
        return
    threads = os.cpu_count() or 1
    blocks = int(os.environ.get("REF_BLOCKS", str(cfg["n_layers"] if cfg["n_layers"] <= 4 else 2)))
    n_prompt = 16
    need = n_prompt + args.warmup + args.steps + 1
    handles = [None] * threads

    def create(i):
        prompt = np.random.default_rng(1000 + i).integers(0, cfg["vocab_size"], n_prompt).astype(np.int32)
        handles[i] = R.ref_decoder_create(cfg["vocab_size"], cfg["d_model"], cfg["n_heads"], cfg["head_dim"], blocks,
                                          cfg["ffn_dim"], need, 7 + i, prompt, n_prompt, 0.5)

    t0 = time.perf_counter()
    ts = [threading.Thread(target=create, args=(i,)) for i in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    build_s = time.perf_counter() - t0
    if any(h is None for h in handles):
        print(json.dumps({"impl": "reference", "unavailable": "reference model build failed: "
                          + oracle_error()}))
        return
    p_meas = R.ref_decoder_params(handles[0])
    scale = params_per_token(cfg) / p_meas  # full 7B-shape token / measured model
    per_step = []
    for i in range(args.warmup + args.steps):
        secs = [0.0] * threads

        def step(j):
            s, pp = C.c_double(), C.c_double()
            R.ref_decoder_step(handles[j], C.byref(s), C.byref(pp))
            secs[j] = s.value

        w0 = time.perf_counter()
        ts = [threading.Thread(target=step, args=(j,)) for j in range(threads)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        wall = time.perf_counter() - w0
        if i >= args.warmup:
            per_step.append(wall)
    for h in handles:
        R.ref_decoder_destroy(h)
    step_s = statistics.mean(per_step)
    value = threads / (step_s * scale)
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 * step_s * scale / threads, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{cfg['name']} greedy decode, W8/W4 50/50 mix (the switched schedule's midpoint), "
                               f"{threads} independent sequences on {threads} host threads",
                   "impl": "reference CPU (oracle/_ref, built from /root/reference/proj/src)",
                   "measured_model": f"reference architecture, d {cfg['d_model']}, {cfg['n_heads']}x{cfg['head_dim']} "
                                     f"heads, ffn {cfg['ffn_dim']}, vocab {cfg['vocab_size']}, {blocks} blocks "
                                     f"({p_meas} linear params)",
                   "scaled_to": f"{params_per_token(cfg)} linear params per 7B-shape token (x{scale:.3f})",
                   "measured_step_s": step_s, "build_s": round(build_s, 1),
                   "same_config": "no: reference architecture (pre-LN, GELU w1/w2, learned positions) at the same "
                                  "dimensions, " + ("all blocks" if blocks == cfg["n_layers"] else
                                                    f"{blocks} of {cfg['n_layers']} blocks, scaled by parameters")},
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "reference",
                         "sample": f"per step: one real forward_decode + softmax statistics + argmax token of a "
                                   f"{blocks}-block reference model at the 7B block dimensions on each of {threads} "
                                   "threads (independent sequences), scaled by parameter count to a 7B-shape token"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def oracle_error():
    import oracle  # noqa: E402
    return oracle.ref().ref_last_error().decode()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=8)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=list(CONFIGS))
    ap.add_argument("--theta", type=float, default=1.05, help="prefill-mode threshold factor")
    ap.add_argument("--window", type=int, default=20)
    ap.add_argument("--layers-per-switch", type=int, default=16)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-chain", action="store_true",
                    help="every token through the host loop (no device-chained blocks while the scheduler cannot switch)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = CONFIGS[args.config]

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # --gpus N without a launcher: start one rank per GPU ourselves (torchrun, loopback
        # rendezvous); NCCL's communicator-init log goes to stderr so the ranks can be counted
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        env = dict(os.environ)
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd, env=env))

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU", file=sys.stderr)
        sys.exit(2)
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist  # noqa: E402
        import torch  # noqa: E402
        if args.impl == "ours":
            torch.cuda.set_device(local)
        dist.init_process_group("nccl" if args.impl == "ours" else "gloo")

    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        if dist is not None:
            dist.destroy_process_group()
        return

    import torch  # noqa: E402
    from paper_2506_12024_b200 import capi  # noqa: E402

    torch.cuda.set_device(local)
    ctx = capi.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream_handle())
    need = cfg["prompt"] + args.warmup + args.steps
    max_seq = max(512, ((need + 63) // 64) * 64)
    model = capi.Model(ctx, arch=capi.ARCH_LLAMA, act_dtype=capi.DT_BF16, max_batch=1, group_size=128,
                       max_seq_len=max_seq, norm_eps=1e-5, rope_theta=10000.0,
                       **{k: cfg[k] for k in ("vocab_size", "d_model", "n_heads", "head_dim", "n_layers", "ffn_dim")})
    t_init = time.perf_counter()
    model.init_random(seed=1234, std=0.02)
    t_init = time.perf_counter() - t_init
    # the switch plan from the logit-KL calibration (BASELINE config 4: KL(softmax(l_w4-block) ||
    # softmax(l_w8)) per block on teacher-forced random tokens, tcgen05 prefill path) on a small
    # sample: blocks ascending by KL, a block's linears by id, build_switch_plan order
    # (src/analyzer.cpp:124-139); the head, which the block calibration does not flip, ranks last
    t_cal = time.perf_counter()
    cal_rng = np.random.default_rng(4)
    cal_toks = cal_rng.integers(0, cfg["vocab_size"], (CAL_SEQS, CAL_LEN)).astype(np.int32)
    kl_blk, _ = model.calibrate_logit_kl(cal_toks, capi.RUNG_INT8, capi.RUNG_INT4)
    t_cal = time.perf_counter() - t_cal
    per_block = len(model.ids) // cfg["n_layers"]
    kl_lin = [float(kl_blk[i // per_block]) if i < cfg["n_layers"] * per_block else float("inf")
              for i in range(len(model.ids))]
    plan = build_plan(model.ids, kl_lin)
    model.set_all_rungs(0, capi.RUNG_INT8)

    from paper_2506_12024_b200 import parallel  # noqa: E402
    # weak scaling: every rank decodes its own sequence(s) (global index = rank), seeded by the
    # global sequence index so the workload per sequence does not depend on the GPU count
    rng = np.random.default_rng(parallel.prompt_seed(1000, parallel.shard(world, rank, world)[0]))
    prompt = rng.integers(0, cfg["vocab_size"], cfg["prompt"]).astype(np.int32)

    # ---- prefill (untimed) and threshold: derive_threshold (src/scheduler.cpp:51-60)
    st = model.prefill(0, prompt)
    W = args.window
    k = min(W, prompt.size)
    thre = args.theta * (sum(float(v) for v in st["ppl_entropy"][-k:]) / k)
    sched = Scheduler(W, thre, len(plan), args.layers_per_switch)
    row = st[-1]
    switches = 0
    l0 = ctx.launches()

    # algorithmic weight bytes of the step (payload + 5 B metadata per group-row of every linear
    # at its current rung, as fq_model_step_bytes counts them), kept current as switches apply so
    # the timed loop does no accounting calls; KV bytes grow by one position per step
    lin_w = []
    for i in range(len(model.ids)):
        L = model.linear(i)
        meta = L.N * L.ng * 5
        lin_w.append((L.N * L.K + meta, (L.N * L.K + 1) // 2 + meta))
    rung_now = [8] * len(model.ids)
    wbytes = [sum(w8 for w8, _ in lin_w)]

    def step(row):
        nonlocal switches
        token = int(row["argmax"])
        _, first, cnt = sched.observe(float(row["ppl_entropy"]))
        for i in range(cnt):
            idx = plan[first + i][1]
            model.set_rung(0, idx, capi.RUNG_INT4)
            if rung_now[idx] == 8:
                wbytes[0] += lin_w[idx][1] - lin_w[idx][0]
                rung_now[idx] = 4
        switches += cnt
        return model.decode_one(0, token)

    for w_i in range(args.warmup):
        # the last warm-up token goes through a device-chained step when the scheduler allows it
        # (builds and captures the chained step outside the timed region)
        if w_i == args.warmup - 1 and not args.no_chain and w_i > 0 and sched.safe_observes() >= 1:
            _, _, cnt = sched.observe(float(row["ppl_entropy"]))
            assert cnt == 0
            row = model.decode_chain(0, 1)[0]
        else:
            row = step(row)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    bytes_w_steps = []
    chained = 0
    wb_check, kb0 = model.step_bytes([0])
    assert wb_check == wbytes[0], (wb_check, wbytes[0])  # the tracked weight bytes match the engine's
    kv_per_pos = cfg["n_layers"] * 2 * cfg["d_model"] * 2
    with ClockSampler(local) as clocks:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        model.step_kernel_time(reset=True)
        launches_before = ctx.launches()
        i = 0
        while i < args.steps:
            # tokens whose scheduler decision cannot switch anything run as one device-chained
            # block (fq_model_decode_chain: the token fed back from the previous argmax on the
            # device, no host round trip); the observes are replayed afterwards and must not fire
            n = min(sched.safe_observes(), args.steps - i, 64) if not args.no_chain else 0
            if n >= 1:
                rows = model.decode_chain(0, n)
                for r in [row] + [rows[k] for k in range(n - 1)]:
                    _, _, cnt = sched.observe(float(r["ppl_entropy"]))
                    assert cnt == 0, "chained step switched"
                row = rows[n - 1]
                chained += n
            else:
                row = step(row)
                n = 1
            for k in range(n):
                bytes_w_steps.append(wbytes[0] + kb0 + (i + k) * kv_per_pos)  # the rungs each step ran at
            i += n
        e1.record(stream)
        torch.cuda.synchronize()
    launches_timed = ctx.launches() - launches_before
    prog_ms, prog_n = model.step_kernel_time(reset=True)
    ms = e0.elapsed_time(e1)
    if dist is not None:
        dist.barrier()
    ms_max = parallel.max_over_ranks(ms, device="cuda")
    sec = ms_max / 1000.0
    value = parallel.aggregate_throughput(args.steps, world, sec)
    hbm, peak_kind = peaks()
    step_bytes = statistics.mean(bytes_w_steps)
    step_frac = (step_bytes / (ms_max / args.steps / 1000.0)) / 1e9 / hbm

    # ---- kernel roofline of the dominant kernel (the GEMV), live CUDA events on the launch stream
    ms_gemv, gemv_per_step, gemv_bytes = model.profile_gemvs(0, 20)
    # DRAM bytes per launch of the step program from the committed ncu --set full capture
    traffic, traffic_note = None, None
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", "ncu_step_traffic.json")))
        if tj.get("config") == args.config:
            traffic = tj["dram_bytes_per_step"]
            traffic_note = (f"ncu --set full, one step launch: {tj['note']}; algorithmic bytes of that launch "
                            f"{tj['algorithmic_bytes_per_step']}")
    except Exception:
        pass
    # the dominant kernel is the step program itself (one launch per decode step): algorithmic
    # bytes of the timed steps / its device time from events around each launch (same stream)
    prog_launch_ms = prog_ms / max(prog_n, 1)
    prog_achieved = step_bytes / (prog_launch_ms / 1000.0) / 1e9 if prog_n else None
    gemv_achieved = gemv_bytes / gemv_per_step / (ms_gemv / 1000.0) / 1e9

    # ---- e2e through the reference-facing C++ API (flexquant::generate, libflexquant_b200.so)
    #      with host buffers: prompt H2D, the 256-token prefill on the tcgen05 path, then the
    #      decode loop with the C++ SchedulerState and the plan above; device events around it
    from paper_2506_12024_b200 import _flexquant as fq  # noqa: E402
    e2e_tokens = min(cfg["decode"], max_seq - cfg["prompt"])
    fc = fq.ModelConfig()
    fc.arch = fq.Arch.Llama
    for k in ("vocab_size", "d_model", "n_heads", "head_dim", "n_layers", "ffn_dim"):
        setattr(fc, k, cfg[k])
    fc.max_seq_len, fc.group_size, fc.max_batch = max_seq, 128, 1
    fmodel = fq.Model(fc)
    fmodel.init_random(1234, 0.02)  # the same device generator and seed: identical weights
    fplan = fq.SwitchPlan()
    ents = []
    for lid, _ in plan:
        e = fq.SwitchEntry()
        e.layer_id, e.from_, e.to, e.kl = lid, fq.Rung.Int8, fq.Rung.Int4, 0.0
        ents.append(e)
    fplan.entries = ents
    gcfg = fq.GenerationConfig()
    gcfg.max_new_tokens = e2e_tokens
    gcfg.start_rung = fq.Rung.Int8
    gcfg.scheduler.threshold_mode = fq.ThresholdMode.Prefill
    gcfg.scheduler.theta = args.theta
    gcfg.scheduler.window_len = W
    gcfg.scheduler.layers_per_switch = args.layers_per_switch
    fstream = torch.cuda.ExternalStream(fq.runtime_stream())
    prompt_host = prompt.copy()  # host buffer: copied to the device by the engine each call
    # warm-up at the timed run's sizes (full prompt: the prefill workspace, step programs and
    # graphs are built here, not inside the timed region)
    wcfg = fq.GenerationConfig()
    wcfg.max_new_tokens = 16
    wcfg.start_rung = fq.Rung.Int8
    wcfg.scheduler.threshold_mode = fq.ThresholdMode.Prefill
    wcfg.scheduler.theta = args.theta
    wcfg.scheduler.window_len = W
    wcfg.scheduler.layers_per_switch = args.layers_per_switch
    fq.generate(prompt_host.copy(), fmodel, fplan, wcfg)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    f0 = torch.cuda.Event(enable_timing=True)
    f1 = torch.cuda.Event(enable_timing=True)
    f0.record(fstream)
    res = fq.generate(prompt_host, fmodel, fplan, gcfg)
    f1.record(fstream)
    torch.cuda.synchronize()
    e2e_ms = parallel.max_over_ranks(f0.elapsed_time(f1), device="cuda")
    e2e_value = parallel.aggregate_throughput(len(res.sequence), world, e2e_ms / 1000.0)
    e2e_switches = sum(len(r.switch_events) for r in res.trace.records)
    # the trace's own per-token wall times (TraceRecord::elapsed_ns; token 1 covers the prefill)
    tok_ns = sorted(int(r.elapsed_ns) for r in res.trace.records[1:])
    e2e_detail = {"prefill_ms": round(int(res.trace.records[0].elapsed_ns) / 1e6, 3),
                  "decode_ms_median": round(tok_ns[len(tok_ns) // 2] / 1e6, 4) if tok_ns else None,
                  "decode_ms_max": round(tok_ns[-1] / 1e6, 3) if tok_ns else None,
                  "decode_ms_sum": round(sum(tok_ns) / 1e6, 2)}
    row_bytes = capi.ROW_STATS_DTYPE.itemsize
    h2d = (cfg["prompt"] * 4 + (e2e_tokens - 1) * 4) / e2e_tokens
    d2h = (cfg["prompt"] + e2e_tokens - 1) * row_bytes / e2e_tokens
    del fmodel

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_decode_sample(cfg)
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "unit": "tokens/s", "cores": 1, "kind": "reference", "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value,
            "unit": "tokens/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic",
            "config": {
                "workload": f"{cfg['name']} (BASELINE config {3 if args.config == 'c3' else 1}): B=1 per GPU, {cfg['prompt']}-token random prompt, "
                            f"decode positions {cfg['prompt']}..{cfg['prompt'] + args.warmup + args.steps}, "
                            f"W8 start, 8->4 plan ordered by the logit-KL calibration (BASELINE config 4 on "
                            f"{CAL_SEQS}x{CAL_LEN} tokens, {t_cal:.1f} s)",
                "model": cfg["name"], "global_batch": world, "seq_len": cfg["prompt"] + args.warmup + args.steps,
                "parallelism": f"dp{world}", "group_size": 128, "kv_cache": "fp16",
                "scheduler": {"mode": "prefill", "theta": args.theta, "threshold": thre, "window": W,
                              "layers_per_switch": args.layers_per_switch, "switches_applied": switches,
                              "device_chained_steps": chained},
                "l2": "no flush needed: >6.5 GB of weights streamed per step (126 MB L2)",
                "weights_init_s": round(t_init, 2),
            },
            "step_hbm_fraction": round(step_frac, 4),
            "step_algorithmic_bytes": int(step_bytes),
            "roofline": {
                "bound": "hbm", "achieved": prog_achieved, "peak": hbm, "unit": "GB/s",
                "frac": (prog_achieved / hbm) if prog_achieved else None, "traffic": traffic,
                "kernel": "program_kernel: the whole decode step (embedding, 225 tiled W8/W4 g128 dequant-GEMVs "
                          "on mma.sync, attention, fused softmax entropy), one launch per step",
                "peak_kind": peak_kind,
                "per_launch_bytes": step_bytes, "per_launch_ms": prog_launch_ms, "launches_timed": prog_n,
                "traffic_note": traffic_note,
                "gemv_only": {"achieved": gemv_achieved, "frac": gemv_achieved / hbm,
                              "per_launch_bytes": gemv_bytes / gemv_per_step, "per_launch_ms": ms_gemv,
                              "note": "the same program with its GEMV phases only (profile_gemvs replay)"},
            },
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "trace": e2e_detail,
                    "note": f"flexquant::generate (C++ API, libflexquant_b200.so) of the full config with host "
                            f"buffers: {cfg['prompt']}-token prefill on the tcgen05 path + {e2e_tokens} decode tokens "
                            f"with the C++ SchedulerState, {e2e_switches} switch events"},
            "gpu_launches": launches_timed,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    model.close()
    ctx.close()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
