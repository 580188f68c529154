"""BASELINE config 4 at full scale: KL layer-sensitivity calibration on the 7B shape.

64 random-token sequences x 512 tokens; for each of the 32 blocks that block's linears are set to
W4 with all others W8, and the mean KL(softmax(logits_q) || softmax(logits_w8)) over the 32000
vocabulary plus the mean entropy are measured (fq_model_calibrate_logit_kl: the prefill runs on
the tcgen05 dequant-GEMM, KL / entropy on the device).  Prints one JSON line: wall time, the
implied tensor throughput (2 * params * tokens * 33 forwards), and the block ranking that
build_switch_plan orders (ascending KL, ties by index).

Multi-GPU: under torchrun each rank calibrates its shard of the sequences
(parallel.shard) and one NCCL all-reduce of the per-block partial sums merges them
(parallel.allreduce_block_kl); the time is the max over ranks.

  python tools/calibrate_c4.py --seqs 64 --len 512
  torchrun --nproc-per-node 8 --master-addr 127.0.0.1 tools/calibrate_c4.py
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_12024_b200 import capi, parallel  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seqs", type=int, default=64)
    ap.add_argument("--len", type=int, default=512)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--full", action="store_true", help="every flipped forward from the embedding (FQ_CALIB_FULL)")
    ap.add_argument("--dump", default="", help="write the per-block KL / entropy arrays (.npy pair prefix)")
    a = ap.parse_args()
    if a.full:
        os.environ["FQ_CALIB_FULL"] = "1"
    ri = parallel.RankInfo.from_env()
    if ri.world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(ri.local_rank)
        dist.init_process_group("nccl")
    ctx = capi.Context(ri.local_rank)
    m = capi.Model(ctx, arch=capi.ARCH_LLAMA, act_dtype=capi.DT_BF16, max_batch=1, group_size=128,
                   max_seq_len=a.len + 8, vocab_size=32000, d_model=4096, n_heads=32, head_dim=128,
                   n_layers=a.layers, ffn_dim=11008)
    m.init_random(1234, 0.02)
    toks = np.random.default_rng(4).integers(0, 32000, (a.seqs, a.len)).astype(np.int32)
    mine = parallel.shard(a.seqs, ri.rank, ri.world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    kl, ent = m.calibrate_logit_kl(toks[mine.start:mine.stop], capi.RUNG_INT8, capi.RUNG_INT4)
    torch.cuda.synchronize()
    dt = parallel.max_over_ranks(time.perf_counter() - t0, device="cuda")
    kl, ent, _ = parallel.allreduce_block_kl(kl, ent, len(mine) * a.len, device="cuda")
    if ri.world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    if ri.rank != 0:
        return
    if a.dump:
        np.save(a.dump + "_kl.npy", np.asarray(kl))
        np.save(a.dump + "_ent.npy", np.asarray(ent))
    lp, hp = 4 * 4096 * 4096 + 3 * 4096 * 11008, 32000 * 4096
    full_flops = 2.0 * (a.layers * lp + hp) * a.seqs * a.len * (a.layers + 1)  # 33 full forwards
    # executed: the base forward, then forward fl runs blocks fl.. only (the blocks below are the
    # base forward's, reused from its residual-stream snapshots) unless --full
    run_layers = a.layers + sum(a.layers if a.full else a.layers - fl for fl in range(a.layers))
    exec_flops = 2.0 * (run_layers * lp + (a.layers + 1) * hp) * a.seqs * a.len
    order = sorted(range(a.layers), key=lambda i: (kl[i], i))
    print(json.dumps({"config": "C4", "seqs": a.seqs, "len": a.len, "n_gpus": ri.world, "blocks": a.layers,
                      "forwards": a.layers + 1,
                      "block_reuse": not a.full, "seconds": round(dt, 2),
                      "tflops_executed": round(exec_flops / dt / 1e12, 1),
                      "full_forward_equivalent_tflops": round(full_flops / dt / 1e12, 1),
                      "kl_min": float(np.min(kl)), "kl_max": float(np.max(kl)),
                      "entropy_mean": float(np.mean(ent)), "switch_order_blocks": order}), flush=True)


if __name__ == "__main__":
    main()
