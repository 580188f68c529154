"""Multi-process (world_size 2, gloo, CPU) tests of the data-parallel plumbing: sequence sharding,
max-over-ranks timing, aggregate throughput and the trace gather."""
import os
import socket

import pytest

from paper_2506_12024_b200 import parallel


def test_shard_partitions_and_balances():
    for n in (0, 1, 7, 8, 256):
        for world in (1, 2, 3, 8):
            shards = [parallel.shard(n, r, world) for r in range(world)]
            flat = [i for s in shards for i in s]
            assert flat == list(range(n))
            sizes = [len(s) for s in shards]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        parallel.shard(4, 2, 2)


def test_prompt_seed_independent_of_world():
    assert parallel.prompt_seed(7, 3) == parallel.prompt_seed(7, 3)
    assert parallel.prompt_seed(7, 3) != parallel.prompt_seed(7, 4)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n_seqs, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = parallel.shard(n_seqs, rank, world)
        # a stand-in per-sequence result: (sequence, seed) from this rank's shard
        results = [(i, parallel.prompt_seed(5, i)) for i in mine]
        t = parallel.max_over_ranks(1.0 + rank)  # rank r "took" 1 + r seconds
        gathered = parallel.gather_objects(results)
        merged = parallel.merge_shards(gathered, n_seqs)
        thr = parallel.aggregate_throughput(len(mine), world, t)
        q.put((rank, t, merged, thr))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sharding_timing_and_gather():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    n = 9
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, t, merged, thr in outs:
        assert t == 2.0  # max over ranks
        assert merged == [(i, parallel.prompt_seed(5, i)) for i in range(n)]
        assert thr == pytest.approx(2 * len(parallel.shard(n, rank, 2)) / 2.0)


def test_bench_gpus_flag_launches_the_ranks():
    """bench.py --gpus N without a launcher starts N ranks itself (torchrun, loopback rendezvous)
    and rank 0 prints one JSON line with n_gpus = N (here the reference arm over gloo: no GPU)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["REF_BLOCKS"] = "1"
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--impl", "reference",
                        "--config", "c1", "--steps", "1", "--warmup", "3"], capture_output=True, text=True,
                       timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["impl"] == "reference" and line["value"] > 0


def _calib_worker(rank, world, port, q):
    import numpy as np
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # per-token KL / entropy of 5 sequences x 4 tokens for 3 blocks, sharded by sequence
        rng = np.random.default_rng(11)
        kl_tok = rng.random((5, 4, 3))
        ent_tok = rng.random((5, 4, 3)) + 5.0
        mine = parallel.shard(5, rank, world)
        kl_loc = kl_tok[mine.start:mine.stop].reshape(-1, 3).mean(axis=0)
        ent_loc = ent_tok[mine.start:mine.stop].reshape(-1, 3).mean(axis=0)
        kl, ent, rows = parallel.allreduce_block_kl(kl_loc, ent_loc, len(mine) * 4)
        q.put((rank, kl.tolist(), ent.tolist(), rows,
               kl_tok.reshape(-1, 3).mean(axis=0).tolist(), ent_tok.reshape(-1, 3).mean(axis=0).tolist()))
    finally:
        dist.destroy_process_group()


def test_two_rank_c4_calibration_merge():
    """C4 sharded by sequence: one all-reduce of the per-block partial sums reproduces the
    per-block means over every token (tools/calibrate_c4.py under torchrun)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_calib_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, kl, ent, rows, kl_want, ent_want in outs:
        assert rows == 20
        assert kl == pytest.approx(kl_want, rel=1e-12, abs=1e-15)
        assert ent == pytest.approx(ent_want, rel=1e-12)
