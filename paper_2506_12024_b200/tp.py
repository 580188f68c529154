"""Tensor-parallel decode (the variant north_star names; SURVEY §8e "TP variant").

The reference has no distribution: one block (src/model.cpp:201-233) runs on one core.  Here a
Llama model of the full config is split over `size` ranks, one GPU each:

* column split: q/k/v of the rank's heads, gate/up of its ffn columns (whole quantization groups);
* row split: o/down over the matching input columns -> an fp32 [B, d] partial per rank, summed by
  one all-reduce after each (2 per block), the sum added to the replicated residual stream;
* vocab split: the head rows of the rank's vocab slice; the fused softmax statistics leave each
  rank as one mergeable partial per row (max, sum e, sum e*l, top-2, argmax), all-gathered and
  merged on the host (fq_tp_merge_stats) into ppl_entropy / fault_tolerance / argmax_token
  (src/scheduler.cpp:13-49, src/engine.cpp:144-155).

Each segment between two exchanges is one launch of the step program (model.cu tp_program).  The
collectives are torch.distributed's (NCCL over NVLink on the GPUs, in place on the rank's partial
buffer, on the stream the engine runs on).  `LocalExchange` runs all ranks in one process on one
device -- the segments of the ranks one after another and the sum on the device -- which checks the
sharded arithmetic against the unsplit oracle; it is not a stand-in for multi-GPU timing.
"""
from __future__ import annotations

from typing import Dict, List, Sequence, Tuple

import numpy as np

from . import capi

LINEARS = ("attn.wq", "attn.wk", "attn.wv", "attn.wo", "ffn.w_gate", "ffn.w_up", "ffn.w_down")


def linear_ranges(lid: str, cfg: capi.ModelConfig, sh: capi.TpShard) -> Tuple[Tuple[int, int], Tuple[int, int]]:
    """(rows, cols) of the full [N, K] weight `lid` that rank `sh` holds."""
    d, hd = cfg.d_model, cfg.head_dim
    name = lid.split(".", 2)[-1] if lid.startswith("blocks.") else lid
    q0, q1 = sh.head0 * hd, (sh.head0 + sh.heads) * hd
    f0, f1 = sh.ffn0, sh.ffn0 + sh.ffn
    if name in ("attn.wq", "attn.wk", "attn.wv"):
        return (q0, q1), (0, d)
    if name == "attn.wo":
        return (0, d), (q0, q1)
    if name in ("ffn.w_gate", "ffn.w_up"):
        return (f0, f1), (0, d)
    if name == "ffn.w_down":
        return (0, d), (f0, f1)
    if name == "head":
        return (sh.vocab0, sh.vocab0 + sh.vocab), (0, d)
    raise ValueError(f"tensor parallel: unknown linear {lid}")


def full_shape(lid: str, cfg: capi.ModelConfig) -> Tuple[int, int]:
    d, f, V = cfg.d_model, cfg.ffn_dim, cfg.vocab_size
    name = lid.split(".", 2)[-1] if lid.startswith("blocks.") else lid
    return {"attn.wq": (d, d), "attn.wk": (d, d), "attn.wv": (d, d), "attn.wo": (d, d), "ffn.w_gate": (f, d),
            "ffn.w_up": (f, d), "ffn.w_down": (d, f), "head": (V, d)}[name]


def upload_shard(model: capi.Model, quantized: Dict[str, Dict[int, tuple]], params: Dict[str, np.ndarray]) -> None:
    """Uploads rank `model`'s slices of the full model: quantized[lid][bits] = (payload, scale, zp)
    of the full [N, K] weight; params: non-switchable parameters (tok_emb, norms), replicated."""
    for idx, lid in enumerate(model.ids):
        upload_shard_one(model, idx, lid, quantized[lid])
    for name, arr in params.items():
        model.set_param(name, arr)


def upload_shard_one(model: capi.Model, idx: int, lid: str, q: Dict[int, tuple]) -> None:
    """Rank `model`'s slice of one linear: q[bits] = (payload, scale, zp) of the full weight."""
    cfg, sh = model.cfg, model.tp_shard()
    N, K = full_shape(lid, cfg)
    rows, cols = linear_ranges(lid, cfg, sh)
    L = model.linear(idx)
    for bits, rung in ((8, capi.RUNG_INT8), (4, capi.RUNG_INT4)):
        if bits in q:
            p, s, z = q[bits]
            sp, ss, sz = capi.shard_quantized(bits, N, K, cfg.group_size, p, s, z, rows, cols)
            L.upload_quantized(rung, sp, ss, sz)


class LocalExchange:
    """All ranks in this process on one device: sum in rank order, copied back to every rank."""

    def __init__(self, size: int):
        self.size = size

    def allreduce(self, bufs: Sequence) -> None:
        total = bufs[0].clone()
        for b in bufs[1:]:
            total += b
        for b in bufs:
            b.copy_(total)

    def allgather(self, parts: Sequence) -> List:
        return list(parts)


class DistExchange:
    """One rank per process: torch.distributed collectives (NCCL over NVLink on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.size = dist.get_world_size(group)

    def allreduce(self, bufs: Sequence) -> None:
        (b,) = bufs
        self.dist.all_reduce(b, group=self.group)

    def allgather(self, parts: Sequence) -> List:
        import torch
        (p,) = parts
        out = [torch.empty_like(p) for _ in range(self.size)]
        self.dist.all_gather(out, p, group=self.group)
        return out


class TpDecoder:
    """Decode steps of the local TP rank models (all ranks with LocalExchange, one with
    DistExchange).  step() returns the merged row statistics of the full vocabulary."""

    def __init__(self, models: Sequence[capi.Model], exchange, max_batch: int = 1, graphs: bool = True):
        import torch
        self.torch = torch
        self.models = list(models)
        self.ex = exchange
        cfg = self.models[0].cfg
        sh = self.models[0].tp_shard()
        self.size = sh.size
        self.nseg = sh.n_segments
        self.vocab0 = [capi.tp_shard_spec(cfg, r, sh.size).vocab0 for r in range(sh.size)]
        self.vocab = [capi.tp_shard_spec(cfg, r, sh.size).vocab for r in range(sh.size)]
        dev = torch.device("cuda", torch.cuda.current_device())
        # one exchange buffer per local rank: a segment reads the reduced sum in its first phase
        # and writes its new partial in its last, so the in-place all-reduce needs no second buffer
        self.part = [torch.zeros(max_batch, cfg.d_model, dtype=torch.float32, device=dev) for _ in self.models]
        self.stat = [torch.zeros(max_batch * 32, dtype=torch.uint8, device=dev) for _ in self.models]
        # the exchange (torch / NCCL) is ordered on the engine's own stream; the local ranks share
        # one context (one stream)
        handles = {m.ctx.stream_handle() for m in self.models}
        if len(handles) != 1:
            raise capi.ConfigError("tp decode: the local rank models must share one context")
        self.stream = torch.cuda.ExternalStream(handles.pop())
        self.max_batch = max_batch
        # the 2L+1 segments and the exchanges between them, captured per batch size after one
        # eager step (which builds the segment programs) and replayed: no host round trip per
        # segment.  Rebuild the decoder after re-uploading weights (the programs bake pointers in).
        self.use_graphs = graphs
        self.graphs = {}
        self.eager_steps = {}

    def begin(self, slots, tokens) -> None:
        for m in self.models:
            m.tp_begin(slots, tokens)

    def segments(self) -> None:
        for seg in range(self.nseg):
            last = seg == self.nseg - 1
            for m, p, st in zip(self.models, self.part, self.stat):
                m.tp_segment(seg, None if seg == 0 else p, st if last else p)
            if not last:
                self.ex.allreduce(self.part)

    def finish(self, B: int) -> np.ndarray:
        gathered = self.ex.allgather([s[: B * 32] for s in self.stat])
        parts = np.stack([g.cpu().numpy().view(capi.STAT_PART_DTYPE) for g in gathered])
        return capi.tp_merge_stats(parts, self.vocab0)

    def step(self, slots, tokens) -> np.ndarray:
        torch = self.torch
        B = len(slots)
        if B > self.max_batch:
            raise capi.InputError("tp decode: batch larger than the exchange buffers")
        self.begin(slots, tokens)
        with torch.cuda.stream(self.stream):
            g = self.graphs.get(B)
            if g is None and self.use_graphs and self.eager_steps.get(B, 0) >= 1:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=self.stream):
                    self.segments()
                self.graphs[B] = g
            if g is not None:
                g.replay()
            else:
                self.segments()
                self.eager_steps[B] = self.eager_steps.get(B, 0) + 1
            for m in self.models:
                m.tp_end()
            return self.finish(B)

    def logits(self, B: int) -> np.ndarray:
        """Full-vocabulary logits [B, V] of the last step, gathered from the local ranks (LocalExchange)."""
        self.stream.synchronize()
        cols = [_device_view(m.logits_ptr(), B * v).view(B, v).cpu().numpy() for m, v in zip(self.models, self.vocab)]
        return np.concatenate(cols, axis=1)


def _device_view(ptr: int, n: int):
    """A torch float32 tensor over n floats of foreign device memory (the caller only reads it)."""
    import torch

    class _Holder:
        def __init__(self, p, n):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (p, False), "version": 2,
                                             "strides": None}

    return torch.as_tensor(_Holder(ptr, n), device="cuda")
