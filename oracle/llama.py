"""numpy restatement of the Llama-shaped decoder the engine runs for the BASELINE configs.

TEST INFRASTRUCTURE ONLY.  Parity unpinned by the reference (it has no RMSNorm / SwiGLU / RoPE,
SURVEY §8c): this follows the reference's numeric conventions (double-accumulated linear of
fp32 dequantized weights, src/tensor.cpp:83-101; dequantize src/quantizer.cpp:205-219;
softmax_double statistics src/scheduler.cpp:13-49) and the engine's documented precision
contract: fp32 residual stream; RMSNorm output, q/k/v, attention output and the
SwiGLU product rounded to bf16; RoPE (rotate-half, theta 10000) in fp32; fp16 K/V cache;
fp32 logits.
"""
from __future__ import annotations

import numpy as np

from . import dequantize, normal, quantize


def bf16(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as float32."""
    x = np.ascontiguousarray(x, np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


def fp16(x: np.ndarray) -> np.ndarray:
    return np.asarray(x, np.float32).astype(np.float16).astype(np.float32)


class _Shape:
    def __init__(self, n, k):
        self.shape = (n, k)


LINEARS = ("attn.wq", "attn.wk", "attn.wv", "attn.wo", "ffn.w_gate", "ffn.w_up", "ffn.w_down")


class LlamaOracle:
    """Weights generated on the host (N(0,std) from oracle.normal), quantized with the oracle
    quantizer, dequantized to fp32 for the reference-style linear."""

    def __init__(self, cfg: dict, seed: int = 0, std: float = 0.02, lean: bool = False, act: str = "bf16",
                 acc: str = "f64"):
        """lean: keep only the quantized copies and fp32 dequantized weights (no fp master, no
        float64 cache) -- the 7B-dimension parity test holds ~0.5e9 parameters.
        act: the activation dtype of the engine contract ("bf16", or "fp16" = Model act_dtype F16).
        acc: "f64" = the reference's double-accumulated linear (src/tensor.cpp:95-96); "f32" = the
        same contract with fp32 accumulation -- not a reference behaviour but the conditioning probe:
        how far the result moves under fp32-level perturbations (the envelope of any fp32 engine)."""
        self.cfg = cfg
        d, f, V, L = cfg["d_model"], cfg["ffn_dim"], cfg["vocab_size"], cfg["n_layers"]
        self.group = cfg.get("group_size", 128)
        self.eps = cfg.get("norm_eps", 1e-5)
        self.theta = cfg.get("rope_theta", 10000.0)
        self.tok_emb = normal(V * d, seed, 0, std).reshape(V, d)
        self.layers = []  # (id, fp weight, {bits: (payload, scale, zp)})
        shapes = []
        for i in range(L):
            for nm in LINEARS:
                n, k = {"ffn.w_gate": (f, d), "ffn.w_up": (f, d), "ffn.w_down": (d, f)}.get(nm, (d, d))
                shapes.append((f"blocks.{i}.{nm}", n, k))
        shapes.append(("head", V, d))
        for idx, (lid, n, k) in enumerate(shapes):
            w = normal(n * k, seed, 100 + idx, std).reshape(n, k)
            q = {bits: quantize(w, self.group, bits) for bits in (8, 4)}
            self.layers.append((lid, w if not lean else _Shape(n, k), q))
        self.ids = [l[0] for l in self.layers]
        self._deq = {}
        self.lean = lean
        self.act = act
        self.acc = acc
        self._round = bf16 if act == "bf16" else fp16

    def variant(self, act: str | None = None, acc: str | None = None) -> "LlamaOracle":
        """The same weights under another activation dtype / accumulation (shares the caches)."""
        import copy
        o = copy.copy(self)
        if act is not None:
            o.act = act
            o._round = bf16 if act == "bf16" else fp16
        if acc is not None:
            o.acc = acc
        return o

    def weight(self, idx: int, bits: int) -> np.ndarray:
        key = (idx, bits)
        if key not in self._deq:
            lid, w, q = self.layers[idx]
            p, s, z = q[bits]
            wd = dequantize(p, w.shape[0], w.shape[1], self.group, bits, s, z)
            self._deq[key] = wd if self.lean else wd.astype(np.float64)
        return self._deq[key]

    def upload(self, model, capi) -> None:
        model.set_param("tok_emb", self.tok_emb)
        for idx, (lid, w, q) in enumerate(self.layers):
            assert model.ids[idx] == lid
            L = model.linear(idx)
            for bits, rung in ((8, capi.RUNG_INT8), (4, capi.RUNG_INT4)):
                p, s, z = q[bits]
                L.upload_quantized(rung, p, s, z)

    # ---------------------------------------------------------------- forward
    def _norm(self, x):
        ms = np.mean(x.astype(np.float64) ** 2)
        rstd = 1.0 / np.sqrt(ms + self.eps)
        return bf16((x.astype(np.float64) * rstd).astype(np.float32))  # gains are 1

    def _lin(self, idx, bits, h):
        return (self.weight(idx, bits) @ h.astype(np.float64)).astype(np.float32)

    def _rope(self, x, pos):
        hd = self.cfg["head_dim"]
        x = x.reshape(-1, hd).astype(np.float32).copy()
        i = np.arange(hd // 2)
        ang = pos * np.power(float(self.theta), -2.0 * i / hd)
        c = np.cos(ang).astype(np.float32)
        s = np.sin(ang).astype(np.float32)
        a, b = x[:, : hd // 2].copy(), x[:, hd // 2:].copy()
        x[:, : hd // 2] = a * c - b * s
        x[:, hd // 2:] = b * c + a * s
        return x.reshape(-1)

    def new_cache(self):
        return {"k": [[] for _ in range(self.cfg["n_layers"])], "v": [[] for _ in range(self.cfg["n_layers"])]}

    def step(self, token: int, cache: dict, rungs: list[int]) -> np.ndarray:
        """One decode step; rungs[i] in {8, 4} per linear; returns fp32 logits."""
        return self.forward([token], cache, rungs)[0]

    def forward(self, tokens, cache: dict, rungs: list[int]) -> np.ndarray:
        """n consecutive positions at once (prefill semantics: row i attends to every cached
        position and rows 0..i of this call, causal as src/model.cpp:100-140); each row is
        computed exactly as step() would compute it.  Returns fp32 logits [n, V]."""
        c = self.cfg
        d, H, hd = c["d_model"], c["n_heads"], c["head_dim"]
        toks = [int(t) for t in tokens]
        n = len(toks)
        pos0 = len(cache["k"][0])
        x = self.tok_emb[toks].astype(np.float32).copy()  # [n, d]
        for l in range(c["n_layers"]):
            b = l * 7
            h = self._norm_rows(x)
            q = self._round(self._lin_rows(b + 0, rungs[b + 0], h))
            k = self._round(self._lin_rows(b + 1, rungs[b + 1], h))
            v = self._round(self._lin_rows(b + 2, rungs[b + 2], h))
            for i in range(n):
                qr = self._rope(q[i], pos0 + i) * np.float32(1.0 / np.sqrt(np.float32(hd)))
                q[i] = qr
                cache["k"][l].append(fp16(self._rope(k[i], pos0 + i)))
                cache["v"][l].append(fp16(v[i]))
            K = np.stack(cache["k"][l]).reshape(pos0 + n, H, hd).astype(np.float64)
            Vv = np.stack(cache["v"][l]).reshape(pos0 + n, H, hd).astype(np.float64)
            qh = q.reshape(n, H, hd).astype(np.float64)
            s = np.einsum("nhd,jhd->nhj", qh, K)
            vis = np.arange(pos0 + n)[None, :] <= (pos0 + np.arange(n))[:, None]  # [n, ctx]
            s = np.where(vis[:, None, :], s, -np.inf)
            p = np.exp(s - s.max(axis=2, keepdims=True))
            o = np.einsum("nhj,jhd->nhd", p, Vv) / p.sum(axis=2, keepdims=True)
            o = self._round(o.reshape(n, d).astype(np.float32))
            x = (x + self._lin_rows(b + 3, rungs[b + 3], o)).astype(np.float32)
            h2 = self._norm_rows(x)
            g = self._lin_rows(b + 4, rungs[b + 4], h2)
            u = self._lin_rows(b + 5, rungs[b + 5], h2)
            mid = self._round((g / (1.0 + np.exp(-g.astype(np.float64)))).astype(np.float32) * u)
            x = (x + self._lin_rows(b + 6, rungs[b + 6], mid)).astype(np.float32)
        hf = self._norm_rows(x)
        return self._lin_rows(len(self.layers) - 1, rungs[-1], hf)

    def _norm_rows(self, x):
        ms = np.mean(x.astype(np.float64) ** 2, axis=1, keepdims=True)
        rstd = 1.0 / np.sqrt(ms + self.eps)
        return self._round((x.astype(np.float64) * rstd).astype(np.float32))  # gains are 1

    def _lin_rows(self, idx, bits, h):
        """Reference linear (double accumulation, src/tensor.cpp:83-101) of every row of h."""
        if self.acc == "f32":
            return (h.astype(np.float32) @ self.weight(idx, bits).astype(np.float32).T).astype(np.float32)
        return (h.astype(np.float64) @ self.weight(idx, bits).T).astype(np.float32)
