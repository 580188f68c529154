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


LINEARS = ("attn.wq", "attn.wk", "attn.wv", "attn.wo", "ffn.w_gate", "ffn.w_up", "ffn.w_down")


class LlamaOracle:
    """Weights generated on the host (N(0,std) from oracle.normal), quantized with the oracle
    quantizer, dequantized to fp32 for the reference-style linear."""

    def __init__(self, cfg: dict, seed: int = 0, std: float = 0.02):
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
            self.layers.append((lid, w, q))
        self.ids = [l[0] for l in self.layers]
        self._deq = {}

    def weight(self, idx: int, bits: int) -> np.ndarray:
        key = (idx, bits)
        if key not in self._deq:
            lid, w, q = self.layers[idx]
            p, s, z = q[bits]
            self._deq[key] = dequantize(p, w.shape[0], w.shape[1], self.group, bits, s, z).astype(np.float64)
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
        c = self.cfg
        d, H, hd = c["d_model"], c["n_heads"], c["head_dim"]
        pos = len(cache["k"][0])
        x = self.tok_emb[token].astype(np.float32).copy()
        for l in range(c["n_layers"]):
            b = l * 7
            h = self._norm(x)
            q = bf16(self._lin(b + 0, rungs[b + 0], h))
            k = bf16(self._lin(b + 1, rungs[b + 1], h))
            v = bf16(self._lin(b + 2, rungs[b + 2], h))
            qr = self._rope(q, pos) * np.float32(1.0 / np.sqrt(np.float32(hd)))
            kr = fp16(self._rope(k, pos))
            cache["k"][l].append(kr)
            cache["v"][l].append(fp16(v))
            K = np.stack(cache["k"][l]).reshape(pos + 1, H, hd)
            Vv = np.stack(cache["v"][l]).reshape(pos + 1, H, hd)
            qh = qr.reshape(H, hd).astype(np.float64)
            s = np.einsum("hd,jhd->hj", qh, K.astype(np.float64))
            p = np.exp(s - s.max(axis=1, keepdims=True))
            o = np.einsum("hj,jhd->hd", p, Vv.astype(np.float64)) / p.sum(axis=1, keepdims=True)
            o = bf16(o.reshape(-1).astype(np.float32))
            x = (x + self._lin(b + 3, rungs[b + 3], o)).astype(np.float32)
            h2 = self._norm(x)
            g = self._lin(b + 4, rungs[b + 4], h2)
            u = self._lin(b + 5, rungs[b + 5], h2)
            mid = bf16((g / (1.0 + np.exp(-g.astype(np.float64)))).astype(np.float32) * u)
            x = (x + self._lin(b + 6, rungs[b + 6], mid)).astype(np.float32)
        hf = self._norm(x)
        return self._lin(len(self.layers) - 1, rungs[-1], hf)
