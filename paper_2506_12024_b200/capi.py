"""ctypes binding of the C-ABI boundary (include/fq_cuda.h).

This is how Python (tests, bench) reaches the CUDA engine; it exercises exactly the entry
points a reference maintainer would bind.  There is no CPU fallback: if the
extension is missing or no B200 is visible, ``load()`` / ``Context()`` raise.

Status codes are mapped onto the reference's exception hierarchy
(/root/reference/proj/include/flexquant/error.hpp:10-49).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FQ_CUDA_LIB", os.path.join(_HERE, "lib", "libfq_cuda.so"))

RUNG_FP, RUNG_INT8, RUNG_INT4 = 0, 1, 2
MODE_ASYM, MODE_SYM = 0, 1
DT_F32, DT_F16, DT_BF16 = 0, 1, 2
ARCH_REFERENCE, ARCH_LLAMA = 0, 1
NUMERICS_FAST, NUMERICS_EXACT = 0, 1

ABI_FUNCTIONS = [
    "fq_last_error", "fq_abi_version", "fq_ctx_create", "fq_ctx_destroy", "fq_ctx_set_stream", "fq_ctx_get_stream",
    "fq_ctx_synchronize", "fq_ctx_launch_count", "fq_layer_create", "fq_layer_destroy", "fq_layer_upload_quantized",
    "fq_layer_download_quantized", "fq_layer_upload_fp", "fq_layer_upload_bias", "fq_layer_quantize_device",
    "fq_layer_has", "fq_layer_shape", "fq_layer_bytes", "fq_gemv", "fq_softmax_stats", "fq_kl_rows", "fq_hist_kl",
    "fq_fill_normal", "fq_model_create", "fq_model_destroy", "fq_model_num_linears", "fq_model_linear_id",
    "fq_model_linear_index", "fq_model_linear", "fq_model_set_param", "fq_model_init_random", "fq_model_set_rung",
    "fq_model_get_rung", "fq_model_set_all_rungs", "fq_model_reset_slot", "fq_model_slot_length", "fq_model_prefill",
    "fq_model_decode", "fq_model_logits", "fq_model_step_bytes", "fq_model_calibrate_logit_kl",
    "fq_model_init_random_kl", "fq_model_profile_gemvs", "fq_model_profile_step", "fq_gemm",
    "fq_model_step_kernel_time", "fq_gemv_chain_time", "fq_tiled_activation_bytes", "fq_tile_activations",
    "fq_gemm_tiled", "fq_model_decode_timed", "fq_layer_download_fp", "fq_layer_download_bias", "fq_model_get_param", "fq_model_param_size",
    "fq_tp_shard_spec", "fq_shard_quantized", "fq_tp_merge_stats", "fq_model_create_tp", "fq_model_tp_shard",
    "fq_model_tp_begin", "fq_model_tp_segment", "fq_model_tp_end", "fq_model_get_rungs", "fq_model_decode_chain",
]


class Error(RuntimeError):
    """flexquant::Error"""


class DimensionError(Error):
    pass


class ConfigError(Error):
    pass


class InputError(Error):
    pass


class StateError(Error):
    pass


class FormatError(Error):
    pass


class CapacityError(Error):
    pass


class CudaError(Error):
    pass


_ERRORS = {1: DimensionError, 2: ConfigError, 3: InputError, 4: StateError, 5: FormatError, 6: CapacityError,
           7: CudaError}


class RowStats(C.Structure):
    _fields_ = [("ppl_entropy", C.c_double), ("entropy", C.c_double), ("p1", C.c_double), ("p2", C.c_double),
                ("fault_tolerance", C.c_double), ("max_logit", C.c_float), ("argmax", C.c_int32)]


ROW_STATS_DTYPE = np.dtype([("ppl_entropy", np.float64), ("entropy", np.float64), ("p1", np.float64),
                            ("p2", np.float64), ("fault_tolerance", np.float64), ("max_logit", np.float32),
                            ("argmax", np.int32)])
assert ROW_STATS_DTYPE.itemsize == C.sizeof(RowStats)


class TpShard(C.Structure):
    _fields_ = [("rank", C.c_int32), ("size", C.c_int32), ("head0", C.c_int64), ("heads", C.c_int64),
                ("ffn0", C.c_int64), ("ffn", C.c_int64), ("vocab0", C.c_int64), ("vocab", C.c_int64),
                ("n_segments", C.c_int32)]


STAT_PART_DTYPE = np.dtype([("S", np.float64), ("T", np.float64), ("m", np.float32), ("v1", np.float32),
                            ("v2", np.float32), ("arg", np.int32)])
assert STAT_PART_DTYPE.itemsize == 32


class ModelConfig(C.Structure):
    _fields_ = [("arch", C.c_int32), ("act_dtype", C.c_int32), ("vocab_size", C.c_int64), ("d_model", C.c_int64),
                ("n_heads", C.c_int64), ("head_dim", C.c_int64), ("n_layers", C.c_int64), ("ffn_dim", C.c_int64),
                ("max_seq_len", C.c_int64), ("tie_embeddings", C.c_int32), ("max_batch", C.c_int32),
                ("group_size", C.c_int64), ("norm_eps", C.c_float), ("rope_theta", C.c_float)]


_lib = None


def load(path: str = LIB_PATH):
    """Loads libfq_cuda.so; raises if it is missing (no fallback path exists).  FQ_CUDA_LIB
    selects another build of the same library (A/B profiling)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("FQ_CUDA_LIB", path)
    if not os.path.exists(path):
        raise ImportError(f"CUDA extension {path} is not built; run `make` or __graft_entry__.build()")
    L = C.CDLL(path)
    v = C.c_void_p
    i32, i64, u64 = C.c_int32, C.c_int64, C.c_uint64
    L.fq_last_error.restype = C.c_char_p
    L.fq_abi_version.restype = i32
    sig = {
        "fq_ctx_create": [i32, C.POINTER(v)],
        "fq_ctx_destroy": [v],
        "fq_ctx_set_stream": [v, v],
        "fq_ctx_get_stream": [v, C.POINTER(v)],
        "fq_ctx_synchronize": [v],
        "fq_ctx_launch_count": [v, C.POINTER(i64)],
        "fq_layer_create": [v, i64, i64, i64, C.POINTER(v)],
        "fq_layer_destroy": [v],
        "fq_layer_upload_quantized": [v, i32, i32, v, i64, v, v, i64],
        "fq_layer_download_quantized": [v, i32, v, v, v],
        "fq_layer_upload_fp": [v, v],
        "fq_layer_upload_bias": [v, v],
        "fq_layer_quantize_device": [v, i32, i32, v],
        "fq_layer_has": [v, i32, C.POINTER(i32)],
        "fq_layer_shape": [v, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)],
        "fq_layer_bytes": [v, i32, i64, C.POINTER(i64)],
        "fq_gemv": [v, v, i32, i64, v, i32, v, i32, i32],
        "fq_gemv_chain_time": [v, C.POINTER(v), i32, i32, i64, v, i32, C.POINTER(v), i32, i32, C.POINTER(C.c_double)],
        "fq_softmax_stats": [v, v, i64, i64, v],
        "fq_kl_rows": [v, v, v, i32, i64, i64, v, v],
        "fq_hist_kl": [v, v, i32, i32, C.POINTER(C.c_double)],
        "fq_fill_normal": [v, v, i64, u64, u64, C.c_float],
        "fq_model_create": [v, C.POINTER(ModelConfig), C.POINTER(v)],
        "fq_model_destroy": [v],
        "fq_model_num_linears": [v, C.POINTER(i32)],
        "fq_model_linear_id": [v, i32, C.c_char_p, i32],
        "fq_model_linear_index": [v, C.c_char_p, C.POINTER(i32)],
        "fq_model_linear": [v, i32, C.POINTER(v)],
        "fq_model_set_param": [v, C.c_char_p, v, i64],
        "fq_model_get_param": [v, C.c_char_p, v, i64],
        "fq_model_init_random": [v, u64, C.c_float],
        "fq_model_init_random_kl": [v, u64, C.c_float, i32, v, v],
        "fq_model_set_rung": [v, i32, i32, i32],
        "fq_model_get_rung": [v, i32, i32, C.POINTER(i32)],
        "fq_model_set_all_rungs": [v, i32, i32],
        "fq_model_reset_slot": [v, i32],
        "fq_model_slot_length": [v, i32, C.POINTER(i64)],
        "fq_model_prefill": [v, i32, v, i64, v, v],
        "fq_model_decode": [v, i32, v, v, v, v],
        "fq_model_logits": [v, C.POINTER(v)],
        "fq_model_step_kernel_time": [v, i32, C.POINTER(C.c_double), C.POINTER(i64)],
        "fq_model_step_bytes": [v, i32, v, C.POINTER(i64), C.POINTER(i64)],
        "fq_model_calibrate_logit_kl": [v, v, i64, i64, i32, i32, v, v],
        "fq_model_profile_gemvs": [v, i32, i32, C.POINTER(C.c_double), C.POINTER(i64), C.POINTER(i64)],
        "fq_model_profile_step": [v, i32, i32, v, i64, C.POINTER(i32), C.POINTER(i32), v],
        "fq_gemm": [v, v, i32, i64, v, i64, v, i64],
        "fq_tp_shard_spec": [C.POINTER(ModelConfig), i32, i32, C.POINTER(TpShard)],
        "fq_shard_quantized": [i32, i64, i64, i64, v, v, v, i64, i64, i64, i64, v, v, v],
        "fq_tp_merge_stats": [v, i32, i32, v, v],
        "fq_model_create_tp": [v, C.POINTER(ModelConfig), i32, i32, C.POINTER(v)],
        "fq_model_tp_shard": [v, C.POINTER(TpShard)],
        "fq_model_tp_begin": [v, i32, v, v],
        "fq_model_tp_segment": [v, i32, v, v],
        "fq_model_tp_end": [v],
        "fq_model_get_rungs": [v, i32, v, i32],
        "fq_model_decode_chain": [v, i32, i32, v],
        "fq_tile_activations": [v, v, i32, i64, i64, i64, i32, v],
        "fq_gemm_tiled": [v, v, i32, i64, v, i32, v, i64, i32],
    }
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = i32
    L.fq_tiled_activation_bytes.argtypes = [i64, i64]
    L.fq_tiled_activation_bytes.restype = i64
    _lib = L
    return L


def check(status: int) -> None:
    if status != 0:
        msg = load().fq_last_error().decode(errors="replace")
        raise _ERRORS.get(status, Error)(msg)


def _ptr(a) -> int | None:
    """Raw pointer of a numpy array or a torch tensor (host or device)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    if isinstance(a, int):
        return a
    raise TypeError(f"cannot take a pointer of {type(a)}")


class Context:
    """fq_ctx: one device + one stream."""

    def __init__(self, device: int = 0, stream=None):
        L = load()
        h = C.c_void_p()
        check(L.fq_ctx_create(device, C.byref(h)))
        self.h = h
        self.L = L
        if stream is not None:
            self.set_stream(stream)

    def set_stream(self, stream) -> None:
        raw = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
        check(self.L.fq_ctx_set_stream(self.h, C.c_void_p(raw)))

    def stream_handle(self) -> int:
        s = C.c_void_p()
        check(self.L.fq_ctx_get_stream(self.h, C.byref(s)))
        return s.value or 0

    def synchronize(self) -> None:
        check(self.L.fq_ctx_synchronize(self.h))

    def launches(self) -> int:
        n = C.c_int64()
        check(self.L.fq_ctx_launch_count(self.h, C.byref(n)))
        return n.value

    def close(self) -> None:
        if self.h:
            check(self.L.fq_ctx_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # stateless kernels -------------------------------------------------------
    def gemv(self, layer: "Layer", rung: int, batch: int, x, x_dtype: int, y, y_dtype: int,
             numerics: int = NUMERICS_FAST) -> None:
        check(self.L.fq_gemv(self.h, layer.h, rung, batch, _ptr(x), x_dtype, _ptr(y), y_dtype, numerics))

    def gemv_chain_time(self, layers, rung: int, batch: int, x, x_dtype: int, ys, y_dtype: int, reps: int) -> float:
        """n independent GEMVs (same x) as one step-program launch without barriers; ms per launch."""
        n = len(layers)
        lh = (C.c_void_p * n)(*[l.h for l in layers])
        yh = (C.c_void_p * n)(*[_ptr(y) for y in ys])
        ms = C.c_double()
        check(self.L.fq_gemv_chain_time(self.h, lh, n, rung, batch, _ptr(x), x_dtype, yh, y_dtype, reps, C.byref(ms)))
        return ms.value

    def gemm(self, layer: "Layer", rung: int, rows: int, x_bf16, y_f32, x_stride: int = 0, y_stride: int = 0) -> None:
        """y[rows, N] = x[rows, K] . dequant(W_rung)^T on the tcgen05 tensor cores."""
        check(self.L.fq_gemm(self.h, layer.h, rung, rows, _ptr(x_bf16), x_stride or layer.K, _ptr(y_f32),
                             y_stride or layer.N))

    def tile_activations(self, x, x_dtype: int, rows: int, K: int, out_dtype: int, xt, x_stride: int = 0) -> None:
        check(self.L.fq_tile_activations(self.h, _ptr(x), x_dtype, x_stride or K, rows, K, out_dtype, _ptr(xt)))

    def tiled_activation_bytes(self, rows: int, K: int) -> int:
        return int(self.L.fq_tiled_activation_bytes(rows, K))

    def gemm_tiled(self, layer: "Layer", rung: int, rows: int, xt, x_dtype: int, y_f32, y_stride: int = 0,
                   accumulate: bool = False) -> None:
        check(self.L.fq_gemm_tiled(self.h, layer.h, rung, rows, _ptr(xt), x_dtype, _ptr(y_f32), y_stride or layer.N,
                                   1 if accumulate else 0))

    def softmax_stats(self, logits, rows: int, vocab: int, stats_dev) -> None:
        check(self.L.fq_softmax_stats(self.h, _ptr(logits), rows, vocab, _ptr(stats_dev)))

    def kl_rows(self, lq, lp, dtype: int, rows: int, vocab: int, kl_dev, ent_dev=None) -> None:
        check(self.L.fq_kl_rows(self.h, _ptr(lq), _ptr(lp), dtype, rows, vocab, _ptr(kl_dev), _ptr(ent_dev)))

    def fill_normal(self, dst_dev, n: int, seed: int, stream_id: int, std: float) -> None:
        check(self.L.fq_fill_normal(self.h, _ptr(dst_dev), n, seed, stream_id, std))


class Layer:
    """fq_layer: resident per-precision copies of one linear."""

    def __init__(self, ctx: Context, out_features: int, in_features: int, group_size: int = 128, handle=None):
        self.ctx = ctx
        self.L = ctx.L
        self.borrowed = handle is not None
        if handle is None:
            h = C.c_void_p()
            check(self.L.fq_layer_create(ctx.h, out_features, in_features, group_size, C.byref(h)))
            self.h = h
        else:
            self.h = handle
        n, k, g = C.c_int64(), C.c_int64(), C.c_int64()
        check(self.L.fq_layer_shape(self.h, C.byref(n), C.byref(k), C.byref(g)))
        self.N, self.K, self.G = n.value, k.value, g.value
        self.ng = (self.K + self.G - 1) // self.G

    def upload_quantized(self, rung: int, payload: np.ndarray, scale: np.ndarray, zp: np.ndarray,
                         mode: int = MODE_ASYM) -> None:
        payload = np.ascontiguousarray(payload, np.uint8)
        scale = np.ascontiguousarray(scale, np.float32).ravel()
        zp = np.ascontiguousarray(zp, np.int32).ravel()
        check(self.L.fq_layer_upload_quantized(self.h, rung, mode, _ptr(payload), payload.size, _ptr(scale),
                                               _ptr(zp), scale.size))

    def download_quantized(self, rung: int):
        bits = 8 if rung == RUNG_INT8 else 4
        payload = np.zeros((self.N * self.K * bits + 7) // 8, np.uint8)
        scale = np.zeros(self.N * self.ng, np.float32)
        zp = np.zeros(self.N * self.ng, np.int32)
        check(self.L.fq_layer_download_quantized(self.h, rung, _ptr(payload), _ptr(scale), _ptr(zp)))
        return payload, scale.reshape(self.N, self.ng), zp.reshape(self.N, self.ng)

    def upload_fp(self, w: np.ndarray) -> None:
        w = np.ascontiguousarray(w, np.float32)
        check(self.L.fq_layer_upload_fp(self.h, _ptr(w)))

    def upload_bias(self, b: np.ndarray) -> None:
        b = np.ascontiguousarray(b, np.float32)
        check(self.L.fq_layer_upload_bias(self.h, _ptr(b)))

    def quantize_device(self, rung: int, w_dev, mode: int = MODE_ASYM) -> None:
        check(self.L.fq_layer_quantize_device(self.h, rung, mode, _ptr(w_dev)))

    def has(self, rung: int) -> bool:
        o = C.c_int32()
        check(self.L.fq_layer_has(self.h, rung, C.byref(o)))
        return bool(o.value)

    def algorithmic_bytes(self, rung: int, batch: int) -> int:
        o = C.c_int64()
        check(self.L.fq_layer_bytes(self.h, rung, batch, C.byref(o)))
        return o.value

    def hist_kl(self, rung: int, bins: int) -> float:
        o = C.c_double()
        check(self.L.fq_hist_kl(self.ctx.h, self.h, rung, bins, C.byref(o)))
        return o.value

    def close(self) -> None:
        if self.h and not self.borrowed:
            check(self.L.fq_layer_destroy(self.h))
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_CFG_KEYS = ["arch", "act_dtype", "vocab_size", "d_model", "n_heads", "head_dim", "n_layers", "ffn_dim",
             "max_seq_len", "tie_embeddings", "max_batch", "group_size", "norm_eps", "rope_theta"]


def model_config(**kw) -> ModelConfig:
    c = ModelConfig()
    c.arch = kw.get("arch", ARCH_LLAMA)
    c.act_dtype = kw.get("act_dtype", DT_BF16 if c.arch == ARCH_LLAMA else DT_F32)
    for k in ["vocab_size", "d_model", "n_heads", "head_dim", "n_layers", "ffn_dim", "max_seq_len"]:
        setattr(c, k, int(kw[k]))
    c.tie_embeddings = int(kw.get("tie_embeddings", 0))
    c.max_batch = int(kw.get("max_batch", 1))
    c.group_size = int(kw.get("group_size", 128))
    c.norm_eps = float(kw.get("norm_eps", 1e-5))
    c.rope_theta = float(kw.get("rope_theta", 10000.0))
    return c


def tp_shard_spec(cfg: ModelConfig, rank: int, size: int) -> TpShard:
    """The shard of TP rank `rank` of `size` (host only, no GPU needed)."""
    sh = TpShard()
    check(load().fq_tp_shard_spec(C.byref(cfg), rank, size, C.byref(sh)))
    return sh


def shard_quantized(bits: int, N: int, K: int, group: int, payload, scale, zp, rows, cols):
    """Rows [r0, r1) x columns [c0, c1) of a g-grouped quantized [N, K] weight (host only)."""
    (r0, r1), (c0, c1) = rows, cols
    ng_out = (c1 - c0 + group - 1) // group
    n = r1 - r0
    pl = np.zeros(n * (c1 - c0) * bits // 8, np.uint8)
    sc = np.zeros(n * ng_out, np.float32)
    z = np.zeros(n * ng_out, np.int32)
    payload = np.ascontiguousarray(payload, np.uint8)
    scale = np.ascontiguousarray(scale, np.float32)
    zp = np.ascontiguousarray(zp, np.int32)
    check(load().fq_shard_quantized(bits, N, K, group, _ptr(payload), _ptr(scale), _ptr(zp), r0, r1, c0, c1,
                                    _ptr(pl), _ptr(sc), _ptr(z)))
    return pl, sc, z


def tp_merge_stats(parts: np.ndarray, vocab0) -> np.ndarray:
    """parts: STAT_PART_DTYPE [nranks, batch] -> ROW_STATS_DTYPE [batch] (host only)."""
    parts = np.ascontiguousarray(parts, STAT_PART_DTYPE)
    nr, b = parts.shape
    v0 = np.ascontiguousarray(vocab0, np.int64)
    out = np.zeros(b, ROW_STATS_DTYPE)
    check(load().fq_tp_merge_stats(_ptr(parts), nr, b, _ptr(v0), _ptr(out)))
    return out


class Model:
    """fq_model: the device-resident decoder (precision table, KV caches, decode step).
    tp=(rank, size): a tensor-parallel rank of the full config (see tp.py)."""

    def __init__(self, ctx: Context, tp=None, **cfg):
        self.ctx = ctx
        self.L = ctx.L
        self.cfg = model_config(**cfg)
        h = C.c_void_p()
        if tp is None:
            check(self.L.fq_model_create(ctx.h, C.byref(self.cfg), C.byref(h)))
        else:
            check(self.L.fq_model_create_tp(ctx.h, C.byref(self.cfg), int(tp[0]), int(tp[1]), C.byref(h)))
        self.h = h
        n = C.c_int32()
        check(self.L.fq_model_num_linears(h, C.byref(n)))
        self.n_linears = n.value
        self.ids = []
        buf = C.create_string_buffer(256)
        for i in range(self.n_linears):
            check(self.L.fq_model_linear_id(h, i, buf, 256))
            self.ids.append(buf.value.decode())
        self.V = self.cfg.vocab_size

    def linear(self, i: int) -> Layer:
        lh = C.c_void_p()
        check(self.L.fq_model_linear(self.h, i, C.byref(lh)))
        return Layer(self.ctx, 0, 0, handle=lh)

    def linear_index(self, layer_id: str) -> int:
        o = C.c_int32()
        check(self.L.fq_model_linear_index(self.h, layer_id.encode(), C.byref(o)))
        return o.value

    def set_param(self, name: str, arr: np.ndarray) -> None:
        a = np.ascontiguousarray(arr, np.float32)
        check(self.L.fq_model_set_param(self.h, name.encode(), _ptr(a), a.size))

    def get_param(self, name: str, numel: int) -> np.ndarray:
        a = np.zeros(numel, np.float32)
        check(self.L.fq_model_get_param(self.h, name.encode(), _ptr(a), a.size))
        return a

    def init_random(self, seed: int, std: float = 0.02, kl_bins: int = 0):
        """Device-side random init; with kl_bins > 0 also returns the weight-histogram KL of the
        W8 and W4 rungs of every linear (reference analyzer, src/analyzer.cpp:83-94)."""
        if kl_bins <= 0:
            check(self.L.fq_model_init_random(self.h, seed, std))
            return None
        kl8 = np.zeros(self.n_linears, np.float64)
        kl4 = np.zeros(self.n_linears, np.float64)
        check(self.L.fq_model_init_random_kl(self.h, seed, std, kl_bins, _ptr(kl8), _ptr(kl4)))
        return kl8, kl4

    def set_rung(self, slot: int, index: int, rung: int) -> None:
        check(self.L.fq_model_set_rung(self.h, slot, index, rung))

    def get_rung(self, slot: int, index: int) -> int:
        o = C.c_int32()
        check(self.L.fq_model_get_rung(self.h, slot, index, C.byref(o)))
        return o.value

    def set_all_rungs(self, slot: int, rung: int) -> None:
        check(self.L.fq_model_set_all_rungs(self.h, slot, rung))

    def reset_slot(self, slot: int) -> None:
        check(self.L.fq_model_reset_slot(self.h, slot))

    def slot_length(self, slot: int) -> int:
        o = C.c_int64()
        check(self.L.fq_model_slot_length(self.h, slot, C.byref(o)))
        return o.value

    def prefill(self, slot: int, tokens, logits_dev=None) -> np.ndarray:
        t = np.ascontiguousarray(tokens, np.int32)
        st = np.zeros(t.size, ROW_STATS_DTYPE)
        check(self.L.fq_model_prefill(self.h, slot, _ptr(t), t.size, _ptr(logits_dev), _ptr(st)))
        return st

    def decode(self, slots, tokens, logits_dev=None) -> np.ndarray:
        s = np.ascontiguousarray(slots, np.int32)
        t = np.ascontiguousarray(tokens, np.int32)
        st = np.zeros(s.size, ROW_STATS_DTYPE)
        check(self.L.fq_model_decode(self.h, s.size, _ptr(s), _ptr(t), _ptr(logits_dev), _ptr(st)))
        return st

    def decode_one(self, slot: int, token: int):
        """decode() for one slot with preallocated argument / result buffers (the per-token call
        of a decode loop); returns the row's stats record (valid until the next call)."""
        if not hasattr(self, "_d1"):
            self._d1 = (np.zeros(1, np.int32), np.zeros(1, np.int32), np.zeros(1, ROW_STATS_DTYPE))
            self._d1p = tuple(a.ctypes.data for a in self._d1)
        s, t, st = self._d1
        s[0] = slot
        t[0] = token
        check(self.L.fq_model_decode(self.h, 1, self._d1p[0], self._d1p[1], None, self._d1p[2]))
        return st[0]

    def decode_chain(self, slot: int, n: int) -> np.ndarray:
        """n device-chained decode steps of `slot` (token = the previous step's argmax)."""
        st = np.zeros(n, ROW_STATS_DTYPE)
        check(self.L.fq_model_decode_chain(self.h, slot, n, _ptr(st)))
        return st

    def step_kernel_time(self, reset: bool = True) -> tuple:
        """(total ms, steps) of the decode-step program kernels since the last reset (device events)."""
        ms, n = C.c_double(), C.c_int64()
        check(self.L.fq_model_step_kernel_time(self.h, 1 if reset else 0, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def logits_ptr(self) -> int:
        p = C.c_void_p()
        check(self.L.fq_model_logits(self.h, C.byref(p)))
        return p.value

    def step_bytes(self, slots) -> tuple:
        s = np.ascontiguousarray(slots, np.int32)
        w, k = C.c_int64(), C.c_int64()
        check(self.L.fq_model_step_bytes(self.h, s.size, _ptr(s), C.byref(w), C.byref(k)))
        return w.value, k.value

    def profile_gemvs(self, slot: int, reps: int):
        """(ms per GEMV launch, launches per step, algorithmic bytes per step) of the step's GEMVs."""
        ms, n, b = C.c_double(), C.c_int64(), C.c_int64()
        check(self.L.fq_model_profile_gemvs(self.h, slot, reps, C.byref(ms), C.byref(n), C.byref(b)))
        return ms.value, n.value, b.value

    def profile_step(self, slot: int, token: int, max_phases: int = 4096):
        """One decode step with per-phase %globaltimer stamps: returns (types[nphases],
        end[nphases, grid], after_barrier[nphases, grid], start[grid]) in ns."""
        nph, grid = C.c_int32(), C.c_int32()
        cap = (max_phases * 2 + 1) * 256 + 3 * 16384 + max_phases * 256 * 8
        ticks = np.zeros(cap, np.uint64)
        types = np.zeros(max_phases, np.int32)
        check(self.L.fq_model_profile_step(self.h, slot, token, _ptr(ticks), cap, C.byref(nph), C.byref(grid),
                                           _ptr(types)))
        n, g = nph.value, grid.value
        t = ticks[: (2 * n + 1) * g].astype(np.int64)
        ph = t[: 2 * n * g].reshape(n, g, 2)
        off = (2 * n + 1) * g
        self.last_ring_trace = ticks[off: off + 3 * 16384].astype(np.int64).reshape(-1, 3)
        self.last_gemv_detail = ticks[off + 3 * 16384: off + 3 * 16384 + n * g * 8].astype(np.int64).reshape(n, g, 8)
        return types[:n], ph[:, :, 0], ph[:, :, 1], t[2 * n * g:]

    def calibrate_logit_kl(self, tokens: np.ndarray, base_rung: int, flip_rung: int):
        t = np.ascontiguousarray(tokens, np.int32)
        n_seqs, length = t.shape
        kl = np.zeros(self.cfg.n_layers, np.float64)
        ent = np.zeros(self.cfg.n_layers, np.float64)
        check(self.L.fq_model_calibrate_logit_kl(self.h, _ptr(t), n_seqs, length, base_rung, flip_rung, _ptr(kl),
                                                 _ptr(ent)))
        return kl, ent

    # ---------------------------------------------------------------- tensor-parallel rank
    def tp_shard(self) -> TpShard:
        sh = TpShard()
        check(self.L.fq_model_tp_shard(self.h, C.byref(sh)))
        return sh

    def tp_begin(self, slots, tokens) -> None:
        self._tp_s = np.ascontiguousarray(slots, np.int32)
        t = np.ascontiguousarray(tokens, np.int32)
        check(self.L.fq_model_tp_begin(self.h, self._tp_s.size, _ptr(self._tp_s), _ptr(t)))

    def tp_segment(self, seg: int, reduced_dev, out_dev) -> None:
        check(self.L.fq_model_tp_segment(self.h, seg, _ptr(reduced_dev), _ptr(out_dev)))

    def tp_end(self) -> None:
        check(self.L.fq_model_tp_end(self.h))

    def close(self) -> None:
        if self.h:
            check(self.L.fq_model_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
