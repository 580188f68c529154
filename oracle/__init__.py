"""CPU oracle for the FlexQuant hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package.  The product (paper_2506_12024_b200) never does.

* ``lib()``  -> ctypes handle on liboracle.so, the plain-C restatement (fq_oracle.c).
* ``ref()``  -> ctypes handle on _ref/libfqref.so, the unmodified reference library compiled
  from /root/reference/proj/src (None when it was not built).
* numpy helpers wrapping both, plus ``llama.py`` (numpy restatement of the Llama-shaped block).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_REF = None

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_i64 = C.c_int64


def build() -> None:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.fqo_quantize.argtypes = [_f32p, _i64, _i64, _i64, C.c_int, C.c_int, _u8p, _f32p, _i32p]
        L.fqo_dequantize.argtypes = [_u8p, _i64, _i64, _i64, C.c_int, C.c_int, _f32p, _i32p, _f32p]
        L.fqo_linear.argtypes = [_f32p, _i64, _i64, _f32p, _i64, C.c_void_p, _f32p]
        L.fqo_quant_linear.argtypes = [_f32p, _i64, _u8p, _i64, _i64, _i64, C.c_int, C.c_int, _f32p, _i32p,
                                       C.c_void_p, _f32p]
        L.fqo_row_stats.argtypes = [_f32p, _i64] + [C.POINTER(C.c_double)] * 5 + [C.POINTER(C.c_int32)]
        L.fqo_derive_threshold.argtypes = [_f32p, _i64, _i64, C.c_int, C.c_double, C.POINTER(C.c_double)]
        L.fqo_scheduler_replay.argtypes = [_f64p, _i64, C.c_int, C.c_double, C.c_int, _i64, _i64p, _i64p, _f64p, _i32p]
        L.fqo_hist_kl.argtypes = [_f32p, _f32p, _i64, C.c_int, C.POINTER(C.c_double)]
        L.fqo_kl_logits.argtypes = [_f32p, _f32p, _i64, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.fqo_fill_normal.argtypes = [_f32p, _i64, C.c_uint64, C.c_uint64, C.c_float]
        L.fqo_random_tokens.argtypes = [_i64, _i64, C.c_uint64, _i32p]
        L.fqo_pack.argtypes = [_u32p, _i64, C.c_int, _u8p]
        L.fqo_unpack.argtypes = [_u8p, _i64, C.c_int, _u32p]
        _LIB = L
    return _LIB


def ref():
    """The reference library itself (None if oracle/_ref was never built)."""
    global _REF
    if _REF is None:
        path = os.path.join(_HERE, "_ref", "libfqref.so")
        if not os.path.exists(path):
            return None
        R = C.CDLL(path)
        R.ref_last_error.restype = C.c_char_p
        R.ref_quantize.argtypes = [_f32p, _i64, _i64, _i64, C.c_int, C.c_int, _u8p, _f32p, _i32p]
        R.ref_dequantize.argtypes = [_u8p, _i64, _i64, _i64, C.c_int, C.c_int, _f32p, _i32p, _f32p]
        R.ref_linear.argtypes = [_f32p, _i64, _i64, _f32p, _i64, C.c_void_p, _f32p]
        R.ref_row_stats.argtypes = [_f32p, _i64, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_int32)]
        R.ref_derive_threshold.argtypes = [_f32p, _i64, _i64, C.c_int, C.c_double, C.POINTER(C.c_double)]
        R.ref_scheduler_replay.argtypes = [_f64p, _i64, C.c_int, C.c_double, C.c_int, _i64, _i64p, _i64p, _f64p, _i32p]
        R.ref_hist_kl.argtypes = [_f32p, _f32p, _i64, C.c_int, C.POINTER(C.c_double)]
        R.ref_kl_divergence.argtypes = [_f64p, _f64p, _i64, C.POINTER(C.c_double)]
        R.ref_make_fixture.argtypes = [C.c_char_p, C.c_uint64, _i64, C.c_char_p]
        R.ref_analyze.argtypes = [C.c_char_p, C.c_int, C.c_char_p]
        R.ref_generate.argtypes = [C.c_char_p, C.c_char_p, _i32p, _i64, _i64, C.c_double, C.c_int, C.c_int, C.c_int,
                                   C.c_int, C.c_char_p, _i32p, C.POINTER(C.c_int64), C.POINTER(C.c_double)]
        R.ref_prefill_logits.argtypes = [C.c_char_p, _i32p, _i64, C.c_int, _f32p]
        R.ref_decode_logits.argtypes = [C.c_char_p, _i32p, _i64, C.c_int, _f32p]
        R.ref_time_quant_linear.argtypes = [_f32p, _i64, _i64, _i64, C.c_int, _f32p, _i64, C.c_int,
                                            C.POINTER(C.c_double)]
        _REF = R
    return _REF


def _check(st: int, who: str = "oracle") -> None:
    if st != 0:
        msg = ""
        if who == "ref" and ref() is not None:
            msg = ref().ref_last_error().decode()
        raise RuntimeError(f"{who} call failed with status {st} {msg}")


# ---------------------------------------------------------------- numpy helpers
def quantize(w: np.ndarray, group: int, bits: int, mode: int = 0, impl: str = "oracle"):
    """Group-wise RTN quantization -> (payload u8, scale f32 [N, ng], zp i32 [N, ng])."""
    w = np.ascontiguousarray(w, dtype=np.float32)
    N, K = w.shape
    G = K if group <= 0 or group > K else group
    ng = (K + G - 1) // G
    payload = np.zeros((N * K * bits + 7) // 8, np.uint8)
    scale = np.zeros(N * ng, np.float32)
    zp = np.zeros(N * ng, np.int32)
    if impl == "ref":
        _check(ref().ref_quantize(w, N, K, G, bits, mode, payload, scale, zp), "ref")
    else:
        _check(lib().fqo_quantize(w, N, K, G, bits, mode, payload, scale, zp))
    return payload, scale.reshape(N, ng), zp.reshape(N, ng)


def dequantize(payload, N, K, group, bits, scale, zp, mode: int = 0) -> np.ndarray:
    out = np.zeros(N * K, np.float32)
    G = K if group <= 0 or group > K else group
    _check(lib().fqo_dequantize(np.ascontiguousarray(payload), N, K, G, bits, mode,
                                np.ascontiguousarray(scale, np.float32).ravel(),
                                np.ascontiguousarray(zp, np.int32).ravel(), out))
    return out.reshape(N, K)


def linear(x: np.ndarray, w: np.ndarray, bias=None) -> np.ndarray:
    """Reference linear(): double accumulation, k ascending, one float cast."""
    x = np.ascontiguousarray(x, np.float32)
    w = np.ascontiguousarray(w, np.float32)
    B, K = x.shape
    N = w.shape[0]
    y = np.zeros((B, N), np.float32)
    b = None if bias is None else np.ascontiguousarray(bias, np.float32)
    lib().fqo_linear(x, B, K, w, N, None if b is None else b.ctypes.data, y)
    return y


def row_stats(logits: np.ndarray) -> dict:
    l = np.ascontiguousarray(logits, np.float32).ravel()
    ppl, ent, ft, p1, p2 = (C.c_double() for _ in range(5))
    am = C.c_int32()
    _check(lib().fqo_row_stats(l, l.size, C.byref(ppl), C.byref(ent), C.byref(ft), C.byref(p1), C.byref(p2),
                               C.byref(am)))
    return dict(ppl_entropy=ppl.value, entropy=ent.value, fault_tolerance=ft.value, p1=p1.value, p2=p2.value,
                argmax=am.value)


def scheduler_replay(ppl, window_len, thre, layers_per_switch, plan_len, impl="oracle"):
    ppl = np.ascontiguousarray(ppl, np.float64)
    n = ppl.size
    ff = np.zeros(n, np.int64)
    fc = np.zeros(n, np.int64)
    mv = np.zeros(n, np.float64)
    vv = np.zeros(n, np.int32)
    fn = ref().ref_scheduler_replay if impl == "ref" else lib().fqo_scheduler_replay
    _check(fn(ppl, n, window_len, thre, layers_per_switch, plan_len, ff, fc, mv, vv), impl)
    return ff, fc, mv, vv.astype(bool)


def hist_kl(w: np.ndarray, wq: np.ndarray, bins: int, impl="oracle") -> float:
    out = C.c_double()
    w = np.ascontiguousarray(w, np.float32).ravel()
    wq = np.ascontiguousarray(wq, np.float32).ravel()
    fn = ref().ref_hist_kl if impl == "ref" else lib().fqo_hist_kl
    _check(fn(w, wq, w.size, bins, C.byref(out)), impl)
    return out.value


def kl_logits(lq, lp):
    kl, h = C.c_double(), C.c_double()
    lq = np.ascontiguousarray(lq, np.float32).ravel()
    lp = np.ascontiguousarray(lp, np.float32).ravel()
    _check(lib().fqo_kl_logits(lq, lp, lq.size, C.byref(kl), C.byref(h)))
    return kl.value, h.value


def normal(n: int, seed: int, stream: int, std: float) -> np.ndarray:
    out = np.zeros(n, np.float32)
    lib().fqo_fill_normal(out, n, seed, stream, std)
    return out


def random_tokens(n: int, vocab: int, seed: int) -> np.ndarray:
    out = np.zeros(n, np.int32)
    lib().fqo_random_tokens(n, vocab, seed, out)
    return out
