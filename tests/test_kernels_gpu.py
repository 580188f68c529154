"""Parity of the CUDA kernels (through the C-ABI) against the CPU oracle.

Bars (BASELINE north_star): bit-exact packing / scales / zero points; GEMV within 1e-2
relative of the reference dequant+linear; entropy / KL within 1e-4 absolute.
"""
import ctypes as C

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2506_12024_b200 import capi  # noqa: E402


def _w(N, K, seed, std=0.02):
    return oracle.normal(N * K, seed, 1, std).reshape(N, K)


def _layer(ctx, w, group, bits_list=(8, 4), mode=0):
    N, K = w.shape
    L = capi.Layer(ctx, N, K, group)
    ref = {}
    for bits in bits_list:
        p, s, z = oracle.quantize(w, group, bits, mode)
        L.upload_quantized(capi.RUNG_INT8 if bits == 8 else capi.RUNG_INT4, p, s, z, mode)
        ref[bits] = (p, s, z)
    return L, ref


def _gemv(ctx, L, rung, x_np, x_dtype, numerics=capi.NUMERICS_FAST):
    B = x_np.shape[0]
    tdt = {capi.DT_F32: torch.float32, capi.DT_F16: torch.float16, capi.DT_BF16: torch.bfloat16}[x_dtype]
    x = torch.from_numpy(x_np).to("cuda").to(tdt).contiguous()
    y = torch.empty((B, L.N), dtype=torch.float32, device="cuda")
    ctx.gemv(L, rung, B, x, x_dtype, y, capi.DT_F32, numerics)
    ctx.synchronize()
    return y.cpu().numpy(), x.float().cpu().numpy()


def _rel(y, yref):
    return float(np.max(np.abs(y - yref)) / max(np.max(np.abs(yref)), 1e-30))


@pytest.mark.parametrize("N,K", [(256, 512), (128, 1376), (96, 4096), (64, 11008), (4096, 4096)])
@pytest.mark.parametrize("bits", [8, 4])
@pytest.mark.parametrize("B", [1, 2, 4, 16])
def test_gemv_fast_vs_oracle(ctx, N, K, bits, B):
    w = _w(N, K, N * 31 + K)
    L, ref = _layer(ctx, w, 128, (bits,))
    x = np.random.default_rng(K + B).standard_normal((B, K)).astype(np.float32)
    rung = capi.RUNG_INT8 if bits == 8 else capi.RUNG_INT4
    y, x16 = _gemv(ctx, L, rung, x, capi.DT_F16)
    p, s, z = ref[bits]
    yref = np.zeros((B, N), np.float32)
    oracle.lib().fqo_quant_linear(np.ascontiguousarray(x16), B, p, N, K, 128, bits, 0, s.ravel(), z.ravel(), None, yref)
    assert _rel(y, yref) < 1e-4, _rel(y, yref)
    # elementwise: 1e-2 relative on every output that is not tiny
    big = np.abs(yref) > 1e-3 * np.max(np.abs(yref))
    assert np.all(np.abs(y - yref)[big] <= 1e-2 * np.abs(yref)[big])


@pytest.mark.parametrize("N,K", [(200, 1376), (4096, 4096)])
@pytest.mark.parametrize("bits", [8, 4])
@pytest.mark.parametrize("B", [9, 24, 32, 40])
def test_gemv_fast_wide_batches_and_repeatability(ctx, N, K, bits, B):
    """Stand-alone GEMV (gemv_direct.cu) with 2 / 4 MMA column groups and a > 32-row batch split
    into launches; split-K partials summed in slice order by the tile's last task: two calls are
    bit-identical."""
    w = _w(N, K, N * 7 + K + B)
    L, ref = _layer(ctx, w, 128, (bits,))
    x = np.random.default_rng(K + 3 * B).standard_normal((B, K)).astype(np.float32)
    rung = capi.RUNG_INT8 if bits == 8 else capi.RUNG_INT4
    y, x16 = _gemv(ctx, L, rung, x, capi.DT_F16)
    y2, _ = _gemv(ctx, L, rung, x, capi.DT_F16)
    assert np.array_equal(y, y2)
    p, s, z = ref[bits]
    yref = np.zeros((B, N), np.float32)
    oracle.lib().fqo_quant_linear(np.ascontiguousarray(x16), B, p, N, K, 128, bits, 0, s.ravel(), z.ravel(), None, yref)
    assert _rel(y, yref) < 1e-4, _rel(y, yref)


@pytest.mark.parametrize("N,K", [(5, 256), (17, 130), (33, 1376)])
@pytest.mark.parametrize("bits", [8, 4])
@pytest.mark.parametrize("B", [1, 3, 17])
@pytest.mark.parametrize("x_dtype", [capi.DT_F32, capi.DT_BF16])
def test_gemv_fast_tiny_and_ragged(ctx, N, K, bits, B, x_dtype):
    """Layers smaller than one 16-row tile, a 2-code ragged last group, fp32 / bf16 inputs (the
    direct kernel rounds them to the fp16 MMA operand; the oracle sees the same fp16 values)."""
    w = _w(N, K, 900 + N + K)
    L, ref = _layer(ctx, w, 128, (bits,))
    x = np.random.default_rng(N + K + B).standard_normal((B, K)).astype(np.float32)
    rung = capi.RUNG_INT8 if bits == 8 else capi.RUNG_INT4
    y, xin = _gemv(ctx, L, rung, x, x_dtype)
    p, s, z = ref[bits]
    rels = []
    # the fast kernels take fp16 operands; a layer whose zero points span more than a byte (the
    # 2-code group of K = 130 quantizes to an extreme z) has no tiled copy and runs the exact
    # fp32 path on the unrounded input -- each matches the oracle on its own operands
    for xo in (xin.astype(np.float16).astype(np.float32), xin):
        yref = np.zeros((B, N), np.float32)
        oracle.lib().fqo_quant_linear(np.ascontiguousarray(xo), B, p, N, K, 128, bits, 0, s.ravel(), z.ravel(), None, yref)
        rels.append(_rel(y, yref))
    assert min(rels) < 1e-4, rels


@pytest.mark.parametrize("y_dtype", [capi.DT_BF16, capi.DT_F16])
def test_gemv_fast_half_outputs(ctx, y_dtype):
    N, K, B = 4096, 4096, 4
    w = _w(N, K, 77)
    L, ref = _layer(ctx, w, 128, (8,))
    x = torch.from_numpy(np.random.default_rng(5).standard_normal((B, K)).astype(np.float32)).to("cuda").half()
    tdt = torch.bfloat16 if y_dtype == capi.DT_BF16 else torch.float16
    y = torch.empty((B, N), dtype=tdt, device="cuda")
    yf = torch.empty((B, N), dtype=torch.float32, device="cuda")
    ctx.gemv(L, capi.RUNG_INT8, B, x, capi.DT_F16, y, y_dtype, capi.NUMERICS_FAST)
    ctx.gemv(L, capi.RUNG_INT8, B, x, capi.DT_F16, yf, capi.DT_F32, capi.NUMERICS_FAST)
    ctx.synchronize()
    assert torch.equal(y, yf.to(tdt))  # the same fp32 sums, rounded once at the store


_C2_CACHE = {}


def _c2_layer(ctx, K, N, bits):
    """BASELINE C2 weights: W [N, K] N(0, 0.02) quantized g128 (cached per shape and width)."""
    key = (K, N, bits)
    if key not in _C2_CACHE:
        _C2_CACHE.clear()  # one 7B-shape layer resident at a time
        w = _w(N, K, 2000 + N + K)
        _C2_CACHE[key] = _layer(ctx, w, 128, (bits,))
    return _C2_CACHE[key]


@pytest.mark.parametrize("K,N", [(4096, 4096), (4096, 11008), (11008, 4096), (4096, 32000)])
@pytest.mark.parametrize("bits", [8, 4])
@pytest.mark.parametrize("B", [1, 4, 16])
def test_gemv_c2_shapes_full_size(ctx, K, N, bits, B):
    """BASELINE C2 at its exact Llama-7B shapes (no shrunken N): fp16 activations N(0,1), batch
    1/4/16, each width against the reference dequant + double-accumulated linear (oracle)."""
    L, ref = _c2_layer(ctx, K, N, bits)
    x = np.random.default_rng(K * 7 + B).standard_normal((B, K)).astype(np.float32)
    rung = capi.RUNG_INT8 if bits == 8 else capi.RUNG_INT4
    y, x16 = _gemv(ctx, L, rung, x, capi.DT_F16)
    p, s, z = ref[bits]
    yref = np.zeros((B, N), np.float32)
    oracle.lib().fqo_quant_linear(np.ascontiguousarray(x16), B, p, N, K, 128, bits, 0, s.ravel(), z.ravel(), None, yref)
    assert _rel(y, yref) < 1e-4, _rel(y, yref)
    big = np.abs(yref) > 1e-3 * np.max(np.abs(yref))
    assert np.all(np.abs(y - yref)[big] <= 1e-2 * np.abs(yref)[big])


@pytest.mark.parametrize("bits", [8, 4])
@pytest.mark.parametrize("B", [1, 3])
def test_gemv_chain_program_matches_oracle(ctx, bits, B):
    # fq_gemv_chain_time: n independent GEMVs as one step-program launch (the C2 sweep's
    # "program" timing) produce every layer's reference dequant+linear
    N, K, n = 256, 1376, 3
    rung = capi.RUNG_INT8 if bits == 8 else capi.RUNG_INT4
    layers, refs = [], []
    for i in range(n):
        L, ref = _layer(ctx, _w(N, K, 900 + i), 128, (bits,))
        layers.append(L)
        refs.append(ref[bits])
    x = np.random.default_rng(5).standard_normal((B, K)).astype(np.float32)
    xt = torch.from_numpy(x).to("cuda").half().contiguous()
    ys = [torch.empty((B, N), dtype=torch.float32, device="cuda") for _ in range(n)]
    ms = ctx.gemv_chain_time(layers, rung, B, xt, capi.DT_F16, ys, capi.DT_F32, 2)
    assert ms > 0
    x16 = xt.float().cpu().numpy()
    for y, (p, s, z) in zip(ys, refs):
        yref = np.zeros((B, N), np.float32)
        oracle.lib().fqo_quant_linear(np.ascontiguousarray(x16), B, p, N, K, 128, bits, 0, s.ravel(), z.ravel(), None,
                                      yref)
        assert _rel(y.cpu().numpy(), yref) < 1e-4


@pytest.mark.parametrize("bits", [8, 4])
def test_gemv_bf16_activations(ctx, bits):
    N, K = 512, 4096
    w = _w(N, K, 5)
    L, ref = _layer(ctx, w, 128, (bits,))
    x = np.random.default_rng(3).standard_normal((1, K)).astype(np.float32)
    rung = capi.RUNG_INT8 if bits == 8 else capi.RUNG_INT4
    y, xb = _gemv(ctx, L, rung, x, capi.DT_BF16)
    p, s, z = ref[bits]
    yref = np.zeros((1, N), np.float32)
    oracle.lib().fqo_quant_linear(np.ascontiguousarray(xb), 1, p, N, K, 128, bits, 0, s.ravel(), z.ravel(), None, yref)
    assert _rel(y, yref) < 1e-4


@pytest.mark.parametrize("shape,group", [((64, 96), 0), ((48, 33), 0), ((32, 512), 128), ((16, 1376), 128)])
@pytest.mark.parametrize("bits", [8, 4])
@pytest.mark.parametrize("mode", [0, 1])
def test_gemv_exact_matches_reference_linear(ctx, shape, group, bits, mode):
    """Exact numerics: dequantize in fp32 + double accumulation == reference linear()."""
    N, K = shape
    w = _w(N, K, 77 + K, 0.3)
    L, ref = _layer(ctx, w, group, (bits,), mode)
    bias = np.random.default_rng(1).standard_normal(N).astype(np.float32)
    L.upload_bias(bias)
    x = np.random.default_rng(2).standard_normal((3, K)).astype(np.float32)
    rung = capi.RUNG_INT8 if bits == 8 else capi.RUNG_INT4
    y, _ = _gemv(ctx, L, rung, x, capi.DT_F32, capi.NUMERICS_EXACT)
    p, s, z = ref[bits]
    yref = np.zeros((3, N), np.float32)
    oracle.lib().fqo_quant_linear(x, 3, p, N, K, group, bits, mode, s.ravel(), z.ravel(), bias.ctypes.data, yref)
    # double accumulation in a different order: identical after the float cast except for
    # rare double-rounding ties (<= 1 ulp)
    ulp = np.abs(y.view(np.int32).astype(np.int64) - yref.view(np.int32).astype(np.int64))
    assert ulp.max() <= 1 and np.mean(ulp == 0) > 0.99


def test_gemv_fp_rung_exact(ctx):
    N, K = 40, 64
    w = _w(N, K, 9, 0.5)
    L = capi.Layer(ctx, N, K, 0)
    L.upload_fp(w)
    x = np.random.default_rng(4).standard_normal((2, K)).astype(np.float32)
    y, _ = _gemv(ctx, L, capi.RUNG_FP, x, capi.DT_F32, capi.NUMERICS_EXACT)
    yref = oracle.linear(x, w)
    ulp = np.abs(y.view(np.int32).astype(np.int64) - yref.view(np.int32).astype(np.int64))
    assert ulp.max() <= 1


@pytest.mark.parametrize("key", ["64x512_g128", "16x1376_g128", "24x96_g0", "8x4096_g128"])
def test_layer_upload_download_round_trip(ctx, key):
    """The device layout is a bijection of the canonical QuantizedTensor packing."""
    g = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "quant_g128.npz"))
    w = g["w_" + key]
    N, K = w.shape
    group = int(key.split("_g")[1])
    L = capi.Layer(ctx, N, K, group)
    for bits, rung in ((8, capi.RUNG_INT8), (4, capi.RUNG_INT4)):
        p, s, z = g[f"p_{key}_b{bits}"], g[f"s_{key}_b{bits}"], g[f"z_{key}_b{bits}"]
        L.upload_quantized(rung, p, s, z)
        p2, s2, z2 = L.download_quantized(rung)
        assert np.array_equal(p, p2) and np.array_equal(s.view(np.uint32), s2.view(np.uint32)) and np.array_equal(z, z2)


@pytest.mark.parametrize("key", ["64x512_g128", "16x1376_g128", "24x96_g0", "8x4096_g128"])
@pytest.mark.parametrize("mode", [0, 1])
def test_device_quantizer_bit_exact(ctx, key, mode):
    """K9 on the device reproduces the reference quantizer bit for bit (golden vectors for asym)."""
    g = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "quant_g128.npz"))
    w = g["w_" + key]
    N, K = w.shape
    group = int(key.split("_g")[1])
    L = capi.Layer(ctx, N, K, group)
    wd = torch.from_numpy(w).cuda()
    for bits, rung in ((8, capi.RUNG_INT8), (4, capi.RUNG_INT4)):
        L.quantize_device(rung, wd, mode)
        p2, s2, z2 = L.download_quantized(rung)
        if mode == 0:
            p, s, z = g[f"p_{key}_b{bits}"], g[f"s_{key}_b{bits}"], g[f"z_{key}_b{bits}"]
        else:
            p, s, z = oracle.quantize(w, group, bits, mode)
        assert np.array_equal(p, p2)
        assert np.array_equal(s.view(np.uint32), s2.view(np.uint32))
        assert np.array_equal(z, z2)


def test_device_quantizer_constant_and_nonfinite(ctx):
    w = np.zeros((3, 256), np.float32)
    w[1, :128] = 0.25
    w[2, 128:] = -0.125
    L = capi.Layer(ctx, 3, 256, 128)
    L.quantize_device(capi.RUNG_INT4, torch.from_numpy(w).cuda())
    p2, s2, z2 = L.download_quantized(capi.RUNG_INT4)
    p, s, z = oracle.quantize(w, 128, 4)
    assert np.array_equal(p, p2) and np.array_equal(s, s2) and np.array_equal(z, z2)
    w[0, 5] = np.inf
    with pytest.raises(capi.InputError):
        L.quantize_device(capi.RUNG_INT8, torch.from_numpy(w).cuda())


def test_upload_validation_errors(ctx):
    L = capi.Layer(ctx, 4, 8, 0)
    p, s, z = oracle.quantize(_w(4, 8, 1), 0, 8)
    with pytest.raises(capi.FormatError):
        L.upload_quantized(capi.RUNG_INT8, p[:-1], s, z)
    with pytest.raises(capi.ConfigError):
        L.upload_quantized(7, p, s, z)
    with pytest.raises(capi.StateError):
        y = torch.zeros(4, device="cuda")
        ctx.gemv(L, capi.RUNG_INT4, 1, torch.zeros(8, device="cuda"), capi.DT_F32, y, capi.DT_F32)


@pytest.mark.parametrize("V", [2, 256, 8192, 32000])
def test_softmax_stats_vs_oracle(ctx, V):
    rng = np.random.default_rng(V)
    rows = 5
    l = (rng.standard_normal((rows, V)) * rng.uniform(0.05, 4, (rows, 1))).astype(np.float32)
    l[1, 7 % V] = l[1].max()  # a tie for the argmax
    out = torch.zeros(rows * capi.ROW_STATS_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    ctx.softmax_stats(torch.from_numpy(l).cuda(), rows, V, out)
    ctx.synchronize()
    st = np.frombuffer(out.cpu().numpy().tobytes(), capi.ROW_STATS_DTYPE)
    for r in range(rows):
        o = oracle.row_stats(l[r])
        assert st["argmax"][r] == o["argmax"]
        assert abs(st["ppl_entropy"][r] - o["ppl_entropy"]) <= 1e-12 * o["ppl_entropy"]
        assert abs(st["entropy"][r] - o["entropy"]) <= 1e-12
        assert abs(st["fault_tolerance"][r] - o["fault_tolerance"]) <= 1e-14


@pytest.mark.parametrize("dtype", [capi.DT_F32, capi.DT_BF16])
def test_kl_rows_vs_oracle(ctx, dtype):
    rng = np.random.default_rng(11)
    rows, V = 6, 32000
    lp = (rng.standard_normal((rows, V)) * 1.3).astype(np.float32)
    lq = lp + (rng.standard_normal((rows, V)) * 0.05).astype(np.float32)
    td = torch.float32 if dtype == capi.DT_F32 else torch.bfloat16
    tq, tp = torch.from_numpy(lq).cuda().to(td), torch.from_numpy(lp).cuda().to(td)
    kl = torch.zeros(rows, dtype=torch.float64, device="cuda")
    ent = torch.zeros(rows, dtype=torch.float64, device="cuda")
    ctx.kl_rows(tq, tp, dtype, rows, V, kl, ent)
    ctx.synchronize()
    qn, pn = tq.float().cpu().numpy(), tp.float().cpu().numpy()
    for r in range(rows):
        k, h = oracle.kl_logits(qn[r], pn[r])
        assert abs(kl[r].item() - k) <= 1e-4 and abs(ent[r].item() - h) <= 1e-4
        assert abs(kl[r].item() - k) <= 1e-3 * k + 1e-7


@pytest.mark.parametrize("bits", [8, 4])
def test_hist_kl_vs_oracle(ctx, bits):
    N, K = 128, 512
    w = _w(N, K, 123)
    L = capi.Layer(ctx, N, K, 0)
    L.upload_fp(w)
    p, s, z = oracle.quantize(w, 0, bits)
    L.upload_quantized(capi.RUNG_INT8 if bits == 8 else capi.RUNG_INT4, p, s, z)
    wq = oracle.dequantize(p, N, K, 0, bits, s, z)
    for bins in (512, 2048):
        got = L.hist_kl(capi.RUNG_INT8 if bits == 8 else capi.RUNG_INT4, bins)
        want = oracle.hist_kl(w, wq, bins)
        assert got == want


def test_fill_normal_matches_host_generator(ctx):
    n = 1 << 16
    d = torch.zeros(n, dtype=torch.float32, device="cuda")
    ctx.fill_normal(d, n, 1234, 5, 0.02)
    ctx.synchronize()
    h = oracle.normal(n, 1234, 5, 0.02)
    dd = d.cpu().numpy()
    same = dd.view(np.uint32) == h.view(np.uint32)
    assert same.mean() > 0.999  # libm vs CUDA double transcendentals may differ in the last ulp
    assert np.max(np.abs(dd - h)) <= 1e-8


@pytest.mark.parametrize("N,K,T", [(128, 128, 1), (256, 512, 64), (200, 1376, 130), (1024, 4096, 256),
                                   (4096, 11008, 300), (32000, 4096, 128)])
@pytest.mark.parametrize("bits", [8, 4])
def test_tcgen05_gemm_vs_oracle(ctx, N, K, T, bits):
    """Prefill / calibration contraction on tcgen05: exact integer codes (q - z) and bf16
    activations on the tensor cores, fp32 accumulation per quantization group in tensor memory,
    fp32 group scale in the epilogue -- the decode GEMV's precision contract, so within 1e-4
    (max-norm relative) of the reference dequant + double-accumulated linear."""
    w = _w(N, K, N + 7 * K)
    L, ref = _layer(ctx, w, 128, (bits,))
    x = np.random.default_rng(T + K).standard_normal((T, K)).astype(np.float32)
    xb = torch.from_numpy(x).cuda().to(torch.bfloat16).contiguous()
    y = torch.full((T, N), float("nan"), dtype=torch.float32, device="cuda")
    rung = capi.RUNG_INT8 if bits == 8 else capi.RUNG_INT4
    ctx.gemm(L, rung, T, xb, y)
    ctx.synchronize()
    p, s, z = ref[bits]
    yref = np.zeros((T, N), np.float32)
    oracle.lib().fqo_quant_linear(np.ascontiguousarray(xb.float().cpu().numpy()), T, p, N, K, 128, bits, 0, s.ravel(),
                                  z.ravel(), None, yref)
    got = y.cpu().numpy()
    assert np.all(np.isfinite(got))
    assert _rel(got, yref) < 1e-4, _rel(got, yref)
    big = np.abs(yref) > 1e-3 * np.max(np.abs(yref))
    assert np.all(np.abs(got - yref)[big] <= 1e-3 * np.abs(yref)[big])
