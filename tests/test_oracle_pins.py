"""Pins the CPU oracle restatement against the reference itself and its known answers.

These tests run without a GPU.  They compare oracle/fq_oracle.c with the reference library
compiled from /root/reference/proj/src (oracle/_ref/libfqref.so) and with the known-answer
tests of the reference suite (proj/tests/*.cpp), and check the committed golden fixtures.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")
needs_ref = pytest.mark.skipif(oracle.ref() is None, reason="oracle/_ref not built (reference sources absent)")


def _rand(shape, seed, std=0.02):
    return oracle.normal(int(np.prod(shape)), seed, 7, std).reshape(shape)


# ------------------------------------------------------------ quantizer known answers
def test_kat_asym_endpoints():
    # proj/tests/test_quantizer.cpp:67-74
    p, s, z = oracle.quantize(np.array([[0.0, 1.0]], np.float32), 0, 8)
    assert s[0, 0] == np.float32(1.0 / 255.0)
    assert z[0, 0] == 0 and p[0] == 0 and p[1] == 255


def test_kat_constant_rows_exact():
    # proj/tests/test_quantizer.cpp:76-90
    for c, bits in [(5.0, 8), (0.37, 4), (-2.75, 4), (-1e-3, 4), (0.0, 8)]:
        w = np.full((1, 4), c, np.float32)
        p, s, z = oracle.quantize(w, 0, bits)
        back = oracle.dequantize(p, 1, 4, 0, bits, s, z)
        assert np.all(back == np.float32(c))


def test_kat_symmetric_endpoints():
    # proj/tests/test_quantizer.cpp:109-121: codes 0/127/254 stored with the +127 offset
    p, s, z = oracle.quantize(np.array([[-1.0, 0.0, 1.0]], np.float32), 0, 8, mode=1)
    assert list(p) == [0, 127, 254] and z[0, 0] == 0


def test_kat_nibble_order():
    # proj/tests/test_quantizer.cpp:251-258
    codes = np.array([1, 2, 3], np.uint32)
    out = np.zeros(2, np.uint8)
    oracle.lib().fqo_pack(codes, 3, 4, out)
    assert list(out) == [0x21, 0x03]
    back = np.zeros(3, np.uint32)
    oracle.lib().fqo_unpack(out, 3, 4, back)
    assert list(back) == [1, 2, 3]


def test_kat_payload_length():
    # proj/tests/test_quantizer.cpp:292-300
    w = _rand((3, 3), 1)
    assert oracle.quantize(w, 0, 4)[0].size == 5
    assert oracle.quantize(w, 0, 8)[0].size == 9


def test_round_trip_bound():
    # acceptance c1 (proj/tests/acceptance.cpp:71-105): |x - x_hat| <= s/2 + eps
    w = _rand((64, 256), 3, 1.0)
    for bits in (8, 4):
        p, s, z = oracle.quantize(w, 128, bits)
        back = oracle.dequantize(p, 64, 256, 128, bits, s, z)
        bound = np.repeat(s, 128, axis=1) / 2 + 1e-6
        assert np.all(np.abs(w - back) <= bound)


@needs_ref
@pytest.mark.parametrize("shape,group", [((64, 512), 128), ((8, 1376), 128), ((16, 96), 0), ((5, 7), 0),
                                         ((32, 4096), 128), ((3, 33), 0)])
@pytest.mark.parametrize("bits", [8, 4])
@pytest.mark.parametrize("mode", [0, 1])
def test_quantize_bit_exact_vs_reference(shape, group, bits, mode):
    w = _rand(shape, 11 + shape[1], 0.02)
    w[0, :3] = [0.5, 0.5, 0.5]  # a near-constant prefix
    if shape[1] % 2 and bits == 4 and group == 0:
        pass  # odd row length: nibbles straddle rows, still the reference layout
    a = oracle.quantize(w, group, bits, mode)
    b = oracle.quantize(w, group, bits, mode, impl="ref")
    assert np.array_equal(a[0], b[0])
    assert np.array_equal(a[1].view(np.uint32), b[1].view(np.uint32))
    assert np.array_equal(a[2], b[2])


@needs_ref
def test_quantize_constant_groups_vs_reference():
    w = np.zeros((4, 256), np.float32)
    w[1, :128] = 0.25
    w[2, 128:] = -0.125
    w[3] = _rand((256,), 5)
    for bits in (8, 4):
        for mode in (0, 1):
            a = oracle.quantize(w, 128, bits, mode)
            b = oracle.quantize(w, 128, bits, mode, impl="ref")
            assert all(np.array_equal(x, y) for x, y in zip(a, b))


@needs_ref
def test_dequant_linear_vs_reference():
    w = _rand((48, 384), 21)
    x = _rand((3, 384), 22, 1.0)
    R = oracle.ref()
    for bits in (8, 4):
        p, s, z = oracle.quantize(w, 128, bits)
        wd = oracle.dequantize(p, 48, 384, 128, bits, s, z)
        wr = np.zeros(48 * 384, np.float32)
        assert R.ref_dequantize(p, 48, 384, 128, bits, 0, s.ravel(), z.ravel(), wr) == 0
        assert np.array_equal(wd.ravel().view(np.uint32), wr.view(np.uint32))
        y = oracle.linear(x, wd)
        yr = np.zeros((3, 48), np.float32)
        assert R.ref_linear(x, 3, 384, wd, 48, None, yr) == 0
        assert np.array_equal(y.view(np.uint32), yr.view(np.uint32))


# ------------------------------------------------------------ scheduler statistics
def _logits_from_probs(p):
    return np.log(np.asarray(p, np.float64)).astype(np.float32)


def test_kat_ppl_entropy():
    # proj/tests/test_scheduler.cpp:49-55
    st = oracle.row_stats(_logits_from_probs([0.7, 0.2, 0.1]))
    assert abs(st["ppl_entropy"] - 2.2295918739204163) <= 2.2295918739204163 * 1e-7
    # :108-111
    assert abs(st["fault_tolerance"] - 0.5) <= 1e-7


def test_ppl_uniform_and_onehot():
    # proj/tests/test_scheduler.cpp:36-47
    for v in (2, 50, 256, 32000):
        assert abs(oracle.row_stats(np.zeros(v, np.float32))["ppl_entropy"] - v) <= 1e-9 * v
    l = np.zeros(8, np.float32)
    l[3] = 1000.0
    st = oracle.row_stats(l)
    assert abs(st["ppl_entropy"] - 1.0) <= 1e-6 and st["argmax"] == 3


def test_argmax_lowest_index_on_ties():
    l = np.array([0.0, 2.0, 1.0, 2.0], np.float32)
    assert oracle.row_stats(l)["argmax"] == 1


@needs_ref
def test_row_stats_vs_reference():
    R = oracle.ref()
    import ctypes as C
    rng = np.random.default_rng(5)
    for V in (2, 17, 256, 8192, 32000):
        for _ in range(3):
            l = (rng.standard_normal(V) * rng.uniform(0.1, 5)).astype(np.float32)
            st = oracle.row_stats(l)
            ppl, ft, am = C.c_double(), C.c_double(), C.c_int32()
            assert R.ref_row_stats(l, V, C.byref(ppl), C.byref(ft), C.byref(am)) == 0
            assert st["ppl_entropy"] == ppl.value  # same arithmetic, same order
            assert st["fault_tolerance"] == ft.value
            assert st["argmax"] == am.value


@needs_ref
def test_derive_threshold_vs_reference():
    import ctypes as C
    rng = np.random.default_rng(9)
    l = rng.standard_normal((33, 300)).astype(np.float32)
    for W in (1, 5, 20, 40):
        a, b = C.c_double(), C.c_double()
        assert oracle.lib().fqo_derive_threshold(l, 33, 300, W, 1.02, C.byref(a)) == 0
        assert oracle.ref().ref_derive_threshold(l, 33, 300, W, 1.02, C.byref(b)) == 0
        assert a.value == b.value


def test_kat_derive_threshold():
    # proj/tests/test_scheduler.cpp:146-157
    import ctypes as C
    l = np.zeros((2, 4), np.float32)
    l[1, 2] = l[1, 3] = -10000.0
    out = C.c_double()
    oracle.lib().fqo_derive_threshold(l, 2, 4, 20, 1.0, C.byref(out))
    assert abs(out.value - 3.0) <= 3e-6
    l = np.zeros((3, 4), np.float32)
    l[0, 0] = 500.0
    oracle.lib().fqo_derive_threshold(l, 3, 4, 2, 1.0, C.byref(out))
    assert abs(out.value - 4.0) <= 4e-6


@needs_ref
def test_scheduler_replay_vs_reference():
    rng = np.random.default_rng(101)
    for _ in range(40):
        W = int(rng.integers(1, 9))
        thre = 2.0 + float(rng.integers(0, 5))
        plan = int(rng.integers(0, 8))
        lps = int(rng.integers(1, 4))
        ppl = 1.0 + rng.integers(0, 500, 300) / 100.0
        a = oracle.scheduler_replay(ppl, W, thre, lps, plan)
        b = oracle.scheduler_replay(ppl, W, thre, lps, plan, impl="ref")
        for x, y in zip(a, b):
            assert np.array_equal(x, y)


def test_scheduler_kats():
    # proj/tests/test_scheduler.cpp:194-291
    ff, fc, mv, vv = oracle.scheduler_replay(np.full(20, 5.0 - 1e-6), 20, 5.0, 1, 10)
    assert fc[:19].sum() == 0 and fc[19] == 1 and not vv[:19].any() and vv[19]
    ff, fc, _, _ = oracle.scheduler_replay(np.full(50, 3.0), 5, 3.0, 1, 10)
    assert fc.sum() == 0  # strict <
    ff, fc, _, _ = oracle.scheduler_replay(np.ones(40), 20, 10.0, 1, 10)
    assert list(np.nonzero(fc)[0]) == [19, 39]
    ff, fc, _, _ = oracle.scheduler_replay(np.ones(12), 3, 100.0, 4, 10)
    assert list(fc[[2, 5, 8, 11]]) == [4, 4, 2, 0]


# ------------------------------------------------------------ analyzer
def test_kat_kl_divergence():
    # proj/tests/test_analyzer.cpp:125-130: KL([.5,.5] || [.25,.75]) = 0.14384
    p = np.array([0.5, 0.5])
    q = np.array([0.25, 0.75])
    kl = float(np.sum(p * np.log(p / q)))
    assert abs(kl - 0.14384103622589045) < 1e-12
    if oracle.ref() is not None:
        import ctypes as C
        out = C.c_double()
        assert oracle.ref().ref_kl_divergence(p, q, 2, C.byref(out)) == 0
        assert out.value == kl


@needs_ref
@pytest.mark.parametrize("bits", [8, 4])
def test_hist_kl_vs_reference(bits):
    w = _rand((96, 256), 31)
    p, s, z = oracle.quantize(w, 0, bits)
    wq = oracle.dequantize(p, 96, 256, 0, bits, s, z)
    for bins in (64, 512, 2048):
        assert oracle.hist_kl(w, wq, bins) == oracle.hist_kl(w, wq, bins, impl="ref")


def test_grid_exact_kl_is_tiny():
    # proj/tests/test_analyzer.cpp:161-165 analogue: a weight already on the grid
    w = _rand((16, 128), 41)
    p, s, z = oracle.quantize(w, 0, 8)
    wg = oracle.dequantize(p, 16, 128, 0, 8, s, z)
    p2, s2, z2 = oracle.quantize(wg, 0, 8)
    wq = oracle.dequantize(p2, 16, 128, 0, 8, s2, z2)
    assert oracle.hist_kl(wg, wq, 512) <= 1e-9


# ------------------------------------------------------------ generators
def test_random_tokens_match_reference_stream():
    # random_tokens (src/fixture.cpp:133-138) = mt19937_64() % V; first outputs of
    # mt19937_64(5489) are a published constant (C++ [rand.predef]: 10000th = 9981545732273789042)
    t = oracle.random_tokens(10000, 1 << 62, 5489)
    assert t.size == 10000  # stream length
    out = np.zeros(1, np.int32)
    import ctypes as C
    L = oracle.lib()
    L.fqo_mt64_size.restype = C.c_size_t
    buf = (C.c_uint8 * L.fqo_mt64_size())()
    L.fqo_mt64_seed.argtypes = [C.c_void_p, C.c_uint64]
    L.fqo_mt64_next.argtypes = [C.c_void_p]
    L.fqo_mt64_next.restype = C.c_uint64
    L.fqo_mt64_seed(buf, 5489)
    v = 0
    for _ in range(10000):
        v = L.fqo_mt64_next(buf)
    assert v == 9981545732273789042


def test_normal_generator_moments():
    x = oracle.normal(1 << 20, 0, 1, 0.02).astype(np.float64)
    assert abs(x.mean()) < 1e-4 and abs(x.std() - 0.02) < 1e-4


# ------------------------------------------------------------ golden artefacts
@needs_ref
def test_golden_plan_and_trace_reproduced_by_reference(tmp_path):
    """Reference build regenerates det.fqp byte-for-byte and det_t0.jsonl minus timing."""
    R = oracle.ref()
    model = str(tmp_path / "det.fqw").encode()
    plan = str(tmp_path / "det.fqp").encode()
    trace = str(tmp_path / "det_t0.jsonl").encode()
    assert R.ref_make_fixture(b"micro", 2, 0, model) == 0
    assert R.ref_analyze(model, 512, plan) == 0
    with open(plan, "rb") as f, open(os.path.join(GOLD, "det.fqp"), "rb") as g:
        assert f.read() == g.read()
    prompt = np.frombuffer(open(os.path.join(GOLD, "p01.txt"), "rb").read(), np.uint8).astype(np.int32)
    import ctypes as C
    toks = np.zeros(96, np.int32)
    cnt, thre = C.c_int64(), C.c_double()
    assert R.ref_generate(model, plan, prompt, prompt.size, 96, 1.02, 0, 20, 1, 0, trace, toks, C.byref(cnt),
                          C.byref(thre)) == 0
    assert abs(thre.value - 157.12635610416251) < 1e-9
    got = [json.loads(x) for x in open(trace)]
    want = [json.loads(x) for x in open(os.path.join(GOLD, "det_t0.jsonl"))]
    assert len(got) == len(want) == 96
    for a, b in zip(got, want):
        for k in ("elapsed_ns", "buckets"):
            a.pop(k)
            b.pop(k)
        assert a == b
