"""The C++ host API (include/flexquant/*.hpp via the _flexquant module) — the drop-in surface for
the reference's hot path.  CPU-only parts run everywhere; device parts are marked gpu.

GPU cases drive the reference's own golden workload through the B200 engine: the reference
fixture model loaded from its weights container, the reference analyzer's plan, and
generate() reproducing proj/acceptance_out/det_t0.jsonl (tokens, PPLE, switch schedule).
"""
import json
import math
import os

import numpy as np
import pytest

import oracle

fq = pytest.importorskip("paper_2506_12024_b200._flexquant")
GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- CPU: quantizer, scheduler, plans
@pytest.mark.parametrize("key", ["64x512_g128", "16x1376_g128", "24x96_g0", "8x4096_g128"])
@pytest.mark.parametrize("bits", [8, 4])
def test_host_quantizer_matches_reference_golden(key, bits):
    g = np.load(os.path.join(GOLD, "quant_g128.npz"))
    w = g["w_" + key]
    group = int(key.split("_g")[1])
    q = fq.quantize(w, bits, fq.QuantMode.Asymmetric, group)
    assert np.array_equal(q.payload, g[f"p_{key}_b{bits}"])
    assert np.array_equal(q.scale.view(np.uint32), g[f"s_{key}_b{bits}"].ravel().view(np.uint32))
    assert np.array_equal(q.zero_point, g[f"z_{key}_b{bits}"].ravel())


def test_host_quantizer_kats():
    q = fq.quantize(np.array([[0.0, 1.0]], np.float32), 8)
    assert q.scale[0] == np.float32(1.0 / 255.0) and q.code_at(0, 0) == 0 and q.code_at(0, 1) == 255
    assert list(fq.pack_codes([1, 2, 3], 4)) == [0x21, 0x03]
    for c in (0.37, -2.75, -1e-3):
        back = fq.dequantize(fq.quantize(np.full((1, 4), c, np.float32), 4))
        assert np.all(back == np.float32(c))
    with pytest.raises(fq.ConfigError):
        fq.quantize(np.zeros((1, 4), np.float32), 3)
    q = fq.quantize(np.ones((2, 8), np.float32), 8)
    q.payload = q.payload[:-1]
    with pytest.raises(fq.FormatError):
        fq.dequantize(q)


def test_host_scheduler_matches_reference_state_machine():
    rng = np.random.default_rng(7)
    for _ in range(25):
        W = int(rng.integers(1, 9))
        thre = 2.0 + float(rng.integers(0, 5))
        plan = int(rng.integers(0, 8))
        lps = int(rng.integers(1, 4))
        ppl = 1.0 + rng.integers(0, 500, 200) / 100.0
        ff, fc, mv, vv = oracle.scheduler_replay(ppl, W, thre, lps, plan)
        cfg = fq.SchedulerConfig()
        cfg.window_len = W
        cfg.layers_per_switch = lps
        st = fq.SchedulerState(cfg, plan)
        st.set_threshold(thre)
        for i, v in enumerate(ppl):
            mean, first, count = st.observe(float(v))
            assert count == fc[i] and (count == 0 or first == ff[i])
            assert (mean is not None) == vv[i]
            if mean is not None:
                assert mean == mv[i]


def test_plan_text_round_trip_and_golden_parse():
    txt = open(os.path.join(GOLD, "det.fqp")).read()
    plan = fq.SwitchPlan.from_text(txt)
    assert plan.size() == 26
    assert plan.to_text() == txt
    r = [fq.LayerKlReport() for _ in range(3)]
    for rep, (lid, kl) in zip(r, [("b", 0.5), ("a", 0.5), ("c", 0.1)]):
        rep.layer_id, rep.kl, rep.bits = lid, kl, fq.Rung.Int8
    p = fq.build_switch_plan(r, fq.Rung.Fp, fq.Rung.Int8)
    assert [e.layer_id for e in p.entries] == ["c", "a", "b"]  # (kl, layer_id) order


def test_histogram_and_kl_match_reference_library():
    """The restated weight_histogram / kl_divergence (host/analyzer.cpp) equal the reference's
    (src/analyzer.cpp:31-79, oracle/_ref) bit for bit, including values exactly on bin edges."""
    if oracle.ref() is None:
        pytest.skip("reference library not built")
    rng = np.random.default_rng(3)
    for bins in (2, 7, 512, 2048):
        w = (rng.standard_normal((64, 96)) * 0.02).astype(np.float32)
        wq = np.round(w * 50).astype(np.float32) / 50  # a coarser copy with many ties
        e = fq.uniform_edges(float(w.min()), float(w.max()), bins)
        w.ravel()[:len(e)] = np.asarray(e, np.float32)[: w.size]  # values on (float-rounded) edges
        p = fq.weight_histogram(w, e)
        q = fq.weight_histogram(wq, fq.uniform_edges(float(w.min()), float(w.max()), bins))
        mine = fq.kl_divergence(p, q)
        assert mine == oracle.hist_kl(w, wq, bins, impl="ref")


def test_kl_and_histogram_host_utilities():
    assert abs(fq.kl_divergence([0.5, 0.5], [0.25, 0.75]) - 0.14384103622589045) < 1e-15
    e = fq.uniform_edges(0.0, 1.0, 4)
    assert e[0] == 0.0 and e[-1] == 1.0 and len(e) == 5


# ---------------------------------------------------------------- GPU: the golden workload
def _golden_model():
    return fq.load_model_file(os.path.join(GOLD, "micro_seed2.fqw"), 1)


@pytest.mark.gpu
def test_analyzer_reproduces_golden_plan():
    m = _golden_model()
    plan = fq.build_ladder_plan(m, [fq.Rung.Int8, fq.Rung.Int4], 512)
    want = fq.SwitchPlan.from_text(open(os.path.join(GOLD, "det.fqp")).read())
    assert [(e.layer_id, e.from_, e.to) for e in plan.entries] == [(e.layer_id, e.from_, e.to) for e in want.entries]
    for a, b in zip(plan.entries, want.entries):
        assert abs(a.kl - b.kl) <= 1e-12 * b.kl


@pytest.mark.gpu
def test_generate_reproduces_golden_trace():
    m = _golden_model()
    plan = fq.SwitchPlan.from_text(open(os.path.join(GOLD, "det.fqp")).read())
    prompt = np.frombuffer(open(os.path.join(GOLD, "p01.txt"), "rb").read(), np.uint8).astype(np.int32)
    cfg = fq.GenerationConfig()
    cfg.max_new_tokens = 96
    cfg.scheduler.theta = 1.02
    cfg.scheduler.threshold_mode = fq.ThresholdMode.Prefill
    r = fq.generate(prompt, m, plan, cfg)
    assert abs(r.threshold - 157.12635610416251) <= 1e-9 * 157.0
    got = [json.loads(l) for l in r.trace.to_jsonl().splitlines()]
    want = [json.loads(l) for l in open(os.path.join(GOLD, "det_t0.jsonl"))]
    assert len(got) == len(want) == 96
    for a, b in zip(got, want):
        for k in ("elapsed_ns", "buckets"):
            a.pop(k)
            b.pop(k)
        assert a["token_id"] == b["token_id"]
        assert a.get("switch_events") == b.get("switch_events")
        assert a["effective_bits"] == b["effective_bits"] and a["weight_bytes_touched"] == b["weight_bytes_touched"]
        assert math.isclose(a["ppl_entropy"], b["ppl_entropy"], rel_tol=1e-9)
        assert abs(a["fault_tolerance"] - b["fault_tolerance"]) <= 1e-12
        if b["moving_average"] is None:
            assert a["moving_average"] is None
        else:
            assert math.isclose(a["moving_average"], b["moving_average"], rel_tol=1e-9)


@pytest.mark.gpu
def test_generate_static_equals_disabled_scheduler():
    # proj/tests/test_engine.cpp:61-71: theta = 0 reproduces the static fp run
    m = _golden_model()
    plan = fq.SwitchPlan.from_text(open(os.path.join(GOLD, "det.fqp")).read())
    prompt = np.frombuffer(b"A small boat crossed the bay before sunrise and turned north.", np.uint8).astype(np.int32)
    cfg = fq.GenerationConfig()
    cfg.max_new_tokens = 48
    cfg.scheduler.theta = 0.0
    dyn = fq.generate(prompt, m, plan, cfg)
    stat = fq.generate_static(prompt, m, fq.Rung.Fp, cfg)
    assert list(dyn.sequence) == list(stat.sequence)
    assert all(r.effective_bits == 16.0 for r in stat.trace.records)


@pytest.mark.gpu
def test_infinite_threshold_cadence():
    # proj/tests/test_engine.cpp:73-97: absolute +inf -> one switch every window length
    m = _golden_model()
    plan = fq.SwitchPlan.from_text(open(os.path.join(GOLD, "det.fqp")).read())
    prompt = np.frombuffer(b"A small boat crossed the bay before sunrise and turned north.", np.uint8).astype(np.int32)
    cfg = fq.GenerationConfig()
    cfg.max_new_tokens = 600
    cfg.scheduler.threshold_mode = fq.ThresholdMode.Absolute
    cfg.scheduler.theta = float("inf")
    cfg.scheduler.window_len = 20
    r = fq.generate(prompt, m, plan, cfg)
    at = [rec.token_index for rec in r.trace.records if rec.switch_events]
    assert at == [20 * (i + 1) for i in range(26)]
    assert r.trace.records[-1].effective_bits == 4.0


@pytest.mark.gpu
def test_plan_validation_errors():
    m = _golden_model()
    bad = fq.SwitchPlan.from_text("flexquant-plan v1\nentry layer_id=head from=8 to=4 kl=1\n")
    cfg = fq.GenerationConfig()
    with pytest.raises(fq.ConfigError):
        fq.generate(np.array([1, 2, 3], np.int32), m, bad, cfg)
    cfg.start_rung = fq.Rung.Int4
    with pytest.raises(fq.ConfigError):
        fq.generate(np.array([1, 2, 3], np.int32), m, fq.SwitchPlan(), cfg)
    with pytest.raises(fq.InputError):
        fq.generate(np.array([], np.int32), m, fq.SwitchPlan(), fq.GenerationConfig())


def _llama(max_batch=3):
    c = fq.ModelConfig()
    c.arch = fq.Arch.Llama
    c.vocab_size, c.d_model, c.n_heads, c.head_dim = 8192, 512, 8, 64
    c.n_layers, c.ffn_dim, c.max_seq_len, c.group_size, c.max_batch = 4, 1376, 128, 128, max_batch
    m = fq.Model(c)
    m.init_random(0, 0.02)
    return m


@pytest.mark.gpu
def test_generate_batch_heterogeneous_matches_single():
    m = _llama()
    ids = m.linear_ids()
    plan = fq.SwitchPlan()
    entries = []
    for lid in ids:
        e = fq.SwitchEntry()
        e.layer_id, e.from_, e.to, e.kl = lid, fq.Rung.Int8, fq.Rung.Int4, 0.0
        entries.append(e)
    plan.entries = entries
    cfg = fq.GenerationConfig()
    cfg.max_new_tokens = 24
    cfg.start_rung = fq.Rung.Int8
    cfg.scheduler.threshold_mode = fq.ThresholdMode.Absolute
    cfg.scheduler.theta = float("inf")
    cfg.scheduler.window_len = 5
    cfg.scheduler.layers_per_switch = 4
    prompts = [list(oracle.random_tokens(12 + 3 * i, 8192, 40 + i)) for i in range(3)]
    batch = fq.generate_batch(prompts, m, plan, cfg)
    for i, p in enumerate(prompts):
        single = fq.generate(np.array(p, np.int32), m, plan, cfg)
        assert list(batch[i].sequence) == list(single.sequence)
        for a, b in zip(batch[i].trace.records, single.trace.records):
            assert abs(a.ppl_entropy - b.ppl_entropy) <= 1e-4 * b.ppl_entropy
            assert [e.layer_id for e in a.switch_events] == [e.layer_id for e in b.switch_events]


@pytest.mark.gpu
def test_weights_container_round_trip_reference_and_llama(tmp_path):
    """save_model_file / load_model_file (src/model_io.cpp:130-258): a reference-architecture
    model round-trips to the reference's own byte layout (the golden micro fixture is rewritten
    byte for byte), and a g128 llama model round-trips through the group-wise extension records
    with identical decode statistics."""
    src = os.path.join(GOLD, "micro_seed2.fqw")
    m = fq.load_model_file(src, 1)
    out = str(tmp_path / "micro.fqw")
    fq.save_model_file(m, out)
    assert open(out, "rb").read() == open(src, "rb").read()
    # llama, g128, random device init: save, load, decode the same tokens
    a = _llama(max_batch=1)
    a.set_all_precision(fq.Rung.Int8)
    for i, lid in enumerate(a.linear_ids()):
        if i % 3 == 0:
            a.set_precision(lid, fq.Rung.Int4)
    path = str(tmp_path / "llama.fqw")
    fq.save_model_file(a, path)
    b = fq.load_model_file(path, 1)
    for i, lid in enumerate(b.linear_ids()):
        b.set_precision(lid, a.precision(i))
    toks = oracle.random_tokens(10, 8192, 77)
    ra = a.prefill_rows(0, toks)
    rb = b.prefill_rows(0, toks)
    assert [r["argmax"] for r in ra] == [r["argmax"] for r in rb]
    assert all(x["ppl_entropy"] == y["ppl_entropy"] for x, y in zip(ra, rb))


@pytest.mark.gpu
def test_sweep_reproduces_golden_csv_rows():
    """Acceptance c9 (proj/tests/acceptance.cpp:410-434): the speed sweep of the tiny fixture
    (seed 1) under its 2048-bin ladder plan, 200 tokens, speeds 1 and 20, on prompt p01, writes
    the reference's golden CSV rows (tests/golden/sweep.csv) character for character."""
    m = fq.make_fixture_model(fq.tiny_config(), 1)
    plan = fq.build_ladder_plan(m, [fq.Rung.Int8, fq.Rung.Int4], 2048)
    prompt = np.frombuffer(open(os.path.join(GOLD, "p01.txt"), "rb").read(), np.uint8).astype(np.int32)
    cfg = fq.GenerationConfig()
    cfg.max_new_tokens = 200
    rows = fq.sweep_switch_speed(prompt, m, plan, [1, 20], cfg)
    got = fq.sweep_csv_header() + "".join(fq.sweep_csv_row("p01", r) for r in rows)
    want = "".join(open(os.path.join(GOLD, "sweep.csv")).readlines()[:3])
    assert got == want, (got, want)


@pytest.mark.gpu
def test_latency_breakdown_c11_analogue():
    """Acceptance c11 (proj/tests/acceptance.cpp:494-501): the trace's per-rung time buckets sum
    to the step time within 5% and the PPLE computation stays under 2% of it."""
    m = fq.make_fixture_model(fq.tiny_config(), 1)
    plan = fq.build_ladder_plan(m, [fq.Rung.Int8, fq.Rung.Int4], 2048)
    prompt = np.frombuffer(open(os.path.join(GOLD, "p01.txt"), "rb").read(), np.uint8).astype(np.int32)
    cfg = fq.GenerationConfig()
    cfg.max_new_tokens = 120
    cfg.scheduler.threshold_mode = fq.ThresholdMode.Absolute
    cfg.scheduler.theta = float("inf")
    r = fq.generate(prompt, m, plan, cfg)
    rep = fq.traffic_report_struct(r.trace)
    print(fq.traffic_report(r.trace))
    assert abs(rep.bucket_sum_over_total - 1.0) <= 0.05
    assert rep.ppl_share < 0.02


@pytest.mark.gpu
def test_latency_breakdown_device_timed_llama():
    """The c11 analogue with device-timed buckets on the llama engine: each decode step's linear
    time comes from the program's phase clock, split by precision (fq_model_decode_timed); the
    buckets still sum to the step time within 5% and the W4 bucket grows as layers switch."""
    m = _llama(max_batch=1)
    ids = m.linear_ids()
    plan = fq.SwitchPlan()
    ents = []
    for lid in ids:
        e = fq.SwitchEntry()
        e.layer_id, e.from_, e.to, e.kl = lid, fq.Rung.Int8, fq.Rung.Int4, 0.0
        ents.append(e)
    plan.entries = ents
    cfg = fq.GenerationConfig()
    cfg.max_new_tokens = 60
    cfg.start_rung = fq.Rung.Int8
    cfg.scheduler.threshold_mode = fq.ThresholdMode.Absolute
    cfg.scheduler.theta = float("inf")
    cfg.scheduler.window_len = 4
    cfg.scheduler.layers_per_switch = 4
    cfg.device_timed_buckets = True
    r = fq.generate(oracle.random_tokens(12, 8192, 3), m, plan, cfg)
    rep = fq.traffic_report_struct(r.trace)
    print(fq.traffic_report(r.trace))
    assert abs(rep.bucket_sum_over_total - 1.0) <= 0.05
    assert rep.ppl_share < 0.02
    late = r.trace.records[-1].buckets
    assert late.ns_int4 > 0 and late.ns_int8 == 0  # every linear switched to W4 by then
