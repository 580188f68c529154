"""Regenerates tests/golden/ from the reference (run in the build container, where
/root/reference exists).  The GPU box only reads the committed outputs.

* det.fqp, det_t0.jsonl, sweep.csv: the reference's own acceptance artefacts
  (proj/acceptance_out, produced by proj/tests/acceptance.cpp c9/c12), copied verbatim.
* p01.txt: the prompt those artefacts were generated from (proj/data/corpus/p01.txt).
* quant_g128.npz: reference-quantizer outputs (oracle/_ref/libfqref.so, the unmodified
  reference compiled from source) on seeded N(0,0.02) matrices, g128 and per-row, W8/W4,
  including the ragged K=1376 case.
* micro_seed2.fqw: the reference fixture model (micro preset, seed 2) in the reference's
  flexquant-weights v1 container (the model behind det.fqp / det_t0.jsonl).
* ref_logits_micro.npz: teacher-forced reference logits of that model at each rung.
"""
import os
import shutil
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402

REF = "/root/reference/proj"


def main():
    for name in ("det.fqp", "det_t0.jsonl", "sweep.csv"):
        shutil.copy(os.path.join(REF, "acceptance_out", name), os.path.join(HERE, name))
    shutil.copy(os.path.join(REF, "data", "corpus", "p01.txt"), os.path.join(HERE, "p01.txt"))
    R = oracle.ref()
    assert R is not None, "build oracle/_ref first (make -C oracle)"
    out = {}
    for (n, k, g) in [(64, 512, 128), (16, 1376, 128), (24, 96, 0), (8, 4096, 128)]:
        w = oracle.normal(n * k, 1000 + k, 3, 0.02).reshape(n, k)
        out[f"w_{n}x{k}_g{g}"] = w
        for bits in (8, 4):
            p, s, z = oracle.quantize(w, g, bits, impl="ref")
            out[f"p_{n}x{k}_g{g}_b{bits}"] = p
            out[f"s_{n}x{k}_g{g}_b{bits}"] = s
            out[f"z_{n}x{k}_g{g}_b{bits}"] = z
    np.savez_compressed(os.path.join(HERE, "quant_g128.npz"), **out)
    fqw = os.path.join(HERE, "micro_seed2.fqw")
    assert R.ref_make_fixture(b"micro", 2, 0, fqw.encode()) == 0
    prompt = np.frombuffer(open(os.path.join(HERE, "p01.txt"), "rb").read(), np.uint8).astype(np.int32)
    logits = {}
    for rung in (0, 1, 2):
        l = np.zeros((prompt.size, 256), np.float32)
        assert R.ref_prefill_logits(fqw.encode(), prompt, prompt.size, rung, l) == 0
        logits[f"prefill_r{rung}"] = l
        d = np.zeros((40, 256), np.float32)
        assert R.ref_decode_logits(fqw.encode(), prompt[:40].copy(), 40, rung, d) == 0
        logits[f"decode_r{rung}"] = d
    np.savez_compressed(os.path.join(HERE, "ref_logits_micro.npz"), **logits)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
