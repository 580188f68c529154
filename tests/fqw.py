"""Reader of the reference's `flexquant-weights v1` container (src/model_io.cpp:130-258) —
test helper used to load the golden fixture model (tests/golden/micro_seed2.fqw)."""
import struct

import numpy as np


def read_fqw(path):
    data = open(path, "rb").read()
    pos = 0

    def line():
        nonlocal pos
        e = data.index(b"\n", pos)
        s = data[pos:e].decode()
        pos = e + 1
        return s

    assert line() == "flexquant-weights v1"
    cfg = dict(kv.split("=") for kv in line().split())
    cfg = {k: int(v) for k, v in cfg.items()}
    count = int(line().split("=")[1])
    tensors, quant = {}, {}

    def u32():
        nonlocal pos
        v = struct.unpack_from("<I", data, pos)[0]
        pos += 4
        return v

    for _ in range(count):
        n = u32()
        name = data[pos:pos + n].decode()
        pos += n
        dtype = data[pos]
        pos += 1
        if dtype == 0:
            nd = u32()
            shape = [u32() for _ in range(nd)]
            numel = int(np.prod(shape))
            tensors[name] = np.frombuffer(data, np.float32, numel, pos).reshape(shape).copy()
            pos += 4 * numel
        else:
            bits, mode = data[pos], data[pos + 1]
            pos += 2
            rows, cols = u32(), u32()
            scale = np.frombuffer(data, np.float32, rows, pos).copy()
            pos += 4 * rows
            zp = np.frombuffer(data, np.int32, rows, pos).copy()
            pos += 4 * rows
            nb = (rows * cols * bits + 7) // 8
            payload = np.frombuffer(data, np.uint8, nb, pos).copy()
            pos += nb
            quant[name] = dict(bits=bits, mode=mode, rows=rows, cols=cols, scale=scale, zp=zp, payload=payload)
    return cfg, tensors, quant


def load_into_model(model, path, capi):
    """Uploads every tensor / rung of a reference container into an fq_model (reference arch)."""
    cfg, T, Q = read_fqw(path)
    model.set_param("tok_emb", T["tok_emb"])
    model.set_param("pos_emb", T["pos_emb"])
    for i in range(cfg["n_layers"]):
        p = f"blocks.{i}."
        for nm in ("ln1.gamma", "ln1.beta", "ln2.gamma", "ln2.beta"):
            model.set_param(p + nm, T[p + nm])
    model.set_param("final_norm.gamma", T["ln_f.gamma"])
    model.set_param("final_norm.beta", T["ln_f.beta"])
    for idx, lid in enumerate(model.ids):
        L = model.linear(idx)
        L.upload_fp(T[lid])
        L.upload_bias(T[lid + ".bias"])
        for tag, rung in ((".w8", capi.RUNG_INT8), (".w4", capi.RUNG_INT4)):
            q = Q[lid + tag]
            L.upload_quantized(rung, q["payload"], q["scale"], q["zp"], q["mode"])
    return cfg
