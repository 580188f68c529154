import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import oracle, oracle.llama
from paper_2506_12024_b200 import capi, tp
cfg = dict(vocab_size=4096, d_model=256, n_heads=2, head_dim=128, n_layers=2, ffn_dim=768, max_seq_len=64)
orc = oracle.llama.LlamaOracle(dict(cfg, group_size=128), seed=0)
ctx = capi.Context(0)
full = capi.Model(ctx, arch=capi.ARCH_LLAMA, act_dtype=capi.DT_BF16, max_batch=1, group_size=128, **cfg)
orc.upload(full, capi)
quant = {lid: q for lid, _, q in orc.layers}
for size in (1, 2):
    ms = []
    for r in range(size):
        m = capi.Model(ctx, tp=(r, size), arch=capi.ARCH_LLAMA, act_dtype=capi.DT_BF16, max_batch=1, group_size=128, **cfg)
        tp.upload_shard(m, quant, {"tok_emb": orc.tok_emb}); ms.append(m)
    dec = tp.TpDecoder(ms, tp.LocalExchange(size))
    full.reset_slot(0)
    out = torch.zeros((1, cfg["vocab_size"]), dtype=torch.float32, device="cuda")
    for i, t in enumerate(oracle.random_tokens(5, cfg["vocab_size"], 7)):
        st = dec.step([0], [int(t)])
        got = dec.logits(1)[0]
        full.decode([0], [int(t)], out); ctx.synchronize()
        ref = out.cpu().numpy()[0]
        print(size, i, "rel vs single", float(np.max(np.abs(got-ref))/np.max(np.abs(ref))), "lens", [m.slot_length(0) for m in ms], full.slot_length(0), flush=True)
    for m in ms: m.close()
full.close(); ctx.close()
