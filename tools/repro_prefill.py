import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2506_12024_b200 import capi
import oracle
ctx = capi.Context(0)
m = capi.Model(ctx, arch=capi.ARCH_LLAMA, act_dtype=capi.DT_BF16, max_batch=3, group_size=128, vocab_size=8192, d_model=512, n_heads=8, head_dim=64, n_layers=4, ffn_dim=1376, max_seq_len=128)
m.init_random(0, 0.02)
for step, (slot, n) in enumerate([(0, 18), (1, 12), (2, 18)]):
    try:
        st = m.prefill(slot, oracle.random_tokens(n, 8192, 40 + slot))
        print("ok", slot, n, st["entropy"][-1], flush=True)
    except Exception as e:
        print("fail", slot, n, e, flush=True)
        break
