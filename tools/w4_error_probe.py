import numpy as np, torch, sys, os
sys.path.insert(0, '/root/repo')
import oracle
from paper_2506_12024_b200 import capi
ctx = capi.Context(0)
for (N, K) in [(256, 512), (128, 1376), (96, 4096), (64, 11008), (4096, 4096)]:
    for B in [1, 4]:
        w = oracle.normal(N * K, N * 31 + K, 1, 0.02).reshape(N, K)
        L = capi.Layer(ctx, N, K, 128)
        p, s, z = oracle.quantize(w, 128, 4, 0)
        L.upload_quantized(capi.RUNG_INT4, p, s, z, 0)
        x = np.random.default_rng(K + B).standard_normal((B, K)).astype(np.float32)
        xt = torch.from_numpy(x).to("cuda").half().contiguous()
        y = torch.empty((B, N), dtype=torch.float32, device="cuda")
        ctx.gemv(L, capi.RUNG_INT4, B, xt, capi.DT_F16, y, capi.DT_F32)
        ctx.synchronize()
        yref = np.zeros((B, N), np.float32)
        oracle.lib().fqo_quant_linear(np.ascontiguousarray(xt.float().cpu().numpy()), B, p, N, K, 128, 4, 0, s.ravel(), z.ravel(), None, yref)
        yy = y.cpu().numpy()
        mx = np.max(np.abs(yref))
        big = np.abs(yref) > 1e-3 * mx
        el = np.max(np.abs(yy - yref)[big] / np.abs(yref)[big])
        print(f"N={N} K={K} B={B}: maxnorm {np.max(np.abs(yy-yref))/mx:.2e}  worst elementwise(>1e-3max) {el:.2e}")
        L.close()
