import sys, os, torch
sys.path.insert(0, os.getcwd())
from paper_2506_12024_b200 import capi
ctx = capi.Context(0)
K, N = int(sys.argv[1]), int(sys.argv[2]); bits = int(sys.argv[3]); B = int(sys.argv[4])
w = torch.empty(N * K, dtype=torch.float32, device="cuda")
ctx.fill_normal(w, N * K, 0, 5, 0.02)
L = capi.Layer(ctx, N, K, 128)
rung = capi.RUNG_INT8 if bits == 8 else capi.RUNG_INT4
L.quantize_device(rung, w)
x = torch.randn(B, K, device="cuda").half(); y = torch.empty(B, N, device="cuda")
for _ in range(5): ctx.gemv(L, rung, B, x, capi.DT_F16, y, capi.DT_F32)
ctx.synchronize(); print("ok")
