// Row-parallel kernels of the tensor-core prefill (llama arch): the T prompt rows of one sequence
// go through each layer at once, the seven linears of a block and the head on the tcgen05 GEMM
// (gemm_tc.cu), everything else here.  Precision contract as in the decode program:
// fp32 residual, bf16-rounded activations (normalised inputs, q/k/v, attention output, SwiGLU
// product), RoPE from the model's cos/sin table, fp16 K/V cache, fp32 softmax.
#include "fq_internal.cuh"

namespace fqc {
namespace {

// rounding to the activation dtype (bf16, or fp16 when f16), as the decode program's round_act
__device__ __forceinline__ float actr(float v, int f16) {
  return f16 ? __half2float(__float2half_rn(v)) : __bfloat162float(__float2bfloat16_rn(v));
}
// GEMM operand: the activation rounded to the activation dtype (the contract), stored as fp16 in
// the tiled layout (tiled_act_offset): exact for bf16 values in fp16's normal range; a value past
// 65504 would not be, so it raises the overflow flag the host checks after the prefill.
__device__ unsigned int g_act_overflow;
__device__ __forceinline__ uint16_t actb(float v, int f16) {
  const float r = actr(v, f16);
  if (fabsf(r) > 65504.f) atomicOr(&g_act_overflow, 1u);
  const __half h = __float2half_rn(r);
  return *reinterpret_cast<const uint16_t*>(&h);
}

__global__ void embed_rows_kernel(const float* __restrict__ tok_emb, const int32_t* __restrict__ tokens, int64_t d,
                                  float* __restrict__ x) {
  const int t = blockIdx.x;
  const float* e = tok_emb + static_cast<int64_t>(tokens[t]) * d;
  for (int64_t i = threadIdx.x; i < d; i += blockDim.x) x[t * d + i] = e[i];
}

// h[t] = bf16(x[t] * rsqrt(mean(x[t]^2) + eps) * g)
__global__ void rmsnorm_rows_kernel(const float* __restrict__ x, int64_t d, const float* __restrict__ g, float eps,
                                    uint16_t* __restrict__ h, int nkb, int f16) {
  // one row per block; d % 4 == 0 (the caller checks): float4 loads, 4 consecutive k -> one 8-byte
  // store in the tiled layout (k & 7 groups of 8 are contiguous)
  const int t = blockIdx.x;
  const float4* xr = reinterpret_cast<const float4*>(x + t * d);
  const int64_t d4 = d / 4;
  float s = 0.f;
  for (int64_t i = threadIdx.x; i < d4; i += blockDim.x) {
    const float4 v = xr[i];
    s += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  __shared__ float red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float rstd = 1.0f / sqrtf(red[0] / static_cast<float>(d) + eps);
  const float4* g4 = reinterpret_cast<const float4*>(g);
  for (int64_t i = threadIdx.x; i < d4; i += blockDim.x) {
    const float4 v = xr[i], w = g4[i];
    const uint32_t lo = actb(v.x * rstd * w.x, f16) | (static_cast<uint32_t>(actb(v.y * rstd * w.y, f16)) << 16);
    const uint32_t hi = actb(v.z * rstd * w.z, f16) | (static_cast<uint32_t>(actb(v.w * rstd * w.w, f16)) << 16);
    *reinterpret_cast<uint2*>(h + tiled_act_offset(t, 4 * i, nkb)) = make_uint2(lo, hi);
  }
}

// q/k/v rows (fp32 GEMM outputs, rounded to bf16 as the decode step stores them) -> RoPE'd and
// pre-scaled q (fp32) and the fp16 K / V cache rows 0..T-1 of the slot.
__global__ void rope_kv_rows_kernel(const float* __restrict__ q, const float* __restrict__ k, const float* __restrict__ v,
                                    int H, int hd, const float2* __restrict__ cs, float* __restrict__ qr,
                                    __half* __restrict__ kv_layer, int64_t max_seq, int f16) {
  const int t = blockIdx.x;
  const int d = H * hd, half = hd / 2;
  const float scale = 1.0f / sqrtf(static_cast<float>(hd));
  for (int idx = threadIdx.x; idx < H * half; idx += blockDim.x) {
    const int h = idx / half, i = idx - h * half;
    const int64_t o0 = static_cast<int64_t>(t) * d + h * hd + i, o1 = o0 + half;
    const float2 c = cs[static_cast<int64_t>(t) * half + i];
    const float q0 = actr(q[o0], f16), q1 = actr(q[o1], f16);
    qr[o0] = (q0 * c.x - q1 * c.y) * scale;
    qr[o1] = (q1 * c.x + q0 * c.y) * scale;
    const float k0 = actr(k[o0], f16), k1 = actr(k[o1], f16);
    __half* kc = kv_layer + static_cast<int64_t>(h) * max_seq * hd + static_cast<int64_t>(t) * hd;
    __half* vc = kc + static_cast<int64_t>(H) * max_seq * hd;
    kc[i] = __float2half_rn(k0 * c.x - k1 * c.y);
    kc[i + half] = __float2half_rn(k1 * c.x + k0 * c.y);
    vc[i] = __float2half_rn(actr(v[o0], f16));
    vc[i + half] = __float2half_rn(actr(v[o1], f16));
  }
}

__global__ void swiglu_rows_kernel(const float* __restrict__ g, const float* __restrict__ u, int64_t n, int64_t f,
                                   uint16_t* __restrict__ out, int nkb, int f16) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float gv = g[i];  // unrounded GEMM sums, as the decode step's SwiGLU epilogue reads them
    const float silu = gv / (1.0f + expf(-gv));
    const int64_t t = i / f;
    out[tiled_act_offset(static_cast<int>(t), i - t * f, nkb)] = actb(silu * u[i], f16);
  }
}

int elem_grid(const fq_ctx* ctx, int64_t n) { return static_cast<int>(std::min<int64_t>(ctx->num_sms * 8, (n + 255) / 256)); }

}  // namespace

bool prefill_overflow_take(fq_ctx* ctx) {
  unsigned int h = 0;
  FQ_CUDA(cudaMemcpyFromSymbolAsync(&h, g_act_overflow, sizeof(h), 0, cudaMemcpyDeviceToHost, ctx->stream));
  FQ_CUDA(cudaStreamSynchronize(ctx->stream));
  if (h) {
    const unsigned int zero = 0;
    FQ_CUDA(cudaMemcpyToSymbolAsync(g_act_overflow, &zero, sizeof(zero), 0, cudaMemcpyHostToDevice, ctx->stream));
  }
  return h != 0;
}

void prefill_embed(fq_ctx* ctx, const float* tok_emb, const int32_t* tokens_dev, int T, int64_t d, float* x) {
  embed_rows_kernel<<<T, 256, 0, ctx->stream>>>(tok_emb, tokens_dev, d, x);
  FQ_CUDA(cudaGetLastError());
  ctx->launches += 1;
}

void prefill_rmsnorm(fq_ctx* ctx, const float* x, int T, int64_t d, const float* g, float eps, void* h16, int act_dtype) {
  if (d % 4 != 0 || (reinterpret_cast<uintptr_t>(g) & 15) != 0) fail(FQ_E_DIMENSION, "rmsnorm rows: d must be a multiple of 4");
  rmsnorm_rows_kernel<<<T, 256, 0, ctx->stream>>>(x, d, g, eps, static_cast<uint16_t*>(h16), ceil_div_i(d, 128),
                                                  act_dtype == FQ_DT_F16 ? 1 : 0);
  FQ_CUDA(cudaGetLastError());
  ctx->launches += 1;
}

void prefill_rope_kv(fq_ctx* ctx, const float* q, const float* k, const float* v, int T, int H, int hd,
                     const float2* cs, float* qr, __half* kv_layer, int64_t max_seq, int act_dtype) {
  rope_kv_rows_kernel<<<T, 256, 0, ctx->stream>>>(q, k, v, H, hd, cs, qr, kv_layer, max_seq, act_dtype == FQ_DT_F16 ? 1 : 0);
  FQ_CUDA(cudaGetLastError());
  ctx->launches += 1;
}

void prefill_swiglu(fq_ctx* ctx, const float* g, const float* u, int64_t n, int64_t f, void* out16, int act_dtype) {
  swiglu_rows_kernel<<<elem_grid(ctx, n), 256, 0, ctx->stream>>>(g, u, n, f, static_cast<uint16_t*>(out16),
                                                                 ceil_div_i(f, 128), act_dtype == FQ_DT_F16 ? 1 : 0);
  FQ_CUDA(cudaGetLastError());
  ctx->launches += 1;
}

}  // namespace fqc
