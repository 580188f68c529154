// Batched decode on the tensor-core path (BASELINE config 5: many sequences per GPU, each with
// its own per-layer precision table).  One step = B rows, one new token per sequence slot:
// RMSNorm / RoPE + cache append / attention over each slot's own history / SwiGLU run here, row
// parallel; every linear runs on the tcgen05 GEMM (gemm_tc.cu) once per precision copy present
// in the batch, each launch writing only the rows at that copy (row_rung mask) -- so every
// resident copy streams from HBM at most once per step whatever the batch size (the grouped
// GEMV of the per-sequence set_precision state, /root/reference/proj/src/model.cpp:268-278,
// applied across a batch).  Precision contract as the decode step program.
#include "fq_internal.cuh"

namespace fqc {
namespace {

__device__ __forceinline__ float actr(float v, int f16) {
  return f16 ? __half2float(__float2half_rn(v)) : __bfloat162float(__float2bfloat16_rn(v));
}

// Row b at position pos[b] of slot slots[b]: q/k/v (fp32 GEMM sums, rounded to the activation
// dtype) -> RoPE'd, pre-scaled q (fp32) and the fp16 K / V cache entries of that position.
__global__ void rope_append_rows_kernel(const float* __restrict__ q, const float* __restrict__ k,
                                        const float* __restrict__ v, int H, int hd, const float2* __restrict__ cs,
                                        const int32_t* __restrict__ pos, const int32_t* __restrict__ slots,
                                        __half* __restrict__ kv, int64_t slot_stride, int64_t layer_off,
                                        int64_t max_seq, float* __restrict__ qr, int f16) {
  const int b = blockIdx.x, h = blockIdx.y;  // one block per (row, head): B x H blocks of hd / 2 threads
  const int d = H * hd, half = hd / 2;
  const int p = pos[b];
  const float scale = 1.0f / sqrtf(static_cast<float>(hd));
  __half* kvl = kv + static_cast<int64_t>(slots[b]) * slot_stride + layer_off;
  for (int i = threadIdx.x; i < half; i += blockDim.x) {
    const int64_t o0 = static_cast<int64_t>(b) * d + h * hd + i, o1 = o0 + half;
    const float2 c = cs[static_cast<int64_t>(p) * half + i];
    const float q0 = actr(q[o0], f16), q1 = actr(q[o1], f16);
    qr[o0] = (q0 * c.x - q1 * c.y) * scale;
    qr[o1] = (q1 * c.x + q0 * c.y) * scale;
    const float k0 = actr(k[o0], f16), k1 = actr(k[o1], f16);
    __half* kc = kvl + static_cast<int64_t>(h) * max_seq * hd + static_cast<int64_t>(p) * hd;
    __half* vc = kc + static_cast<int64_t>(H) * max_seq * hd;
    kc[i] = __float2half_rn(k0 * c.x - k1 * c.y);
    kc[i + half] = __float2half_rn(k1 * c.x + k0 * c.y);
    vc[i] = __float2half_rn(actr(v[o0], f16));
    vc[i + half] = __float2half_rn(actr(v[o1], f16));
  }
}

// Attention of row b, head h over keys 0..pos[b] of its slot, one warp per (row, head), 32 keys
// per round: lane j scores key j (its own 256-byte K row), the round's softmax statistics merge
// into the running (max, sum), then the lanes own DPL dimensions each for P.V.  Output: the
// activation-rounded fp16 GEMM operand in the tiled layout.
template <int DPL>
__global__ void attn_decode_rows_kernel(const float* __restrict__ qr, const __half* __restrict__ kv, int B, int H,
                                        const int32_t* __restrict__ pos, const int32_t* __restrict__ slots,
                                        int64_t slot_stride, int64_t layer_off, int64_t max_seq,
                                        uint16_t* __restrict__ out, int nkb, int f16, int slot0) {
  constexpr int hd = DPL * 32;
  __shared__ float qs[8][hd];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x * (blockDim.x >> 5) + wib;
  if (item >= B * H) return;
  const int b = item / H, h = item - b * H;
  const int d = H * hd;
  for (int e = lane; e < hd; e += 32) qs[wib][e] = qr[static_cast<int64_t>(b) * d + h * hd + e];
  __syncwarp();
  // pos / slots null: the rows of one prompt (row b at position b of slot slot0)
  const int64_t slot = slots ? slots[b] : slot0;
  const __half* kc = kv + slot * slot_stride + layer_off + static_cast<int64_t>(h) * max_seq * hd;
  const __half* vc = kc + static_cast<int64_t>(H) * max_seq * hd;
  const int n = (pos ? pos[b] : b) + 1;
  float m = -INFINITY, l = 0.f, o[DPL];
#pragma unroll
  for (int e = 0; e < DPL; ++e) o[e] = 0.f;
  for (int j0 = 0; j0 < n; j0 += 32) {
    const int j = j0 + lane;
    float s = -INFINITY;
    if (j < n) {
      const uint4* kr = reinterpret_cast<const uint4*>(kc + static_cast<int64_t>(j) * hd);
      // the lane's whole K row in flight at once (one memory latency per round, not hd / 32)
      uint4 kw[hd / 8];
#pragma unroll
      for (int c = 0; c < hd / 8; ++c) kw[c] = kr[c];
      float acc = 0.f;
#pragma unroll
      for (int c = 0; c < hd / 8; ++c) {
        const uint4 w = kw[c];
        const __half2* h2 = reinterpret_cast<const __half2*>(&w);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __half22float2(h2[e]);
          acc = fmaf(qs[wib][8 * c + 2 * e], f.x, acc);
          acc = fmaf(qs[wib][8 * c + 2 * e + 1], f.y, acc);
        }
      }
      s = acc;
    }
    float mx = s;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    const float mn = fmaxf(m, mx);
    const float p = j < n ? expf(s - mn) : 0.f;
    float ps = p;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, off);
    const float fa = m == -INFINITY ? 0.f : expf(m - mn);
    l = l * fa + ps;
#pragma unroll
    for (int e = 0; e < DPL; ++e) o[e] *= fa;
    // P.V: the lanes own DPL dimensions; the round's V rows load 16 at a time, all in flight
    // together (p_j of keys past the history is 0, their rows are not read)
    const int cnt = min(32, n - j0);
#pragma unroll
    for (int jb = 0; jb < 32; jb += 16) {
      if (jb >= cnt) break;
      float vv[16][DPL];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int jj = min(jb + u, cnt - 1);
        const __half* vr = vc + static_cast<int64_t>(j0 + jj) * hd + DPL * lane;
        if constexpr (DPL == 4) {
          const uint2 raw = *reinterpret_cast<const uint2*>(vr);
          const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&raw.x));
          const float2 c = __half22float2(*reinterpret_cast<const __half2*>(&raw.y));
          vv[u][0] = a.x; vv[u][1] = a.y; vv[u][2] = c.x; vv[u][3] = c.y;
        } else {
          const float2 a = __half22float2(*reinterpret_cast<const __half2*>(vr));
          vv[u][0] = a.x; vv[u][1] = a.y;
        }
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const float pj = __shfl_sync(0xffffffffu, p, jb + u);  // 0 for keys past the history
#pragma unroll
        for (int e = 0; e < DPL; ++e) o[e] = fmaf(pj, vv[u][e], o[e]);
      }
    }
    m = mn;
  }
#pragma unroll
  for (int e = 0; e < DPL; ++e) {
    const float r = actr(o[e] / l, f16);
    const __half hv = __float2half_rn(r);
    out[tiled_act_offset(b, h * hd + DPL * lane + e, nkb)] = *reinterpret_cast<const uint16_t*>(&hv);
  }
}

}  // namespace

void batched_rope_append(fq_ctx* ctx, const float* q, const float* k, const float* v, int B, int H, int hd,
                         const float2* cs, const int32_t* pos, const int32_t* slots, __half* kv, int64_t slot_stride,
                         int64_t layer_off, int64_t max_seq, float* qr, int act_dtype) {
  rope_append_rows_kernel<<<dim3(B, H), hd / 2, 0, ctx->stream>>>(q, k, v, H, hd, cs, pos, slots, kv, slot_stride, layer_off, max_seq,
                                                      qr, act_dtype == FQ_DT_F16 ? 1 : 0);
  FQ_CUDA(cudaGetLastError());
  ctx->launches += 1;
}

void batched_attention(fq_ctx* ctx, const float* qr, const __half* kv, int B, int H, int hd, const int32_t* pos,
                       const int32_t* slots, int64_t slot_stride, int64_t layer_off, int64_t max_seq, void* out16,
                       int act_dtype, int slot0) {
  const int items = B * H, per = 8;
  const int blocks = (items + per - 1) / per;
  const int nkb = ceil_div_i(static_cast<int64_t>(H) * hd, 128), f16 = act_dtype == FQ_DT_F16 ? 1 : 0;
  if (hd == 128)
    attn_decode_rows_kernel<4><<<blocks, per * 32, 0, ctx->stream>>>(qr, kv, B, H, pos, slots, slot_stride, layer_off,
                                                                     max_seq, static_cast<uint16_t*>(out16), nkb, f16,
                                                                     slot0);
  else if (hd == 64)
    attn_decode_rows_kernel<2><<<blocks, per * 32, 0, ctx->stream>>>(qr, kv, B, H, pos, slots, slot_stride, layer_off,
                                                                     max_seq, static_cast<uint16_t*>(out16), nkb, f16,
                                                                     slot0);
  else
    fail(FQ_E_CONFIG, "batched decode: head_dim must be 64 or 128");
  FQ_CUDA(cudaGetLastError());
  ctx->launches += 1;
}

}  // namespace fqc
