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

// Causal attention of the T rows of one prompt (row r at position r of slot slot0) on the tensor
// cores: one CTA = 64 query rows (4 warps x 16) of one head; 64-key tiles of K and V go through
// shared memory (two buffers, rows padded to 272 B: conflict-free fragment loads);
// S = Q K^T and O += P V run as mma.sync m16n8k16 (fp16 in, fp32 accumulate) with online
// softmax in the accumulator registers (the S accumulator layout is P's A-fragment layout).  The
// tiles are filled with plain 16-byte loads and stores (a cp.async version returned rows that
// differed between repeats of the same prompt; the plain fill costs < 2 % of the prefill).
// Precision: K and V are exact fp16 (the cache format); q (fp32, RoPE'd, pre-scaled) and P (fp32)
// are split into fp16 hi + lo parts and both products issued, so S and P.V carry ~22 significant
// bits -- the fp32 contract of the row kernel within its own rounding.
namespace fa {
constexpr int kRows = 64, kKeys = 64, kWarps = 4;

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// (x, y) -> fp16x2 hi and the fp16x2 of the remainders
__device__ __forceinline__ void split2(float x, float y, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(x, y);
  const float2 hf = __half22float2(h);
  const __half2 l = __floats2half2_rn(x - hf.x, y - hf.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}
}  // namespace fa

template <int HD>
__global__ void __launch_bounds__(fa::kWarps * 32)
    attn_prompt_tc_kernel(const float* __restrict__ qr, const __half* __restrict__ kv, int T, int H,
                          int64_t slot_stride, int64_t layer_off, int64_t max_seq, uint16_t* __restrict__ out, int nkb,
                          int f16, int slot0) {
  using namespace fa;
  constexpr int KC = HD / 16;      // 16-dim chunks
  constexpr int LD = HD + 8;       // padded smem row (halves): 272 B at HD = 128
  constexpr int NT = kKeys / 8;    // 8-key tiles of S
  constexpr int DT = HD / 8;       // 8-dim tiles of O
  extern __shared__ __align__(16) __half fsm[];
  __half* ks = fsm;                       // [2][kKeys][LD]
  __half* vs = fsm + 2 * kKeys * LD;      // [2][kKeys][LD]
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int h = blockIdx.y;
  const int r0 = blockIdx.x * kRows, wr = r0 + 16 * w;  // the warp's first row
  const int d = H * HD;
  const __half* kc = kv + static_cast<int64_t>(slot0) * slot_stride + layer_off + static_cast<int64_t>(h) * max_seq * HD;
  const __half* vc = kc + static_cast<int64_t>(H) * max_seq * HD;
  const int last_row = min(r0 + kRows, T) - 1;
  const int n_tiles = last_row / kKeys + 1;
  auto load_tile = [&](int tile, int buf) {
    const int k0 = tile * kKeys;
    constexpr int chunks = kKeys * HD / 8;  // 16-byte chunks per matrix
    for (int c = threadIdx.x; c < chunks; c += blockDim.x) {
      const int row = c / (HD / 8), col = (c % (HD / 8)) * 8;
      const int key = min(k0 + row, T - 1);  // rows past the prompt: any valid row (masked)
      *reinterpret_cast<uint4*>(ks + (buf * kKeys + row) * LD + col) = *reinterpret_cast<const uint4*>(kc + static_cast<int64_t>(key) * HD + col);
      *reinterpret_cast<uint4*>(vs + (buf * kKeys + row) * LD + col) = *reinterpret_cast<const uint4*>(vc + static_cast<int64_t>(key) * HD + col);
    }
  };
  load_tile(0, 0);
  // q A-fragments, hi and lo (rows past T read row T-1: their outputs are not written)
  uint32_t qh[KC][4], ql[KC][4];
  {
    const int ra = min(wr + g, T - 1), rb = min(wr + g + 8, T - 1);
    const float* qa = qr + static_cast<int64_t>(ra) * d + h * HD;
    const float* qb = qr + static_cast<int64_t>(rb) * d + h * HD;
#pragma unroll
    for (int c = 0; c < KC; ++c) {
      const float2 x0 = *reinterpret_cast<const float2*>(qa + 16 * c + 2 * t);
      const float2 x1 = *reinterpret_cast<const float2*>(qb + 16 * c + 2 * t);
      const float2 x2 = *reinterpret_cast<const float2*>(qa + 16 * c + 2 * t + 8);
      const float2 x3 = *reinterpret_cast<const float2*>(qb + 16 * c + 2 * t + 8);
      split2(x0.x, x0.y, qh[c][0], ql[c][0]);
      split2(x1.x, x1.y, qh[c][1], ql[c][1]);
      split2(x2.x, x2.y, qh[c][2], ql[c][2]);
      split2(x3.x, x3.y, qh[c][3], ql[c][3]);
    }
  }
  float o[DT][4];
#pragma unroll
  for (int j = 0; j < DT; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;  // rows wr+g, wr+g+8
  const int row_a = wr + g, row_b = wr + g + 8;
  for (int tile = 0; tile < n_tiles; ++tile) {
    const int buf = tile & 1;
    __syncthreads();  // tile `tile` is in buf
    if (tile + 1 < n_tiles) load_tile(tile + 1, buf ^ 1);  // the other buffer, released at the end of tile - 1
    const int k0 = tile * kKeys;
    if (k0 <= wr + 15) {  // some key of the tile is visible to some row of the warp
      const __half* kt = ks + buf * kKeys * LD;
      const __half* vt = vs + buf * kKeys * LD;
      float sc[NT][4];
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        sc[j][0] = sc[j][1] = sc[j][2] = sc[j][3] = 0.f;
        const __half* kr = kt + (8 * j + g) * LD + 2 * t;
#pragma unroll
        for (int c = 0; c < KC; ++c) {
          const uint32_t b0 = *reinterpret_cast<const uint32_t*>(kr + 16 * c);
          const uint32_t b1 = *reinterpret_cast<const uint32_t*>(kr + 16 * c + 8);
          mma16816(sc[j], qh[c], b0, b1);
          mma16816(sc[j], ql[c], b0, b1);
        }
      }
      // causal mask + tile max per row
      float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const int key = k0 + 8 * j + 2 * t;
        if (key > row_a) sc[j][0] = -INFINITY;
        if (key + 1 > row_a) sc[j][1] = -INFINITY;
        if (key > row_b) sc[j][2] = -INFINITY;
        if (key + 1 > row_b) sc[j][3] = -INFINITY;
        mx0 = fmaxf(mx0, fmaxf(sc[j][0], sc[j][1]));
        mx1 = fmaxf(mx1, fmaxf(sc[j][2], sc[j][3]));
      }
#pragma unroll
      for (int off = 1; off <= 2; off <<= 1) {
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, off));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, off));
      }
      const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
      // every row has key 0 visible, so mn is finite from the first tile on
      const float fa0 = m0 == -INFINITY ? 0.f : expf(m0 - mn0), fa1 = m1 == -INFINITY ? 0.f : expf(m1 - mn1);
      float ps0 = 0.f, ps1 = 0.f;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        sc[j][0] = expf(sc[j][0] - mn0);
        sc[j][1] = expf(sc[j][1] - mn0);
        sc[j][2] = expf(sc[j][2] - mn1);
        sc[j][3] = expf(sc[j][3] - mn1);
        ps0 += sc[j][0] + sc[j][1];
        ps1 += sc[j][2] + sc[j][3];
      }
#pragma unroll
      for (int off = 1; off <= 2; off <<= 1) {
        ps0 += __shfl_xor_sync(0xffffffffu, ps0, off);
        ps1 += __shfl_xor_sync(0xffffffffu, ps1, off);
      }
      l0 = l0 * fa0 + ps0;
      l1 = l1 * fa1 + ps1;
      m0 = mn0;
      m1 = mn1;
#pragma unroll
      for (int j = 0; j < DT; ++j) {
        o[j][0] *= fa0;
        o[j][1] *= fa0;
        o[j][2] *= fa1;
        o[j][3] *= fa1;
      }
      // O += P V: k-chunk kc = keys 16kc.., A from S tiles 2kc / 2kc+1, B from V by ldmatrix.trans
#pragma unroll
      for (int kc2 = 0; kc2 < kKeys / 16; ++kc2) {
        uint32_t ph[4], pl[4];
        split2(sc[2 * kc2][0], sc[2 * kc2][1], ph[0], pl[0]);
        split2(sc[2 * kc2][2], sc[2 * kc2][3], ph[1], pl[1]);
        split2(sc[2 * kc2 + 1][0], sc[2 * kc2 + 1][1], ph[2], pl[2]);
        split2(sc[2 * kc2 + 1][2], sc[2 * kc2 + 1][3], ph[3], pl[3]);
        const __half* vrow = vt + (16 * kc2 + (lane & 15)) * LD;
#pragma unroll
        for (int j = 0; j < DT; ++j) {
          uint32_t b0, b1;
          asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0, %1}, [%2];"
                       : "=r"(b0), "=r"(b1)
                       : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(vrow + 8 * j))));
          mma16816(o[j], ph, b0, b1);
          mma16816(o[j], pl, b0, b1);
        }
      }
    }
    __syncthreads();  // the buffer is refilled by the next iteration's load
  }
  const float inv0 = 1.f / l0, inv1 = 1.f / l1;
#pragma unroll
  for (int j = 0; j < DT; ++j) {
    const int col = h * HD + 8 * j + 2 * t;
    if (row_a < T) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const __half hv = __float2half_rn(actr(o[j][e] * inv0, f16));
        out[tiled_act_offset(row_a, col + e, nkb)] = *reinterpret_cast<const uint16_t*>(&hv);
      }
    }
    if (row_b < T) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const __half hv = __float2half_rn(actr(o[j][2 + e] * inv1, f16));
        out[tiled_act_offset(row_b, col + e, nkb)] = *reinterpret_cast<const uint16_t*>(&hv);
      }
    }
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
  if (pos == nullptr && slots == nullptr && (hd == 128 || hd == 64)) {
    // the rows of one prompt: tensor-core flash attention (64 rows x one head per CTA)
    const dim3 grid(static_cast<unsigned>(ceil_div_i(B, fa::kRows)), static_cast<unsigned>(H));
    const int smem = 4 * fa::kKeys * (hd + 8) * static_cast<int>(sizeof(__half));
    if (hd == 128) {
      static bool cfg = false;
      if (!cfg) {
        FQ_CUDA(cudaFuncSetAttribute(attn_prompt_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        cfg = true;
      }
      attn_prompt_tc_kernel<128><<<grid, fa::kWarps * 32, smem, ctx->stream>>>(
          qr, kv, B, H, slot_stride, layer_off, max_seq, static_cast<uint16_t*>(out16), nkb, f16, slot0);
    } else {
      attn_prompt_tc_kernel<64><<<grid, fa::kWarps * 32, smem, ctx->stream>>>(
          qr, kv, B, H, slot_stride, layer_off, max_seq, static_cast<uint16_t*>(out16), nkb, f16, slot0);
    }
    FQ_CUDA(cudaGetLastError());
    ctx->launches += 1;
    return;
  }
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
