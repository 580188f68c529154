// Dequant-fused weight-only GEMV over resident W8/W4 copies (K1/K2 of SURVEY §2.1).
//
// Replaces MultiPrecisionLayer::forward (/root/reference/proj/src/model.cpp:77-98), which
// dequantizes the active rung (src/quantizer.cpp:205-219) and runs a double-accumulated
// linear (src/tensor.cpp:83-101).  Two numerics:
//
//  * fast  — the decode hot path.  Each lane streams 16 codes per row per step with one
//    coalesced 128-bit (W8) or 64-bit (W4) load, unpacks them in registers and accumulates
//    sum_j q_j x_j with packed FFMA2.  Unpacking is a single LOP/SHF per code: the masked
//    code bits (q << s), s < 24, reinterpreted as an fp32 bit pattern are exactly
//    q * 2^(s-149) (subnormal / first binade), so multiplying by x * 2^(109-s) yields
//    q*x*2^-40 with no int->float conversion.  The zero point is folded per group:
//    sum_j (q_j - z) x_j = sum_j q_j x_j - z * sum_j x_j, with sum_j x_j precomputed per lane.
//    fp32 accumulation; deterministic (fixed reduction order, no atomics).
//  * exact — golden/parity mode: w = float(code - z) * s in fp32 exactly as dequantize()
//    does, then double accumulation as linear() does.  Any group size, fp rung, bias.
//
// Work split (fast): a persistent-style grid of (#SM x CTAs/SM) CTAs; CTA c owns a balanced
// contiguous row range of every matrix of the launch; the CTA's W warps split the K-steps
// (512 codes each) so each warp keeps its activations in registers for the whole kernel and
// reuses them across all of the CTA's rows; per-row partials are reduced across warps through
// shared memory in warp order.
#include "fq_internal.cuh"

#include <algorithm>
#include <cstdio>
#include <map>
#include <mutex>

namespace fqc {
namespace {

constexpr int kStepCodes = 512;  // codes per row per warp step (32 lanes x 16)
constexpr int kSegCodes = 16;    // codes per lane per step
constexpr int kMaxB = 4;         // batch rows per fast launch
constexpr float kTwo109 = 649037107316853453566312041152512.0f;  // 2^109
constexpr float kTwo40 = 1099511627776.0f;                        // 2^40
constexpr float kTwoM40 = 9.094947017729282379150390625e-13f;     // 2^-40

__device__ __forceinline__ void ffma2(float2& acc, float a0, float a1, float b0, float b1) {
  asm("{\n\t.reg .b64 pa, pb, pc;\n\t"
      "mov.b64 pa, {%2, %3};\n\t"
      "mov.b64 pb, {%4, %5};\n\t"
      "mov.b64 pc, {%0, %1};\n\t"
      "fma.rn.f32x2 pc, pa, pb, pc;\n\t"
      "mov.b64 {%0, %1}, pc;\n\t}"
      : "+f"(acc.x), "+f"(acc.y)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}

__device__ __forceinline__ uint4 ldg_stream16(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ldg_stream8(const void* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
               : "=r"(r.x), "=r"(r.y)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;");
}

__device__ __forceinline__ float f32(uint32_t u) { return __uint_as_float(u); }

// Bit shift (s) of code j of a 16-code segment after extraction, per bit-width.
__device__ __forceinline__ int seg_shift(int bits, int j) {
  if (bits == 8) {
    const int p = j & 3;
    return p == 3 ? 0 : 8 * p;
  }
  const int p = j & 7;
  return p < 6 ? 4 * p : 4 * (p - 6);
}

// sum_j q_j * xs_j for one 16-code W8 segment (4 words); xs pre-scaled by 2^(109-s_j).
__device__ __forceinline__ float dot_seg8(const uint4 w, const float* xs) {
  float2 a = make_float2(0.f, 0.f), b = make_float2(0.f, 0.f);
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t v = ws[i];
    ffma2(i & 1 ? b : a, f32(v & 0xFFu), f32(v & 0xFF00u), xs[4 * i + 0], xs[4 * i + 1]);
    ffma2(i & 1 ? a : b, f32(v & 0xFF0000u), f32(v >> 24), xs[4 * i + 2], xs[4 * i + 3]);
  }
  return (a.x + a.y) + (b.x + b.y);
}

// sum_j q_j * xs_j for one 16-code W4 segment (2 words, low nibble = even element).
__device__ __forceinline__ float dot_seg4(const uint2 w, const float* xs) {
  float2 a = make_float2(0.f, 0.f), b = make_float2(0.f, 0.f);
  const uint32_t ws[2] = {w.x, w.y};
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const uint32_t v = ws[i];
    const uint32_t t = v >> 24;
    ffma2(a, f32(v & 0xFu), f32(v & 0xF0u), xs[8 * i + 0], xs[8 * i + 1]);
    ffma2(b, f32(v & 0xF00u), f32(v & 0xF000u), xs[8 * i + 2], xs[8 * i + 3]);
    ffma2(a, f32(v & 0xF0000u), f32(v & 0xF00000u), xs[8 * i + 4], xs[8 * i + 5]);
    ffma2(b, f32(t & 0xFu), f32(t & 0xF0u), xs[8 * i + 6], xs[8 * i + 7]);
  }
  return (a.x + a.y) + (b.x + b.y);
}

__device__ __forceinline__ float load_act(const void* x, int dtype, int64_t i) {
  if (dtype == FQ_DT_F32) return static_cast<const float*>(x)[i];
  if (dtype == FQ_DT_BF16) return __bfloat162float(static_cast<const __nv_bfloat16*>(x)[i]);
  return __half2float(static_cast<const __half*>(x)[i]);
}

__device__ __forceinline__ float round_act(float v, int dtype) {
  if (dtype == FQ_DT_BF16) return __bfloat162float(__float2bfloat16_rn(v));
  if (dtype == FQ_DT_F16) return __half2float(__float2half_rn(v));
  return v;
}

__device__ __forceinline__ void store_out(void* y, int dtype, int64_t i, float v) {
  if (dtype == FQ_DT_F32) static_cast<float*>(y)[i] = v;
  else if (dtype == FQ_DT_BF16) static_cast<__nv_bfloat16*>(y)[i] = __float2bfloat16_rn(v);
  else static_cast<__half*>(y)[i] = __float2half_rn(v);
}

struct DevMat {
  const uint8_t* payload8;
  const uint8_t* payload4;
  const float* scale8;
  const float* scale4;
  const uint8_t* zp8_8;
  const uint8_t* zp8_4;
  int32_t zpbase8, zpbase4;
  const uint8_t* rung_table;  // per batch row, or null
  int64_t rung_stride;
  int rung;                   // when no table
  void* y;
};

struct DevArgs {
  DevMat mat[3];
  int nmat;
  int B;
  int64_t N, K, G, ng;
  int nsteps;
  const void* x;
  int x_dtype;
  int64_t x_stride;
  const float* norm_gain;
  const float* norm_partials;
  int n_partials;
  float norm_eps;
  int act_dtype;
  int epi;
  void* y;
  int y_dtype;
  int64_t y_stride;
  float* resid;
  int64_t resid_stride;
  float* out_partials;
  int out_n_partials;
};

__device__ __forceinline__ int mat_rung(const DevMat& m, int b) {
  return m.rung_table ? static_cast<int>(m.rung_table[b * m.rung_stride]) : m.rung;
}

__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Streams rows [0, rows) of one matrix at one bit-width through this warp's K-steps and
// deposits the warp's per-row partial sums in shared memory.
template <int BITS, int SW, int BB>
__device__ __forceinline__ void stream_rows(const DevArgs& a, const DevMat& M, int m, int rows,
                                            int64_t r0, int bmask, const bool (&step_ok)[SW],
                                            const int64_t (&seg_k)[SW], const int (&gidx)[SW],
                                            const float (&xs)[SW][BB][kSegCodes],
                                            const float (&sig)[SW][BB], float* red) {
  constexpr int U = (SW >= 3 ? 2 : (SW == 2 ? 4 : 8));
  constexpr int NW = BITS == 8 ? 4 : 2;
  constexpr int kPrefetchBatches = 2;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int W = blockDim.x >> 5;
  const uint8_t* payload = BITS == 8 ? M.payload8 : M.payload4;
  const float* scale = BITS == 8 ? M.scale8 : M.scale4;
  const uint8_t* zp = BITS == 8 ? M.zp8_8 : M.zp8_4;
  const float zbase = static_cast<float>(BITS == 8 ? M.zpbase8 : M.zpbase4);
  const int64_t row_bytes = BITS == 8 ? a.K : a.K / 2;

  for (int rb = 0; rb < rows; rb += U) {
    if (threadIdx.x == 0) {
      const int ahead = rb + U * (kPrefetchBatches + 1);
      if (ahead < rows) {
        const int cnt = min(U, rows - ahead);
        prefetch_l2_bulk(payload + (r0 + ahead) * row_bytes,
                         static_cast<uint32_t>((cnt * row_bytes) & ~int64_t(15)));
      }
    }
    uint32_t wv[U][SW][NW];
    float sc[U][SW];
    float zf[U][SW];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t row = r0 + rb + u;
      const bool rok = rb + u < rows;
#pragma unroll
      for (int s = 0; s < SW; ++s) {
        const bool ok = rok && step_ok[s];
        const int64_t meta = row * a.ng + gidx[s];
        if constexpr (BITS == 8) {
          const uint4 v = ok ? ldg_stream16(payload + row * row_bytes + seg_k[s]) : make_uint4(0, 0, 0, 0);
          wv[u][s][0] = v.x; wv[u][s][1] = v.y; wv[u][s][2] = v.z; wv[u][s][3] = v.w;
        } else {
          const uint2 v = ok ? ldg_stream8(payload + row * row_bytes + seg_k[s] / 2) : make_uint2(0, 0);
          wv[u][s][0] = v.x; wv[u][s][1] = v.y;
        }
        sc[u][s] = ok ? __ldg(scale + meta) : 0.f;
        zf[u][s] = ok ? static_cast<float>(__ldg(zp + meta)) + zbase : 0.f;
      }
    }
    float acc[U][BB];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int b = 0; b < BB; ++b) acc[u][b] = 0.f;
#pragma unroll
    for (int s = 0; s < SW; ++s) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int b = 0; b < BB; ++b) {
          if (!((bmask >> b) & 1)) continue;
          float p;
          if constexpr (BITS == 8) p = dot_seg8(make_uint4(wv[u][s][0], wv[u][s][1], wv[u][s][2], wv[u][s][3]), xs[s][b]);
          else p = dot_seg4(make_uint2(wv[u][s][0], wv[u][s][1]), xs[s][b]);
          acc[u][b] = fmaf(sc[u][s], fmaf(-zf[u][s], sig[s][b], p), acc[u][b]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int b = 0; b < BB; ++b) {
        float v = acc[u][b];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && rb + u < rows && ((bmask >> b) & 1))
          red[((m * rows + rb + u) * W + warp) * BB + b] = v;
      }
    }
  }
}

template <int BITS, int SW, int BB>
__device__ __forceinline__ void load_acts(const DevArgs& a, const bool (&step_ok)[SW],
                                          const int64_t (&seg_k)[SW], const float (&rstd)[BB],
                                          float (&xs)[SW][BB][kSegCodes], float (&sig)[SW][BB]) {
#pragma unroll
  for (int s = 0; s < SW; ++s) {
#pragma unroll
    for (int b = 0; b < BB; ++b) {
      float acc = 0.f;
#pragma unroll
      for (int j = 0; j < kSegCodes; ++j) {
        float v = 0.f;
        if (step_ok[s] && b < a.B) {
          const int64_t k = seg_k[s] + j;
          v = load_act(a.x, a.x_dtype, b * a.x_stride + k);
          if (a.norm_gain != nullptr) v = round_act(v * rstd[b] * a.norm_gain[k], a.act_dtype);
        }
        acc += v;
        xs[s][b][j] = v * (kTwo109 / static_cast<float>(1u << seg_shift(BITS, j)));
      }
      sig[s][b] = acc * kTwoM40;
    }
  }
}

// Fast kernel.  SW = K-steps per warp (compile time), BB = batch rows (compile time bound).
template <int SW, int BB>
__global__ void __launch_bounds__(512) gemv_fast_kernel(const DevArgs a) {
  constexpr int U0 = (SW >= 3 ? 2 : (SW == 2 ? 4 : 8));
  extern __shared__ float red[];  // [nmat][rows_cta][W][BB]
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int W = blockDim.x >> 5;
  const int cta = blockIdx.x;
  const int ncta = gridDim.x;
  const int64_t r0 = (a.N * cta) / ncta;
  const int64_t r1 = (a.N * (cta + 1)) / ncta;
  const int rows = static_cast<int>(r1 - r0);

  bool step_ok[SW];
  int64_t seg_k[SW];
  int gidx[SW];
#pragma unroll
  for (int s = 0; s < SW; ++s) {
    const int step = warp + s * W;
    seg_k[s] = static_cast<int64_t>(step) * kStepCodes + lane * kSegCodes;
    step_ok[s] = step < a.nsteps && seg_k[s] < a.K;
    gidx[s] = step_ok[s] ? static_cast<int>(seg_k[s] / a.G) : 0;
  }

  // Weight streams do not depend on the previous kernel: pull the first row batches of every
  // matrix into L2 with TMA bulk prefetches before waiting on the dependency.
  if (threadIdx.x == 0 && rows > 0) {
    for (int m = 0; m < a.nmat; ++m) {
      for (int b = 0; b < a.B; ++b) {
        const int rr = mat_rung(a.mat[m], b);
        if (rr != FQ_RUNG_INT8 && rr != FQ_RUNG_INT4) continue;
        const uint8_t* base = rr == FQ_RUNG_INT8 ? a.mat[m].payload8 : a.mat[m].payload4;
        const int64_t rbytes = rr == FQ_RUNG_INT8 ? a.K : a.K / 2;
        const int cnt = min(rows, U0 * 3);
        prefetch_l2_bulk(base + r0 * rbytes, static_cast<uint32_t>((cnt * rbytes) & ~int64_t(15)));
        break;
      }
    }
  }

  pdl_wait();

  float rstd[BB];
#pragma unroll
  for (int b = 0; b < BB; ++b) {
    rstd[b] = 1.f;
    if (a.norm_gain != nullptr && b < a.B) {
      float s = 0.f;
      for (int i = lane; i < a.n_partials; i += 32) s += a.norm_partials[b * a.n_partials + i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      rstd[b] = 1.0f / sqrtf(s / static_cast<float>(a.K) + a.norm_eps);
    }
  }

  float xs[SW][BB][kSegCodes];
  float sig[SW][BB];
  int xs_bits = 0;
  for (int m = 0; m < a.nmat; ++m) {
    const DevMat& M = a.mat[m];
    int want8 = 0, want4 = 0;
    for (int b = 0; b < a.B; ++b) {
      const int r = mat_rung(M, b);
      want8 |= (r == FQ_RUNG_INT8) << b;
      want4 |= (r == FQ_RUNG_INT4) << b;
    }
    if (want8) {
      if (xs_bits != 8) { load_acts<8, SW, BB>(a, step_ok, seg_k, rstd, xs, sig); xs_bits = 8; }
      stream_rows<8, SW, BB>(a, M, m, rows, r0, want8, step_ok, seg_k, gidx, xs, sig, red);
    }
    if (want4) {
      if (xs_bits != 4) { load_acts<4, SW, BB>(a, step_ok, seg_k, rstd, xs, sig); xs_bits = 4; }
      stream_rows<4, SW, BB>(a, M, m, rows, r0, want4, step_ok, seg_k, gidx, xs, sig, red);
    }
  }
  // the next kernel in the stream may start its prologue (weight prefetch) now
  pdl_launch_dependents();
  __syncthreads();

  // cross-warp reduction in warp order + epilogue
  const int items = rows * BB;
  float local_sq[BB];
#pragma unroll
  for (int b = 0; b < BB; ++b) local_sq[b] = 0.f;
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int r = it / BB;
    const int b = it % BB;
    if (b >= a.B) continue;
    const int64_t row = r0 + r;
    float v[3] = {0.f, 0.f, 0.f};
    for (int m = 0; m < a.nmat; ++m) {
      float s = 0.f;
      for (int w = 0; w < W; ++w) s += red[((m * rows + r) * W + w) * BB + b];
      v[m] = s * kTwo40;
    }
    if (a.epi == EPI_STORE) {
      for (int m = 0; m < a.nmat; ++m) store_out(a.y, a.y_dtype, b * a.y_stride + m * a.N + row, v[m]);
    } else if (a.epi == EPI_SPLIT3) {
      for (int m = 0; m < a.nmat; ++m) store_out(a.mat[m].y, a.y_dtype, b * a.y_stride + row, v[m]);
    } else if (a.epi == EPI_SWIGLU) {
      const float g = v[0];
      const float silu = g / (1.0f + expf(-g));
      store_out(a.y, a.y_dtype, b * a.y_stride + row, round_act(silu * v[1], a.act_dtype));
    } else {  // EPI_RESIDUAL
      float* xp = a.resid + b * a.resid_stride + row;
      const float nv = *xp + v[0];
      *xp = nv;
      local_sq[b] += nv * nv;
    }
  }
  if (a.epi == EPI_RESIDUAL) {
    __shared__ float sq_red[kMaxB][16];
#pragma unroll
    for (int b = 0; b < BB; ++b) {
      float v = local_sq[b];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) sq_red[b][warp] = v;
    }
    __syncthreads();
    if (static_cast<int>(threadIdx.x) < a.B) {
      float s = 0.f;
      for (int w = 0; w < W; ++w) s += sq_red[threadIdx.x][w];
      a.out_partials[threadIdx.x * a.out_n_partials + cta] = s;
    }
  }
}

// Exact kernel: one warp per (row, batch row), lanes stride K, double accumulation.
__global__ void gemv_exact_kernel(const int64_t N, const int64_t K, const int64_t G, const int64_t ng,
                                  const int bits, const uint8_t* payload, const float* scale,
                                  const int32_t* zp, const float* fpw, const float* bias, const int B,
                                  const void* x, const int x_dtype, void* y, const int y_dtype) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (gw >= N * B) return;
  const int64_t row = gw / B;
  const int b = static_cast<int>(gw % B);
  double acc = 0.0;
  for (int64_t k = lane; k < K; k += 32) {
    float w;
    if (bits == 0) {
      w = fpw[row * K + k];
    } else {
      const int64_t idx = row * K + k;
      uint32_t code;
      if (bits == 8) code = payload[idx];
      else code = (idx & 1) ? (payload[idx >> 1] >> 4) : (payload[idx >> 1] & 0xFu);
      const int64_t g = row * ng + k / G;
      w = static_cast<float>(static_cast<int32_t>(code) - zp[g]) * scale[g];
    }
    acc += static_cast<double>(load_act(x, x_dtype, b * K + k)) * static_cast<double>(w);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) {
    if (bias) acc += static_cast<double>(bias[row]);
    store_out(y, y_dtype, b * N + row, static_cast<float>(acc));
  }
}

int pick_warps(int nsteps, int* sw_out) {
  // warps per CTA (4..8) dividing the step count as evenly as possible, <= 4 steps per warp
  int best_w = 8, best_sw = (nsteps + 7) / 8;
  double best_eff = -1.0;
  for (int w = 4; w <= 8; ++w) {
    const int sw = (nsteps + w - 1) / w;
    if (sw > 4) continue;
    const double eff = static_cast<double>(nsteps) / (static_cast<double>(sw) * w);
    if (eff > best_eff + 1e-9 || (eff > best_eff - 1e-9 && w > best_w)) {
      best_eff = eff;
      best_w = w;
      best_sw = sw;
    }
  }
  *sw_out = best_sw;
  return best_w;
}

template <int SW, int BB>
int launch_fast_t(fq_ctx* ctx, const DevArgs& d, int W, size_t smem, bool pdl) {
  auto kern = gemv_fast_kernel<SW, BB>;
  // occupancy is a pure function of (kernel, block, smem): cache it, host queries cost microseconds
  static std::map<std::pair<int, size_t>, int> occ_cache;
  static std::mutex occ_mu;
  int per_sm = 0;
  {
    std::lock_guard<std::mutex> lk(occ_mu);
    auto it = occ_cache.find({W, smem});
    if (it == occ_cache.end()) {
      if (smem > 48 * 1024)
        FQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      FQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, W * 32, smem));
      occ_cache[{W, smem}] = per_sm;
    } else {
      per_sm = it->second;
    }
  }
  per_sm = std::max(1, std::min(per_sm, 4));
  const int grid = static_cast<int>(std::min<int64_t>(static_cast<int64_t>(ctx->num_sms) * per_sm, d.N));
  if (d.epi == EPI_RESIDUAL && d.out_n_partials < grid) fail(FQ_E_STATE, "gemv: residual partial buffer too small");
  DevArgs dd = d;
  dd.out_n_partials = d.epi == EPI_RESIDUAL ? grid : d.out_n_partials;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(W * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  FQ_CUDA(cudaLaunchKernelEx(&cfg, kern, dd));
  ctx->launches += 1;
  return grid;
}

template <int SW>
int launch_fast_sw(fq_ctx* ctx, const DevArgs& d, int W, size_t smem_per_b, bool pdl) {
  if constexpr (SW == 1) {
    if (d.B == 1) return launch_fast_t<SW, 1>(ctx, d, W, smem_per_b, pdl);
    if (d.B == 2) return launch_fast_t<SW, 2>(ctx, d, W, smem_per_b * 2, pdl);
    return launch_fast_t<SW, 4>(ctx, d, W, smem_per_b * 4, pdl);
  } else if constexpr (SW == 2) {
    if (d.B == 1) return launch_fast_t<SW, 1>(ctx, d, W, smem_per_b, pdl);
    return launch_fast_t<SW, 2>(ctx, d, W, smem_per_b * 2, pdl);
  } else {
    return launch_fast_t<SW, 1>(ctx, d, W, smem_per_b, pdl);
  }
}

}  // namespace

bool gemv_fast_supported(const fq_layer* L, int rung) {
  if (rung != FQ_RUNG_INT8 && rung != FQ_RUNG_INT4) return false;
  const fq_rung_store& s = L->store(rung);
  return s.present && s.zp_fits_u8 && L->K % 32 == 0 && L->G % kSegCodes == 0 && L->G >= kSegCodes;
}

int launch_gemv_fast(fq_ctx* ctx, const GemvLaunch& g) {
  const fq_layer* L0 = g.mat[0].layer;
  DevArgs d = {};
  d.nmat = g.nmat;
  d.N = L0->N;
  d.K = L0->K;
  d.G = L0->G;
  d.ng = L0->ng;
  d.nsteps = ceil_div_i(L0->K, kStepCodes);
  d.x = g.x;
  d.x_dtype = g.x_dtype;
  d.x_stride = g.x_stride ? g.x_stride : L0->K;
  d.norm_gain = g.norm_gain;
  d.norm_partials = g.norm_partials;
  d.n_partials = g.n_partials;
  d.norm_eps = g.norm_eps;
  d.act_dtype = g.act_dtype;
  d.epi = g.epi;
  d.y = g.y;
  d.y_dtype = g.y_dtype;
  d.y_stride = g.y_stride;
  d.resid = g.resid;
  d.resid_stride = g.resid_stride;
  d.out_partials = g.out_partials;
  d.out_n_partials = g.out_n_partials;
  for (int m = 0; m < g.nmat; ++m) {
    const fq_layer* L = g.mat[m].layer;
    if (L->N != d.N || L->K != d.K || L->G != d.G) fail(FQ_E_DIMENSION, "multi-gemv: matrices differ in shape");
    DevMat& M = d.mat[m];
    M.payload8 = L->r8.payload;
    M.payload4 = L->r4.payload;
    M.scale8 = L->r8.scale;
    M.scale4 = L->r4.scale;
    M.zp8_8 = L->r8.zp8;
    M.zp8_4 = L->r4.zp8;
    M.zpbase8 = L->r8.zp_base;
    M.zpbase4 = L->r4.zp_base;
    M.rung_table = g.mat[m].rung_table;
    M.rung_stride = g.mat[m].rung_stride;
    M.rung = g.mat[m].rung;
    M.y = g.mat[m].y;
  }
  int sw = 1;
  const int W = pick_warps(d.nsteps, &sw);
  // rows per CTA is bounded by ceil(N / #SM) (at least one CTA per SM)
  const int64_t rows_max = (d.N + ctx->num_sms - 1) / ctx->num_sms;
  const size_t smem_per_b = static_cast<size_t>(g.nmat) * rows_max * W * sizeof(float);
  // registers hold SW x B x 16 activations: keep SW*B <= 4 by chunking the batch
  const int64_t bchunk = sw == 1 ? kMaxB : (sw == 2 ? 2 : 1);
  int grid = 0;
  for (int64_t b0 = 0; b0 < g.batch; b0 += bchunk) {
    DevArgs c = d;
    c.B = static_cast<int>(std::min<int64_t>(bchunk, g.batch - b0));
    c.x = static_cast<const char*>(g.x) + b0 * d.x_stride * (g.x_dtype == FQ_DT_F32 ? 4 : 2);
    const int ysz = g.y_dtype == FQ_DT_F32 ? 4 : 2;
    if (g.y) c.y = static_cast<char*>(g.y) + b0 * d.y_stride * ysz;
    for (int m = 0; m < g.nmat; ++m) {
      if (g.mat[m].y) c.mat[m].y = static_cast<char*>(g.mat[m].y) + b0 * d.y_stride * ysz;
      if (g.mat[m].rung_table) c.mat[m].rung_table = g.mat[m].rung_table + b0 * g.mat[m].rung_stride;
    }
    if (g.resid) c.resid = g.resid + b0 * g.resid_stride;
    if (g.out_partials) c.out_partials = g.out_partials + b0 * g.out_n_partials;
    if (g.norm_partials) c.norm_partials = g.norm_partials + b0 * g.n_partials;
    switch (sw) {
      case 1: grid = launch_fast_sw<1>(ctx, c, W, smem_per_b, g.pdl); break;
      case 2: grid = launch_fast_sw<2>(ctx, c, W, smem_per_b, g.pdl); break;
      case 3: grid = launch_fast_sw<3>(ctx, c, W, smem_per_b, g.pdl); break;
      default: grid = launch_fast_sw<4>(ctx, c, W, smem_per_b, g.pdl); break;
    }
  }
  return grid;
}

void launch_gemv_exact(fq_ctx* ctx, const fq_layer* L, int rung, int64_t batch, const void* x,
                       int x_dtype, void* y, int y_dtype) {
  if (!L->has(rung)) fail(FQ_E_STATE, "gemv: rung not resident on the device");
  const int threads = 256;
  const int64_t warps = L->N * batch;
  const int blocks = ceil_div_i(warps * 32, threads);
  const fq_rung_store* s = rung == FQ_RUNG_FP ? nullptr : &L->store(rung);
  gemv_exact_kernel<<<blocks, threads, 0, ctx->stream>>>(
      L->N, L->K, L->G, L->ng, s ? s->bits : 0, s ? s->payload : nullptr, s ? s->scale : nullptr,
      s ? s->zp32 : nullptr, L->fp, L->bias, static_cast<int>(batch), x, x_dtype, y, y_dtype);
  FQ_CUDA(cudaGetLastError());
  ctx->launches += 1;
}

}  // namespace fqc
