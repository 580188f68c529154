// Persistent TMA-fed program kernel (see gemv.cu for the design):
//   warp kNCW        producer: streams every GEMV phase's row ranges through the smem ring
//   warps 0..kNCW-1  consumers: GEMV compute (kSplit warps split K, kRG row groups),
//                    embedding, attention (groups of 4 warps) and row statistics, with a
//                    grid-wide barrier between dependent phases.
#include "gemv_program.cuh"

#include <algorithm>
#include <cfloat>
#include <cstring>
#include <map>
#include <mutex>

namespace fqc {
namespace {

// ---------------------------------------------------------------- PTX helpers
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
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;"); }
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void named_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ unsigned int ld_acquire(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ float f32(uint32_t u) { return __uint_as_float(u); }

__host__ __device__ constexpr int seg_shift(int bits, int j) {
  return bits == 8 ? ((j & 3) == 3 ? 0 : 8 * (j & 3)) : ((j & 7) < 6 ? 4 * (j & 7) : 4 * ((j & 7) - 6));
}

__device__ __forceinline__ float dot_seg8(const uint4 w, const float* xs) {
  float2 a = make_float2(0.f, 0.f), b = make_float2(0.f, 0.f);
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t v = ws[i];
    ffma2(i & 1 ? b : a, f32(v & 0xFFu), f32(v & 0xFF00u), xs[4 * i + 0], xs[4 * i + 1]);
    ffma2(i & 1 ? a : b, f32(v & 0xFF0000u), f32(v >> 24), xs[4 * i + 2], xs[4 * i + 3]);
  }
  a.x += b.x;
  a.y += b.y;
  return a.x + a.y;
}

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
  a.x += b.x;
  a.y += b.y;
  return a.x + a.y;
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

__device__ __forceinline__ int mat_rung(const DevMat& m, int b) {
  return m.rung_table ? static_cast<int>(m.rung_table[b * m.rung_stride]) : m.rung;
}
__device__ __forceinline__ int pass_mask(const Phase& P, int m, int w) {
  int mask = 0;
  const int want = w == 0 ? FQ_RUNG_INT8 : FQ_RUNG_INT4;
  for (int b = 0; b < P.B; ++b) mask |= (mat_rung(P.mat[m], b) == want) << b;
  return mask;
}

__device__ __forceinline__ void cta_rows(int64_t N, int64_t& r0, int& rows) {
  r0 = (N * blockIdx.x) / gridDim.x;
  rows = static_cast<int>((N * (blockIdx.x + 1)) / gridDim.x - r0);
}

// Reduces v[0..7] across the 32 lanes (9 shuffles); afterwards lane l holds the warp sum of
// row (l>>2)&7.
__device__ __forceinline__ float reduce8(const float (&v)[8], int lane) {
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
  float k[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float keep = b4 ? v[4 + i] : v[i], send = b4 ? v[i] : v[4 + i];
    k[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
  float m[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float keep = b3 ? k[2 + i] : k[i], send = b3 ? k[i] : k[2 + i];
    m[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  const float keep = b2 ? m[1] : m[0], send = b2 ? m[0] : m[1];
  float r = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  r += __shfl_xor_sync(0xffffffffu, r, 2);
  r += __shfl_xor_sync(0xffffffffu, r, 1);
  return r;
}

// Reduces v[0..1] across the 32 lanes; afterwards lane l holds the warp sum of row (l>>4)&1.
__device__ __forceinline__ float reduce2(const float (&v)[2], int lane) {
  const bool b4 = lane & 16;
  float k = b4 ? v[1] : v[0];
  const float t = b4 ? v[0] : v[1];
  k += __shfl_xor_sync(0xffffffffu, t, 16);
  k += __shfl_xor_sync(0xffffffffu, k, 8);
  k += __shfl_xor_sync(0xffffffffu, k, 4);
  k += __shfl_xor_sync(0xffffffffu, k, 2);
  k += __shfl_xor_sync(0xffffffffu, k, 1);
  return k;
}

// Reduces v[0..3] across the 32 lanes; afterwards lane l holds the warp sum of row (l>>3)&3.
__device__ __forceinline__ float reduce4(const float (&v)[4], int lane) {
  const bool b4 = lane & 16, b3 = lane & 8;
  float k0 = b4 ? v[2] : v[0], k1 = b4 ? v[3] : v[1];
  const float t0 = b4 ? v[0] : v[2], t1 = b4 ? v[1] : v[3];
  k0 += __shfl_xor_sync(0xffffffffu, t0, 16);
  k1 += __shfl_xor_sync(0xffffffffu, t1, 16);
  float k = b3 ? k1 : k0;
  const float t = b3 ? k0 : k1;
  k += __shfl_xor_sync(0xffffffffu, t, 8);
  k += __shfl_xor_sync(0xffffffffu, k, 4);
  k += __shfl_xor_sync(0xffffffffu, k, 2);
  k += __shfl_xor_sync(0xffffffffu, k, 1);
  return k;
}

struct Ring {
  uint8_t* base;
  uint64_t* full;
  uint64_t* empty;
  int stage_bytes;
  int nstages;
};

// ---------------------------------------------------------------- producer
// All phase fields are copied into registers before the stage loop: the asm statements carry
// "memory" clobbers, so anything left in memory would be reloaded after every copy / wait.
__device__ __forceinline__ void produce_phase(const Phase& P, const Ring R, int& slot_i, uint32_t& phase_bit) {
  int64_t r0;
  int rows;
  cta_rows(P.N, r0, rows);
  if (rows <= 0) return;
  const int nmat = P.nmat;
  const int64_t K = P.K, ng_pad = P.ng_pad, zp_pad = P.zp_pad;
  for (int m = 0; m < nmat; ++m) {
    for (int w = 0; w < 2; ++w) {
      if (pass_mask(P, m, w) == 0) continue;
      const int rps = P.rows_per_stage[w];
      const int64_t row_bytes = w == 0 ? K : K / 2;
      const uint8_t* pay_src = P.mat[m].payload[w] + r0 * row_bytes;
      const uint8_t* sc_src = reinterpret_cast<const uint8_t*>(P.mat[m].scale[w] + r0 * ng_pad);
      const uint8_t* zp_src = P.mat[m].zp[w] + r0 * zp_pad;
      const uint32_t sc_off = static_cast<uint32_t>(P.sc_off[w]), zp_off = static_cast<uint32_t>(P.zp_off[w]);
      const uint32_t pay_row = static_cast<uint32_t>(row_bytes), sc_row = static_cast<uint32_t>(ng_pad * 4),
                     zp_row = static_cast<uint32_t>(zp_pad);
      for (int rb = 0; rb < rows; rb += rps) {
        const int s = slot_i;
        mbar_wait(&R.empty[s], phase_bit ^ 1u);
        if (++slot_i == R.nstages) {
          slot_i = 0;
          phase_bit ^= 1u;
        }
        const uint32_t nr = static_cast<uint32_t>(min(rps, rows - rb));
        uint8_t* dst = R.base + static_cast<size_t>(s) * R.stage_bytes;
        mbar_expect_tx(&R.full[s], nr * (pay_row + sc_row + zp_row));
        bulk_g2s(dst, pay_src + static_cast<int64_t>(rb) * pay_row, nr * pay_row, &R.full[s]);
        bulk_g2s(dst + sc_off, sc_src + static_cast<int64_t>(rb) * sc_row, nr * sc_row, &R.full[s]);
        bulk_g2s(dst + zp_off, zp_src + static_cast<int64_t>(rb) * zp_row, nr * zp_row, &R.full[s]);
      }
    }
  }
}

// ---------------------------------------------------------------- consumers: GEMV
// Activations of a GEMV phase are staged once per phase (and bit-width) in shared memory,
// pre-scaled by the bit pattern of the rung: xsm[b][step][j4][lane] float4 (a lane's 16 values
// of a step as four conflict-free 16-byte chunks) and sigm[b][step][lane] = sum of the 16 values
// * 2^-40 (zero-point folding).  All consumer threads cooperate.
template <int BB>
__device__ void stage_acts(const Phase& P, int bits, const float (&rstd)[BB], float4* xsm, float* sigm) {
  const int nsteps = P.nsteps;
  const int nseg = nsteps * 32;
  const int64_t K = P.K;
  const void* x = P.x;
  const int xdt = P.x_dtype, adt = P.act_dtype;
  const int64_t xstride = P.x_stride;
  const float* gain = P.norm_gain;
  for (int i = threadIdx.x; i < nseg * BB; i += kNCW * 32) {
    const int b = i / nseg, seg = i - b * nseg;
    const int step = seg >> 5, ln = seg & 31;
    const int64_t k0 = static_cast<int64_t>(step) * kStepCodes + ln * kSegCodes;
    float v[kSegCodes];
    float acc = 0.f;
#pragma unroll
    for (int j = 0; j < kSegCodes; ++j) {
      float t = 0.f;
      if (k0 + j < K && b < P.B) {
        t = load_act(x, xdt, b * xstride + k0 + j);
        if (gain != nullptr) t = round_act(t * rstd[b] * gain[k0 + j], adt);
      }
      acc += t;
      const float sc8 = kTwo109 / static_cast<float>(1u << seg_shift(8, j));
      const float sc4 = kTwo109 / static_cast<float>(1u << seg_shift(4, j));
      v[j] = t * (bits == 8 ? sc8 : sc4);
    }
    float4* dst = xsm + (static_cast<size_t>(b * nsteps + step) * 4) * 32 + ln;
#pragma unroll
    for (int j4 = 0; j4 < 4; ++j4) dst[j4 * 32] = make_float4(v[4 * j4], v[4 * j4 + 1], v[4 * j4 + 2], v[4 * j4 + 3]);
    sigm[static_cast<size_t>(b * nsteps + step) * 32 + ln] = acc * kTwoM40;
  }
}

// Consumes one ring slot holding `nrows` rows at bit-width BITS: row quads are split between the
// kRG row groups; within a quad the loop runs over this warp's K-steps (activations loaded from
// shared memory once per step) and then the four rows.
template <int BITS, int SW, int BB, int QR>
__device__ __forceinline__ void consume_stage(const uint8_t* __restrict__ slot, int nrows, int rg, int row_bytes,
                                              int sc_off, int zp_off, int sc_row, int zp_row, const int (&pay_l)[SW],
                                              const int (&sc_l)[SW], const int (&zp_l)[SW], const int (&step_of)[SW],
                                              const bool (&step_ok)[SW], int nsteps, float zmagic,
                                              const float4* __restrict__ xsm, const float* __restrict__ sigm,
                                              float* red_row, int bmask, int lane) {
  const uint8_t* pa = slot + rg * QR * row_bytes;
  const uint8_t* sa = slot + sc_off + rg * QR * sc_row;
  const uint8_t* za = slot + zp_off + rg * QR * zp_row;
  const int red_step = kSplit * BB;
  for (int r0 = rg * QR; r0 < nrows; r0 += QR * kRG) {
    float acc[BB][QR];
#pragma unroll
    for (int b = 0; b < BB; ++b)
#pragma unroll
      for (int u = 0; u < QR; ++u) acc[b][u] = 0.f;
#pragma unroll
    for (int s = 0; s < SW; ++s) {
      if (!step_ok[s]) continue;
      float xs[BB][kSegCodes];
      float sg[BB];
#pragma unroll
      for (int b = 0; b < BB; ++b) {
        const float4* src = xsm + (static_cast<size_t>(b * nsteps + step_of[s]) * 4) * 32 + lane;
#pragma unroll
        for (int j4 = 0; j4 < 4; ++j4) {
          const float4 f = src[j4 * 32];
          xs[b][4 * j4] = f.x;
          xs[b][4 * j4 + 1] = f.y;
          xs[b][4 * j4 + 2] = f.z;
          xs[b][4 * j4 + 3] = f.w;
        }
        sg[b] = sigm[static_cast<size_t>(b * nsteps + step_of[s]) * 32 + lane];
      }
#pragma unroll
      for (int u = 0; u < QR; ++u) {
        const float sc = *reinterpret_cast<const float*>(sa + u * sc_row + sc_l[s]);
        const uint32_t zq = za[u * zp_row + zp_l[s]];
        const float zf = __uint_as_float(0x4B000000u | zq) - zmagic;  // exact: zq + zp_base
        float p[BB];
        if constexpr (BITS == 8) {
          const uint4 w = *reinterpret_cast<const uint4*>(pa + u * row_bytes + pay_l[s]);
#pragma unroll
          for (int b = 0; b < BB; ++b) p[b] = dot_seg8(w, xs[b]);
        } else {
          const uint2 w = *reinterpret_cast<const uint2*>(pa + u * row_bytes + pay_l[s]);
#pragma unroll
          for (int b = 0; b < BB; ++b) p[b] = dot_seg4(w, xs[b]);
        }
#pragma unroll
        for (int b = 0; b < BB; ++b) acc[b][u] = fmaf(sc, fmaf(-zf, sg[b], p[b]), acc[b][u]);
      }
    }
    const int u = QR == 8 ? ((lane >> 2) & 7) : QR == 4 ? ((lane >> 3) & 3) : ((lane >> 4) & 1);
    const bool writer = QR == 8 ? (lane & 3) == 0 : QR == 4 ? (lane & 7) == 0 : (lane & 15) == 0;
#pragma unroll
    for (int b = 0; b < BB; ++b) {
      float v;
      if constexpr (QR == 8) v = reduce8(acc[b], lane);
      else if constexpr (QR == 4) v = reduce4(acc[b], lane);
      else v = reduce2(acc[b], lane);
      if (writer && r0 + u < nrows && ((bmask >> b) & 1)) red_row[(r0 + u) * red_step + b] = v;
    }
    pa += QR * kRG * row_bytes;
    sa += QR * kRG * sc_row;
    za += QR * kRG * zp_row;
  }
}

template <int SW, int BB>
__device__ __forceinline__ void consume_gemv(const Phase& P, const Ring R, float* red, float4* xsm, float* sigm,
                                             int& slot_i, uint32_t& phase_bit) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int kw = warp % kSplit, rg = warp / kSplit;
  int64_t r0;
  int rows;
  cta_rows(P.N, r0, rows);
  const int nsteps = P.nsteps;
  const int64_t K = P.K, G = P.G;
  bool step_ok[SW];
  int step_of[SW], seg_k[SW], gidx[SW];
#pragma unroll
  for (int s = 0; s < SW; ++s) {
    step_of[s] = kw + s * kSplit;
    seg_k[s] = step_of[s] * kStepCodes + lane * kSegCodes;
    step_ok[s] = step_of[s] < nsteps;
    gidx[s] = (step_ok[s] && seg_k[s] < K) ? static_cast<int>(seg_k[s] / G) : 0;
    if (!step_ok[s] || seg_k[s] >= K) seg_k[s] = 0;
    if (!step_ok[s]) step_of[s] = 0;
  }
  float rstd[BB];
#pragma unroll
  for (int b = 0; b < BB; ++b) {
    rstd[b] = 1.f;
    if (P.norm_gain != nullptr && b < P.B) {
      float s = 0.f;
      for (int i = lane; i < P.n_partials; i += 32) s += P.norm_partials[b * P.partials_stride + i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      rstd[b] = 1.0f / sqrtf(s / static_cast<float>(K) + P.norm_eps);
    }
  }
  int xs_bits = 0;
  const int nmat = P.nmat;
  for (int m = 0; m < nmat; ++m) {
    for (int w = 0; w < 2; ++w) {
      const int bmask = pass_mask(P, m, w);
      if (bmask == 0) continue;
      const int bits = w == 0 ? 8 : 4;
      if (xs_bits != bits) {
        named_sync(1, kNCW * 32);  // previous users of the staging area are done
        stage_acts<BB>(P, bits, rstd, xsm, sigm);
        named_sync(1, kNCW * 32);
        xs_bits = bits;
      }
      if (rows == 0) continue;
      const float zmagic = 8388608.0f - static_cast<float>(P.mat[m].zpbase[w]);
      const int rps = P.rows_per_stage[w];
      const int row_bytes = static_cast<int>(w == 0 ? K : K / 2);
      int pay_l[SW], sc_l[SW], zp_l[SW];
#pragma unroll
      for (int s = 0; s < SW; ++s) {
        pay_l[s] = w == 0 ? seg_k[s] : seg_k[s] / 2;
        sc_l[s] = gidx[s] * 4;
        zp_l[s] = gidx[s];
      }
      const int sco = P.sc_off[w], zpo = P.zp_off[w], scr = P.sc_row, zpr = P.zp_row;
      for (int rb = 0; rb < rows; rb += rps) {
        mbar_wait(&R.full[slot_i], phase_bit);
        const uint8_t* slot = R.base + static_cast<size_t>(slot_i) * R.stage_bytes;
        float* red_row = red + ((m * rows + rb) * kSplit + kw) * BB;
        const int nr = min(rps, rows - rb);
        constexpr int QR = SW == 1 ? (BB == 1 ? 8 : 4) : 2;
        if (bits == 8)
          consume_stage<8, SW, BB, QR>(slot, nr, rg, row_bytes, sco, zpo, scr, zpr, pay_l, sc_l, zp_l, step_of, step_ok,
                                   nsteps, zmagic, xsm, sigm, red_row, bmask, lane);
        else
          consume_stage<4, SW, BB, QR>(slot, nr, rg, row_bytes, sco, zpo, scr, zpr, pay_l, sc_l, zp_l, step_of, step_ok,
                                   nsteps, zmagic, xsm, sigm, red_row, bmask, lane);
        __syncwarp();
        if (lane == 0) mbar_arrive(&R.empty[slot_i]);
        if (++slot_i == R.nstages) {
          slot_i = 0;
          phase_bit ^= 1u;
        }
      }
    }
  }
}

// Cross-warp reduction (kSplit partials per row, warp order) + epilogue, consumer threads only.
template <int BB>
__device__ void gemv_epilogue(const Phase& P, const float* red, float (*sq_red)[kNCW]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t r0;
  int rows;
  cta_rows(P.N, r0, rows);
  const int items = rows * BB;
  float local_sq[BB];
#pragma unroll
  for (int b = 0; b < BB; ++b) local_sq[b] = 0.f;
  for (int it = threadIdx.x; it < items; it += kNCW * 32) {
    const int r = it / BB;
    const int b = it % BB;
    if (b >= P.B) continue;
    const int64_t row = r0 + r;
    float v[3] = {0.f, 0.f, 0.f};
    for (int m = 0; m < P.nmat; ++m) {
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < kSplit; ++w) s += red[((m * rows + r) * kSplit + w) * BB + b];
      v[m] = s * kTwo40;
    }
    if (P.epi == EPI_STORE) {
      for (int m = 0; m < P.nmat; ++m) store_out(P.y, P.y_dtype, b * P.y_stride + m * P.N + row, v[m]);
    } else if (P.epi == EPI_SPLIT3) {
      for (int m = 0; m < P.nmat; ++m) store_out(P.mat[m].y, P.y_dtype, b * P.y_stride + row, v[m]);
    } else if (P.epi == EPI_SWIGLU) {
      const float g = v[0];
      const float silu = g / (1.0f + expf(-g));
      store_out(P.y, P.y_dtype, b * P.y_stride + row, round_act(silu * v[1], P.act_dtype));
    } else {
      float* xp = P.resid + b * P.resid_stride + row;
      const float nv = *xp + v[0];
      *xp = nv;
      local_sq[b] += nv * nv;
    }
  }
  if (P.epi == EPI_RESIDUAL) {
#pragma unroll
    for (int b = 0; b < BB; ++b) {
      float v = local_sq[b];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) sq_red[b][warp] = v;
    }
    named_sync(1, kNCW * 32);
    if (static_cast<int>(threadIdx.x) < P.B) {
      float s = 0.f;
      for (int w = 0; w < kNCW; ++w) s += sq_red[threadIdx.x][w];
      P.out_partials[threadIdx.x * P.out_partials_stride + blockIdx.x] = s;
    }
  }
  named_sync(1, kNCW * 32);  // red / sq_red are reused by the next phase
}

template <int BB>
__device__ __forceinline__ void run_gemv_phase(const Phase& P, const Ring R, float* red, float (*sq_red)[kNCW],
                                               float4* xsm, float* sigm, int& slot_i, uint32_t& phase_bit) {
  switch (P.sw) {
    case 1: consume_gemv<1, BB>(P, R, red, xsm, sigm, slot_i, phase_bit); break;
    case 2:
      if constexpr (BB <= 2) consume_gemv<2, BB>(P, R, red, xsm, sigm, slot_i, phase_bit);
      break;
    case 3:
      if constexpr (BB == 1) consume_gemv<3, BB>(P, R, red, xsm, sigm, slot_i, phase_bit);
      break;
    default:
      if constexpr (BB == 1) consume_gemv<4, BB>(P, R, red, xsm, sigm, slot_i, phase_bit);
      break;
  }
  named_sync(1, kNCW * 32);
  gemv_epilogue<BB>(P, red, sq_red);
}

// ---------------------------------------------------------------- consumers: embedding
__device__ void run_embed(const Phase& P, float (*sq_red)[kNCW]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t c0;
  int cnt;
  cta_rows(P.d, c0, cnt);
  for (int b = 0; b < P.B; ++b) {
    const float* e = P.tok_emb + static_cast<int64_t>(P.tokens[b]) * P.d;
    float sq = 0.f;
    for (int i = threadIdx.x; i < cnt; i += kNCW * 32) {
      const float v = e[c0 + i];
      P.resid[b * P.resid_stride + c0 + i] = v;
      sq += v * v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    if (lane == 0) sq_red[0][warp] = sq;
    named_sync(1, kNCW * 32);
    if (threadIdx.x == 0) {
      float s = 0.f;
      for (int w = 0; w < kNCW; ++w) s += sq_red[0][w];
      P.out_partials[b * P.out_partials_stride + blockIdx.x] = s;
    }
    named_sync(1, kNCW * 32);
  }
}

// ---------------------------------------------------------------- consumers: attention
struct AttnSmem {
  float qs[256];
  float knew[256];
  float sc[kAttnChunk];
  int last;
};

__device__ __forceinline__ void rope_pair(float& a, float& b, int i, int hd, int pos, float theta) {
  const double inv = pow(static_cast<double>(theta), -2.0 * i / hd);
  double sn, cs;
  sincos(static_cast<double>(pos) * inv, &sn, &cs);
  const float c = static_cast<float>(cs), s = static_cast<float>(sn);
  const float x0 = a, x1 = b;
  a = x0 * c - x1 * s;
  b = x1 * c + x0 * s;
}

// One (row, head, key chunk) item on a 128-thread group (4 warps, named barrier `bar`).
__device__ void attn_item(const Phase& P, int b, int h, int chunk, int nch, AttnSmem& S, int gtid, int bar) {
  const int hd = P.head_dim, H = P.n_heads;
  const int d = H * hd;
  const int pos = P.pos[b];
  const int slot = P.slots[b];
  const int j0 = chunk * kAttnChunk;
  const int j1 = min(j0 + kAttnChunk, pos + 1);
  __half* kc = P.kv + slot * P.slot_stride + P.layer_off + static_cast<int64_t>(h) * P.max_seq * hd;
  __half* vc = kc + static_cast<int64_t>(H) * P.max_seq * hd;
  float* wsp = P.attn_ws + ((static_cast<int64_t>(b) * H + h) * nch + chunk) * (hd + 2);
  const int adt = P.act_dtype;
  const float scale = 1.0f / sqrtf(static_cast<float>(hd));
  for (int i = gtid; i < hd / 2; i += 128) {
    float a0 = load_act(P.q, adt, static_cast<int64_t>(b) * d + h * hd + i);
    float a1 = load_act(P.q, adt, static_cast<int64_t>(b) * d + h * hd + i + hd / 2);
    rope_pair(a0, a1, i, hd, pos, P.rope_theta);
    S.qs[i] = a0 * scale;
    S.qs[i + hd / 2] = a1 * scale;
  }
  const bool owns_new = pos >= j0 && pos < j0 + kAttnChunk;
  if (owns_new) {
    for (int i = gtid; i < hd / 2; i += 128) {
      float a0 = load_act(P.k, adt, static_cast<int64_t>(b) * d + h * hd + i);
      float a1 = load_act(P.k, adt, static_cast<int64_t>(b) * d + h * hd + i + hd / 2);
      rope_pair(a0, a1, i, hd, pos, P.rope_theta);
      const __half h0 = __float2half_rn(a0), h1 = __float2half_rn(a1);
      kc[static_cast<int64_t>(pos) * hd + i] = h0;
      kc[static_cast<int64_t>(pos) * hd + i + hd / 2] = h1;
      S.knew[i] = __half2float(h0);
      S.knew[i + hd / 2] = __half2float(h1);
    }
    for (int i = gtid; i < hd; i += 128)
      vc[static_cast<int64_t>(pos) * hd + i] = __float2half_rn(load_act(P.v, adt, static_cast<int64_t>(b) * d + h * hd + i));
  }
  named_sync(bar, 128);
  const int lane = gtid & 31, gw = gtid >> 5;
  for (int j = j0 + gw; j < j1; j += 4) {
    float s = 0.f;
    if (j == pos) {
      for (int i = lane; i < hd; i += 32) s += S.qs[i] * S.knew[i];
    } else {
      const __half* kr = kc + static_cast<int64_t>(j) * hd;
      for (int i = lane; i < hd; i += 32) s += S.qs[i] * __half2float(kr[i]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) S.sc[j - j0] = s;
  }
  named_sync(bar, 128);
  float m = -INFINITY;
  for (int j = 0; j < j1 - j0; ++j) m = fmaxf(m, S.sc[j]);
  for (int i = gtid; i < hd; i += 128) {
    float acc = 0.f, l = 0.f;
    for (int j = j0; j < j1; ++j) {
      const float p = expf(S.sc[j - j0] - m);
      const float vv = (j == pos) ? __half2float(__float2half_rn(load_act(P.v, adt, static_cast<int64_t>(b) * d + h * hd + i)))
                                  : __half2float(vc[static_cast<int64_t>(j) * hd + i]);
      acc += p * vv;
      l += p;
    }
    wsp[2 + i] = acc;
    if (i == 0) {
      wsp[0] = m;
      wsp[1] = l;
    }
  }
  __threadfence();
  named_sync(bar, 128);
  if (gtid == 0) {
    const unsigned int prev = atomicAdd(&P.tickets[b * H + h], 1u);
    S.last = prev == static_cast<unsigned int>(nch - 1);
  }
  named_sync(bar, 128);
  if (S.last) {
    __threadfence();
    const float* base = P.attn_ws + (static_cast<int64_t>(b) * H + h) * nch * (hd + 2);
    float M = -INFINITY;
    for (int c = 0; c < nch; ++c) M = fmaxf(M, __ldcg(base + c * (hd + 2)));
    for (int i = gtid; i < hd; i += 128) {
      float L = 0.f, O = 0.f;
      for (int c = 0; c < nch; ++c) {
        const float f = expf(__ldcg(base + c * (hd + 2)) - M);
        L += __ldcg(base + c * (hd + 2) + 1) * f;
        O += __ldcg(base + c * (hd + 2) + 2 + i) * f;
      }
      store_out(P.attn_out, adt, static_cast<int64_t>(b) * d + h * hd + i, O / L);
    }
    if (gtid == 0) P.tickets[b * H + h] = 0u;
  }
  named_sync(bar, 128);
}

__device__ void run_attn(const Phase& P, AttnSmem* S) {
  const int group = threadIdx.x >> 7;  // 4 groups of 4 warps
  const int gtid = threadIdx.x & 127;
  const int groups = kNCW / 4;
  // items: for every row b and head h, the active key chunks of that row
  int total = 0;
  for (int b = 0; b < P.B; ++b) total += P.n_heads * ((P.pos[b] + kAttnChunk) / kAttnChunk);
  for (int item = blockIdx.x * groups + group; item < total; item += gridDim.x * groups) {
    int rem = item, b = 0;
    for (;; ++b) {
      const int per = P.n_heads * ((P.pos[b] + kAttnChunk) / kAttnChunk);
      if (rem < per) break;
      rem -= per;
    }
    const int nch = (P.pos[b] + kAttnChunk) / kAttnChunk;
    attn_item(P, b, rem / nch, rem % nch, nch, S[group], gtid, 2 + group);
  }
}

// ---------------------------------------------------------------- consumers: row statistics
// softmax_double / ppl_entropy / fault_tolerance / argmax_token of logits row b on CTA b.
__device__ void run_stats(const Phase& P, double* shd) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nthreads = kNCW * 32;
  for (int b = blockIdx.x; b < P.B; b += gridDim.x) {
    const float* l = P.logits + b * P.vocab;
    float bv = -INFINITY;
    int bi = 0x7fffffff;
    for (int64_t i = threadIdx.x; i < P.vocab; i += nthreads) {
      const float x = l[i];
      if (x > bv || (x == bv && i < bi)) { bv = x; bi = static_cast<int>(i); }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    float* shv = reinterpret_cast<float*>(shd + 3 * kNCW);
    int* shi = reinterpret_cast<int*>(shv + kNCW);
    if (lane == 0) { shv[warp] = bv; shi[warp] = bi; }
    named_sync(1, nthreads);
    float mxv = shv[0];
    int mxi = shi[0];
    for (int w = 1; w < kNCW; ++w)
      if (shv[w] > mxv || (shv[w] == mxv && shi[w] < mxi)) { mxv = shv[w]; mxi = shi[w]; }
    const double mx = mxv;
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < P.vocab; i += nthreads) s += exp(static_cast<double>(l[i]) - mx);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    named_sync(1, nthreads);
    if (lane == 0) shd[warp] = s;
    named_sync(1, nthreads);
    double sum = 0.0;
    for (int w = 0; w < kNCW; ++w) sum += shd[w];
    double h = 0.0, t1 = -1.0, t2 = -1.0;
    for (int64_t i = threadIdx.x; i < P.vocab; i += nthreads) {
      const double p = exp(static_cast<double>(l[i]) - mx) / sum;
      if (p > 0.0) h -= p * log(p);
      if (p > t1) { t2 = t1; t1 = p; } else if (p > t2) { t2 = p; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      h += __shfl_xor_sync(0xffffffffu, h, o);
      const double o1 = __shfl_xor_sync(0xffffffffu, t1, o), o2 = __shfl_xor_sync(0xffffffffu, t2, o);
      const double n1 = fmax(t1, o1), n2 = fmax(fmin(t1, o1), fmax(t2, o2));
      t1 = n1;
      t2 = n2;
    }
    named_sync(1, nthreads);
    if (lane == 0) { shd[warp] = h; shd[kNCW + warp] = t1; shd[2 * kNCW + warp] = t2; }
    named_sync(1, nthreads);
    if (threadIdx.x == 0) {
      double H = 0.0, a1 = -1.0, a2 = -1.0;
      for (int w = 0; w < kNCW; ++w) {
        H += shd[w];
        const double n1 = fmax(a1, shd[kNCW + w]), n2 = fmax(fmin(a1, shd[kNCW + w]), fmax(a2, shd[2 * kNCW + w]));
        a1 = n1;
        a2 = n2;
      }
      fq_row_stats st;
      st.entropy = H;
      st.ppl_entropy = exp(H);
      st.p1 = a1;
      st.p2 = a2;
      st.fault_tolerance = a1 - a2;
      st.max_logit = mxv;
      st.argmax = mxi;
      P.stats[b] = st;
    }
    named_sync(1, nthreads);
  }
}

// ---------------------------------------------------------------- grid barrier (consumers)
__device__ void grid_barrier(unsigned int* counter, unsigned int& epoch) {
  named_sync(1, kNCW * 32);
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(counter, 1u);
    const unsigned int target = (++epoch) * gridDim.x;
    while (ld_acquire(counter) < target) __nanosleep(32);
    __threadfence();
  } else {
    ++epoch;
  }
  named_sync(1, kNCW * 32);
}

// ---------------------------------------------------------------- the program kernel
template <int BB>
__device__ void run_program(const Phase* phases, int nphases, unsigned int* barrier, int stage_bytes, int nstages,
                            int red_floats, int xs_floats) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ float sq_red[kMaxB][kNCW];
  __shared__ AttnSmem attn_smem[kNCW / 4];
  __shared__ double stat_smem[5 * kNCW];
  Ring R;
  R.base = smem;
  R.full = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(nstages) * stage_bytes);
  R.empty = R.full + kMaxStages;
  R.stage_bytes = stage_bytes;
  R.nstages = nstages;
  float* red = reinterpret_cast<float*>(R.empty + kMaxStages);
  float4* xsm = reinterpret_cast<float4*>(red + ((red_floats + 3) & ~3));
  float* sigm = reinterpret_cast<float*>(xsm + xs_floats / 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nstages; ++s) {
      mbar_init(&R.full[s], 1);
      mbar_init(&R.empty[s], kNCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == kNCW) {
    // the weight stream depends on nothing produced at run time: start immediately
    if (lane == 0) {
      int slot_i = 0;
      uint32_t phase_bit = 0;
      for (int i = 0; i < nphases; ++i)
        if (phases[i].type == PH_GEMV) produce_phase(phases[i], R, slot_i, phase_bit);
    }
    return;
  }
  pdl_wait();
  int slot_i = 0;
  uint32_t phase_bit = 0;
  unsigned int epoch = 0;
  for (int i = 0; i < nphases; ++i) {
    const Phase& P = phases[i];
    if (P.type == PH_GEMV) run_gemv_phase<BB>(P, R, red, sq_red, xsm, sigm, slot_i, phase_bit);
    else if (P.type == PH_EMBED) run_embed(P, sq_red);
    else if (P.type == PH_ATTN) run_attn(P, attn_smem);
    else run_stats(P, stat_smem);
    if (P.barrier_after && i + 1 < nphases) grid_barrier(barrier, epoch);
  }
}

template <int BB>
__global__ void __launch_bounds__(kThreads, 1) program_kernel(const Phase* phases, int nphases, unsigned int* barrier,
                                                              int stage_bytes, int nstages, int red_floats,
                                                              int xs_floats) {
  run_program<BB>(phases, nphases, barrier, stage_bytes, nstages, red_floats, xs_floats);
}

template <int BB>
__global__ void __launch_bounds__(kThreads, 1) program_kernel_inline(const __grid_constant__ InlineProgram prog,
                                                                     int nphases, unsigned int* barrier,
                                                                     int stage_bytes, int nstages, int red_floats,
                                                                     int xs_floats) {
  run_program<BB>(prog.phases, nphases, barrier, stage_bytes, nstages, red_floats, xs_floats);
}

template <int BB>
void launch_t(fq_ctx* ctx, const ProgramRun& run, unsigned int* barrier, bool pdl) {
  static std::mutex mu;
  static bool configured = false;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!configured) {
      FQ_CUDA(cudaFuncSetAttribute(program_kernel<BB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      FQ_CUDA(cudaFuncSetAttribute(program_kernel_inline<BB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      configured = true;
    }
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(run.grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = run.smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  if (run.dev_phases)
    FQ_CUDA(cudaLaunchKernelEx(&cfg, program_kernel<BB>, static_cast<const Phase*>(run.dev_phases), run.nphases,
                               barrier, run.stage_bytes, run.nstages, run.red_floats, run.xs_floats));
  else
    FQ_CUDA(cudaLaunchKernelEx(&cfg, program_kernel_inline<BB>, run.inl, run.nphases, barrier, run.stage_bytes,
                               run.nstages, run.red_floats, run.xs_floats));
  ctx->launches += 1;
}

}  // namespace

ProgramRun upload_program(fq_ctx* ctx, const ProgramBuilder& pb, bool transient) {
  ProgramRun r;
  r.nphases = static_cast<int>(pb.phases.size());
  r.grid = pb.grid;
  r.bb = pb.max_bb;
  const int64_t stage = std::max<int64_t>(pb.stage_bytes, 128);
  r.red_floats = static_cast<int>((pb.red_floats + 3) & ~int64_t(3));
  const int bbk = pb.max_bb <= 1 ? 1 : (pb.max_bb <= 2 ? 2 : 4);  // kernel instantiation's batch bound
  r.xs_floats = static_cast<int>(static_cast<int64_t>(pb.max_nsteps) * kStepCodes * bbk);
  const size_t red_bytes = static_cast<size_t>(r.red_floats) * sizeof(float);
  const size_t xs_bytes = static_cast<size_t>(r.xs_floats) * sizeof(float) +
                          static_cast<size_t>(pb.max_nsteps) * 32 * bbk * sizeof(float);
  const int64_t budget = 200 * 1024 - static_cast<int64_t>(red_bytes + xs_bytes) - 2 * kMaxStages * 8 - 256;
  r.nstages = static_cast<int>(std::min<int64_t>(kMaxStages, budget / stage));
  if (r.nstages < 2) fail(FQ_E_CONFIG, "gemv: layer rows too large for the shared-memory ring");
  r.stage_bytes = static_cast<int>(stage);
  r.smem = static_cast<size_t>(r.nstages) * r.stage_bytes + 2 * kMaxStages * 8 + red_bytes + xs_bytes;
  if (r.nphases <= kInlinePhases && transient) {
    for (int i = 0; i < r.nphases; ++i) r.inl.phases[i] = pb.phases[i];
  } else {
    r.dev_phases = static_cast<Phase*>(dmalloc(sizeof(Phase) * r.nphases));
    FQ_CUDA(cudaMemcpyAsync(r.dev_phases, pb.phases.data(), sizeof(Phase) * r.nphases, cudaMemcpyHostToDevice,
                            ctx->stream));
    FQ_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  return r;
}

void launch_program(fq_ctx* ctx, const ProgramRun& run, unsigned int* barrier, bool pdl) {
  if (run.bb <= 1) launch_t<1>(ctx, run, barrier, pdl);
  else if (run.bb == 2) launch_t<2>(ctx, run, barrier, pdl);
  else launch_t<4>(ctx, run, barrier, pdl);
}

}  // namespace fqc
