// Dequant-fused weight-only GEMV over resident W8/W4 copies (K1/K2 of SURVEY §2.1).
//
// Replaces MultiPrecisionLayer::forward (/root/reference/proj/src/model.cpp:77-98), which
// dequantizes the active rung (src/quantizer.cpp:205-219) and runs a double-accumulated
// linear (src/tensor.cpp:83-101).  Two numerics:
//
//  * fast  — the decode hot path, a TMA-fed streaming kernel:
//      - one CTA per SM owns a balanced, contiguous row range of every matrix of the launch;
//        that range is one contiguous byte range of the row-major payload (plus its padded
//        scale / zero-point rows), so a producer warp streams it through a shared-memory ring
//        with 1-D TMA bulk copies (cp.async.bulk + mbarrier complete_tx).  Bytes in flight per
//        SM are set by the ring size, not by registers.  The producer never depends on the
//        previous kernel, so under programmatic dependent launch it starts pulling weights
//        while the previous kernel is still finishing.
//      - consumer warps split the K-steps of a row (512 codes per step, 16 per lane) and keep
//        their activations in registers for the whole kernel.  Unpacking is one LOP/SHF per
//        code: the masked code bits (q << s), s < 24, reinterpreted as fp32 are exactly
//        q * 2^(s-149) (subnormal / first binade), so an FFMA2 with x * 2^(109-s) accumulates
//        q*x*2^-40 without any int->float conversion.  The zero point is folded per group:
//        sum_j (q_j - z) x_j = sum_j q_j x_j - z * sum_j x_j.
//      - fp32 accumulation; deterministic (fixed reduction order, no atomics).
//  * exact — golden/parity mode: one thread per output, w = float(code - z) * s in fp32 as
//    dequantize() does, then a sequential double accumulation in k order as linear() does:
//    bit-identical to the reference.  Any group size, fp rung, bias.
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
constexpr int kMaxStages = 8;
constexpr int kSplit = 8;  // consumer warps splitting the K-steps of a row
constexpr float kTwo109 = 649037107316853453566312041152512.0f;  // 2^109
constexpr float kTwo40 = 1099511627776.0f;                        // 2^40
constexpr float kTwoM40 = 9.094947017729282379150390625e-13f;     // 2^-40

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

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
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
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ float f32(uint32_t u) { return __uint_as_float(u); }

// Bit shift (s) of code j of a 16-code segment after extraction, per bit-width.
__host__ __device__ constexpr int seg_shift(int bits, int j) {
  return bits == 8 ? ((j & 3) == 3 ? 0 : 8 * (j & 3)) : ((j & 7) < 6 ? 4 * (j & 7) : 4 * ((j & 7) - 6));
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
  a.x += b.x;
  a.y += b.y;
  return a.x + a.y;
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

// ---------------------------------------------------------------- launch descriptor
struct DevMat {
  const uint8_t* payload[2];  // [0] = W8, [1] = W4
  const float* scale[2];
  const uint8_t* zp[2];
  int32_t zpbase[2];
  const uint8_t* rung_table;  // per batch row, or null
  int64_t rung_stride;
  int rung;                   // when no table
  void* y;
};

struct DevArgs {
  DevMat mat[3];
  int nmat;
  int B;
  int64_t N, K, G, ng_pad, zp_pad;
  int nsteps;
  int rows_per_stage[2];  // [0] = W8, [1] = W4
  int sc_off[2], zp_off[2];  // byte offsets of the scale / zero-point blocks in a slot
  int sc_row, zp_row;        // bytes per row of the scale / zero-point blocks
  int stage_bytes;        // ring slot size (bytes, multiple of 128)
  int nstages;
  const void* x;
  int x_dtype;
  int64_t x_stride;
  const float* norm_gain;
  const float* norm_partials;
  int n_partials;
  int partials_stride;
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

// Batch-row mask (bit b) of matrix m wanting bit-width slot w (0 = W8, 1 = W4).
__device__ __forceinline__ int pass_mask(const DevArgs& a, int m, int w) {
  int mask = 0;
  const int want = w == 0 ? FQ_RUNG_INT8 : FQ_RUNG_INT4;
  for (int b = 0; b < a.B; ++b) mask |= (mat_rung(a.mat[m], b) == want) << b;
  return mask;
}

// One ring slot (per bit-width w): [payload: rows_pad rows][scales: rows_pad x ng_pad f32]
// [zero points: rows_pad x zp_pad u8]; rows_pad = rows per stage rounded up to 4.  A partial
// stage copies fewer rows; the trailing rows are stale and their results are discarded.
struct StageLayout {
  int rows;
  int row_bytes;
  uint32_t pay_bytes, sc_bytes, zp_bytes;  // bytes actually copied
};
__device__ __forceinline__ StageLayout stage_layout(const DevArgs& a, int w, int rows) {
  StageLayout L;
  L.rows = rows;
  L.row_bytes = static_cast<int>(w == 0 ? a.K : a.K / 2);
  L.pay_bytes = static_cast<uint32_t>(rows * L.row_bytes);
  L.sc_bytes = static_cast<uint32_t>(rows * a.ng_pad * 4);
  L.zp_bytes = static_cast<uint32_t>(rows * a.zp_pad);
  return L;
}

template <int SW, int BB>
__device__ __forceinline__ void load_acts(const DevArgs& a, int bits, const bool (&step_ok)[SW], const int (&seg_k)[SW],
                                          const float (&rstd)[BB], float (&xs)[SW][BB][kSegCodes],
                                          float (&sig)[SW][BB]) {
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
        const float sc8 = kTwo109 / static_cast<float>(1u << seg_shift(8, j));
        const float sc4 = kTwo109 / static_cast<float>(1u << seg_shift(4, j));
        xs[s][b][j] = v * (bits == 8 ? sc8 : sc4);
      }
      sig[s][b] = acc * kTwoM40;
    }
  }
}

// Reduces v[0..3] (four rows) across the 32 lanes with 6 shuffles; afterwards lane l holds the
// warp sum of row ((l >> 3) & 3).
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

// Consumes one ring slot holding `nrows` rows at bit-width BITS.  Lane-constant offsets:
// pay_l = byte offset of the lane's segment in a row, sc_l / zp_l = the lane's group column.
// red_row points at red[(first row)][warp][0] of this slot; rows are W*BB floats apart.
template <int BITS, int SW, int BB, int RG>
__device__ __forceinline__ void consume_stage(const uint8_t* __restrict__ slot, int nrows, int rg, int row_bytes,
                                              int sc_off, int zp_off, int sc_row, int zp_row,
                                              const int (&pay_l)[SW], const int (&sc_l)[SW], const int (&zp_l)[SW],
                                              float zmagic, const float (&xs)[SW][BB][kSegCodes],
                                              const float (&sig)[SW][BB], float* red_row, int bmask, int lane) {
  const uint8_t* pa = slot + rg * 4 * row_bytes;
  const uint8_t* sa = slot + sc_off + rg * 4 * sc_row;
  const uint8_t* za = slot + zp_off + rg * 4 * zp_row;
  const int red_step = kSplit * BB;
  for (int r0 = rg * 4; r0 < nrows; r0 += 4 * RG) {
    float acc[BB][4];
#pragma unroll
    for (int b = 0; b < BB; ++b)
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[b][u] = 0.f;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int s = 0; s < SW; ++s) {
        const float sc = *reinterpret_cast<const float*>(sa + u * sc_row + sc_l[s]);
        const uint32_t zq = za[u * zp_row + zp_l[s]];
        const float zf = __uint_as_float(0x4B000000u | zq) - zmagic;  // exact: zq + zp_base
        float p[BB];
        if constexpr (BITS == 8) {
          const uint4 w = *reinterpret_cast<const uint4*>(pa + u * row_bytes + pay_l[s]);
#pragma unroll
          for (int b = 0; b < BB; ++b) p[b] = dot_seg8(w, xs[s][b]);
        } else {
          const uint2 w = *reinterpret_cast<const uint2*>(pa + u * row_bytes + pay_l[s]);
#pragma unroll
          for (int b = 0; b < BB; ++b) p[b] = dot_seg4(w, xs[s][b]);
        }
#pragma unroll
        for (int b = 0; b < BB; ++b) acc[b][u] = fmaf(sc, fmaf(-zf, sig[s][b], p[b]), acc[b][u]);
      }
    }
    const int u = (lane >> 3) & 3;
#pragma unroll
    for (int b = 0; b < BB; ++b) {
      const float v = reduce4(acc[b], lane);
      if ((lane & 7) == 0 && r0 + u < nrows && ((bmask >> b) & 1)) red_row[(r0 + u) * red_step + b] = v;
    }
    pa += 4 * RG * row_bytes;
    sa += 4 * RG * sc_row;
    za += 4 * RG * zp_row;
  }
}

// Fast kernel.  SW = K-steps per consumer warp, BB = batch rows (compile-time bounds).
template <int SW, int BB, int RG>
__global__ void __launch_bounds__((kSplit * RG + 1) * 32, RG == 1 ? 2 : 1) gemv_tma_kernel(const DevArgs a) {
  constexpr int NCW = kSplit * RG;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(a.nstages) * a.stage_bytes);
  uint64_t* empty = full + kMaxStages;
  float* red = reinterpret_cast<float*>(empty + kMaxStages);
  __shared__ float sq_red[kMaxB][NCW + 1];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int cta = blockIdx.x;
  const int ncta = gridDim.x;
  const int64_t r0 = (a.N * cta) / ncta;
  const int64_t r1 = (a.N * (cta + 1)) / ncta;
  const int rows = static_cast<int>(r1 - r0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < a.nstages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // Let the next kernel of the stream become resident beside this one (two CTAs fit per SM):
  // its producer warp then streams the next weights while this kernel finishes.
  pdl_launch_dependents();

  if (warp == NCW) {
    // ---------------- producer: stream this CTA's rows of every matrix through the ring
    if (lane == 0 && rows > 0) {
      int t = 0;
      for (int m = 0; m < a.nmat; ++m) {
        for (int w = 0; w < 2; ++w) {
          if (pass_mask(a, m, w) == 0) continue;
          const int rps = a.rows_per_stage[w];
          const DevMat& M = a.mat[m];
          for (int rb = 0; rb < rows; rb += rps, ++t) {
            const int s = t % a.nstages;
            const uint32_t ph = (t / a.nstages) & 1;
            mbar_wait(&empty[s], ph ^ 1);
            const StageLayout L = stage_layout(a, w, min(rps, rows - rb));
            uint8_t* dst = ring + static_cast<size_t>(s) * a.stage_bytes;
            const int64_t row = r0 + rb;
            mbar_expect_tx(&full[s], L.pay_bytes + L.sc_bytes + L.zp_bytes);
            bulk_g2s(dst, M.payload[w] + row * L.row_bytes, L.pay_bytes, &full[s]);
            bulk_g2s(dst + a.sc_off[w], M.scale[w] + row * a.ng_pad, L.sc_bytes, &full[s]);
            bulk_g2s(dst + a.zp_off[w], M.zp[w] + row * a.zp_pad, L.zp_bytes, &full[s]);
          }
        }
      }
    }
    pdl_wait();  // the epilogue below reads buffers written by the previous kernel
  } else {
    // ---------------- consumers
    bool step_ok[SW];
    int seg_k[SW];
    int gidx[SW];
#pragma unroll
    for (int s = 0; s < SW; ++s) {
      const int step = (warp % kSplit) + s * kSplit;
      seg_k[s] = step * kStepCodes + lane * kSegCodes;
      step_ok[s] = step < a.nsteps && seg_k[s] < a.K;
      gidx[s] = step_ok[s] ? static_cast<int>(seg_k[s] / a.G) : 0;
      if (!step_ok[s]) seg_k[s] = 0;
    }
    pdl_wait();  // activations come from the previous kernel
    float rstd[BB];
#pragma unroll
    for (int b = 0; b < BB; ++b) {
      rstd[b] = 1.f;
      if (a.norm_gain != nullptr && b < a.B) {
        float s = 0.f;
        for (int i = lane; i < a.n_partials; i += 32) s += a.norm_partials[b * a.partials_stride + i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        rstd[b] = 1.0f / sqrtf(s / static_cast<float>(a.K) + a.norm_eps);
      }
    }
    float xs[SW][BB][kSegCodes];
    float sig[SW][BB];
    int xs_bits = 0;
    int t = 0;
    for (int m = 0; m < a.nmat; ++m) {
      for (int w = 0; w < 2; ++w) {
        const int bmask = pass_mask(a, m, w);
        if (bmask == 0 || rows == 0) continue;
        const int bits = w == 0 ? 8 : 4;
        if (xs_bits != bits) {
          load_acts<SW, BB>(a, bits, step_ok, seg_k, rstd, xs, sig);
          xs_bits = bits;
        }
        const float zmagic = 8388608.0f - static_cast<float>(a.mat[m].zpbase[w]);
        const int rps = a.rows_per_stage[w];
        const int row_bytes = static_cast<int>(w == 0 ? a.K : a.K / 2);
        int pay_l[SW], sc_l[SW], zp_l[SW];
#pragma unroll
        for (int s = 0; s < SW; ++s) {
          pay_l[s] = w == 0 ? seg_k[s] : seg_k[s] / 2;
          sc_l[s] = gidx[s] * 4;
          zp_l[s] = gidx[s];
        }
        for (int rb = 0; rb < rows; rb += rps, ++t) {
          const int s = t % a.nstages;
          const uint32_t ph = (t / a.nstages) & 1;
          mbar_wait(&full[s], ph);
          const uint8_t* slot = ring + static_cast<size_t>(s) * a.stage_bytes;
          float* red_row = red + ((m * rows + rb) * kSplit + (warp % kSplit)) * BB;
          const int nr = min(rps, rows - rb);
          if (bits == 8)
            consume_stage<8, SW, BB, RG>(slot, nr, warp / kSplit, row_bytes, a.sc_off[0], a.zp_off[0], a.sc_row, a.zp_row, pay_l, sc_l,
                                     zp_l, zmagic, xs, sig, red_row, bmask, lane);
          else
            consume_stage<4, SW, BB, RG>(slot, nr, warp / kSplit, row_bytes, a.sc_off[1], a.zp_off[1], a.sc_row, a.zp_row, pay_l, sc_l,
                                     zp_l, zmagic, xs, sig, red_row, bmask, lane);
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[s]);
        }
      }
    }
  }
  __syncthreads();

  // ---------------- cross-warp reduction in warp order + epilogue
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
      for (int w = 0; w < kSplit; ++w) s += red[((m * rows + r) * kSplit + w) * BB + b];
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
      for (int w = 0; w <= NCW; ++w) s += sq_red[threadIdx.x][w];
      a.out_partials[threadIdx.x * a.out_n_partials + cta] = s;
    }
  }
}

// Exact kernel: one thread per (row, batch row); sequential k, double accumulation.
__global__ void gemv_exact_kernel(const int64_t N, const int64_t K, const int64_t G, const int64_t ng,
                                  const int64_t ng_pad, const int bits, const uint8_t* payload, const float* scale,
                                  const int32_t* zp, const float* fpw, const float* bias, const int B, const void* x,
                                  const int x_dtype, void* y, const int y_dtype) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= N * B) return;
  const int64_t row = t % N;
  const int b = static_cast<int>(t / N);
  double acc = bias ? static_cast<double>(bias[row]) : 0.0;
  for (int64_t k = 0; k < K; ++k) {
    float w;
    if (bits == 0) {
      w = fpw[row * K + k];
    } else {
      const int64_t idx = row * K + k;
      uint32_t code;
      if (bits == 8) code = payload[idx];
      else code = (idx & 1) ? (payload[idx >> 1] >> 4) : (payload[idx >> 1] & 0xFu);
      const int64_t g = k / G;
      w = static_cast<float>(static_cast<int32_t>(code) - zp[row * ng + g]) * scale[row * ng_pad + g];
    }
    acc += static_cast<double>(load_act(x, x_dtype, b * K + k)) * static_cast<double>(w);
  }
  store_out(y, y_dtype, b * N + row, static_cast<float>(acc));
}

struct Plan {
  int sw;
  int rg;
  int grid;
  int rps[2];
  int sc_off[2], zp_off[2];
  int stage_bytes;
  int nstages;
  size_t smem;
};

Plan plan_fast(const fq_ctx* ctx, const fq_layer* L, int nmat, int bb) {
  Plan p{};
  const int nsteps = ceil_div_i(L->K, kStepCodes);
  p.sw = (nsteps + kSplit - 1) / kSplit;
  p.rg = 1;  // 9 warps x <= 112 registers: two CTAs (this kernel + the next) co-reside per SM
  p.grid = static_cast<int>(std::min<int64_t>(ctx->num_sms, L->N));
  const int64_t rows_max = (L->N + p.grid - 1) / p.grid;
  const int64_t target = 24 * 1024;
  int64_t slot = 0;
  for (int w = 0; w < 2; ++w) {
    const int64_t row_bytes = w == 0 ? L->K : L->K / 2;
    const int64_t per_row = row_bytes + L->ng_pad * 4 + L->zp_pad;
    int rps = static_cast<int>(std::max<int64_t>(1, target / per_row));
    rps = std::min(rps, 16);
    const int quantum = 4 * p.rg;
    rps = rps >= quantum ? rps / quantum * quantum : quantum;
    const int64_t pad = (rps + 3) / 4 * 4;
    p.rps[w] = rps;
    p.sc_off[w] = static_cast<int>(pad * row_bytes);
    p.zp_off[w] = static_cast<int>(pad * row_bytes + pad * L->ng_pad * 4);
    slot = std::max<int64_t>(slot, pad * per_row);
  }
  p.stage_bytes = static_cast<int>((slot + 127) / 128 * 128);
  const size_t red_bytes = static_cast<size_t>(nmat) * rows_max * kSplit * bb * sizeof(float);
  const int64_t budget = 100 * 1024 - static_cast<int64_t>(red_bytes) - 2 * kMaxStages * 8 - 256;
  p.nstages = static_cast<int>(std::min<int64_t>(kMaxStages, budget / p.stage_bytes));
  if (p.nstages < 2) fail(FQ_E_CONFIG, "gemv: layer rows too large for the shared-memory ring");
  p.smem = static_cast<size_t>(p.nstages) * p.stage_bytes + 2 * kMaxStages * 8 + red_bytes;
  return p;
}

template <int SW, int BB, int RG>
void launch_fast_t(fq_ctx* ctx, const DevArgs& d, const Plan& p, bool pdl) {
  auto kern = gemv_tma_kernel<SW, BB, RG>;
  static std::mutex mu;
  static bool configured = false;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!configured) {
      FQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024));
      configured = true;
    }
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.grid);
  cfg.blockDim = dim3((kSplit * RG + 1) * 32);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  FQ_CUDA(cudaLaunchKernelEx(&cfg, kern, d));
  ctx->launches += 1;
}

template <int SW>
void launch_fast_sw(fq_ctx* ctx, const DevArgs& d, const Plan& p, bool pdl) {
  if constexpr (SW == 1) {
    if (d.B == 1) {
      if (p.rg == 2) launch_fast_t<SW, 1, 2>(ctx, d, p, pdl);
      else launch_fast_t<SW, 1, 1>(ctx, d, p, pdl);
    } else if (d.B == 2) {
      launch_fast_t<SW, 2, 1>(ctx, d, p, pdl);
    } else {
      launch_fast_t<SW, 4, 1>(ctx, d, p, pdl);
    }
  } else if constexpr (SW == 2) {
    if (d.B == 1) launch_fast_t<SW, 1, 1>(ctx, d, p, pdl);
    else launch_fast_t<SW, 2, 1>(ctx, d, p, pdl);
  } else {
    launch_fast_t<SW, 1, 1>(ctx, d, p, pdl);
  }
}

}  // namespace

bool gemv_fast_supported(const fq_layer* L, int rung) {
  if (rung != FQ_RUNG_INT8 && rung != FQ_RUNG_INT4) return false;
  const fq_rung_store& s = L->store(rung);
  const int nsteps = ceil_div_i(L->K, kStepCodes);
  return s.present && s.zp_fits_u8 && L->K % 32 == 0 && L->G % kSegCodes == 0 && L->G >= kSegCodes &&
         nsteps <= 4 * kSplit;
}

int gemv_fast_grid(const fq_ctx* ctx, int64_t N) {
  return static_cast<int>(std::min<int64_t>(ctx->num_sms, N));
}

int launch_gemv_fast(fq_ctx* ctx, const GemvLaunch& g) {
  const fq_layer* L0 = g.mat[0].layer;
  DevArgs d = {};
  d.nmat = g.nmat;
  d.N = L0->N;
  d.K = L0->K;
  d.G = L0->G;
  d.ng_pad = L0->ng_pad;
  d.zp_pad = L0->zp_pad;
  d.nsteps = ceil_div_i(L0->K, kStepCodes);
  d.x = g.x;
  d.x_dtype = g.x_dtype;
  d.x_stride = g.x_stride ? g.x_stride : L0->K;
  d.norm_gain = g.norm_gain;
  d.norm_partials = g.norm_partials;
  d.n_partials = g.n_partials;
  d.partials_stride = g.partials_stride ? g.partials_stride : g.n_partials;
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
    const fq_rung_store* st[2] = {&L->r8, &L->r4};
    for (int w = 0; w < 2; ++w) {
      M.payload[w] = st[w]->payload;
      M.scale[w] = st[w]->scale;
      M.zp[w] = st[w]->zp8;
      M.zpbase[w] = st[w]->zp_base;
    }
    M.rung_table = g.mat[m].rung_table;
    M.rung_stride = g.mat[m].rung_stride;
    M.rung = g.mat[m].rung;
    M.y = g.mat[m].y;
  }
  const int sw0 = (d.nsteps + kSplit - 1) / kSplit;
  const int64_t bchunk = sw0 == 1 ? kMaxB : (sw0 == 2 ? 2 : 1);
  const int64_t bb = std::min<int64_t>(bchunk, g.batch);
  const Plan p = plan_fast(ctx, L0, g.nmat, static_cast<int>(bb == 3 ? 4 : bb));
  d.rows_per_stage[0] = p.rps[0];
  d.rows_per_stage[1] = p.rps[1];
  for (int w = 0; w < 2; ++w) {
    d.sc_off[w] = p.sc_off[w];
    d.zp_off[w] = p.zp_off[w];
  }
  d.sc_row = static_cast<int>(L0->ng_pad * 4);
  d.zp_row = static_cast<int>(L0->zp_pad);
  d.stage_bytes = p.stage_bytes;
  d.nstages = p.nstages;
  if (g.epi == EPI_RESIDUAL && g.out_n_partials < p.grid) fail(FQ_E_STATE, "gemv: residual partial buffer too small");
  d.out_n_partials = g.out_n_partials;
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
    if (g.norm_partials) c.norm_partials = g.norm_partials + b0 * d.partials_stride;
    switch (p.sw) {
      case 1: launch_fast_sw<1>(ctx, c, p, g.pdl); break;
      case 2: launch_fast_sw<2>(ctx, c, p, g.pdl); break;
      case 3: launch_fast_sw<3>(ctx, c, p, g.pdl); break;
      default: launch_fast_sw<4>(ctx, c, p, g.pdl); break;
    }
  }
  return p.grid;
}

void launch_gemv_exact(fq_ctx* ctx, const fq_layer* L, int rung, int64_t batch, const void* x, int x_dtype, void* y,
                       int y_dtype) {
  if (!L->has(rung)) fail(FQ_E_STATE, "gemv: rung not resident on the device");
  const int threads = 128;
  const int64_t n = L->N * batch;
  const fq_rung_store* s = rung == FQ_RUNG_FP ? nullptr : &L->store(rung);
  gemv_exact_kernel<<<ceil_div_i(n, threads), threads, 0, ctx->stream>>>(
      L->N, L->K, L->G, L->ng, L->ng_pad, s ? s->bits : 0, s ? s->payload : nullptr, s ? s->scale : nullptr,
      s ? s->zp32 : nullptr, L->fp, L->bias, static_cast<int>(batch), x, x_dtype, y, y_dtype);
  FQ_CUDA(cudaGetLastError());
  ctx->launches += 1;
}

}  // namespace fqc
