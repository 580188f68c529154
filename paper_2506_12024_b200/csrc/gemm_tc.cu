// Prefill / calibration contraction on the 5th-generation tensor cores (tcgen05 + TMEM):
//   Y[T, N] (fp32) = X[T, K] (bf16) . dequant(W_rung[N, K])^T
// straight from the tiled W8 / W4 copy the decode GEMV streams (fq_internal.cuh), so prefill and
// calibration use the same resident weights.  This is the dense contraction of SURVEY §7 step 6
// (BASELINE config 4): MultiPrecisionLayer::forward on many rows at once
// (/root/reference/proj/src/model.cpp:77-98 = dequantize src/quantizer.cpp:205-219 + linear
// src/tensor.cpp:83-101).
//
// One CTA = 128 weight rows x 256 tokens, 8 warps:
//   * every k-step (128 codes = one quantization group) all threads dequantize the 8 tiled
//     16x128 blocks of the CTA's rows to bf16 (q - z) * s into shared memory in the UMMA canonical
//     K-major layout (no swizzle: 8x16-byte core matrices, LBO = 128 B along K, SBO = 2 KB along
//     M/N), while the 256x128 bf16 activation tile arrives by cp.async in the same layout;
//   * one elected thread issues 8 tcgen05.mma (M=128, N=256, K=16, fp32 accumulate in TMEM) and
//     commits them to the stage's mbarrier; two stages, so the dequantisation of step k+1
//     overlaps the MMAs of step k;
//   * the global loads of step k+1 (code words, scales, activations) are issued into registers
//     before step k's operands are written, so their latency hides behind the previous step;
//   * epilogue: tcgen05.ld of the 128x128 fp32 accumulator (warps w and w+4 read TMEM lanes
//     32w..32w+31, half of the token columns each).
#include "gemv_program.cuh"

namespace fqc {
namespace {

#ifndef FQ_GEMM_TN
#define FQ_GEMM_TN 256
#endif
#ifndef FQ_GEMM_STAGES
#define FQ_GEMM_STAGES 2
#endif
constexpr int kTM = 128;   // weight rows per CTA (UMMA M)
constexpr int kTN = FQ_GEMM_TN;  // tokens per CTA (UMMA N)
constexpr int kStagesG = FQ_GEMM_STAGES;  // smem stages: activations are loaded kStagesG - 1 k-steps ahead
constexpr int kTK = 128;   // codes per k-step (one tiled block / quantization group)
constexpr int kATileBytes = kTM * kTK * 2;  // bf16 weight tile: 32 KB
constexpr int kBTileBytes = kTN * kTK * 2;  // bf16 activation tile: 64 KB
constexpr int kStageBytesG = kATileBytes + kBTileBytes;
constexpr int kGemmThreads = 256;

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// canonical K-major no-swizzle offset of element (row, k) inside a 128x128 fp16 tile
__device__ __forceinline__ uint32_t kmajor_off(int row, int k) {
  return static_cast<uint32_t>((row >> 3) * 2048 + (k >> 3) * 128 + (row & 7) * 16 + (k & 7) * 2);
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);          // start address
  d |= static_cast<uint64_t>(128u >> 4) << 16;                  // LBO: K-adjacent core matrices
  d |= static_cast<uint64_t>(2048u >> 4) << 32;                 // SBO: 8-row groups
  d |= static_cast<uint64_t>(1u) << 46;                         // descriptor version (sm_100)
  return d;                                                     // base offset 0, SWIZZLE_NONE
}

// kind::f16 instruction descriptor: D f32, A/B bf16 (F16 = 0) or fp16 (F16 = 1), both K-major,
// N = kTN, M = kTM
template <int F16>
constexpr uint32_t idesc() {
  return (1u << 4) | ((F16 ? 0u : 1u) << 7) | ((F16 ? 0u : 1u) << 10) | ((kTN >> 3) << 17) | ((kTM >> 4) << 24);
}

__device__ __forceinline__ void mbar_init1(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)));
}
__device__ __forceinline__ void mbar_wait1(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  unsigned long long t0 = 0;
  for (uint32_t spins = 0;; ++spins) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    if (ok) return;
    if ((spins & 1023u) == 1023u) {  // deadlock watchdog: report and trap instead of hanging
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t0 == 0) t0 = t;
      else if (t - t0 > 4000000000ull) {
        printf("fq gemm watchdog: mma barrier stuck (cta %d,%d parity %u)\n", blockIdx.x, blockIdx.y, parity);
        __trap();
      }
    }
  }
}

template <int F16>
__device__ __forceinline__ uint32_t pack_b2(float a, float b) {
  if constexpr (F16) {
    const __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
  } else {
    const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
  }
}

// Global-side raw data of one k-step for one thread: its 16-byte code words of the 8 tiled blocks
// (+ the two rows' scale / zero point) and its 16-byte chunks of the activation tile.  Loaded one
// k-step ahead (registers), so the global latency hides behind the previous step.
template <int W>
struct StepRaw {
  static constexpr int kWords = W == 0 ? 4 : 2;                       // 16-byte code words per lane per block
  static constexpr int kA = 8 * kWords * 32 / kGemmThreads;           // per thread
  uint4 w[kA];
  float s0[kA], s1[kA], z0[kA], z1[kA];
};

// Activation tile of a k-step straight into shared memory (cp.async, 16-byte chunks = one core-
// matrix row; rows past T / codes past K are zero-filled), bf16 as stored.
__device__ __forceinline__ void load_tokens_async(const uint16_t* __restrict__ x, int64_t x_stride, int T, int64_t K,
                                                  int t0, int kb, uint8_t* b_tile) {
#pragma unroll 4
  for (int it = threadIdx.x; it < kTN * (kTK / 8); it += kGemmThreads) {
    const int tok = it >> 4, kc = it & 15;
    const int t = t0 + tok;
    const int64_t k = static_cast<int64_t>(kb) * kTK + kc * 8;
    const bool in = t < T && k < K;
    const uint16_t* src = in ? x + static_cast<int64_t>(t) * x_stride + k : x;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(b_tile + kmajor_off(tok, kc * 8))),
                 "l"(src), "r"(in ? 16 : 0)
                 : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

template <int W>
__device__ __forceinline__ void load_step(const uint8_t* __restrict__ tiles, int64_t tile0, int n_tiles, int nkb, int kb,
                                          int32_t zbase, StepRaw<W>& r) {
  constexpr int bb = W == 0 ? kBlockBytes8 : kBlockBytes4;
  constexpr int cbytes = W == 0 ? 2048 : 1024;
  constexpr int words = StepRaw<W>::kWords;
#pragma unroll
  for (int u = 0; u < StepRaw<W>::kA; ++u) {
    const int it = threadIdx.x + u * kGemmThreads;
    const int rt = it / (words * 32), rem = it - rt * words * 32;
    const int i = rem >> 5, t = rem & 31;
    const int64_t tile = min(tile0 + rt, static_cast<int64_t>(n_tiles) - 1);  // rows past N masked at store
    const uint8_t* blk = tiles + (tile * nkb + kb) * bb;
    const int rr = t >> 2;
    r.w[u] = reinterpret_cast<const uint4*>(blk)[i * 32 + t];
    r.s0[u] = reinterpret_cast<const float*>(blk + cbytes)[rr];
    r.s1[u] = reinterpret_cast<const float*>(blk + cbytes)[rr + 8];
    r.z0[u] = static_cast<float>(static_cast<int32_t>(blk[cbytes + 64 + rr]) + zbase);
    r.z1[u] = static_cast<float>(static_cast<int32_t>(blk[cbytes + 64 + rr + 8]) + zbase);
  }
}

// Writes one k-step's weight operand into the stage's shared-memory tile (UMMA K-major layout):
// A = 16-bit (q - z) * s of the CTA's 128 weight rows.
template <int W, int F16>
__device__ __forceinline__ void store_step(const StepRaw<W>& r, int64_t tile0, int n_tiles, uint8_t* a_tile) {
  constexpr int words = StepRaw<W>::kWords;
#pragma unroll
  for (int u = 0; u < StepRaw<W>::kA; ++u) {
    const int it = threadIdx.x + u * kGemmThreads;
    const int rt = it / (words * 32), rem = it - rt * words * 32;
    const int i = rem >> 5, t = rem & 31;
    const bool live = tile0 + rt < n_tiles;
    const int rrow = t >> 2, c2 = 2 * (t & 3);
    const int row = rt * 16 + rrow;
    const float s0 = live ? r.s0[u] : 0.f, s1 = live ? r.s1[u] : 0.f, z0 = r.z0[u], z1 = r.z1[u];
    const uint32_t q4[4] = {r.w[u].x, r.w[u].y, r.w[u].z, r.w[u].w};
    if constexpr (W == 0) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int k0 = 16 * (2 * i + h) + c2;
#pragma unroll
        for (int e = 0; e < 2; ++e) {  // e = 0: codes at k0, k0+1; e = 1: at k0+8, k0+9
          const uint32_t q = q4[2 * h + e];
          const float a0 = (static_cast<float>(q & 0xFFu) - z0) * s0, a1 = (static_cast<float>((q >> 8) & 0xFFu) - z0) * s0;
          const float b0 = (static_cast<float>((q >> 16) & 0xFFu) - z1) * s1, b1 = (static_cast<float>(q >> 24) - z1) * s1;
          *reinterpret_cast<uint32_t*>(a_tile + kmajor_off(row, k0 + 8 * e)) = pack_b2<F16>(a0, a1);
          *reinterpret_cast<uint32_t*>(a_tile + kmajor_off(row + 8, k0 + 8 * e)) = pack_b2<F16>(b0, b1);
        }
      }
    } else {
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int k0 = 16 * (4 * i + v) + c2;
        const uint32_t q = q4[v];
        // nibbles (low to high): (r,k0) (r,k0+8) (r+8,k0) (r+8,k0+8) (r,k0+1) (r,k0+9) (r+8,k0+1) (r+8,k0+9)
        auto nib = [&](int n) { return static_cast<float>((q >> (4 * n)) & 0xFu); };
        *reinterpret_cast<uint32_t*>(a_tile + kmajor_off(row, k0)) = pack_b2<F16>((nib(0) - z0) * s0, (nib(4) - z0) * s0);
        *reinterpret_cast<uint32_t*>(a_tile + kmajor_off(row, k0 + 8)) = pack_b2<F16>((nib(1) - z0) * s0, (nib(5) - z0) * s0);
        *reinterpret_cast<uint32_t*>(a_tile + kmajor_off(row + 8, k0)) = pack_b2<F16>((nib(2) - z1) * s1, (nib(6) - z1) * s1);
        *reinterpret_cast<uint32_t*>(a_tile + kmajor_off(row + 8, k0 + 8)) = pack_b2<F16>((nib(3) - z1) * s1, (nib(7) - z1) * s1);
      }
    }
  }
}

template <int W, int F16>
__global__ void __launch_bounds__(kGemmThreads, 1) gemm_dq_kernel(const uint8_t* __restrict__ tiles, int n_tiles, int nkb,
                                                                  int32_t zbase, int64_t N, int64_t K,
                                                                  const uint16_t* __restrict__ x, int64_t x_stride, int T,
                                                                  float* __restrict__ y, int64_t y_stride, int accumulate,
                                                                  int splits, int64_t split_stride) {
  extern __shared__ __align__(1024) uint8_t gsm[];
  __shared__ uint64_t mma_done[kStagesG];
  __shared__ uint32_t tmem_base_s;
  uint8_t* stage_base = gsm;  // kStagesG stages x (A 32 KB | B kTN x 256 B)
  const int warp = threadIdx.x >> 5;
  const int64_t tile0 = static_cast<int64_t>(blockIdx.x) * (kTM / kTileRows);
  const int t0 = blockIdx.y * kTN;
  // split-K: this CTA's k-steps [kb0, kb1); partial sums go to y + z * split_stride
  const int kb0 = static_cast<int>(static_cast<int64_t>(nkb) * blockIdx.z / splits);
  const int kb1 = static_cast<int>(static_cast<int64_t>(nkb) * (blockIdx.z + 1) / splits);
  y += blockIdx.z * split_stride;
  if (threadIdx.x == 0) {
    for (int q = 0; q < kStagesG; ++q) mbar_init1(&mma_done[q]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tmem_base_s)),
                 "r"(kTN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_s;
  uint32_t phase[kStagesG];
#pragma unroll
  for (int q = 0; q < kStagesG; ++q) phase[q] = 0u;
  StepRaw<W> cur, nxt;
  // activation tiles of the first kStagesG - 1 k-steps (one cp.async group each, empty past kb1)
#pragma unroll
  for (int q = 0; q < kStagesG - 1; ++q) {
    if (kb0 + q < kb1) load_tokens_async(x, x_stride, T, K, t0, kb0 + q, stage_base + q * kStageBytesG + kATileBytes);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  }
  load_step<W>(tiles, tile0, n_tiles, nkb, kb0, zbase, cur);
  // Pipeline: k-step kb dequantises into stage s = kb & 1 while the MMAs of kb - 1 run; right
  // after kb's MMAs are issued, the MMAs of kb - 1 (the other stage's last reader) are waited for
  // and that stage's activation tile refilled for kb + 1, so neither the tensor pipe nor the
  // dequantisation waits on the other in steady state.
  for (int kb = kb0; kb < kb1; ++kb) {
    const int i = kb - kb0;
    const int s = i % kStagesG;
    const bool more = kb + 1 < kb1;
    uint8_t* at = stage_base + s * kStageBytesG;
    if (more) load_step<W>(tiles, tile0, n_tiles, nkb, kb + 1, zbase, nxt);
    store_step<W, F16>(cur, tile0, n_tiles, at);
    // this step's activation group is complete; the kStagesG - 2 newer ones may still be in flight
    asm volatile("cp.async.wait_group %0;" ::"n"(kStagesG - 2) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy writes -> tensor core
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a0 = smem_addr(at), b0 = smem_addr(at + kATileBytes);
#pragma unroll
      for (int j = 0; j < kTK / 16; ++j) {
        const uint64_t da = umma_desc(a0 + j * 256), db = umma_desc(b0 + j * 256);
        const uint32_t acc = (i > 0 || j > 0) ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
            ::"r"(tmem), "l"(da), "l"(db), "r"(idesc<F16>()), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_addr(&mma_done[s]))
                   : "memory");
    }
    // the stage of step i - 1 (= that of step i + kStagesG - 1) is free once MMA(i - 1) is done:
    // refill its activation tile kStagesG - 1 steps ahead (an empty group past kb1)
    if (i >= 1) {
      const int sp = (i - 1) % kStagesG;
      mbar_wait1(&mma_done[sp], phase[sp]);
      phase[sp] ^= 1u;
    }
    if (kb + kStagesG - 1 < kb1)
      load_tokens_async(x, x_stride, T, K, t0, kb + kStagesG - 1,
                        stage_base + ((i + kStagesG - 1) % kStagesG) * kStageBytesG + kATileBytes);
    else
      asm volatile("cp.async.commit_group;" ::: "memory");
    if (more) cur = nxt;
  }
  // wait for the last commit (it covers every earlier MMA of this thread)
  const int last = (kb1 - kb0 - 1) % kStagesG;
  mbar_wait1(&mma_done[last], phase[last]);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // epilogue: warp w (of the first four) owns accumulator lanes 32w .. 32w+31 (weight rows);
  // warps 4..7 take the second half of the token columns
  const int lane = threadIdx.x & 31;
  const int wl = warp & 3;
  const int64_t n = static_cast<int64_t>(blockIdx.x) * kTM + wl * 32 + lane;
  const int cbeg = (warp >> 2) * (kTN / 2);
#pragma unroll 1
  for (int c0 = cbeg; c0 < cbeg + kTN / 2 && t0 + c0 < T; c0 += 8) {
    uint32_t v[8];
    const uint32_t taddr = tmem + (static_cast<uint32_t>(wl * 32) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (n < N) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int t = t0 + c0 + e;
        if (t < T) {
          float* yp = y + static_cast<int64_t>(t) * y_stride + n;
          *yp = accumulate ? *yp + __uint_as_float(v[e]) : __uint_as_float(v[e]);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTN));
}

// y[t][n] (+)= sum over the splits in order of ws[z][t][n] (deterministic split-K reduction)
__global__ void split_reduce_kernel(const float* __restrict__ ws, int splits, int64_t T, int64_t N, float* __restrict__ y,
                                    int64_t y_stride, int accumulate) {
  const int64_t total = T * N;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = i / N, n = i - t * N;
    float v = ws[i];
    for (int z = 1; z < splits; ++z) v += ws[z * total + i];
    float* yp = y + t * y_stride + n;
    *yp = accumulate ? *yp + v : v;
  }
}

template <int W, int F16>
void configure_gemm(size_t smem) {
  static bool done = false;
  if (!done) {
    FQ_CUDA(cudaFuncSetAttribute(gemm_dq_kernel<W, F16>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    done = true;
  }
}

}  // namespace

void launch_gemm_dq(fq_ctx* ctx, const fq_layer* L, int rung, int64_t T, const void* x, int x_dtype, int64_t x_stride,
                    float* y, int64_t y_stride, bool accumulate) {
  if (rung != FQ_RUNG_INT8 && rung != FQ_RUNG_INT4) fail(FQ_E_CONFIG, "gemm: rung must be 8 or 4");
  if (x_dtype != FQ_DT_BF16 && x_dtype != FQ_DT_F16) fail(FQ_E_CONFIG, "gemm: activations must be bf16 or fp16");
  const fq_rung_store& st = L->store(rung);
  if (!st.present || st.tiles == nullptr) fail(FQ_E_STATE, "gemm: rung not resident in the tiled layout");
  if (T < 1) fail(FQ_E_DIMENSION, "gemm: no rows");
  if (x_stride % 8 != 0 || (reinterpret_cast<uintptr_t>(x) & 15) != 0)
    fail(FQ_E_CONFIG, "gemm: activation rows must be 16-byte aligned (row stride a multiple of 8)");
  const int n_tiles = ceil_div_i(L->N, kTileRows), nkb = ceil_div_i(L->K, kBlockK);
  const int gx = ceil_div_i(L->N, kTM), gy = ceil_div_i(T, kTN);
  // split K when the output tiles alone leave SMs idle: the fewest splits with the lowest
  // (waves x work per split), at least 4 k-steps per split
  int splits = 1;
  {
    const int64_t cta = gx * static_cast<int64_t>(gy);
    double best = static_cast<double>((cta + ctx->num_sms - 1) / ctx->num_sms);
    for (int sp = 2; sp <= 8 && nkb / sp >= 4; ++sp) {
      const double cost = static_cast<double>((cta * sp + ctx->num_sms - 1) / ctx->num_sms) / sp;
      if (cost < best - 1e-9) {
        best = cost;
        splits = sp;
      }
    }
  }
  float* out = y;
  int64_t out_stride = y_stride, split_stride = 0;
  if (splits > 1) {
    const size_t need = sizeof(float) * static_cast<size_t>(splits) * T * L->N;
    if (ctx->gemm_ws_bytes < need) {
      dfree(ctx->gemm_ws);
      ctx->gemm_ws = static_cast<float*>(dmalloc(need));
      ctx->gemm_ws_bytes = need;
    }
    out = ctx->gemm_ws;
    out_stride = L->N;
    split_stride = T * L->N;
  }
  const dim3 grid(static_cast<unsigned>(gx), static_cast<unsigned>(gy), static_cast<unsigned>(splits));
  const size_t smem = static_cast<size_t>(kStagesG) * kStageBytesG;
  const auto* xs = static_cast<const uint16_t*>(x);
  const int acc = splits > 1 ? 0 : (accumulate ? 1 : 0);
  const int Ti = static_cast<int>(T);
#define FQ_GEMM_LAUNCH(Wv, Fv)                                                                                     \
  do {                                                                                                             \
    configure_gemm<Wv, Fv>(smem);                                                                                  \
    gemm_dq_kernel<Wv, Fv><<<grid, kGemmThreads, smem, ctx->stream>>>(st.tiles, n_tiles, nkb, st.zp_base, L->N, L->K, \
                                                                      xs, x_stride, Ti, out, out_stride, acc,       \
                                                                      splits, split_stride);                        \
  } while (0)
  const bool f16 = x_dtype == FQ_DT_F16;
  if (rung == FQ_RUNG_INT8) {
    if (f16) FQ_GEMM_LAUNCH(0, 1);
    else FQ_GEMM_LAUNCH(0, 0);
  } else {
    if (f16) FQ_GEMM_LAUNCH(1, 1);
    else FQ_GEMM_LAUNCH(1, 0);
  }
#undef FQ_GEMM_LAUNCH
  FQ_CUDA(cudaGetLastError());
  ctx->launches += 1;
  if (splits > 1) {
    const int64_t total = T * L->N;
    const int blocks = static_cast<int>(std::min<int64_t>(ctx->num_sms * 8, (total + 255) / 256));
    split_reduce_kernel<<<blocks, 256, 0, ctx->stream>>>(ctx->gemm_ws, splits, T, L->N, y, y_stride, accumulate ? 1 : 0);
    FQ_CUDA(cudaGetLastError());
    ctx->launches += 1;
  }
}

}  // namespace fqc
