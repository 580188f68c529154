// Stand-alone dequant-GEMV (fq_gemv FAST, BASELINE config 2): y[b] = x[b] . dequant(W)^T for one
// linear at one precision, B <= 32 rows per launch, straight from the tiled copy in HBM.
//
// The decode step streams its linears through the persistent step program (program.cu), whose
// ring / grid-barrier machinery is built for a chain of dependent phases.  A single GEMV needs
// none of it; what bounds it is keeping enough bytes in flight from the first microsecond:
//   * the work is (16-row tile, k-slice) tasks, one per warp, sized so the grid covers every SM
//     once with 12 warps per CTA (split-K only when the layer has too few tiles for the warps);
//   * a CTA stages its k-slice of the activations once, in fp16 B-fragment order, with the
//     per-group sums the zero-point fold needs (sum (q-z)x = sum (off+q)x - (off + z) sum x);
//   * a warp loads U whole blocks (16 rows x 128 codes + their 16 scales / zero points) into
//     registers with 128-bit non-allocating loads -- all U in flight together -- then runs the
//     mma.sync m16n8k16 chains on them (the blocks are stored in A-fragment order: no shuffles,
//     W8 unpacked by byte permute to fp16 1024+q, W4 by one LOP3 per pair to fp16 64+q);
//   * split-K partials go to a workspace; the last task of a tile (arrival counter) sums them in
//     slice order and writes y -- one launch, deterministic.
// Numerics are those of the step program's GEMV (fp16 activations, exact products, fp32
// accumulation per 128-code group, fp32 group scale): src/quantizer.cpp:205-219 dequantize +
// src/tensor.cpp:83-101 linear within the FAST tolerance.
#include <atomic>

#include "fq_internal.cuh"

namespace fqc {
namespace {

constexpr int kWarps = 12;

struct DirectArgs {
  const uint8_t* tiles;
  int64_t N, K;
  int n_tiles, nkb, zp_base;
  const void* x;
  int x_dtype;
  int64_t x_stride;
  int B;
  void* y;
  int y_dtype;
  int64_t y_stride;
  int S, kb_per;
  float* ws;      // [S][B][n_tiles * 16]
  unsigned* cnt;  // [n_tiles]
};

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

__device__ __forceinline__ uint32_t nib_f16(uint32_t v) {  // nibbles at bits 4-7 / 20-23 -> fp16 64 + q
  uint32_t r;
  asm("lop3.b32 %0, %1, 0x00F000F0, 0x54005400, 0xEA;" : "=r"(r) : "r"(v));
  return r;
}

__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ float load_x(const void* x, int dtype, int64_t i) {
  if (dtype == FQ_DT_F32) return static_cast<const float*>(x)[i];
  if (dtype == FQ_DT_BF16) return __bfloat162float(static_cast<const __nv_bfloat16*>(x)[i]);
  return __half2float(static_cast<const __half*>(x)[i]);
}

__device__ __forceinline__ void store_y(void* y, int dtype, int64_t i, float v) {
  if (dtype == FQ_DT_F32) static_cast<float*>(y)[i] = v;
  else if (dtype == FQ_DT_BF16) static_cast<__nv_bfloat16*>(y)[i] = __float2bfloat16_rn(v);
  else static_cast<__half*>(y)[i] = __float2half_rn(v);
}

constexpr int kRing = 3;  // stages per warp

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
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
// one bulk copy global -> shared for a whole batch of consecutive blocks, completion on `bar`
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// The warp's stream of batches: for each of its tiles, the slice's blocks in groups of U.
struct Stream {
  int tile, kb;  // next batch to issue
  int step;      // tile stride between this warp's tiles
};

template <int W, int U>
__device__ __forceinline__ bool issue(Stream& st, const DirectArgs& a, int k0, int nk, uint8_t* stage, uint64_t* bar) {
  constexpr int BB = W == 0 ? kBlockBytes8 : kBlockBytes4;
  if (st.tile >= a.n_tiles) return false;
  const int nb = min(U, nk - st.kb);
  bulk_copy(stage, a.tiles + (static_cast<int64_t>(st.tile) * a.nkb + k0 + st.kb) * BB, static_cast<uint32_t>(nb * BB),
            bar);
  st.kb += U;
  if (st.kb >= nk) {
    st.kb = 0;
    st.tile += st.step;
  }
  return true;
}

// MMAs of one staged batch (blocks kb .. kb+U-1 of the slice) against the staged activations, then
// the per-group fold y += s * (acc - (off * X + z * X)) (X = the group's activation sum, off =
// 1024 for the W8 byte-permute operands, 64 for the W4 nibble operands).
template <int W, int NG, int U>
__device__ __forceinline__ void compute_batch(const uint8_t* stage, int kb, int nk, const uint4* __restrict__ xs,
                                              const float4* __restrict__ dx, int rs, int bmax, int zp_base, int lane,
                                              float (&y)[NG][4]);

// NB blocks of a staged batch, interleaved block by block at every k-step so the NB accumulator
// chains (and their shared-memory loads) overlap; then the per-group fold
// y += s * (acc - (off * X + z * X)) (X = the group's activation sum, off = 1024 for the W8
// byte-permute operands, 64 for the W4 nibble operands).
template <int W, int NG, int NB>
__device__ __forceinline__ void compute_blocks(const uint8_t* stage, int kl0, const uint4* __restrict__ xs,
                                               const float4* __restrict__ dx, int rs, int bmax, int zp_base,
                                               int lane, float (&y)[NG][4]) {
  constexpr int BR = 8 * NG;
  constexpr int BB = W == 0 ? kBlockBytes8 : kBlockBytes4;
  constexpr int CB = W == 0 ? 2048 : 1024;
  const int g = lane >> 2, tig = lane & 3;
  float c[NB][NG][4];
#pragma unroll
  for (int n = 0; n < NB; ++n)
#pragma unroll
    for (int cg = 0; cg < NG; ++cg)
#pragma unroll
      for (int e = 0; e < 4; ++e) c[n][cg][e] = 0.f;
  if constexpr (W == 0) {
#pragma unroll
    for (int p = 0; p < 4; ++p) {
#pragma unroll
      for (int n = 0; n < NB; ++n) {
        const uint4 q = reinterpret_cast<const uint4*>(stage + n * BB)[p * 32 + lane];
        const uint32_t a0 = prmt(q.x, 0x64646464u, 0x4140u), a1 = prmt(q.x, 0x64646464u, 0x4342u);
        const uint32_t a2 = prmt(q.y, 0x64646464u, 0x4140u), a3 = prmt(q.y, 0x64646464u, 0x4342u);
        const uint32_t a4 = prmt(q.z, 0x64646464u, 0x4140u), a5 = prmt(q.z, 0x64646464u, 0x4342u);
        const uint32_t a6 = prmt(q.w, 0x64646464u, 0x4140u), a7 = prmt(q.w, 0x64646464u, 0x4342u);
#pragma unroll
        for (int cg = 0; cg < NG; ++cg) {
          const uint4 xv = xs[min(cg * 8 + g, bmax) * rs + (kl0 + n) * 16 + p * 4 + tig];
          mma16816(c[n][cg], a0, a1, a2, a3, xv.x, xv.y);
          mma16816(c[n][cg], a4, a5, a6, a7, xv.z, xv.w);
        }
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
#pragma unroll
      for (int n = 0; n < NB; ++n) {
        const uint4 wv = reinterpret_cast<const uint4*>(stage + n * BB)[i * 32 + lane];
        const uint32_t qs[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
        for (int uu = 0; uu < 4; ++uu) {
          const uint32_t q = qs[uu];
          const uint32_t a0 = nib_f16(q << 4), a1 = nib_f16(q >> 4), a2 = nib_f16(q), a3 = nib_f16(q >> 8);
#pragma unroll
          for (int cg = 0; cg < NG; ++cg) {
            const uint4 xv = xs[min(cg * 8 + g, bmax) * rs + (kl0 + n) * 16 + (2 * i + (uu >> 1)) * 4 + tig];
            mma16816(c[n][cg], a0, a1, a2, a3, (uu & 1) ? xv.z : xv.x, (uu & 1) ? xv.w : xv.y);
          }
        }
      }
    }
  }
#pragma unroll
  for (int n = 0; n < NB; ++n) {
    const uint8_t* blk = stage + n * BB;
    const int kl = kl0 + n;
    const float s0 = reinterpret_cast<const float*>(blk + CB)[g], s1 = reinterpret_cast<const float*>(blk + CB)[g + 8];
    const float zf0 = static_cast<float>(static_cast<int>(blk[CB + 64 + g]) + zp_base);
    const float zf1 = static_cast<float>(static_cast<int>(blk[CB + 64 + g + 8]) + zp_base);
#pragma unroll
    for (int cg = 0; cg < NG; ++cg) {
      const float4 d0 = dx[kl * BR + cg * 8 + 2 * tig], d1 = dx[kl * BR + cg * 8 + 2 * tig + 1];
      const float D0 = W == 0 ? d0.x : d0.y, D1 = W == 0 ? d1.x : d1.y;
      y[cg][0] = fmaf(s0, c[n][cg][0] - fmaf(zf0, d0.z, D0), y[cg][0]);
      y[cg][1] = fmaf(s0, c[n][cg][1] - fmaf(zf0, d1.z, D1), y[cg][1]);
      y[cg][2] = fmaf(s1, c[n][cg][2] - fmaf(zf1, d0.z, D0), y[cg][2]);
      y[cg][3] = fmaf(s1, c[n][cg][3] - fmaf(zf1, d1.z, D1), y[cg][3]);
    }
  }
}

// One staged batch: blocks kb .. min(kb + U, nk) - 1; full batches interleave all U blocks, a
// tail batch goes block by block.
template <int W, int NG, int U>
__device__ __forceinline__ void compute_batch(const uint8_t* stage, int kb, int nk, const uint4* __restrict__ xs,
                                              const float4* __restrict__ dx, int rs, int bmax, int zp_base, int lane,
                                              float (&y)[NG][4]) {
  constexpr int BB = W == 0 ? kBlockBytes8 : kBlockBytes4;
  if (kb + U <= nk) {
    compute_blocks<W, NG, U>(stage, kb, xs, dx, rs, bmax, zp_base, lane, y);
  } else {
    for (int u = 0; kb + u < nk; ++u) compute_blocks<W, NG, 1>(stage + u * BB, kb + u, xs, dx, rs, bmax, zp_base, lane, y);
  }
}

// Finished tile: store y (one slice) or publish the slice's partial; the tile's last slice sums
// the partials in slice order and stores (deterministic).
template <int NG>
__device__ __forceinline__ void finish_tile(const DirectArgs& a, int tile, int ks, int lane, float (&y)[NG][4]) {
  const int g = lane >> 2, tig = lane & 3;
  const int64_t r0 = static_cast<int64_t>(tile) * kTileRows + g, r1 = r0 + 8;
  if (a.S == 1) {
#pragma unroll
    for (int cg = 0; cg < NG; ++cg)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int col = cg * 8 + 2 * tig + (e & 1);
        const int64_t row = (e & 2) ? r1 : r0;
        if (col < a.B && row < a.N) store_y(a.y, a.y_dtype, col * a.y_stride + row, y[cg][e]);
      }
    return;
  }
  const int64_t npad = static_cast<int64_t>(a.n_tiles) * kTileRows;
#pragma unroll
  for (int cg = 0; cg < NG; ++cg)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int col = cg * 8 + 2 * tig + (e & 1);
      if (col < a.B) __stcg(a.ws + (static_cast<int64_t>(ks) * a.B + col) * npad + ((e & 2) ? r1 : r0), y[cg][e]);
    }
  __threadfence();
  __syncwarp();
  unsigned prev = 0;
  if (lane == 0) prev = atomicAdd(&a.cnt[tile], 1u);
  prev = __shfl_sync(0xffffffffu, prev, 0);
  if (prev != static_cast<unsigned>(a.S - 1)) return;
  __threadfence();
#pragma unroll
  for (int cg = 0; cg < NG; ++cg)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int col = cg * 8 + 2 * tig + (e & 1);
      const int64_t row = (e & 2) ? r1 : r0;
      if (col >= a.B) continue;
      float sum = 0.f;
      for (int sl = 0; sl < a.S; ++sl) sum += __ldcg(a.ws + (static_cast<int64_t>(sl) * a.B + col) * npad + row);
      if (row < a.N) store_y(a.y, a.y_dtype, col * a.y_stride + row, sum);
    }
  __syncwarp();
  if (lane == 0) a.cnt[tile] = 0u;  // ready for the next launch (stream-ordered)
}

// Persistent: CTA (ks, cy) of a (S, Y) grid, one per SM; warp w streams tiles cy*12 + w,
// (cy + Y)*12 + w, ... of k-slice ks through its own ring of kRing stages (U blocks each, one bulk
// copy per stage), so the weight stream continues across its tiles and their epilogues.
template <int W, int NG, int U>
__global__ void __launch_bounds__(kWarps * 32, 1) gemv_direct_kernel(const DirectArgs a) {
  constexpr int BR = 8 * NG;
  constexpr int BB = W == 0 ? kBlockBytes8 : kBlockBytes4;
  constexpr int kStage = U * BB;
  extern __shared__ __align__(128) uint8_t smem[];  // ring [warp][stage] | xs fragments | dx
  __shared__ __align__(8) uint64_t bars[kWarps][kRing];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ks = blockIdx.x;
  const int k0 = static_cast<int>(static_cast<int64_t>(a.nkb) * ks / a.S);
  const int k1 = static_cast<int>(static_cast<int64_t>(a.nkb) * (ks + 1) / a.S);
  const int nk = k1 - k0;
  uint8_t* ring = smem + static_cast<size_t>(warp) * kRing * kStage;
  uint4* xs = reinterpret_cast<uint4*>(smem + static_cast<size_t>(kWarps) * kRing * kStage);
  // activation rows padded by 16 bytes: the 8 rows x 4 lanes of a fragment load hit 8 distinct
  // bank quads (4 wavefronts for 32 lanes); columns past the batch read the last row (broadcast)
  const int rs = a.kb_per * 16 + 1;
  float4* dx = reinterpret_cast<float4*>(xs + static_cast<size_t>(BR) * rs);

  // the weight stream depends on nothing: start it before staging the activations
  Stream st{static_cast<int>(blockIdx.y) * kWarps + warp, 0, static_cast<int>(gridDim.y) * kWarps};
  int issued = 0;
  if (lane == 0) {
    for (int s = 0; s < kRing; ++s) mbar_init(&bars[warp][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < kRing; ++s) issued += issue<W, U>(st, a, k0, nk, ring + s * kStage, &bars[warp][s]) ? 1 : 0;
  }
  issued = __shfl_sync(0xffffffffu, issued, 0);

  // ---- stage the k-slice of x: one warp per (row, block), lane l holds codes 4l..4l+3
  __half* xh = reinterpret_cast<__half*>(xs);
  for (int item = warp; item < BR * nk; item += kWarps) {
    const int b = item / nk, kl = item - b * nk;
    float v[4];
    float sum = 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t k = static_cast<int64_t>(k0 + kl) * kBlockK + 4 * lane + e;
      const float f = (b < a.B && k < a.K) ? load_x(a.x, a.x_dtype, b * a.x_stride + k) : 0.f;
      v[e] = __half2float(__float2half_rn(f));  // the MMA's operand value
      sum += v[e];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) dx[kl * BR + b] = make_float4(1024.f * sum, 64.f * sum, sum, 0.f);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int r = 4 * lane + e, j16 = r >> 4, r16 = r & 15;
      const int p = j16 >> 1, hh = j16 & 1, tig = (r16 & 7) >> 1, comp = 2 * hh + (r16 >> 3);
      xh[(static_cast<size_t>(b) * rs + kl * 16 + p * 4 + tig) * 8 + comp * 2 + (r16 & 1)] = __float2half_rn(v[e]);
    }
  }
  __syncthreads();
  if (issued == 0) return;

  float y[NG][4];
#pragma unroll
  for (int cg = 0; cg < NG; ++cg)
#pragma unroll
    for (int e = 0; e < 4; ++e) y[cg][e] = 0.f;
  int tile = static_cast<int>(blockIdx.y) * kWarps + warp, kb = 0, s = 0;
  uint32_t parity = 0;
  while (tile < a.n_tiles) {
    mbar_wait(&bars[warp][s], parity);
    compute_batch<W, NG, U>(ring + s * kStage, kb, nk, xs, dx, rs, a.B - 1, a.zp_base, lane, y);
    __syncwarp();  // every lane is done with the stage: refill it
    if (lane == 0) issue<W, U>(st, a, k0, nk, ring + s * kStage, &bars[warp][s]);
    if (++s == kRing) {
      s = 0;
      parity ^= 1u;
    }
    kb += U;
    if (kb >= nk) {
      finish_tile<NG>(a, tile, ks, lane, y);
#pragma unroll
      for (int cg = 0; cg < NG; ++cg)
#pragma unroll
        for (int e = 0; e < 4; ++e) y[cg][e] = 0.f;
      kb = 0;
      tile += static_cast<int>(gridDim.y) * kWarps;
    }
  }
}

template <int W, int NG, int U>
void launch_t(fq_ctx* ctx, const DirectArgs& a, int Y) {
  constexpr int BB = W == 0 ? kBlockBytes8 : kBlockBytes4;
  const size_t smem = static_cast<size_t>(kWarps) * kRing * U * BB +
                      static_cast<size_t>(8 * NG) * (a.kb_per * (16 * 16 + 16) + 16);
  // the shared-memory opt-in is a per-device attribute: set once per device this process uses
  static std::atomic<uint64_t> set_on{0};
  const uint64_t bit = 1ull << (ctx->device & 63);
  if (!(set_on.load() & bit)) {
    FQ_CUDA(cudaFuncSetAttribute(gemv_direct_kernel<W, NG, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    set_on.fetch_or(bit);
  }
  if (smem > 220 * 1024) fail(FQ_E_CONFIG, "gemv: activation slice does not fit shared memory");
  gemv_direct_kernel<W, NG, U><<<dim3(a.S, Y), kWarps * 32, smem, ctx->stream>>>(a);
  FQ_CUDA(cudaGetLastError());
  ctx->launches += 1;
}

}  // namespace

void launch_gemv_direct(fq_ctx* ctx, const fq_layer* L, int rung, int64_t batch, const void* x, int x_dtype, void* y,
                        int y_dtype) {
  const fq_rung_store& st = L->store(rung);
  if (!st.present || st.tiles == nullptr) fail(FQ_E_STATE, "gemv: no tiled copy for this precision");
  const int w = rung == FQ_RUNG_INT4 ? 1 : 0;
  const int n_tiles = ceil_div_i(L->N, kTileRows), nkb = ceil_div_i(L->K, kBlockK);
  const size_t xsz = x_dtype == FQ_DT_F32 ? 4 : 2, ysz = y_dtype == FQ_DT_F32 ? 4 : 2;
  for (int64_t b0 = 0; b0 < batch; b0 += 32) {
    const int B = static_cast<int>(std::min<int64_t>(32, batch - b0));
    const int ng = B <= 8 ? 1 : B <= 16 ? 2 : 4;
    // k-slices and CTAs: one 12-warp CTA per SM, (S, Y) with S * Y <= #SM; S splits K when the
    // layer has too few tiles to give every warp work, and is chosen (with Y) to balance the
    // tiles per warp; the activation slice must fit next to the rings
    const int U = w == 0 ? (ng == 4 ? 1 : 2) : (ng == 4 ? 2 : 4);
    const int64_t ring = static_cast<int64_t>(kWarps) * kRing * U * (w == 0 ? kBlockBytes8 : kBlockBytes4);
    const int64_t per_kb = static_cast<int64_t>(8 * ng) * (16 * 16 + 16);  // fragments + dx per k-block
    const int64_t budget = 220 * 1024 - ring - 16 * 8 * ng;
    const int s_min = std::max<int>(1, static_cast<int>((nkb * per_kb + budget - 1) / budget));
    const int sms = ctx->num_sms;
    int S = s_min, Y = 1;
    double best = 1e30;
    for (int s = s_min; s <= std::min(nkb, 16); ++s) {
      const int y = std::max(1, std::min(sms / s, ceil_div_i(n_tiles, kWarps)));
      const int64_t warps = static_cast<int64_t>(y) * kWarps;
      const int64_t tiles_per_warp = (n_tiles + warps - 1) / warps;
      const double cost = static_cast<double>(tiles_per_warp) * (ceil_div_i(nkb, s) + (s > 1 ? 3.0 : 0.0));
      if (cost < best - 1e-9) {
        best = cost;
        S = s;
        Y = y;
      }
    }
    DirectArgs a{};
    a.tiles = st.tiles;
    a.N = L->N;
    a.K = L->K;
    a.n_tiles = n_tiles;
    a.nkb = nkb;
    a.zp_base = st.zp_base;
    a.x = static_cast<const char*>(x) + b0 * L->K * xsz;
    a.x_dtype = x_dtype;
    a.x_stride = L->K;
    a.B = B;
    a.y = static_cast<char*>(y) + b0 * L->N * ysz;
    a.y_dtype = y_dtype;
    a.y_stride = L->N;
    a.S = S;
    a.kb_per = ceil_div_i(nkb, S);
    if (S > 1) {
      const size_t ws = sizeof(float) * static_cast<size_t>(S) * B * n_tiles * kTileRows;
      const size_t cn = sizeof(unsigned) * static_cast<size_t>(n_tiles);
      if (ctx->direct_ws_bytes < ws || ctx->direct_cnt_n < static_cast<size_t>(n_tiles)) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(ctx->stream, &cs);
        if (cs != cudaStreamCaptureStatusNone) fail(FQ_E_STATE, "gemv: workspace must be sized before graph capture");
        FQ_CUDA(cudaStreamSynchronize(ctx->stream));
        if (ctx->direct_ws_bytes < ws) {
          dfree(ctx->direct_ws);
          ctx->direct_ws = static_cast<float*>(dmalloc(ws));
          ctx->direct_ws_bytes = ws;
        }
        if (ctx->direct_cnt_n < static_cast<size_t>(n_tiles)) {
          dfree(ctx->direct_cnt);
          ctx->direct_cnt = static_cast<unsigned*>(dmalloc(cn));
          FQ_CUDA(cudaMemset(ctx->direct_cnt, 0, cn));
          ctx->direct_cnt_n = n_tiles;
        }
      }
      a.ws = ctx->direct_ws;
      a.cnt = ctx->direct_cnt;
    }
    if (w == 0) {
      if (ng == 1) launch_t<0, 1, 2>(ctx, a, Y);
      else if (ng == 2) launch_t<0, 2, 2>(ctx, a, Y);
      else launch_t<0, 4, 1>(ctx, a, Y);
    } else {
      if (ng == 1) launch_t<1, 1, 4>(ctx, a, Y);
      else if (ng == 2) launch_t<1, 2, 4>(ctx, a, Y);
      else launch_t<1, 4, 2>(ctx, a, Y);
    }
  }
}

}  // namespace fqc
