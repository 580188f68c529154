// Stand-alone dequant-fused GEMV (fq_gemv FAST numerics, the per-layer drop-in path of
// MultiPrecisionLayer::forward, /root/reference/proj/src/model.cpp:77-98): one ordinary launch,
// no persistent program.  The step program (program.cu) amortises its start-up (ring, partition
// table, barriers) over a whole decode step; a single GEMV call cannot, so this kernel keeps
// only what one GEMV needs:
//   * every CTA stages the activations once (fp16 in the m16n8k16 B-fragment order, the
//     per-block sums for the zero-point fold), then walks 16-row tiles of the tiled copy;
//   * its 8 warps split a tile's 128-code k-blocks, loading each block's codes straight from
//     global memory into the A-fragment registers (coalesced 16-byte words, two blocks in flight
//     per warp), unpacking with the byte permute (W8, fp16 1024 + q) / one LOP3 (W4, 64 + q) and
//     running mma.sync with the batch rows as the MMA's columns;
//   * fold per block: sum (q - z) x = acc - (D + z X); fixed-order cross-warp sum per tile.
// Numerics identical in kind to the step program's GEMV phases (fp32 accumulation per group).
#include "fq_internal.cuh"

namespace fqc {
namespace {

constexpr int kDWarps = 8;
constexpr int kDThreads = kDWarps * 32;

__device__ __forceinline__ uint32_t prmt_d(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}
__device__ __forceinline__ uint32_t nib_d(uint32_t v) {  // (v & 0x00F000F0) | 0x54005400: fp16 64 + q
  uint32_t r;
  asm("lop3.b32 %0, %1, 0x00F000F0, 0x54005400, 0xEA;" : "=r"(r) : "r"(v));
  return r;
}
__device__ __forceinline__ void mma_d(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                      uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint4 ldg_nc(const uint8_t* p) {
  uint4 v;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

__device__ __forceinline__ float act_in(const void* x, int dt, int64_t i) {
  if (dt == FQ_DT_F32) return static_cast<const float*>(x)[i];
  if (dt == FQ_DT_BF16) return __bfloat162float(static_cast<const __nv_bfloat16*>(x)[i]);
  return __half2float(static_cast<const __half*>(x)[i]);
}

// One k-block of one tile on one warp: codes from global, B fragments from shared memory.
template <int W>
__device__ __forceinline__ void block_mma(const uint4 (&wv)[4], const uint4* __restrict__ xb, float (&c)[4]) {
  if constexpr (W == 0) {
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const uint4 xv = xb[p * 4];
      mma_d(c, prmt_d(wv[p].x, 0x64646464u, 0x4140u), prmt_d(wv[p].x, 0x64646464u, 0x4342u),
            prmt_d(wv[p].y, 0x64646464u, 0x4140u), prmt_d(wv[p].y, 0x64646464u, 0x4342u), xv.x, xv.y);
      mma_d(c, prmt_d(wv[p].z, 0x64646464u, 0x4140u), prmt_d(wv[p].z, 0x64646464u, 0x4342u),
            prmt_d(wv[p].w, 0x64646464u, 0x4140u), prmt_d(wv[p].w, 0x64646464u, 0x4342u), xv.z, xv.w);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const uint4 x0 = xb[(2 * i) * 4], x1 = xb[(2 * i + 1) * 4];
      const uint32_t qs[4] = {wv[i].x, wv[i].y, wv[i].z, wv[i].w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t q = qs[u];
        const uint4 xv = u < 2 ? x0 : x1;
        mma_d(c, nib_d(q << 4), nib_d(q >> 4), nib_d(q), nib_d(q >> 8), (u & 1) ? xv.z : xv.x, (u & 1) ? xv.w : xv.y);
      }
    }
  }
}

template <int W>
__global__ void __launch_bounds__(kDThreads) gemv_direct_kernel(const uint8_t* __restrict__ tiles, int n_tiles, int nkb,
                                                                 int32_t zbase, int64_t N, int64_t K, int B,
                                                                 const void* __restrict__ x, int x_dtype,
                                                                 int64_t x_stride, void* __restrict__ y, int y_dtype,
                                                                 int64_t y_stride) {
  constexpr int bb = W == 0 ? kBlockBytes8 : kBlockBytes4;
  constexpr int cbytes = W == 0 ? 2048 : 1024;
  constexpr int words = W == 0 ? 4 : 2;
  extern __shared__ __align__(16) uint8_t dsm[];
  uint4* xs = reinterpret_cast<uint4*>(dsm);                                  // [B][nkb][16] fragments
  float4* dx = reinterpret_cast<float4*>(dsm + static_cast<size_t>(B) * nkb * 256);  // [nkb][B]
  float* red = reinterpret_cast<float*>(dx + static_cast<size_t>(nkb) * B);  // [warps][16][B]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // ---- stage x: element (b, k) -> fp16 at its B-fragment slot; per-block sums
  __half* xh = reinterpret_cast<__half*>(xs);
  for (int64_t i = tid; i < static_cast<int64_t>(B) * nkb * kBlockK; i += kDThreads) {
    const int b = static_cast<int>(i / (static_cast<int64_t>(nkb) * kBlockK));
    const int64_t k = i - static_cast<int64_t>(b) * nkb * kBlockK;
    const float v = k < K ? act_in(x, x_dtype, b * x_stride + k) : 0.f;
    const int kb = static_cast<int>(k >> 7), r = static_cast<int>(k & 127);
    const int k16 = r >> 4, rr = r & 15;
    const int p = k16 >> 1, hh = k16 & 1, tig = (rr & 7) >> 1, half = rr >> 3, lo = rr & 1;
    xh[(((static_cast<int64_t>(b) * nkb + kb) * 16 + p * 4 + tig) * 8) + 2 * (2 * hh + half) + lo] = __float2half_rn(v);
  }
  __syncthreads();
  for (int blk = warp; blk < B * nkb; blk += kDWarps) {
    const uint2 h4 = reinterpret_cast<const uint2*>(xs + static_cast<size_t>(blk) * 16)[lane];
    const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&h4.x));
    const float2 c = __half22float2(*reinterpret_cast<const __half2*>(&h4.y));
    float sum = (a.x + a.y) + (c.x + c.y);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const int b = blk / nkb, kb = blk - b * nkb;
    if (lane == 0) dx[kb * B + b] = make_float4(1024.f * sum, 64.f * sum, sum, 0.f);
  }
  __syncthreads();
  const int g = lane >> 2, tig = lane & 3;
  const uint4* xl = xs + static_cast<size_t>(min(g, B - 1)) * nkb * 16 + tig;
  const bool ca = 2 * tig < B, cb = 2 * tig + 1 < B;
  const float zm = 8388608.0f - static_cast<float>(zbase);
  for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    float yv[4] = {0.f, 0.f, 0.f, 0.f};
    const uint8_t* tb = tiles + static_cast<int64_t>(t) * nkb * bb;
    // this warp's k-blocks kb = warp, warp + 8, ...: the next block's codes load while the current
    // one computes
    uint4 cur[4], nxt[4];
    int kb = warp;
    if (kb < nkb) {
#pragma unroll
      for (int i = 0; i < words; ++i) cur[i] = ldg_nc(tb + static_cast<int64_t>(kb) * bb + i * 512 + lane * 16);
    }
    for (; kb < nkb; kb += kDWarps) {
      const int kn = kb + kDWarps;
      if (kn < nkb) {
#pragma unroll
        for (int i = 0; i < words; ++i) nxt[i] = ldg_nc(tb + static_cast<int64_t>(kn) * bb + i * 512 + lane * 16);
      }
      const uint8_t* bk = tb + static_cast<int64_t>(kb) * bb;
      const float s0 = __ldg(reinterpret_cast<const float*>(bk + cbytes) + g);
      const float s1 = __ldg(reinterpret_cast<const float*>(bk + cbytes) + g + 8);
      const float z0 = __uint_as_float(0x4B000000u | __ldg(bk + cbytes + 64 + g)) - zm;
      const float z1 = __uint_as_float(0x4B000000u | __ldg(bk + cbytes + 64 + g + 8)) - zm;
      float c[4] = {0.f, 0.f, 0.f, 0.f};
      block_mma<W>(cur, xl + kb * 16, c);
      const float4* dxa = dx + static_cast<size_t>(kb) * B + 2 * tig;
      if (ca) {
        const float4 d = dxa[0];
        const float D = W == 0 ? d.x : d.y;
        yv[0] = fmaf(s0, c[0] - fmaf(z0, d.z, D), yv[0]);
        yv[2] = fmaf(s1, c[2] - fmaf(z1, d.z, D), yv[2]);
      }
      if (cb) {
        const float4 d = dxa[1];
        const float D = W == 0 ? d.x : d.y;
        yv[1] = fmaf(s0, c[1] - fmaf(z0, d.z, D), yv[1]);
        yv[3] = fmaf(s1, c[3] - fmaf(z1, d.z, D), yv[3]);
      }
#pragma unroll
      for (int i = 0; i < words; ++i) cur[i] = nxt[i];
    }
    // fixed-order sum over the warps: red[warp][row][b]
    float* r = red + static_cast<size_t>(warp) * 16 * B;
    if (ca) {
      r[g * B + 2 * tig] = yv[0];
      r[(g + 8) * B + 2 * tig] = yv[2];
    }
    if (cb) {
      r[g * B + 2 * tig + 1] = yv[1];
      r[(g + 8) * B + 2 * tig + 1] = yv[3];
    }
    __syncthreads();
    if (tid < 16 * B) {
      const int row = tid / B, b = tid - row * B;
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < kDWarps; ++w) s += red[(static_cast<size_t>(w) * 16 + row) * B + b];
      const int64_t n = static_cast<int64_t>(t) * kTileRows + row;
      if (n < N) {
        const int64_t o = b * y_stride + n;
        if (y_dtype == FQ_DT_F32) static_cast<float*>(y)[o] = s;
        else if (y_dtype == FQ_DT_BF16) static_cast<__nv_bfloat16*>(y)[o] = __float2bfloat16_rn(s);
        else static_cast<__half*>(y)[o] = __float2half_rn(s);
      }
    }
    __syncthreads();
  }
}

}  // namespace

// Rows per launch of the direct kernel: the staged activations fit in 96 KB of shared memory.
int gemv_direct_rows(int64_t K) {
  const int64_t nkb = (K + kBlockK - 1) / kBlockK;
  const int64_t per_row = nkb * 256 + nkb * 16;  // fragments + block sums
  return static_cast<int>(std::max<int64_t>(0, std::min<int64_t>(8, (96 * 1024) / per_row)));
}

void launch_gemv_direct(fq_ctx* ctx, const fq_layer* L, int rung, int64_t batch, const void* x, int x_dtype,
                        int64_t x_stride, void* y, int y_dtype, int64_t y_stride) {
  const fq_rung_store& st = L->store(rung);
  const int n_tiles = ceil_div_i(L->N, kTileRows), nkb = ceil_div_i(L->K, kBlockK);
  const int rows = gemv_direct_rows(L->K);
  if (rows < 1) fail(FQ_E_DIMENSION, "gemv: row too long for the direct kernel");
  const size_t esz = x_dtype == FQ_DT_F32 ? 4 : 2, ysz = y_dtype == FQ_DT_F32 ? 4 : 2;
  for (int64_t b0 = 0; b0 < batch; b0 += rows) {
    const int B = static_cast<int>(std::min<int64_t>(rows, batch - b0));
    const size_t smem = static_cast<size_t>(B) * nkb * 256 + static_cast<size_t>(nkb) * B * 16 +
                        static_cast<size_t>(kDWarps) * 16 * B * 4;
    // ~4 CTAs per SM, each walking a share of the tiles (the activations are staged once per CTA)
    const int grid = std::max(1, std::min(n_tiles, ctx->num_sms * 4));
    const void* xb = static_cast<const uint8_t*>(x) + b0 * x_stride * esz;
    void* yb = static_cast<uint8_t*>(y) + b0 * y_stride * ysz;
    if (rung == FQ_RUNG_INT8) {
      FQ_CUDA(cudaFuncSetAttribute(gemv_direct_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
      gemv_direct_kernel<0><<<grid, kDThreads, smem, ctx->stream>>>(st.tiles, n_tiles, nkb, st.zp_base, L->N, L->K, B, xb,
                                                                    x_dtype, x_stride, yb, y_dtype, y_stride);
    } else {
      FQ_CUDA(cudaFuncSetAttribute(gemv_direct_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
      gemv_direct_kernel<1><<<grid, kDThreads, smem, ctx->stream>>>(st.tiles, n_tiles, nkb, st.zp_base, L->N, L->K, B, xb,
                                                                    x_dtype, x_stride, yb, y_dtype, y_stride);
    }
    FQ_CUDA(cudaGetLastError());
    ctx->launches += 1;
  }
}

}  // namespace fqc
