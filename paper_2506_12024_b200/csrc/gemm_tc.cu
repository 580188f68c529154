// Prefill / calibration contraction on the 5th-generation tensor cores (tcgen05 + TMEM):
//   Y[T, N] (fp32) = X[T, K] (fp16 operands) . dequant(W_rung[N, K])^T
// straight from the tiled W8 / W4 copy the decode GEMV streams (fq_internal.cuh), so prefill and
// calibration use the same resident weights.  This is the dense contraction of BASELINE config 4:
// MultiPrecisionLayer::forward on many rows at once (/root/reference/proj/src/model.cpp:77-98 =
// dequantize src/quantizer.cpp:205-219 + linear src/tensor.cpp:83-101).
//
// Numerics (the decode GEMV's contract): the tensor cores see the EXACT integer codes q - z (|q - z|
// <= 255, exact in fp16) and the activations (bf16-rounded values stored as fp16, exact in fp16's
// normal range; the producers flag anything past 65504); each 128-code k-block is one quantization group,
// accumulated alone in fp32 in tensor memory, and the group's fp32 scale is applied in the
// epilogue: y = sum_kb s[n, kb] * (sum_{k in kb} (q - z) x).  No weight is ever rounded.
//
// One CTA = 128 weight rows (UMMA M) x 128 tokens (UMMA N), warp-specialised, 12 warps:
//   warp 0     producer: per k-block one 1-D bulk copy (cp.async.bulk) of the 32 KB activation
//              tile (X is stored pre-tiled in the UMMA canonical K-major layout, see
//              tiled_act_offset) and eight bulk copies of the CTA's raw 16x128 weight blocks
//              into a 3-deep ring, completion by mbarrier transaction bytes;
//   warps 6-11 dequantisers: raw codes -> fp16 (q - z) into a 2-deep A-operand ring (canonical
//              K-major, no swizzle), fence.proxy.async, one arrival per k-block;
//   warp 1     MMA issuer (one thread): 8 x tcgen05.mma (M128 N128 K16) per k-block into one of
//              two TMEM accumulators, tcgen05.commit releases the A / input slots and hands the
//              accumulator to the epilogue;
//   warps 2-5  epilogue: tcgen05.ld of the k-block's accumulator (lane quarter = warp % 4), then
//              y[128 tokens] += s[row, kb] * D in registers; the accumulator slot is returned as
//              soon as it is read, so the MMAs of k-block kb+1 overlap the scaling of kb.
#include "gemv_program.cuh"

namespace fqc {
namespace {

constexpr int kTM = 128;                      // weight rows per CTA (UMMA M)
constexpr int kTN = 128;                      // tokens per activation tile (the tiled layout's row block)
constexpr int kTK = 128;                      // codes per k-block (one tiled block / group)
constexpr int kTileBytes = kTM * kTK * 2;     // bf16 128 x 128 tile: 32 KB (A and B alike)
constexpr int kInStages = 3;                  // activation + raw-weight ring
constexpr int kAStages = 2;                   // dequantised A ring
constexpr int kGemmThreads = 384;             // 12 warps (3 per SM sub-partition: 168 registers each)
constexpr int kDequantThreads = 192;          // warps 6..11
constexpr int kRawBytes = 8 * kBlockBytes8;   // 8 raw 16x128 blocks (W8 size; W4 uses half)
// tokens per CTA (UMMA N): 128, or 32 for decode-sized batches (the first 32 rows of a 128-row
// tile are its first 8 KB in the canonical layout, so the same tiled activations serve both)
template <int TN>
constexpr int smem_gemm() { return kInStages * (TN * 256 + kRawBytes) + kAStages * kTileBytes + 1024; }

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// canonical K-major no-swizzle byte offset of element (row, k) inside a 128x128 16-bit tile:
// 8x16-byte core matrices, LBO = 128 B (K-adjacent core matrices), SBO = 2 KB (8-row groups)
__device__ __forceinline__ uint32_t kmajor_off(int row, int k) {
  return static_cast<uint32_t>((row >> 3) * 2048 + (k >> 3) * 128 + (row & 7) * 16 + (k & 7) * 2);
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);  // start address
  d |= static_cast<uint64_t>(128u >> 4) << 16;          // LBO: K-adjacent core matrices
  d |= static_cast<uint64_t>(2048u >> 4) << 32;         // SBO: 8-row groups
  d |= static_cast<uint64_t>(1u) << 46;                 // descriptor version (sm_100)
  return d;                                             // base offset 0, SWIZZLE_NONE
}

// kind::f16 instruction descriptor: D f32, A/B bf16 (F16 = 0) or fp16 (F16 = 1), both K-major,
// N = TN, M = kTM
template <int F16, int TN>
constexpr uint32_t idesc() {
  return (1u << 4) | ((F16 ? 0u : 1u) << 7) | ((F16 ? 0u : 1u) << 10) | ((TN >> 3) << 17) | ((kTM >> 4) << 24);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity, int who) {
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
        printf("fq gemm watchdog: role %d stuck (cta %d,%d,%d parity %u)\n", who, blockIdx.x, blockIdx.y, blockIdx.z, parity);
        __trap();
      }
    }
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(bar))
               : "memory");
}

// Dequantiser threads (128): raw 16x128 blocks of the stage -> fp16 (q - z) A tile.  The raw
// block is in mma.sync A-fragment order (fq_internal.cuh); thread d always converts word
// (i, t) = (d >> 5, d & 31) of its blocks (W8) / word (d >> 5 & 1, d & 31) of block pairs (W4).
// Codes become fp16 1024 + q by a byte permute (W8) or one LOP3 (W4: the nibble pair of a
// register lands in bits 0-3 / 16-19), and one HSUB2 of {1024 + z, 1024 + z} leaves the exact
// integer q - z (|q - z| <= 255).
__device__ __forceinline__ uint32_t hsub2(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}
__device__ __forceinline__ uint32_t nib_pair(uint32_t v) {  // (v & 0x000F000F) | 0x64006400
  uint32_t r;
  asm("lop3.b32 %0, %1, 0x000F000F, 0x64006400, 0xEA;" : "=r"(r) : "r"(v));
  return r;
}
__device__ __forceinline__ uint32_t zpair(const uint8_t* zp8, int r, int32_t zbase) {
  const uint32_t z = 1024u + static_cast<uint32_t>(static_cast<int32_t>(zp8[r]) + zbase);
  const __half h = __uint2half_rn(z);
  const uint32_t u = *reinterpret_cast<const uint16_t*>(&h);
  return u | (u << 16);
}

template <int W>
__device__ __forceinline__ void dequant_stage(const uint8_t* raw, int32_t zbase, uint8_t* a_tile, int d) {
  constexpr int bb = W == 0 ? kBlockBytes8 : kBlockBytes4;
  constexpr int cbytes = W == 0 ? 2048 : 1024;
  constexpr int words = W == 0 ? 4 : 2;  // 16-byte code words per lane per block
  constexpr int units = 8 * words * 32;  // (block, word, lane) units of the stage
  constexpr int per = (units + kDequantThreads - 1) / kDequantThreads;
  // every load of the thread's units first (independent, all in flight), then the conversions
  uint4 wv[per];
  uint32_t z0v[per], z1v[per];
#pragma unroll
  for (int j = 0; j < per; ++j) {
    const int u = d + j * kDequantThreads;
    if (u < units) {
      const int rt = u / (words * 32), rem = u - rt * (words * 32);
      const int i = rem >> 5, t = rem & 31, r = t >> 2;
      const uint8_t* blk = raw + rt * bb;
      wv[j] = reinterpret_cast<const uint4*>(blk)[i * 32 + t];
      z0v[j] = zpair(blk + cbytes + 64, r, zbase);
      z1v[j] = zpair(blk + cbytes + 64, r + 8, zbase);
    }
  }
#pragma unroll
  for (int j = 0; j < per; ++j) {
    const int u = d + j * kDequantThreads;
    if (u >= units) break;
    const int rt = u / (words * 32), rem = u - rt * (words * 32);
    const int i = rem >> 5, t = rem & 31;
    const int r = t >> 2, c2 = 2 * (t & 3);
    const uint32_t q4[4] = {wv[j].x, wv[j].y, wv[j].z, wv[j].w};
    const uint32_t z0 = z0v[j], z1 = z1v[j];
    const int row = rt * 16 + r;
    if constexpr (W == 0) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {  // bytes (r, k0), (r, k0+1), (r+8, k0), (r+8, k0+1)
          const int k0 = 16 * (2 * i + h) + c2 + 8 * e;
          const uint32_t q = q4[2 * h + e];
          *reinterpret_cast<uint32_t*>(a_tile + kmajor_off(row, k0)) = hsub2(prmt(q, 0x64646464u, 0x4140u), z0);
          *reinterpret_cast<uint32_t*>(a_tile + kmajor_off(row + 8, k0)) = hsub2(prmt(q, 0x64646464u, 0x4342u), z1);
        }
      }
    } else {
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        // nibbles (low to high): (r,k0) (r,k0+8) (r+8,k0) (r+8,k0+8) (r,k0+1) (r,k0+9) (r+8,k0+1) (r+8,k0+9)
        const int k0 = 16 * (4 * i + v) + c2;
        const uint32_t q = q4[v];
        *reinterpret_cast<uint32_t*>(a_tile + kmajor_off(row, k0)) = hsub2(nib_pair(q), z0);
        *reinterpret_cast<uint32_t*>(a_tile + kmajor_off(row, k0 + 8)) = hsub2(nib_pair(q >> 4), z0);
        *reinterpret_cast<uint32_t*>(a_tile + kmajor_off(row + 8, k0)) = hsub2(nib_pair(q >> 8), z1);
        *reinterpret_cast<uint32_t*>(a_tile + kmajor_off(row + 8, k0 + 8)) = hsub2(nib_pair(q >> 12), z1);
      }
    }
  }
}

template <int W, int TN>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_ws_kernel(const uint8_t* __restrict__ tiles, int n_tiles, int nkb, int32_t zbase, int64_t N,
                   const uint8_t* __restrict__ xt, int T, float* __restrict__ y, int64_t y_stride, int accumulate,
                   int splits, int64_t split_stride, const uint8_t* __restrict__ row_rung, int64_t rr_stride,
                   int want_rung) {
  constexpr int kBBytes = TN * 256;  // activation bytes per k-block
  constexpr int bb = W == 0 ? kBlockBytes8 : kBlockBytes4;
  constexpr int cbytes = W == 0 ? 2048 : 1024;
  extern __shared__ __align__(1024) uint8_t gsm[];
  __shared__ uint64_t in_full[kInStages], in_empty[kInStages], a_full[kAStages], a_empty[kAStages];
  __shared__ uint64_t d_full[2], d_empty[2];
  __shared__ uint32_t tmem_base_s;
  uint8_t* base = gsm + ((1024u - (smem_addr(gsm) & 1023u)) & 1023u);  // 1 KB aligned, still a shared pointer
  uint8_t* b_ring = base;                                        // kInStages x 32 KB activations
  uint8_t* raw_ring = b_ring + kInStages * kBBytes;              // kInStages x 8 raw blocks
  uint8_t* a_ring = raw_ring + kInStages * kRawBytes;            // kAStages x 32 KB bf16 (q - z)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t tile0 = static_cast<int64_t>(blockIdx.x) * (kTM / kTileRows);
  const int tt = blockIdx.y;  // token tile of TN rows
  const int64_t b_src = static_cast<int64_t>(tt * TN / kTN) * nkb * kTileBytes + (tt * TN % kTN) * 256;
  const int kb0 = static_cast<int>(static_cast<int64_t>(nkb) * blockIdx.z / splits);
  const int kb1 = static_cast<int>(static_cast<int64_t>(nkb) * (blockIdx.z + 1) / splits);
  const int nk = kb1 - kb0;
  y += blockIdx.z * split_stride;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kInStages; ++s) {
      mbar_init(&in_full[s], 1);
      mbar_init(&in_empty[s], 2);  // dequantisers done with the raw blocks + MMAs done with B
    }
    for (int s = 0; s < kAStages; ++s) {
      mbar_init(&a_full[s], 1);
      mbar_init(&a_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&d_full[s], 1);
      mbar_init(&d_empty[s], 4);  // one arrival per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tmem_base_s)),
                 "r"(2 * TN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_s;

  if (warp == 0) {
    // ---------------- producer
    if (lane == 0) {
      auto weights = [&](int s, int kb) {
#pragma unroll 1
        for (int r = 0; r < 8; ++r) {
          const int64_t tile = min(tile0 + r, static_cast<int64_t>(n_tiles) - 1);  // rows past N masked at store
          bulk_g2s(raw_ring + s * kRawBytes + r * bb, tiles + (tile * nkb + kb) * bb, bb, &in_full[s]);
        }
      };
      // the weights do not depend on the previous kernel: the first stages' blocks go out before
      // the programmatic-dependency wait (the launch overlaps the previous kernel's tail), the
      // activation tiles only after it
      const int pre = min(nk, kInStages);
      for (int i = 0; i < pre; ++i) {
        mbar_expect_tx(&in_full[i], kBBytes + 8 * bb);
        weights(i, kb0 + i);
      }
      asm volatile("griddepcontrol.wait;" ::: "memory");
      for (int i = 0; i < pre; ++i)
        bulk_g2s(b_ring + i * kBBytes, xt + b_src + static_cast<int64_t>(kb0 + i) * kTileBytes, kBBytes, &in_full[i]);
      for (int i = pre; i < nk; ++i) {
        const int s = i % kInStages, kb = kb0 + i;
        mbar_wait(&in_empty[s], ((i / kInStages) - 1) & 1, 0);
        mbar_expect_tx(&in_full[s], kBBytes + 8 * bb);
        bulk_g2s(b_ring + s * kBBytes, xt + b_src + static_cast<int64_t>(kb) * kTileBytes, kBBytes, &in_full[s]);
        weights(s, kb);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (lane == 0) {
      for (int i = 0; i < nk; ++i) {
        const int s = i % kInStages, a = i % kAStages, dbuf = i & 1;
        mbar_wait(&in_full[s], (i / kInStages) & 1, 1);
        mbar_wait(&a_full[a], (i / kAStages) & 1, 1);
        if (i >= 2) mbar_wait(&d_empty[dbuf], ((i >> 1) - 1) & 1, 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t a0 = smem_addr(a_ring + a * kTileBytes), b0 = smem_addr(b_ring + s * kBBytes);
        const uint32_t dt = tmem + static_cast<uint32_t>(dbuf * TN);
#pragma unroll
        for (int j = 0; j < kTK / 16; ++j) {
          const uint64_t da = umma_desc(a0 + j * 256), db = umma_desc(b0 + j * 256);
          const uint32_t acc = j > 0 ? 1u : 0u;
          asm volatile(
              "{\n\t.reg .pred p;\n\t"
              "setp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(dt),
              "l"(da), "l"(db), "r"(idesc<1, TN>()), "r"(acc));
        }
        tc_commit(&d_full[dbuf]);
        tc_commit(&a_empty[a]);
        tc_commit(&in_empty[s]);
      }
      asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    }
  } else if (warp >= 6) {
    // ---------------- dequantisers
    const int d = threadIdx.x - 6 * 32;
    for (int i = 0; i < nk; ++i) {
      const int s = i % kInStages, a = i % kAStages;
      mbar_wait(&in_full[s], (i / kInStages) & 1, 2);
      if (i >= kAStages) mbar_wait(&a_empty[a], ((i / kAStages) - 1) & 1, 2);
      dequant_stage<W>(raw_ring + s * kRawBytes, zbase, a_ring + a * kTileBytes, d);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core
      asm volatile("bar.sync 1, %0;" ::"n"(kDequantThreads) : "memory");
      if (d == 0) {
        mbar_arrive(&a_full[a]);
        mbar_arrive(&in_empty[s]);
      }
    }
  } else {
    // ---------------- epilogue (warps 2..5): TMEM lane quarter q = warp % 4 = weight rows 32q..
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int64_t n = static_cast<int64_t>(blockIdx.x) * kTM + row;
    const int64_t tile = min(tile0 + row / kTileRows, static_cast<int64_t>(n_tiles) - 1);
    const float* sc = reinterpret_cast<const float*>(tiles + tile * nkb * bb + cbytes) + (row % kTileRows);
    const int64_t sstride = bb / 4;  // floats between the scales of consecutive k-blocks
    float acc[TN];
#pragma unroll
    for (int c = 0; c < TN; ++c) acc[c] = 0.f;
    float s_next = nk > 0 ? sc[kb0 * sstride] : 0.f;
    for (int i = 0; i < nk; ++i) {
      const int dbuf = i & 1;
      const float s_kb = s_next;
      if (i + 1 < nk) s_next = sc[(kb0 + i + 1) * sstride];
      mbar_wait(&d_full[dbuf], (i >> 1) & 1, 3);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t taddr = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(dbuf * TN);
#pragma unroll
      for (int c0 = 0; c0 < TN; c0 += 16) {
        uint32_t v[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
            "%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr + static_cast<uint32_t>(c0)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int e = 0; e < 16; ++e) acc[c0 + e] = fmaf(s_kb, __uint_as_float(v[e]), acc[c0 + e]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&d_empty[dbuf]);
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");  // y / row table may come from the previous kernel
    if (n < N) {
      const int t0 = tt * TN;
#pragma unroll
      for (int c = 0; c < TN; ++c) {
        const int t = t0 + c;
        // row_rung: this launch covers only the rows decoding at want_rung (grouped batches)
        if (t < T && (row_rung == nullptr || row_rung[t * rr_stride] == want_rung)) {
          float* yp = y + static_cast<int64_t>(t) * y_stride + n;
          *yp = accumulate ? *yp + acc[c] : acc[c];
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * TN));
}

// y[t][n] (+)= sum over the splits in order of ws[z][t][n] (deterministic split-K reduction)
__global__ void split_reduce_kernel(const float* __restrict__ ws, int splits, int64_t T, int64_t N, float* __restrict__ y,
                                    int64_t y_stride, int accumulate, const uint8_t* __restrict__ row_rung,
                                    int64_t rr_stride, int want_rung) {
  asm volatile("griddepcontrol.launch_dependents;");  // the next GEMM may start prefetching weights
  const int64_t total = T * N;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = i / N, n = i - t * N;
    if (row_rung != nullptr && row_rung[t * rr_stride] != want_rung) continue;
    float v = ws[i];
    for (int z = 1; z < splits; ++z) v += ws[z * total + i];
    float* yp = y + t * y_stride + n;
    *yp = accumulate ? *yp + v : v;
  }
}

// row-major [T, K] (bf16 / fp16 / f32, row stride x_stride) -> tiled bf16 (tiled_act_offset)
__global__ void tile_acts_kernel(const void* __restrict__ x, int dtype, int64_t x_stride, int T, int64_t K, int nkb,
                                 int out_f16, uint16_t* __restrict__ xt) {
  asm volatile("griddepcontrol.launch_dependents;");  // the next GEMM may start prefetching weights
  const int64_t total = static_cast<int64_t>(T) * K;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = i / K, k = i - t * K;
    float v;
    if (dtype == FQ_DT_BF16) v = __bfloat162float(static_cast<const __nv_bfloat16*>(x)[t * x_stride + k]);
    else if (dtype == FQ_DT_F16) v = __half2float(static_cast<const __half*>(x)[t * x_stride + k]);
    else v = static_cast<const float*>(x)[t * x_stride + k];
    uint16_t bits;
    if (out_f16) {
      const __half h = __float2half_rn(v);
      bits = *reinterpret_cast<const uint16_t*>(&h);
    } else {
      const __nv_bfloat16 b = __float2bfloat16_rn(v);
      bits = *reinterpret_cast<const uint16_t*>(&b);
    }
    xt[tiled_act_offset(static_cast<int>(t), k, nkb)] = bits;
  }
}

template <int W, int TN>
void configure_gemm() {
  static bool done = false;
  if (!done) {
    FQ_CUDA(cudaFuncSetAttribute(gemm_ws_kernel<W, TN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_gemm<TN>()));
    done = true;
  }
}

}  // namespace

int64_t tiled_act_elems(int64_t T, int64_t K) {
  return (T + kTN - 1) / kTN * kTN * ((K + kTK - 1) / kTK * kTK);
}

void launch_tile_acts(fq_ctx* ctx, const void* x, int x_dtype, int64_t x_stride, int64_t T, int64_t K, void* xt,
                      int out_dtype) {
  const int64_t total = T * K;
  const int blocks = static_cast<int>(std::min<int64_t>(ctx->num_sms * 8, (total + 255) / 256));
  tile_acts_kernel<<<std::max(blocks, 1), 256, 0, ctx->stream>>>(x, x_dtype, x_stride, static_cast<int>(T), K,
                                                                 ceil_div_i(K, kTK), out_dtype == FQ_DT_F16 ? 1 : 0,
                                                                 static_cast<uint16_t*>(xt));
  FQ_CUDA(cudaGetLastError());
  ctx->launches += 1;
}

void launch_gemm_dq(fq_ctx* ctx, const fq_layer* L, int rung, int64_t T, const void* xt, int x_dtype, float* y,
                    int64_t y_stride, bool accumulate, const uint8_t* row_rung, int64_t rr_stride) {
  if (rung != FQ_RUNG_INT8 && rung != FQ_RUNG_INT4) fail(FQ_E_CONFIG, "gemm: rung must be 8 or 4");
  if (x_dtype != FQ_DT_F16) fail(FQ_E_CONFIG, "gemm: the tiled activations are fp16 (bf16 values stored exactly)");
  const fq_rung_store& st = L->store(rung);
  if (!st.present || st.tiles == nullptr) fail(FQ_E_STATE, "gemm: rung not resident in the tiled layout");
  if (T < 1) fail(FQ_E_DIMENSION, "gemm: no rows");
  if ((reinterpret_cast<uintptr_t>(xt) & 15) != 0) fail(FQ_E_CONFIG, "gemm: tiled activations must be 16-byte aligned");
  const int n_tiles = ceil_div_i(L->N, kTileRows), nkb = ceil_div_i(L->K, kBlockK);
  const int tn = T <= 32 ? 32 : kTN;  // decode-sized batches: 32-token MMAs, a quarter of the activation traffic
  const int gx = ceil_div_i(L->N, kTM), gy = ceil_div_i(T, tn);
  // split K when the output tiles alone leave SMs idle: the fewest splits with the lowest
  // (waves x work per split), at least 4 k-blocks per split
  // the split-K reduction is a separate pass over splits x T x N floats: split only grids that
  // leave more than half the SMs idle (decode-sized batches), not to even out waves
  int splits = 1;
  if (static_cast<int64_t>(gx) * gy * 2 <= ctx->num_sms) {
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
  const int acc = splits > 1 ? 0 : (accumulate ? 1 : 0);
  const auto* xb = static_cast<const uint8_t*>(xt);
#define FQ_GEMM_LAUNCH(Wv, TNv)                                                                              \
  do {                                                                                                      \
    configure_gemm<Wv, TNv>();                                                                              \
    FQ_CUDA(cudaLaunchKernelEx(&lc, gemm_ws_kernel<Wv, TNv>, st.tiles, n_tiles, nkb, st.zp_base, L->N, xb,     \
                               static_cast<int>(T), out, out_stride, acc, splits, split_stride,                \
                               splits > 1 ? nullptr : row_rung, rr_stride, rung));                          \
  } while (0)
  // programmatic dependent launch: the kernel may start while the previous one drains (its
  // producer prefetches weights, then waits on the dependency before reading activations)
  cudaLaunchAttribute pdl[1];
  pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = grid;
  lc.blockDim = dim3(kGemmThreads);
  lc.stream = ctx->stream;
  lc.attrs = pdl;
  lc.numAttrs = 1;
  if (rung == FQ_RUNG_INT8) {
    if (tn == 32) {
      lc.dynamicSmemBytes = smem_gemm<32>();
      FQ_GEMM_LAUNCH(0, 32);
    } else {
      lc.dynamicSmemBytes = smem_gemm<128>();
      FQ_GEMM_LAUNCH(0, 128);
    }
  } else {
    if (tn == 32) {
      lc.dynamicSmemBytes = smem_gemm<32>();
      FQ_GEMM_LAUNCH(1, 32);
    } else {
      lc.dynamicSmemBytes = smem_gemm<128>();
      FQ_GEMM_LAUNCH(1, 128);
    }
  }
#undef FQ_GEMM_LAUNCH
  FQ_CUDA(cudaGetLastError());
  ctx->launches += 1;
  if (splits > 1) {
    const int64_t total = T * L->N;
    const int blocks = static_cast<int>(std::min<int64_t>(ctx->num_sms * 8, (total + 255) / 256));
    split_reduce_kernel<<<blocks, 256, 0, ctx->stream>>>(ctx->gemm_ws, splits, T, L->N, y, y_stride, accumulate ? 1 : 0,
                                                         row_rung, rr_stride, rung);
    FQ_CUDA(cudaGetLastError());
    ctx->launches += 1;
  }
}

}  // namespace fqc
