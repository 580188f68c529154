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
// One CTA = 128 weight rows (UMMA M) x TN tokens (UMMA N = 128, or 32 for decode-sized
// batches), warp-specialised; every hand-off is an mbarrier:
//   producer   (warp 0) per k-block: lane 0 arms the stage's barrier with the byte count, lanes 0-7
//              bulk-copy (cp.async.bulk) the CTA's eight raw 16x128 weight blocks and lane 8 the
//              activation tile (X is stored pre-tiled in the UMMA canonical K-major layout, see
//              tiled_act_offset) into the input ring;
//   dequantisers (groups of 8 warps, one raw block per warp): raw codes -> exact fp16 (q - z)
//              into the A-operand ring (canonical K-major, no swizzle) and the block's row scales
//              into a scale ring; fence.proxy.async, named barrier, one arrival on a_full;
//   MMA issuers (one thread each): 8 x tcgen05.mma (K16) per k-block into one of the TMEM
//              accumulator buffers, then ONE tcgen05.commit on mma_done[k-block], which is at once
//              the epilogue's "accumulator full", the dequantisers' "A slot free" and the
//              producer's "stage free";
//   epilogue   (4 or 8 warps): tcgen05.ld of the k-block's accumulator (lane quarter = warp % 4),
//              y += s[row, kb] * D in registers, d_empty arrival.
// Measured (clock64 traces of one CTA, tools/gemm_bench.py): an mbarrier wait costs 150-450 cycles
// even when the phase is already complete, a bulk-copy issue ~150, a tcgen05.mma issue ~65, so the
// loop is shaped to put as few of them as possible on any one thread per k-block; at TN = 32 two
// dequantiser groups and two MMA issuers take alternating k-blocks.
#include "gemv_program.cuh"


namespace fqc {
namespace {

constexpr int kTM = 128;                      // weight rows per CTA (UMMA M)
constexpr int kTN = 128;                      // tokens per activation tile (the tiled layout's row block)
constexpr int kTK = 128;                      // codes per k-block (one tiled block / group)
constexpr int kTileBytes = kTM * kTK * 2;     // bf16 128 x 128 tile: 32 KB (A and B alike)
// ring depths (shared memory: 227 KB per CTA): input stages of raw blocks + activation tile (49 KB
// at TN = 128, 25 KB at TN = 32), dequantised A slots (32 KB), TMEM accumulator buffers (the
// epilogue scales every k-block's D by its own per-row scale, so MMA k-block i waits for the
// epilogue of i - d_bufs)
template <int TN>
constexpr int in_stages() { return TN == 32 ? 5 : 3; }
constexpr int kMaxInStages = 6;
template <int TN>
constexpr int a_stages() { return TN == 32 ? 3 : 2; }
constexpr int kMaxAStages = 4;
template <int TN>
constexpr int d_bufs() { return TN == 32 ? 8 : 4; }
constexpr int kMaxDBufs = 16;
// warps: 0 producer, then MI MMA issuers, E epilogue warps, and G groups of 8 dequantisers (one
// raw block per warp).  Every mbarrier hand-off costs a few hundred cycles of wake-up, so at
// TN = 32 (where a k-block's MMAs are short) two dequantiser groups and two MMA issuers work on
// alternating k-blocks: 1 + 2 + 4 + 16 = 23 warps (<= 88 registers; 32 fp32 sums per epilogue
// thread).  At TN = 128 the MMAs themselves pace the loop: 1 + 1 + 8 + 8 = 18 warps (<= 112), two
// epilogue warps per TMEM lane quarter with 64 columns each.
template <int TN>
constexpr int mma_issuers() { return TN == 32 ? 2 : 1; }
template <int TN>
constexpr int epi_warps() { return TN == 128 ? 8 : 4; }
template <int TN>
constexpr int dq_groups() { return TN == 32 ? 2 : 1; }
template <int TN>
constexpr int gemm_threads() { return 32 * (1 + mma_issuers<TN>() + epi_warps<TN>() + 8 * dq_groups<TN>()); }
constexpr int kDequantThreads = 256;  // per group
constexpr int kRawBytes = 8 * kBlockBytes8;   // 8 raw 16x128 blocks (W8 size; W4 uses half)
// tokens per CTA (UMMA N): 128, or 32 for decode-sized batches (the first 32 rows of a 128-row
// tile are its first 8 KB in the canonical layout, so the same tiled activations serve both)
template <int TN>
constexpr int smem_gemm() { return in_stages<TN>() * (TN * 256 + kRawBytes) + a_stages<TN>() * kTileBytes + 1024; }

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// canonical K-major no-swizzle layout of a 128x128 16-bit tile: element (row, k) at byte
// (row >> 3) * 2048 + (k >> 3) * 128 + (row & 7) * 16 + (k & 7) * 2 -- 8x16-byte core matrices,
// LBO = 128 B (K-adjacent core matrices), SBO = 2 KB (8-row groups)
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

// One dequantiser warp per raw 16x128 block of the stage (rt = 0..7): lane (r, c2) = (lane >> 2,
// 2 (lane & 3)) holds, in every 16-byte code word of the block, codes of rows r and r + 8 only, so
// its two zero-point pairs are loaded once per k-block and every store lands at a compile-time
// offset from one per-thread base (row 16 rt + r, k & 7 = c2 of the canonical K-major tile).
template <int W>
__device__ __forceinline__ void dequant_block(const uint8_t* raw, int32_t zbase, uint8_t* a_tile, int rt, int lane) {
  constexpr int bb = W == 0 ? kBlockBytes8 : kBlockBytes4;
  constexpr int cbytes = W == 0 ? 2048 : 1024;
  constexpr int words = W == 0 ? 4 : 2;  // 16-byte code words per lane
  const uint8_t* blk = raw + rt * bb;
  const int r = lane >> 2, c2 = 2 * (lane & 3);
  uint4 wv[words];
#pragma unroll
  for (int i = 0; i < words; ++i) wv[i] = reinterpret_cast<const uint4*>(blk)[i * 32 + lane];
  const uint32_t z0 = zpair(blk + cbytes + 64, r, zbase), z1 = zpair(blk + cbytes + 64, r + 8, zbase);
  uint8_t* base = a_tile + rt * 4096 + r * 16 + c2 * 2;  // + (k >> 3) * 128, + 2048 for row + 8
#pragma unroll
  for (int i = 0; i < words; ++i) {
    const uint32_t q4[4] = {wv[i].x, wv[i].y, wv[i].z, wv[i].w};
    if constexpr (W == 0) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {  // word j = (h, e): bytes (r, k0), (r, k0+1), (r+8, k0), (r+8, k0+1)
        const int col = 4 * i + j;   // k0 = 16 (2i + h) + c2 + 8e  ->  k0 >> 3 = 4i + 2h + e
        *reinterpret_cast<uint32_t*>(base + col * 128) = hsub2(prmt(q4[j], 0x64646464u, 0x4140u), z0);
        *reinterpret_cast<uint32_t*>(base + 2048 + col * 128) = hsub2(prmt(q4[j], 0x64646464u, 0x4342u), z1);
      }
    } else {
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        // nibbles (low to high): (r,k0) (r,k0+8) (r+8,k0) (r+8,k0+8) (r,k0+1) (r,k0+9) (r+8,k0+1) (r+8,k0+9),
        // k0 = 16 (4i + v) + c2
        const int col = 2 * (4 * i + v);
        const uint32_t q = q4[v];
        *reinterpret_cast<uint32_t*>(base + col * 128) = hsub2(nib_pair(q), z0);
        *reinterpret_cast<uint32_t*>(base + (col + 1) * 128) = hsub2(nib_pair(q >> 4), z0);
        *reinterpret_cast<uint32_t*>(base + 2048 + col * 128) = hsub2(nib_pair(q >> 8), z1);
        *reinterpret_cast<uint32_t*>(base + 2048 + (col + 1) * 128) = hsub2(nib_pair(q >> 12), z1);
      }
    }
  }
}

// One launch covers a GROUP of products of the same tiled activations (q/k/v, gate/up, the
// precision copies of one linear in a mixed batch): blockIdx.z = problem * splits + split; CTAs
// past a problem's own row count exit at once.  Each problem carries its copy's code width, so W8
// and W4 products share a launch.
constexpr int kMaxProblems = 8;
struct GemmProblem {
  const uint8_t* tiles;
  float* y;
  const uint8_t* row_rung;  // rows (tokens) of this problem: row_rung[t * rr_stride] == want_rung, or all
  int64_t N, y_stride, rr_stride;
  int n_tiles;  // 16-row tiles of the tiled copy
  int32_t zbase;
  int bits, accumulate, want_rung;
};
struct GemmGroup {
  GemmProblem p[kMaxProblems];
  const uint8_t* xt;     // tiled fp16 activations [T, K]
  int64_t split_stride;  // floats between split partial outputs (splits > 1: one problem only)
  int T, nkb, splits;
};

template <int TN>
__global__ void __launch_bounds__(gemm_threads<TN>(), 1) gemm_ws_kernel(const __grid_constant__ GemmGroup g) {
  constexpr int kBBytes = TN * 256;  // activation bytes per k-block
  constexpr int kInStages = in_stages<TN>();
  constexpr int kAStages = a_stages<TN>();
  const int prob = blockIdx.z / g.splits, split = blockIdx.z - prob * g.splits;
  const uint8_t* tiles = nullptr;
  float* y = nullptr;
  const uint8_t* row_rung = nullptr;
  int64_t N = 0, y_stride = 0, rr_stride = 0;
  int n_tiles = 0, bits = 8, accumulate = 0, want_rung = 0;
  int32_t zbase = 0;
#pragma unroll
  for (int k = 0; k < kMaxProblems; ++k)  // static indices only: the table stays in parameter space
    if (k == prob) {
      tiles = g.p[k].tiles;
      y = g.p[k].y;
      row_rung = g.p[k].row_rung;
      N = g.p[k].N;
      y_stride = g.p[k].y_stride;
      rr_stride = g.p[k].rr_stride;
      n_tiles = g.p[k].n_tiles;
      zbase = g.p[k].zbase;
      bits = g.p[k].bits;
      accumulate = g.p[k].accumulate;
      want_rung = g.p[k].want_rung;
    }
  if (static_cast<int64_t>(blockIdx.x) * kTM >= N) return;  // shorter problem of the group
  const int nkb = g.nkb, T = g.T, splits = g.splits;
  const uint8_t* xt = g.xt;
  const int64_t split_stride = g.split_stride;
  const int bb = bits == 8 ? kBlockBytes8 : kBlockBytes4;
  const int cbytes = bits == 8 ? 2048 : 1024;
  extern __shared__ __align__(1024) uint8_t gsm[];
  constexpr int kDBufs = d_bufs<TN>();
  // mma_done[i % kR] completes (one tcgen05.commit) when k-block i's MMAs are done: it is the
  // epilogue's "accumulator full", the dequantisers' "A slot free" (lag kAStages) and the
  // producer's "stage free" (lag kInStages; the MMAs ran after the dequant of the raw blocks).  A
  // waiter must never fall a whole phase behind: MMA i + kR needs the epilogue of i + kR - kDBufs
  // and the bytes of k-block i + kR - kAStages (loaded in order, at most kInStages ahead of the
  // slowest dequant), so kR >= max(kDBufs, kAStages + kInStages) suffices; twice that is used.
  constexpr int kR0 = kDBufs > kAStages + kInStages ? kDBufs : kAStages + kInStages;
  constexpr int kR = 2 * kR0 > kMaxDBufs ? kMaxDBufs : 2 * kR0;
  static_assert(kR >= kR0, "mma_done ring too short");
  __shared__ uint64_t in_full[kMaxInStages], a_full[kMaxAStages], mma_done[kMaxDBufs], d_empty[kMaxDBufs];
  constexpr int kScSlots = kAStages + kDBufs;
  __shared__ float sc_ring[kScSlots * kTM];
  __shared__ uint32_t tmem_base_s;
  uint8_t* base = gsm + ((1024u - (smem_addr(gsm) & 1023u)) & 1023u);  // 1 KB aligned, still a shared pointer
  uint8_t* b_ring = base;                                        // kInStages x 32 KB activations
  uint8_t* raw_ring = b_ring + kInStages * kBBytes;              // kInStages x 8 raw blocks
  uint8_t* a_ring = raw_ring + kInStages * kRawBytes;            // kAStages x 32 KB bf16 (q - z)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t tile0 = static_cast<int64_t>(blockIdx.x) * (kTM / kTileRows);
  const int tt = blockIdx.y;  // token tile of TN rows
  const int64_t b_src = static_cast<int64_t>(tt * TN / kTN) * nkb * kTileBytes + (tt * TN % kTN) * 256;
  const int kb0 = static_cast<int>(static_cast<int64_t>(nkb) * split / splits);
  const int kb1 = static_cast<int>(static_cast<int64_t>(nkb) * (split + 1) / splits);
  const int nk = kb1 - kb0;
  y += split * split_stride;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kInStages; ++s) mbar_init(&in_full[s], 1);
    for (int s = 0; s < kAStages; ++s) mbar_init(&a_full[s], 1);
    for (int s = 0; s < kR; ++s) mbar_init(&mma_done[s], 1);
    for (int s = 0; s < kDBufs; ++s) mbar_init(&d_empty[s], epi_warps<TN>());  // one arrival per epilogue warp
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tmem_base_s)),
                 "r"(kDBufs * TN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_s;
#ifdef FQ_GEMM_TRACE
  __shared__ long long trc[9][24];
  const bool trace_cta = blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0;
#define TRC(k, i) do { if (trace_cta && (i) < 24) trc[k][i] = clock64(); } while (0)
  TRC(6, 0);
#else
#define TRC(k, i) do {} while (0)
#endif

  if (warp == 0) {
    // ---------------- producer: lane 0 arms the stage barrier, then lanes 0-7 issue the eight
    // raw-block copies and lane 8 the activation tile in parallel (bulk copies issued back to back
    // by one thread cost ~150 cycles each: nine of them took longer than the k-block)
    auto issue = [&](int s, int kb) {
      if (lane < 8) {
        const int64_t tile = min(tile0 + lane, static_cast<int64_t>(n_tiles) - 1);
        bulk_g2s(raw_ring + s * kRawBytes + lane * bb, tiles + (tile * nkb + kb) * bb, bb, &in_full[s]);
      } else if (lane == 8) {
        bulk_g2s(b_ring + s * kBBytes, xt + b_src + static_cast<int64_t>(kb) * kTileBytes, kBBytes, &in_full[s]);
      }
    };
    for (int i = 0; i < nk; ++i) {
      const int s = i % kInStages;
      if (lane == 0) {
        if (i >= kInStages) mbar_wait(&mma_done[(i - kInStages) % kR], ((i - kInStages) / kR) & 1, 0);
        mbar_expect_tx(&in_full[s], kBBytes + 8 * bb);
      }
      __syncwarp();
      issue(s, kb0 + i);
    }
  } else if (warp <= mma_issuers<TN>()) {
    // ---------------- MMA issuers: issuer m = warp - 1 takes k-blocks i = m (mod MI); each
    // tcgen05.commit tracks only its own thread's MMAs
    if (lane == 0) {
      for (int i = warp - 1; i < nk; i += mma_issuers<TN>()) {
        const int s = i % kInStages, a = i % kAStages, dbuf = i % kDBufs;
        // a_full(i) implies in_full(i): the dequantisers waited for the stage's bytes before
        // converting them
        mbar_wait(&a_full[a], (i / kAStages) & 1, 1);
        if (i >= kDBufs) mbar_wait(&d_empty[dbuf], ((i / kDBufs) - 1) & 1, 1);
        TRC(3, i);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint64_t da = umma_desc(smem_addr(a_ring + a * kTileBytes)), db = umma_desc(smem_addr(b_ring + s * kBBytes));
        const uint32_t dt = tmem + static_cast<uint32_t>(dbuf * TN);
#pragma unroll
        for (int j = 0; j < kTK / 16; ++j) {  // K step of 16 = 256 B = +16 in the descriptors' address field
          asm volatile(
              "{\n\t.reg .pred p;\n\t"
              "setp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(dt),
              "l"(da + 16u * j), "l"(db + 16u * j), "r"(idesc<1, TN>()), "r"(j > 0 ? 1u : 0u));
        }
        TRC(7, i);
        tc_commit(&mma_done[i % kR]);
        TRC(8, i);
      }
    }
  } else if (warp >= 1 + mma_issuers<TN>() + epi_warps<TN>()) {
    // ---------------- dequantisers: group g takes k-blocks i = g (mod G); its warp rt converts
    // raw block rt of the stage
    const int dw = warp - 1 - mma_issuers<TN>() - epi_warps<TN>();
    const int g = dw >> 3, rt = dw & 7;
    for (int i = g; i < nk; i += dq_groups<TN>()) {
      const int s = i % kInStages, a = i % kAStages;
      mbar_wait(&in_full[s], (i / kInStages) & 1, 2);
      if (i >= kAStages) mbar_wait(&mma_done[(i - kAStages) % kR], ((i - kAStages) / kR) & 1, 2);
      if (g == 0 && rt == 0 && lane == 0) TRC(1, i);
      const uint8_t* raw = raw_ring + s * kRawBytes;
      if (bits == 8) dequant_block<0>(raw, zbase, a_ring + a * kTileBytes, rt, lane);
      else dequant_block<1>(raw, zbase, a_ring + a * kTileBytes, rt, lane);
      // the block's 16 row scales into the scale ring the epilogue reads: the slot is rewritten by
      // the dequant of k-block i + kScSlots, which waits for MMA i + kDBufs, which
      // waited (d_empty) for this k-block's epilogue
      if (lane < 16) sc_ring[(i % kScSlots) * kTM + rt * 16 + lane] = reinterpret_cast<const float*>(raw + rt * bb + cbytes)[lane];
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core
      asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "n"(kDequantThreads) : "memory");
      if (rt == 0 && lane == 0) {
        if (g == 0) TRC(2, i);
        mbar_arrive(&a_full[a]);
      }
    }
  } else {
    // ---------------- epilogue: TMEM lane quarter q = warp % 4 = weight rows 32q.., columns
    // [half * EC, half * EC + EC) of the k-block's accumulator
    constexpr int EC = TN * 4 / epi_warps<TN>();
    const int q = warp & 3, half = (warp - 1 - mma_issuers<TN>()) >> 2;
    const int row = q * 32 + lane;
    const int64_t n = static_cast<int64_t>(blockIdx.x) * kTM + row;
    float acc[EC];
#pragma unroll
    for (int c = 0; c < EC; ++c) acc[c] = 0.f;
    for (int i = 0; i < nk; ++i) {
      const int dbuf = i % kDBufs;
      mbar_wait(&mma_done[i % kR], (i / kR) & 1, 3);
      if (q == 0 && lane == 0) TRC(4, i);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const float s_kb = sc_ring[(i % kScSlots) * kTM + row];
      const uint32_t taddr = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(dbuf * TN + half * EC);
#pragma unroll
      for (int c0 = 0; c0 < EC; c0 += 16) {
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
      if (q == 0 && lane == 0) TRC(5, i);
    }
    if (n < N) {
      const int t0 = tt * TN + half * EC;
#pragma unroll
      for (int c = 0; c < EC; ++c) {
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
#ifdef FQ_GEMM_TRACE
  if (trace_cta && threadIdx.x == 0) {
    printf("TRACE nk=%d start=%lld\n", nk, trc[6][0]);
    for (int i = 0; i < min(nk, 24); ++i) {
      printf("TRACE %d P %lld D0 %lld D1 %lld M %lld Mi %lld Mc %lld E0 %lld E1 %lld\n", i, trc[0][i] - trc[6][0], trc[1][i] - trc[6][0],
             trc[2][i] - trc[6][0], trc[3][i] - trc[6][0], trc[7][i] - trc[6][0], trc[8][i] - trc[6][0], trc[4][i] - trc[6][0], trc[5][i] - trc[6][0]);
    }
  }
#endif
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kDBufs * TN));
}

// y[t][n] (+)= sum over the splits in order of ws[z][t][n] (deterministic split-K reduction)
__global__ void split_reduce_kernel(const float* __restrict__ ws, int splits, int64_t T, int64_t N, float* __restrict__ y,
                                    int64_t y_stride, int accumulate, const uint8_t* __restrict__ row_rung,
                                    int64_t rr_stride, int want_rung) {
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

template <int TN>
void configure_gemm() {
  static bool done = false;
  if (!done) {
    FQ_CUDA(cudaFuncSetAttribute(gemm_ws_kernel<TN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_gemm<TN>()));
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

namespace {
// launch-time model (measured, tools/gemm_bench.py): a CTA streams a k-block in ~0.6 us whatever
// the grid, a launch costs ~6 us of prologue / drain, a split-K reduction pass ~3 us
constexpr double kUsPerKb = 0.63, kUsLaunch = 6.0, kUsReduce = 3.0;
int best_splits(int64_t ctas, int nkb, int sms, double* cost) {
  int splits = 1;
  double best = static_cast<double>((ctas + sms - 1) / sms) * nkb * kUsPerKb;
  if (ctas * 2 <= sms)
    for (int sp = 2; sp <= 8 && nkb / sp >= 4; ++sp) {
      const double c = static_cast<double>((ctas * sp + sms - 1) / sms) * ((nkb + sp - 1) / sp) * kUsPerKb + kUsReduce;
      if (c < best - 1e-9) {
        best = c;
        splits = sp;
      }
    }
  if (cost != nullptr) *cost = best + kUsLaunch;
  return splits;
}
}  // namespace

void launch_gemm_group(fq_ctx* ctx, const GemmJob* jobs, int n_jobs, int64_t T, const void* xt) {
  if (n_jobs < 1 || n_jobs > kMaxProblems) fail(FQ_E_CONFIG, "gemm: 1..8 products per launch");
  if (n_jobs > 1) {
    // one launch for all, or one (possibly split-K) launch each: whichever the model says is faster
    const int tn0 = T <= 32 ? 32 : kTN;
    const int gy0 = ceil_div_i(T, tn0), nkb0 = ceil_div_i(jobs[0].L->K, kBlockK);
    int64_t ctas = 0;
    double separate = 0.0;
    for (int j = 0; j < n_jobs; ++j) {
      const int64_t c = static_cast<int64_t>(ceil_div_i(jobs[j].L->N, kTM)) * gy0;
      ctas += c;
      double cj = 0.0;
      best_splits(c, nkb0, ctx->num_sms, &cj);
      separate += cj;
    }
    const double grouped = static_cast<double>((ctas + ctx->num_sms - 1) / ctx->num_sms) * nkb0 * kUsPerKb + kUsLaunch;
    if (separate < grouped) {
      for (int j = 0; j < n_jobs; ++j) launch_gemm_group(ctx, jobs + j, 1, T, xt);
      return;
    }
  }
  if (T < 1) fail(FQ_E_DIMENSION, "gemm: no rows");
  if ((reinterpret_cast<uintptr_t>(xt) & 15) != 0) fail(FQ_E_CONFIG, "gemm: tiled activations must be 16-byte aligned");
  const int64_t K = jobs[0].L->K;
  const int tn = T <= 32 ? 32 : kTN;  // decode-sized batches: 32-token MMAs, a quarter of the activation traffic
  GemmGroup g = {};
  g.xt = static_cast<const uint8_t*>(xt);
  g.T = static_cast<int>(T);
  g.nkb = ceil_div_i(K, kBlockK);
  int gx = 0;
  for (int j = 0; j < n_jobs; ++j) {
    const GemmJob& jb = jobs[j];
    if (jb.rung != FQ_RUNG_INT8 && jb.rung != FQ_RUNG_INT4) fail(FQ_E_CONFIG, "gemm: rung must be 8 or 4");
    if (jb.L->K != K) fail(FQ_E_DIMENSION, "gemm: products of one launch share K");
    const fq_rung_store& st = jb.L->store(jb.rung);
    if (!st.present || st.tiles == nullptr) fail(FQ_E_STATE, "gemm: rung not resident in the tiled layout");
    GemmProblem& P = g.p[j];
    P.tiles = st.tiles;
    P.y = jb.y;
    P.row_rung = jb.row_rung;
    P.N = jb.L->N;
    P.y_stride = jb.y_stride;
    P.rr_stride = jb.rr_stride;
    P.n_tiles = ceil_div_i(jb.L->N, kTileRows);
    P.zbase = st.zp_base;
    P.bits = st.bits;
    P.accumulate = jb.accumulate ? 1 : 0;
    P.want_rung = jb.rung;
    gx = std::max(gx, ceil_div_i(jb.L->N, kTM));
  }
  const int gy = ceil_div_i(T, tn);
  // split K (one product only) when the output tiles alone leave more than half the SMs idle
  // (decode-sized batches), per the launch-time model; the partial sums are reduced by a separate
  // deterministic pass
  const int splits = n_jobs == 1 ? best_splits(static_cast<int64_t>(gx) * gy, g.nkb, ctx->num_sms, nullptr) : 1;
  g.splits = splits;
  const GemmJob& j0 = jobs[0];
  if (splits > 1) {
    const size_t need = sizeof(float) * static_cast<size_t>(splits) * T * j0.L->N;
    if (ctx->gemm_ws_bytes < need) {
      if (ctx->gemm_ws != nullptr) ctx->retired.push_back(ctx->gemm_ws);  // captured graphs may hold it
      ctx->gemm_ws = static_cast<float*>(dmalloc(need));
      ctx->gemm_ws_bytes = need;
    }
    g.p[0].y = ctx->gemm_ws;  // partials [split][T][N], reduced below
    g.p[0].y_stride = j0.L->N;
    g.p[0].accumulate = 0;
    g.p[0].row_rung = nullptr;
    g.split_stride = T * j0.L->N;
  }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(static_cast<unsigned>(gx), static_cast<unsigned>(gy), static_cast<unsigned>(splits * n_jobs));
  lc.stream = ctx->stream;
  if (tn == 32) {
    configure_gemm<32>();
    lc.blockDim = dim3(gemm_threads<32>());
    lc.dynamicSmemBytes = smem_gemm<32>();
    FQ_CUDA(cudaLaunchKernelEx(&lc, gemm_ws_kernel<32>, g));
  } else {
    configure_gemm<128>();
    lc.blockDim = dim3(gemm_threads<128>());
    lc.dynamicSmemBytes = smem_gemm<128>();
    FQ_CUDA(cudaLaunchKernelEx(&lc, gemm_ws_kernel<128>, g));
  }
  FQ_CUDA(cudaGetLastError());
  ctx->launches += 1;
  if (splits > 1) {
    const int64_t total = T * j0.L->N;
    const int blocks = static_cast<int>(std::min<int64_t>(ctx->num_sms * 8, (total + 255) / 256));
    split_reduce_kernel<<<std::max(blocks, 1), 256, 0, ctx->stream>>>(ctx->gemm_ws, splits, T, j0.L->N, j0.y, j0.y_stride,
                                                                   j0.accumulate ? 1 : 0, j0.row_rung, j0.rr_stride,
                                                                   j0.rung);
    FQ_CUDA(cudaGetLastError());
    ctx->launches += 1;
  }
}

void launch_gemm_dq(fq_ctx* ctx, const fq_layer* L, int rung, int64_t T, const void* xt, int x_dtype, float* y,
                    int64_t y_stride, bool accumulate, const uint8_t* row_rung, int64_t rr_stride) {
  if (x_dtype != FQ_DT_F16) fail(FQ_E_CONFIG, "gemm: the tiled activations are fp16 (bf16 values stored exactly)");
  const GemmJob job{L, rung, y, y_stride, accumulate, row_rung, rr_stride};
  launch_gemm_group(ctx, &job, 1, T, xt);
}

}  // namespace fqc
