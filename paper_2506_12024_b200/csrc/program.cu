// Persistent TMA-fed program kernel (see gemv.cu for the design):
//   warp kNCW        producer: streams every GEMV phase's block range through the smem ring
//   warps 0..kNCW-1  consumers: GEMV compute (tensor-core m16n8k16 over the unpacked codes, one
//                    16x128 block per warp at a time), embedding, attention (groups of 4 warps)
//                    and row statistics, with a grid-wide barrier between dependent phases.
#include "gemv_program.cuh"

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <type_traits>
#ifndef FQ_DBG
#define FQ_DBG 0
#endif
// once-per-step phases (embedding, statistics, prefill append): out of line unless FQ_STEP_INLINE
#ifndef FQ_STEP_INLINE
#define FQ_STEP_INLINE 0
#endif
#if FQ_STEP_INLINE
#define FQ_ONCE __device__ __forceinline__
#else
#define FQ_ONCE __device__ __noinline__
#endif
#ifndef FQ_GEMV_HOOKS
#define FQ_GEMV_HOOKS 1  // per-phase GEMV detail stamps (tools/phase_profile.py); 0 compiles them out
#endif
#ifndef FQ_SQ_B
#define FQ_SQ_B 1  // residual tail: shuffle only the batch rows present
#endif
#include <cfloat>
#include <cstring>
#include <map>
#include <mutex>

namespace fqc {

// Per-phase timing hook (profiling only): when set, consumer thread 0 of every CTA records
// %globaltimer at the end of each phase and after the grid barrier that follows it:
// prof[(phase * grid + cta) * 2 + {0, 1}], kernel entry at prof[nphases * grid * 2 + cta].
__device__ unsigned long long* g_phase_prof = nullptr;
// GEMV phase detail (profiling only): [(phase * grid + cta) * 8 + k], k = 0 setup done (warp 1),
// 1 norm factors done (warp 0), 2 first barrier, 3 staged, 4 weight loop done, 5 final reduction
// done, 6 phase done.
__device__ unsigned long long* g_gemv_prof = nullptr;
__device__ int g_cur_phase = 0;
// Ring trace (profiling only): for CTA g_trace_cta, stage s of the whole program records
// [3s] = producer got the empty slot, [3s+1] = consumer warp 0 saw the data, [3s+2] = consumer warp
// 0 released the slot; up to kTraceStages stages.
constexpr int kTraceStages = 16384;
__device__ unsigned long long* g_ring_trace = nullptr;
__device__ int g_trace_cta = 0;

void set_phase_profile(unsigned long long* dev) {
  FQ_CUDA(cudaMemcpyToSymbol(g_phase_prof, &dev, sizeof(dev)));
}
void set_gemv_profile(unsigned long long* dev) {
  FQ_CUDA(cudaMemcpyToSymbol(g_gemv_prof, &dev, sizeof(dev)));
}
void set_ring_trace(unsigned long long* dev, int cta) {
  FQ_CUDA(cudaMemcpyToSymbol(g_ring_trace, &dev, sizeof(dev)));
  FQ_CUDA(cudaMemcpyToSymbol(g_trace_cta, &cta, sizeof(cta)));
}

namespace {

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
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
__device__ __forceinline__ unsigned long long gtimer_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Deadlock watchdog: a wait that has not completed after kWatchdogNs reports where it is stuck
// and traps (the launch fails with an error instead of hanging the device).
constexpr unsigned long long kWatchdogNs = 4000000000ull;
__device__ __noinline__ void watchdog_fire(const char* what, int a, int b) {
  printf("fq watchdog: %s stuck (cta %d, thread %d, %d, %d)\n", what, blockIdx.x, threadIdx.x, a, b);
  __trap();
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  unsigned long long t0 = 0;
  for (uint32_t spins = 0;; ++spins) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return;
    if ((spins & 1023u) == 1023u) {
      const unsigned long long t = gtimer_now();
      if (t0 == 0) t0 = t;
      else if (t - t0 > kWatchdogNs) watchdog_fire("mbarrier", static_cast<int>(parity), static_cast<int>(spins));
    }
  }
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
__device__ __forceinline__ float2 ld_volatile_f2(const float2* p) {
  float2 v;
  asm volatile("ld.volatile.global.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

// (v & 0x00F000F0) | 0x54005400 in one LOP3: the two nibbles at bits 4-7 / 20-23 as fp16 64 + q.
// Written as PTX with both constants immediate so ptxas keeps one in a register instead of
// splitting the AND and the OR (the W4 unpack is ALU-bound).
__device__ __forceinline__ uint32_t nib_f16(uint32_t v) {
  uint32_t r;
  asm("lop3.b32 %0, %1, 0x00F000F0, 0x54005400, 0xEA;" : "=r"(r) : "r"(v));
  return r;
}

// D += A(16x16 f16, row) * B(16x8 f16, col), fp32 accumulators.
__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
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

// Activation k of batch row b in B-fragment order (the smem xs layout, fp16): block kb = k/128,
// k16 = (k%128)/16 -> (p, hh) = (k16>>1, k16&1), r = k%16 -> (tig, half, lo) = ((r&7)>>1, r>>3, r&1);
// uint4 (b*nkb + kb)*16 + p*4 + tig, half-word 2*(2*hh + half) + lo.
__device__ __forceinline__ void frag_store(__half* frag, int nkb, int b, int64_t k, float v) {
  const int kb = static_cast<int>(k >> 7), r = static_cast<int>(k & 127), j16 = r >> 4, r16 = r & 15;
  const int p = j16 >> 1, hh = j16 & 1, tig = (r16 & 7) >> 1, comp = 2 * hh + (r16 >> 3);
  frag[((static_cast<int64_t>(b) * nkb + kb) * 16 + p * 4 + tig) * 8 + comp * 2 + (r16 & 1)] = __float2half_rn(v);
}


// ---------------------------------------------------------------- the block sequence
// A GEMV phase is a sequence of 16x128 blocks: tile-major, and inside a tile one segment of nkb
// blocks per (matrix, copy) the batch needs.  CTA c owns the blocks whose first byte lies in
// [c, c+1) * total / grid (byte-balanced across the grid, a tile may be shared by neighbours).
struct Segs {
  int n;
  int m[2 * kMaxMat], w[2 * kMaxMat], mask[2 * kMaxMat];
  int64_t tile_bytes;
};

__device__ __forceinline__ int blk_bytes(int w) { return w == 0 ? kBlockBytes8 : kBlockBytes4; }

__device__ __noinline__ void phase_segs(const Phase& P, Segs& S) {  // one copy: setup paths only
  // all rung bytes are loaded first (independent loads, one round trip), then the masks
  uint8_t rg[kMaxMat][kMaxB];
#pragma unroll
  for (int m = 0; m < kMaxMat; ++m)
#pragma unroll
    for (int b = 0; b < kMaxB; ++b)
      rg[m][b] = (m < P.nmat && b < P.B)
                     ? (P.mat[m].rung_table ? P.mat[m].rung_table[b * P.mat[m].rung_stride] : static_cast<uint8_t>(P.mat[m].rung))
                     : static_cast<uint8_t>(0xFF);
  S.n = 0;
  S.tile_bytes = 0;
#pragma unroll
  for (int m = 0; m < kMaxMat; ++m)
#pragma unroll
    for (int w = 0; w < 2; ++w) {
      const uint8_t want = w == 0 ? FQ_RUNG_INT8 : FQ_RUNG_INT4;
      int mask = 0;
#pragma unroll
      for (int b = 0; b < kMaxB; ++b) mask |= (rg[m][b] == want) << b;
      if (mask == 0) continue;
      S.m[S.n] = m;
      S.w[S.n] = w;
      S.mask[S.n] = mask;
      S.tile_bytes += static_cast<int64_t>(P.nkb) * blk_bytes(w);
      ++S.n;
    }
}

#ifndef FQ_TILE_PART
#define FQ_TILE_PART 1
#endif
// 32-bit arithmetic: the builder guarantees a phase's bytes fit in 32 bits.
// FQ_TILE_PART: whole 16-row tiles per CTA (floor/ceil of n_tiles / grid): no tile is split, so no
// CTA waits for another's stream-K part; the <= 1 tile of imbalance is absorbed by the weight
// stream running ahead.  Otherwise byte-balanced ranges with stream-K fix-up of split tiles.
__device__ int64_t cta_start(const Phase& P, const Segs& S, int c) {
  if (S.n == 0) return 0;
  if (FQ_TILE_PART) {
    const int64_t t = (static_cast<int64_t>(P.n_tiles) * c) / gridDim.x;
    return t * S.n * P.nkb;
  }
  const uint32_t tb = static_cast<uint32_t>(S.tile_bytes);
  const uint32_t total = static_cast<uint32_t>(P.n_tiles) * tb;
  const uint32_t grid = gridDim.x;
  const uint32_t target = (total / grid) * c + ((total % grid) * c) / grid;
  const uint32_t t = target / tb;
  uint32_t r = target - t * tb;
  int64_t gb = static_cast<int64_t>(t) * S.n * P.nkb;
  for (int s = 0; s < S.n; ++s) {
    const uint32_t bb = blk_bytes(S.w[s]);
    const uint32_t sb = static_cast<uint32_t>(P.nkb) * bb;
    if (r < sb) return gb + (r + bb - 1) / bb;
    r -= sb;
    gb += P.nkb;
  }
  return gb;
}

struct StageRef {
  int64_t tile;
  int seg, kb, nb;
};

__device__ __forceinline__ StageRef next_stage(const Phase& P, const Segs& S, int64_t gb, int64_t gend) {
  const int64_t bpt = static_cast<int64_t>(S.n) * P.nkb;
  StageRef r;
  r.tile = gb / bpt;
  const int rem = static_cast<int>(gb - r.tile * bpt);
  r.seg = rem / P.nkb;
  r.kb = rem - r.seg * P.nkb;
  const int cap = S.w[r.seg] == 0 ? kStageBlocks8 : kStageBlocks4;
  r.nb = static_cast<int>(min(static_cast<int64_t>(min(cap, P.nkb - r.kb)), gend - gb));
  return r;
}

struct Ring {
  uint8_t* base;
  uint64_t* full;
  uint64_t* empty;
  int nstages;
};

// ---------------------------------------------------------------- producer
// Walks the weight stages of every GEMV phase of the program in order.
struct StageWalk {
  const Phase* phases;
  int nphases, ph;
  Segs S;
  int64_t gb, g1;

  __device__ void init(const Phase* p, int n) {
    phases = p;
    nphases = n;
    ph = -1;
    gb = g1 = 0;
  }
  // Next stage: source address and byte count; false at the end of the program.
  __device__ bool next(const uint8_t*& src, uint32_t& bytes) {
    while (gb >= g1) {
      if (++ph >= nphases) return false;
      const Phase& P = phases[ph];
      if (P.type != PH_GEMV) continue;
      phase_segs(P, S);
      if (S.n == 0) continue;
      gb = cta_start(P, S, blockIdx.x);
      g1 = cta_start(P, S, blockIdx.x + 1);
    }
    const Phase& P = phases[ph];
    const StageRef st = next_stage(P, S, gb, g1);
    gb += st.nb;
    const int w = S.w[st.seg];
    const int bb = blk_bytes(w);
    src = P.mat[S.m[st.seg]].tiles[w] + (st.tile * P.nkb + st.kb) * bb;
    bytes = static_cast<uint32_t>(st.nb * bb);
    return true;
  }
};

__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// The producer streams every stage through the ring; a second walk runs kPrefetchStages ahead
// and issues L2 prefetches, so HBM keeps streaming while the ring is full (the consumers are in a
// grid barrier, the activation staging or a non-GEMV phase) and ring refills hit L2.

__device__ void produce_all(const Phase* phases, int nphases, const Ring R, unsigned long long* tr, int prefetch) {
  StageWalk main, ahead;
  main.init(phases, nphases);
  ahead.init(phases, nphases);
  const uint8_t* psrc;
  uint32_t pbytes;
  bool more_ahead = prefetch > 0;  // < 0: no loads at all (FQ_PREFETCH=-1, profiling only)
  for (int i = 0; i < prefetch && more_ahead; ++i)
    if ((more_ahead = ahead.next(psrc, pbytes))) prefetch_l2(psrc, pbytes);
  int slot_i = 0, tn = 0;
  uint32_t phase_bit = 0;
  const uint8_t* src;
  uint32_t bytes;
  while (main.next(src, bytes)) {
    if (more_ahead && (more_ahead = ahead.next(psrc, pbytes))) prefetch_l2(psrc, pbytes);
    const int s = slot_i;
    mbar_wait(&R.empty[s], phase_bit ^ 1u);
    if (tr && tn < kTraceStages) tr[3 * tn] = gtimer();
    ++tn;
    if (++slot_i == R.nstages) {
      slot_i = 0;
      phase_bit ^= 1u;
    }
    if (prefetch < 0) {  // profiling: consumer-only timing, the ring keeps whatever it holds
      mbar_arrive(&R.full[s]);
      continue;
    }
    mbar_expect_tx(&R.full[s], bytes);
    bulk_g2s(R.base + static_cast<size_t>(s) * kStageBytes, src, bytes, &R.full[s]);
  }
}

// ---------------------------------------------------------------- consumers: GEMV
#ifndef FQ_RING_TRACE
#define FQ_RING_TRACE 0  // consumer-side ring stamps (tools/phase_profile.py; build with -DFQ_RING_TRACE=1)
#endif
// Shared-memory staging of a GEMV phase's activations (once per phase, all consumer threads):
//   xs[((b*nkb + kb)*4 + p)*4 + tig] = uint4 (batch-major: a lane's fragments sit at immediate offsets): the m16n8k16 B fragments {b0b1, b2b3} of MMAs 2p and
//       2p+1 of block kb for batch column b and thread-in-group tig (fp16, x converted exactly
//       from bf16/fp16 activations);
//   dx[kb*B + b] = {1024*X, 64*X, X, 0}: X = sum of the block's activations; the offsets the
//       magic-number unpack adds per block (fp16 0x6400|q = 1024+q for W8 bytes, 0x5400|q<<4 =
//       64+q for W4 nibbles).
struct GemvSmem {
  uint4* xs;
  float4* dx;
  float* red;   // reduction window: [slot][nmat][kNCW][16][B]
  float* sq;    // [kNCW * 32]
  float* rstd;  // [kMaxB]
  float* mbuf;  // [kMaxMat][16][B] owner's part of a shared tile
  unsigned long long* tr;  // ring trace (profiling) or null
  int* tn;
};

// Issue order: every global load of the first item batch (activations, norm gains) and the RMSNorm
// partials go out together, so the phase pays one round trip before its first MMA; warp b reduces
// row b's partials while the activation loads are in flight.
#ifndef FQ_STAGE_ITEMS
#define FQ_STAGE_ITEMS 2
#endif
constexpr int kStageItems = FQ_STAGE_ITEMS;  // items per thread per batch (loads in flight together)
static_assert(kMaxB <= kNCW, "one consumer warp per batch row computes its RMSNorm factor");

// Staging of the O projection's input when the attention phase ran split (attn_splits > 1): the
// splits' unnormalised partials are merged here, x = sum_s O_s e^(m_s - M) / sum_s l_s e^(m_s - M),
// rounded to the activation dtype exactly as the unsplit attention rounds its output.  All loads
// (every split's O values of this thread's items and the (m, l) pairs) go out together.

// Vectorised staging (16-byte loads of 8 consecutive activations): one load per 8 values (two
// for fp32 inputs / gains), every load of the phase in flight together when they fit VB vectors
// per thread (K = 11008 at B = 1: 6), so the phase pays one round trip.  Vector v covers
// k = kb*128 + 8c .. +7 of batch row b (v = (b*nkb + kb)*16 + c); its pairs (k, k+1) land in
// fragment slot xs[(b*nkb + kb)*16 + (c>>2)*4 + i].comp[c&3] for pair i (the m16n8k16 B layout:
// k16 = c>>1 -> (p, hh) = (c>>2, (c>>1)&1), half c&1, thread-in-group i).
template <int VB, bool F32, bool norm>
__device__ __forceinline__ void stage_vec(const Phase& P, const GemvSmem& G, unsigned long long* gp, const float (&pv)[8]) {
  const int B = P.B;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NT = kNCW * 32;
  const float* gain = P.norm_gain;
  const int nkb = P.nkb;
  const int nvec = B * nkb * 16;
  const int64_t K = P.K;
  const int adt = P.act_dtype;
  for (int base = 0;; base += NT * VB) {
    uint4 raw[VB][F32 ? 2 : 1];
    float4 gv[VB][norm ? 2 : 1];
#pragma unroll
    for (int s = 0; s < VB; ++s) {
      const int v = base + s * NT + tid;
      const int b = v / (nkb * 16), r = v - b * nkb * 16;
      const int64_t k0 = static_cast<int64_t>(r >> 4) * kBlockK + (r & 15) * 8;
      const bool on = v < nvec && k0 < K;
      const int64_t off = on ? b * P.x_stride + k0 : 0;
      if (F32) {
        const uint4* src = reinterpret_cast<const uint4*>(static_cast<const float*>(P.x) + off);
        raw[s][0] = src[0];
        raw[s][1] = src[1];
      } else {
        raw[s][0] = *reinterpret_cast<const uint4*>(static_cast<const unsigned short*>(P.x) + off);
      }
      if (norm) {
        const float4* g4 = reinterpret_cast<const float4*>(gain + (on ? k0 : 0));
        gv[s][0] = g4[0];
        gv[s][1] = g4[1];
      }
    }
    if (base == 0) {
      if (warp < B) {
        float r = 1.f;
        if (norm) {
          float sm = 0.f;
#pragma unroll
          for (int j = 0; j < 8; ++j) sm += pv[j];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, o);
          r = 1.0f / sqrtf(sm / static_cast<float>(P.K) + P.norm_eps);
        }
        if (lane == 0) G.rstd[warp] = r;
      }
      if (gp) gp[1] = gtimer();
      named_sync(1, NT);
      if (gp) gp[2] = gtimer();
    }
#pragma unroll
    for (int s = 0; s < VB; ++s) {
      const int v = base + s * NT + tid;
      const int b = v / (nkb * 16), r = v - b * nkb * 16;
      const int kb = r >> 4, c = r & 15;
      const int64_t k0 = static_cast<int64_t>(kb) * kBlockK + c * 8;
      const bool on = v < nvec && k0 < K;
      float x[8];
      if (F32) {
        const float* f = reinterpret_cast<const float*>(&raw[s][0]);
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = f[i];
      } else {
        const unsigned short* u = reinterpret_cast<const unsigned short*>(&raw[s][0]);
#pragma unroll
        for (int i = 0; i < 8; ++i)
          x[i] = P.x_dtype == FQ_DT_BF16 ? __uint_as_float(static_cast<uint32_t>(u[i]) << 16)
                                         : __half2float(__ushort_as_half(u[i]));
      }
      const float rs = G.rstd[on ? b : 0];
      const float* g8 = norm ? reinterpret_cast<const float*>(&gv[s][0]) : nullptr;
      float sum = 0.f;
      uint32_t hp[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float a = x[2 * i], bq = x[2 * i + 1];
        if (norm) {
          a = round_act(a * rs * g8[2 * i], adt);
          bq = round_act(bq * rs * g8[2 * i + 1], adt);
        }
        a = on ? __half2float(__float2half_rn(a)) : 0.f;
        bq = on ? __half2float(__float2half_rn(bq)) : 0.f;
        sum += a + bq;
        const __half2 h2 = __floats2half2_rn(a, bq);
        hp[i] = *reinterpret_cast<const uint32_t*>(&h2);
      }
      if (v < nvec) {
        uint32_t* dst = reinterpret_cast<uint32_t*>(G.xs + (static_cast<size_t>(b) * nkb + kb) * 16 + (c >> 2) * 4) + (c & 3);
#pragma unroll
        for (int i = 0; i < 4; ++i) dst[4 * i] = hp[i];
      }
      // the 16 vectors of a block sit on 16 consecutive lanes (v is 16-aligned per half-warp)
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      if (v < nvec && c == 0) G.dx[kb * B + b] = make_float4(1024.f * sum, 64.f * sum, sum, 0.f);
    }
    if (base + NT * VB >= nvec) break;
  }
  named_sync(1, NT);
}

__device__ __forceinline__ bool stage_vec_ok(const Phase& P) {
  const size_t es = P.x_dtype == FQ_DT_F32 ? 4 : 2;
  return (reinterpret_cast<uintptr_t>(P.x) & 15) == 0 && ((P.x_stride * es) & 15) == 0 && (P.K & 7) == 0 &&
         (P.norm_gain == nullptr || (reinterpret_cast<uintptr_t>(P.norm_gain) & 15) == 0);
}

// Per-block activation sums dx from fragment-ordered activations in shared memory (one warp per
// 128-block: four halves per lane, shuffle tree), then a consumer barrier.
__device__ __forceinline__ void frag_block_sums(const Phase& P, const GemvSmem& G) {
  const int B = P.B, nkb = P.nkb, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int blk = warp; blk < B * nkb; blk += kNCW) {
    const uint2 h4 = reinterpret_cast<const uint2*>(G.xs + static_cast<size_t>(blk) * 16)[lane];
    const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&h4.x));
    const float2 c = __half22float2(*reinterpret_cast<const __half2*>(&h4.y));
    float sum = (a.x + a.y) + (c.x + c.y);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const int b = blk / nkb, kb = blk - b * nkb;
    if (lane == 0) G.dx[kb * B + b] = make_float4(1024.f * sum, 64.f * sum, sum, 0.f);
  }
  named_sync(1, kNCW * 32);
}


// Staging of an input the producing phase already wrote in fragment order: a straight copy (all
// loads of the phase in flight together), then the per-block sums dx from shared memory (one warp
// per 128-block: four halves per lane, shuffle tree).
constexpr int kCopyVec = 6;  // uint4s per thread per round (K = 11008 at B = 1: 1376 -> one round)
#ifndef FQ_COPY_INLINE
#define FQ_COPY_INLINE 1  // measured -1.8% per step vs an out-of-line call
#endif
#if FQ_COPY_INLINE
__device__ __forceinline__
#else
__device__ __noinline__
#endif
void stage_frag_copy(const Phase& P, const GemvSmem& G, unsigned long long* gp, unsigned int tag) {
  const int B = P.B, nkb = P.nkb;
  const int tid = threadIdx.x;
  constexpr int NT = kNCW * 32;
  const int n = B * nkb * 16;
  for (int base = 0; base < n; base += NT * kCopyVec) {
    uint4 v[kCopyVec];
#pragma unroll
    for (int s = 0; s < kCopyVec; ++s) {
      const int i = base + s * NT + tid;
      v[s] = i < n ? P.xfrag[i] : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int s = 0; s < kCopyVec; ++s) {
      const int i = base + s * NT + tid;
      if (i < n) G.xs[i] = v[s];
    }
  }
  if (gp) gp[1] = gtimer();
  named_sync(1, NT);
  if (gp) gp[2] = gtimer();
  frag_block_sums(P, G);
}

#ifndef FQ_VEC_STAGE
#define FQ_VEC_STAGE 1  // one round trip for K = 11008 (measured -0.6% per step at 11 consumer warps)
#endif
// LEAN (the decode / prefill step program, checked by the host builder): every GEMV input is either
// pre-staged fragments or the aligned fp32 residual under an RMSNorm, so only those two staging
// paths are compiled into that kernel (less code around the weight loop)
template <bool LEAN>
__device__ void stage_acts(const Phase& P, const GemvSmem& G, unsigned long long* gp, unsigned int xtag) {
  if (P.xfrag != nullptr) {
    stage_frag_copy(P, G, gp, xtag);
    return;
  }
  if constexpr (LEAN) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float pv[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int i = lane + 32 * j;
      pv[j] = (warp < P.B && i < P.n_partials) ? P.norm_partials[warp * P.partials_stride + i] : 0.f;
    }
    stage_vec<4, true, true>(P, G, gp, pv);
    return;
  }
  if (P.attn_splits > 1) __trap();  // the builder never splits attention (measured slower)
  const bool vnorm = P.norm_gain != nullptr;
  if (FQ_VEC_STAGE && stage_vec_ok(P) && vnorm == (P.x_dtype == FQ_DT_F32)) {
    const bool norm = vnorm;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float pv[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int i = lane + 32 * j;
      pv[j] = (norm && warp < P.B && i < P.n_partials) ? P.norm_partials[warp * P.partials_stride + i] : 0.f;
    }
    // the two shapes of the decode step: fp32 residual + RMSNorm, bf16/fp16 activations
    if (norm) stage_vec<4, true, true>(P, G, gp, pv);
    else stage_vec<6, false, false>(P, G, gp, pv);
    return;
  }
  const int B = P.B;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NT = kNCW * 32;
  const float* gain = P.norm_gain;
  // RMSNorm partials of row `warp` (fixed-order sums, as before)
  constexpr int kMaxParts = 8;  // 8 x 32 >= partials (grid <= 256)
  float pv[kMaxParts];
  if (warp < B && gain != nullptr) {
#pragma unroll
    for (int j = 0; j < kMaxParts; ++j) {
      const int i = lane + 32 * j;
      pv[j] = i < P.n_partials ? P.norm_partials[warp * P.partials_stride + i] : 0.f;
    }
  }
  const int items = P.nkb * B * 16;
  const int64_t K = P.K;
  const void* x = P.x;
  const int xdt = P.x_dtype, adt = P.act_dtype;
  for (int base = 0;; base += NT * kStageItems) {
    float raw[kStageItems][8], gn[kStageItems][8];
#pragma unroll
    for (int s = 0; s < kStageItems; ++s) {
      const int it = base + s * NT + tid;
      const bool active = it < items;
      const int kb = it / (B * 16);
      const int rem = it - kb * B * 16;
      const int b = active ? rem >> 4 : 0, p = (rem >> 2) & 3, tig = rem & 3;
      int64_t kc[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int hh = e >> 2, q = e & 3;
        const int64_t kk = static_cast<int64_t>(kb) * kBlockK + 16 * (2 * p + hh) + 2 * tig + (q & 1) + 8 * (q >> 1);
        kc[e] = active ? min(kk, K - 1) : 0;
      }
      // loads are unconditional (index clamped into the row) so they issue back to back; one
      // dtype branch around all eight
      if (xdt == FQ_DT_F32) {
        const float* xf = static_cast<const float*>(x) + b * P.x_stride;
#pragma unroll
        for (int e = 0; e < 8; ++e) raw[s][e] = xf[kc[e]];
      } else {
        const unsigned short* xh = static_cast<const unsigned short*>(x) + b * P.x_stride;
        unsigned short u[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) u[e] = xh[kc[e]];
#pragma unroll
        for (int e = 0; e < 8; ++e)
          raw[s][e] = xdt == FQ_DT_BF16 ? __uint_as_float(static_cast<uint32_t>(u[e]) << 16)
                                        : __half2float(__ushort_as_half(u[e]));
      }
      if (gain != nullptr) {
#pragma unroll
        for (int e = 0; e < 8; ++e) gn[s][e] = gain[kc[e]];
      }
    }
    if (base == 0) {
      if (warp < B) {
        float r = 1.f;
        if (gain != nullptr) {
          float sm = 0.f;
#pragma unroll
          for (int j = 0; j < kMaxParts; ++j) sm += pv[j];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, o);
          r = 1.0f / sqrtf(sm / static_cast<float>(P.K) + P.norm_eps);
        }
        if (lane == 0) G.rstd[warp] = r;
      }
      if (gp) gp[1] = gtimer();
      named_sync(1, NT);
      if (gp) gp[2] = gtimer();
    }
#pragma unroll
    for (int s = 0; s < kStageItems; ++s) {
      const int it = base + s * NT + tid;
      const bool active = it < items;
      const int kb = it / (B * 16);
      const int rem = it - kb * B * 16;
      const int b = active ? rem >> 4 : 0, p = (rem >> 2) & 3, tig = rem & 3;
      const float rs = G.rstd[b];
      float lo = 0.f, hi = 0.f;
      uint32_t h[4];
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        float v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int e = 4 * hh + q;
          const int64_t kk = static_cast<int64_t>(kb) * kBlockK + 16 * (2 * p + hh) + 2 * tig + (q & 1) + 8 * (q >> 1);
          float t = raw[s][e];
          if (gain != nullptr) t = round_act(t * rs * gn[s][e], adt);
          t = (active && kk < K) ? t : 0.f;
          v[q] = __half2float(__float2half_rn(t));
        }
        lo += v[0] + v[1];
        hi += v[2] + v[3];
        const __half2 p01 = __floats2half2_rn(v[0], v[1]), p89 = __floats2half2_rn(v[2], v[3]);
        h[2 * hh] = *reinterpret_cast<const uint32_t*>(&p01);
        h[2 * hh + 1] = *reinterpret_cast<const uint32_t*>(&p89);
      }
      if (active) G.xs[(static_cast<size_t>(b) * P.nkb + kb) * 16 + p * 4 + tig] = make_uint4(h[0], h[1], h[2], h[3]);
      // the 16 lanes of an item group share (kb, b): items are 16-aligned and NT is a multiple of 16
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) {
        lo += __shfl_xor_sync(0xffffffffu, lo, o);
        hi += __shfl_xor_sync(0xffffffffu, hi, o);
      }
      if (active && (rem & 15) == 0)
        G.dx[kb * B + b] = make_float4(1024.f * (lo + hi), 64.f * (lo + hi), lo + hi, 0.f);
    }
    if (base + NT * kStageItems >= items) break;
  }
  named_sync(1, NT);
}

// NBLK 16x128 blocks on one warp (interleaved: independent MMA chains): 8 MMAs per block over
// the unpacked codes, then the per-row group fold y += s * (acc - (D + z*X)) for the columns
// (batch rows) that use this copy.  xl: this lane's B-fragment base for the first block (null
// when its column is past the batch); blocks are kbs apart in the block sequence.
template <int W, int NBLK>
__device__ __forceinline__ void gemv_blocks(const uint8_t* __restrict__ blk, const uint4* __restrict__ xl,
                                            const float4* __restrict__ dxa, int dxstep, int lane,
                                            bool ca, bool cb_, float zmagic, float (&y)[4]) {
  const int g = lane >> 2;
  // blocks j and j + kNCW of a stage: codes kNCW blocks apart, activations kNCW * 16 uint4s apart
  constexpr int bstride = (W == 0 ? kBlockBytes8 : kBlockBytes4) * kNCW;
  constexpr int kXBlk = kNCW * 16;
  float c[NBLK][4];
#pragma unroll
  for (int n = 0; n < NBLK; ++n)
#pragma unroll
    for (int e = 0; e < 4; ++e) c[n][e] = 0.f;
  if constexpr (W == 0) {
#pragma unroll
    for (int p = 0; p < 4; ++p) {
#pragma unroll
      for (int n = 0; n < NBLK; ++n) {
        const uint4 wv = reinterpret_cast<const uint4*>(blk + n * bstride)[p * 32 + lane];
        const uint4 xv = xl[n * kXBlk + p * 4];
        mma16816(c[n], prmt(wv.x, 0x64646464u, 0x4140u), prmt(wv.x, 0x64646464u, 0x4342u),
                 prmt(wv.y, 0x64646464u, 0x4140u), prmt(wv.y, 0x64646464u, 0x4342u), xv.x, xv.y);
        mma16816(c[n], prmt(wv.z, 0x64646464u, 0x4140u), prmt(wv.z, 0x64646464u, 0x4342u),
                 prmt(wv.w, 0x64646464u, 0x4140u), prmt(wv.w, 0x64646464u, 0x4342u), xv.z, xv.w);
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
#pragma unroll
      for (int n = 0; n < NBLK; ++n) {
        const uint4 wv = reinterpret_cast<const uint4*>(blk + n * bstride)[i * 32 + lane];
        const uint4 x0 = xl[n * kXBlk + (2 * i) * 4];
        const uint4 x1 = xl[n * kXBlk + (2 * i + 1) * 4];
        const uint32_t qs[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          // every nibble pair is moved to bits 4-7 / 20-23 of the halves: fp16 0x5400 | q<<4 = 64 + q
          const uint32_t q = qs[u];
          const uint4 xv = u < 2 ? x0 : x1;
          mma16816(c[n], nib_f16(q << 4), nib_f16(q >> 4), nib_f16(q), nib_f16(q >> 8), (u & 1) ? xv.z : xv.x,
                   (u & 1) ? xv.w : xv.y);
        }
      }
    }
  }

  constexpr int cbytes = W == 0 ? 2048 : 1024;
#pragma unroll
  for (int n = 0; n < NBLK; ++n) {
    const uint8_t* bk = blk + n * bstride;
    const float s0 = *reinterpret_cast<const float*>(bk + cbytes + 4 * g);
    const float s1 = *reinterpret_cast<const float*>(bk + cbytes + 4 * (g + 8));
    const float z0 = __uint_as_float(0x4B000000u | bk[cbytes + 64 + g]) - zmagic;  // exact: zq + zp_base
    const float z1 = __uint_as_float(0x4B000000u | bk[cbytes + 64 + g + 8]) - zmagic;
    if (ca) {
      const float4 d = dxa[n * dxstep];
      const float D = W == 0 ? d.x : d.y;
      y[0] = fmaf(s0, c[n][0] - fmaf(z0, d.z, D), y[0]);
      y[2] = fmaf(s1, c[n][2] - fmaf(z1, d.z, D), y[2]);
    }
    if (cb_) {
      const float4 d = dxa[n * dxstep + 1];
      const float D = W == 0 ? d.x : d.y;
      y[1] = fmaf(s0, c[n][1] - fmaf(z0, d.z, D), y[1]);
      y[3] = fmaf(s1, c[n][3] - fmaf(z1, d.z, D), y[3]);
    }
  }
}

// Per-phase control block, computed once per phase by consumer thread 0.
struct PhaseCtl {
  Segs S;
  float zmagic[2 * kMaxMat];
  int64_t g0, g1;      // this CTA's block range
  int64_t tile0;       // first tile of the range
  int ntiles;          // tiles the range touches
  int cap;             // tiles per reduction window
  int head_shared;     // first tile started on an earlier CTA: publish its part
  int nfollow;         // later CTAs holding parts of our last tile (we own it)
  unsigned int tag;    // (launch epoch, phase) stamp of this phase's stream-K parts
  short follow[512];
};

// Writes this warp's partial of local tile `loc` into its window slot.
__device__ __forceinline__ void flush_partial(const GemvSmem& G, int slot, int nmat, int B, int warp, int lane,
                                              const float (&y)[kMaxMat][4]) {
  const int g = lane >> 2, tig = lane & 3;
#pragma unroll
  for (int m = 0; m < kMaxMat; ++m) {
    if (m >= nmat) break;
    float* r = G.red + (static_cast<size_t>(slot * nmat + m) * kNCW + warp) * 16 * B;
    if (2 * tig < B) {
      r[g * B + 2 * tig] = y[m][0];
      r[(g + 8) * B + 2 * tig] = y[m][2];
    }
    if (2 * tig + 1 < B) {
      r[g * B + 2 * tig + 1] = y[m][1];
      r[(g + 8) * B + 2 * tig + 1] = y[m][3];
    }
  }
}

// ---------------------------------------------------------------- fused softmax statistics
// Running softmax statistics of a set of logits (softmax_double / ppl_entropy /
// fault_tolerance / argmax_token, src/scheduler.cpp:13-49, src/engine.cpp:144-155), mergeable:
//   m = max, S = sum exp(l - m), T = sum exp(l - m) (l - m)  (double),
//   v1 >= v2 the two largest logits (duplicates count), arg = lowest index of the max.
// H = ln S - T / S, PPLE = exp(H), p1 = exp(v1 - m) / S, p2 = exp(v2 - m) / S.
struct StatPart {
  double S, T;
  float m, v1, v2;
  int arg;
};
static_assert(sizeof(StatPart) == 32, "StatPart layout");

__device__ __forceinline__ void stat_init(StatPart& a) {
  a.S = 0.0;
  a.T = 0.0;
  a.m = -INFINITY;
  a.v1 = -INFINITY;
  a.v2 = -INFINITY;
  a.arg = 0x7fffffff;
}

__device__ __forceinline__ void stat_add(StatPart& a, float l, int idx) {
  if (l > a.m) {
    if (a.m != -INFINITY) {
      const double d = static_cast<double>(a.m) - static_cast<double>(l);
      const double e = exp(d);
      a.T = e * (a.T + d * a.S);
      a.S *= e;
    }
    a.S += 1.0;
    a.m = l;
  } else {
    const double d = static_cast<double>(l) - static_cast<double>(a.m);
    const double e = exp(d);
    a.S += e;
    a.T += e * d;
  }
  if (l > a.v1) {
    a.v2 = a.v1;
    a.v1 = l;
    a.arg = idx;
  } else if (l > a.v2) {
    a.v2 = l;
  }
}

#ifndef FQ_MERGE_INLINE
#define FQ_MERGE_INLINE 0
#endif
#if FQ_MERGE_INLINE
__device__ __forceinline__
#else
__device__ __noinline__
#endif
StatPart stat_merge(const StatPart& a, const StatPart& b) {
  if (b.m == -INFINITY) return a;
  if (a.m == -INFINITY) return b;
  StatPart r;
  r.m = fmaxf(a.m, b.m);
  const double da = static_cast<double>(a.m) - r.m, db = static_cast<double>(b.m) - r.m;
  const double ea = exp(da), eb = exp(db);
  r.S = a.S * ea + b.S * eb;
  r.T = ea * (a.T + da * a.S) + eb * (b.T + db * b.S);
  r.v1 = fmaxf(a.v1, b.v1);
  r.v2 = fmaxf(fminf(a.v1, b.v1), fmaxf(a.v2, b.v2));
  r.arg = a.v1 > b.v1 ? a.arg : (b.v1 > a.v1 ? b.arg : min(a.arg, b.arg));
  return r;
}

__device__ __forceinline__ StatPart stat_shfl(const StatPart& a, int src_lane_xor) {
  StatPart r;
  r.S = __shfl_xor_sync(0xffffffffu, a.S, src_lane_xor);
  r.T = __shfl_xor_sync(0xffffffffu, a.T, src_lane_xor);
  r.m = __shfl_xor_sync(0xffffffffu, a.m, src_lane_xor);
  r.v1 = __shfl_xor_sync(0xffffffffu, a.v1, src_lane_xor);
  r.v2 = __shfl_xor_sync(0xffffffffu, a.v2, src_lane_xor);
  r.arg = __shfl_xor_sync(0xffffffffu, a.arg, src_lane_xor);
  return r;
}

__device__ __forceinline__ void gemv_epilogue(const Phase& P, int64_t tile, int r, int b, const float (&v)[kMaxMat],
                                              float (&sqb)[kMaxB], StatPart& st) {
  const int64_t row = tile * kTileRows + r;
  if (row >= P.N) return;
  if (P.epi == EPI_STORE) {
    for (int m = 0; m < P.nmat; ++m) store_out(P.y, P.y_dtype, b * P.y_stride + m * P.N + row, v[m]);
    if (P.stat_part) stat_add(st, v[0], static_cast<int>(row));
  } else if (P.epi == EPI_SPLIT3) {
    for (int m = 0; m < P.nmat; ++m) store_out(P.mat[m].y, P.y_dtype, b * P.y_stride + row, v[m]);
  } else if (P.epi == EPI_SWIGLU) {
    const float gt = v[0];
    const float silu = gt / (1.0f + expf(-gt));
    const float o = round_act(silu * v[1], P.act_dtype);
    store_out(P.y, P.y_dtype, b * P.y_stride + row, o);
    if (P.yfrag && P.yfrag_nkb > 0) frag_store(P.yfrag, P.yfrag_nkb, b, row, o);
  } else {
    float* xp = P.resid + b * P.resid_stride + row;
    const float nv = *xp + v[0];
    *xp = nv;
#pragma unroll
    for (int bb = 0; bb < kMaxB; ++bb)
      if (bb == b) sqb[bb] += nv * nv;
  }
}

// Reduces the window of local tiles [lo, hi): fixed-order sums over the warps, then per tile the
// publication (a later part of a tile owned by an earlier CTA), the merge of the later parts
// (our last tile continues on following CTAs) or the epilogue.
__device__ void reduce_window(const Phase& P, const PhaseCtl& C, const GemvSmem& G, int lo, int hi, float (&sqb)[kMaxB],
                              StatPart& st, unsigned long long* gp = nullptr) {
  named_sync(1, kNCW * 32);
  if (gp) gp[7] = gtimer();
  const int B = P.B, nmat = P.nmat;
  const int per = 16 * B;
  const int fstride = kMaxMat * 16 * B;
  const bool merge_last = !FQ_TILE_PART && C.nfollow > 0 && hi == C.ntiles;  // stream-K only
  // stream-K parts travel as (value, tag) pairs in one 8-byte store: the tag (launch epoch and
  // phase) tells the owner the value is current, no flag / fence / extra round trip
  float2* fix = reinterpret_cast<float2*>(P.fix);
  // item stride a multiple of `per` (and so of B): a thread's items all belong to batch row
  // threadIdx.x % B (the fused softmax statistics rely on it)
  const int stride = (kNCW * 32 / per) * per;
  for (int it = threadIdx.x; threadIdx.x < stride && it < (hi - lo) * per; it += stride) {
    const int l = lo + it / per, i = it % per;
    float v[kMaxMat] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int m = 0; m < kMaxMat; ++m) {
      if (m >= nmat) break;
      const float* r = G.red + (static_cast<size_t>(((l - lo) * nmat + m) * kNCW)) * per + i;
      float a = 0.f;
#pragma unroll
      for (int w = 0; w < kNCW; ++w) a += r[w * per];
      v[m] = a;
    }
    if (!FQ_TILE_PART && l == 0 && C.head_shared) {
      for (int m = 0; m < nmat; ++m)
        __stcg(fix + static_cast<size_t>(blockIdx.x) * fstride + m * per + i, make_float2(v[m], __uint_as_float(C.tag)));
    } else if (merge_last && l == hi - 1) {
      // owner of the last tile: add the followers' parts in CTA order (each thread polls its own
      // (value, tag) words)
      for (int f = 0; f < C.nfollow; ++f) {
        const int c = C.follow[f];
        for (int m = 0; m < nmat; ++m) {
          const float2* src = fix + static_cast<size_t>(c) * fstride + m * per + i;
          float2 w = ld_volatile_f2(src);
          if (__float_as_uint(w.y) != C.tag) {
            const unsigned long long t0 = gtimer_now();
            do {
              __nanosleep(20);
              w = ld_volatile_f2(src);
              if (gtimer_now() - t0 > kWatchdogNs) watchdog_fire("stream-K part", c, f);
            } while (__float_as_uint(w.y) != C.tag);
          }
          v[m] += w.x;
        }
      }
      gemv_epilogue(P, C.tile0 + l, i / B, i % B, v, sqb, st);
    } else {
      gemv_epilogue(P, C.tile0 + l, i / B, i % B, v, sqb, st);
    }
  }
  named_sync(1, kNCW * 32);  // the window's slots are rewritten next
}

__device__ __forceinline__ int64_t cta_start_or_end(const Phase& P, const Segs& S, int c) {
  return c <= static_cast<int>(gridDim.x) ? cta_start(P, S, c) : INT64_MAX;
}

// Compact per-phase partition of this CTA, computed for every phase of the program at kernel
// start (one consumer thread per phase, in parallel) so no phase pays for it on its critical path.
constexpr int kCtlFollow = FQ_TILE_PART ? 1 : 4;
struct alignas(16) CtlEntry {
  int g0, g1, tile0;
  short ntiles;
  uint8_t nseg, head_shared, nfollow, valid;  // nfollow 0xFF: more than kCtlFollow, recompute
  uint8_t segmw[2 * kMaxMat], mask[2 * kMaxMat];
  short follow[kCtlFollow];  // whole-tile partition: never used (kept 32 bytes per entry)
};

__device__ __noinline__ void compute_ctl(const Phase& P, CtlEntry& E) {
  E.valid = 0;
  if (P.type != PH_GEMV) return;
  Segs S;
  phase_segs(P, S);
  E.nseg = static_cast<uint8_t>(S.n);
  E.g0 = E.g1 = E.tile0 = 0;
  E.ntiles = 0;
  E.head_shared = 0;
  E.nfollow = 0;
  for (int s = 0; s < S.n; ++s) {
    E.segmw[s] = static_cast<uint8_t>(S.m[s] << 1 | S.w[s]);
    E.mask[s] = static_cast<uint8_t>(S.mask[s]);
  }
  E.valid = 1;
  if (S.n == 0) return;
  const int64_t bpt = static_cast<int64_t>(S.n) * P.nkb;
  const int64_t g0 = cta_start(P, S, blockIdx.x), g1 = cta_start(P, S, blockIdx.x + 1);
  E.g0 = static_cast<int>(g0);
  E.g1 = static_cast<int>(g1);
  if (g0 >= g1) return;
  const int64_t tile0 = g0 / bpt, tl = (g1 - 1) / bpt;
  E.tile0 = static_cast<int>(tile0);
  E.ntiles = static_cast<short>(tl - tile0 + 1);
  E.head_shared = g0 > tile0 * bpt;
  const int64_t t1 = (tl + 1) * bpt;
  if (t1 > g1 && tl * bpt >= g0) {
    int64_t cs = g1;
    for (int c = blockIdx.x + 1; c < static_cast<int>(gridDim.x) && cs < t1; ++c) {
      const int64_t cn = cta_start(P, S, c + 1);
      if (cn > cs) {
        if (E.nfollow < kCtlFollow) E.follow[E.nfollow++] = static_cast<short>(c);
        else { E.nfollow = 0xFF; break; }
      }
      cs = cn;
    }
  }
}

// Table-driven producer: the per-phase partition comes from the shared-memory control table the
// consumers fill at kernel start (CtlEntry), so a stage costs a few integer ops (no divisions, no
// rung-table or descriptor loads on the issue path).  The tile base pointers of the next GEMV phase
// are loaded into registers one phase ahead, so a phase switch never waits on global memory.
struct ProdPhase {
  const uint8_t* t[2 * kMaxMat];  // [m * 2 + w]
  int nkb;
};

__device__ __forceinline__ void prod_load(const Phase& P, ProdPhase& q) {
#pragma unroll
  for (int m = 0; m < kMaxMat; ++m)
#pragma unroll
    for (int w = 0; w < 2; ++w) q.t[m * 2 + w] = P.mat[m].tiles[w];
  q.nkb = P.nkb;
}

__device__ __forceinline__ int next_gemv_phase(const CtlEntry* ctab, int from, int nphases) {
  for (int p = from; p < nphases; ++p)
    if (ctab[p].valid && ctab[p].nseg > 0 && ctab[p].g1 > ctab[p].g0) return p;
  return nphases;
}

// Second walk of the same stage sequence, `prefetch` stages ahead of the ring: L2 prefetches keep
// HBM streaming while the ring is full (consumers in a grid barrier, staging, a reduction or a
// non-GEMV phase), so ring refills hit L2.  Its descriptor loads block, which is fine: it is ahead.
struct AheadWalk {
  const Phase* phases;
  const CtlEntry* ctab;
  const uint8_t** tab;  // shared [2 * kMaxMat]
  int nphases, ph, nseg, nkb, tile, seg, kb, left, mw;
  __device__ void init(const Phase* p, const CtlEntry* c, int n, const uint8_t** t) {
    phases = p;
    ctab = c;
    nphases = n;
    tab = t;
    ph = -1;
    left = 0;
  }
  __device__ bool next(const uint8_t*& src, uint32_t& bytes) {
    if (left == 0) {
      ph = next_gemv_phase(ctab, ph + 1, nphases);
      if (ph >= nphases) return false;
      const Phase& P = phases[ph];
#pragma unroll
      for (int m = 0; m < kMaxMat; ++m)
#pragma unroll
        for (int w = 0; w < 2; ++w) tab[m * 2 + w] = P.mat[m].tiles[w];
      nkb = P.nkb;
      const CtlEntry& E = ctab[ph];
      nseg = E.nseg;
      const int bpt = nseg * nkb;
      tile = E.g0 / bpt;
      const int rem = E.g0 - tile * bpt;
      seg = rem / nkb;
      kb = rem - seg * nkb;
      left = E.g1 - E.g0;
      mw = E.segmw[seg];
    }
    const int w = mw & 1;
    const int bb = w == 0 ? kBlockBytes8 : kBlockBytes4;
    const int nb = min(min(w == 0 ? kStageBlocks8 : kStageBlocks4, nkb - kb), left);
    src = tab[mw] + (static_cast<int64_t>(tile) * nkb + kb) * bb;
    bytes = static_cast<uint32_t>(nb * bb);
    left -= nb;
    kb += nb;
    if (kb == nkb) {
      kb = 0;
      if (++seg == nseg) {
        seg = 0;
        ++tile;
      }
      mw = ctab[ph].segmw[seg];
    }
    return true;
  }
};

__device__ void produce_table(const Phase* phases, int nphases, const CtlEntry* ctab, const Ring R,
                              unsigned long long* tr, const uint8_t** s_base, bool noload, int prefetch,
                              const uint8_t** s_base2) {
  AheadWalk ahead;
  ahead.init(phases, ctab, nphases, s_base2);
  bool more_ahead = prefetch > 0;
  for (int i = 0; i < prefetch && more_ahead; ++i) {
    const uint8_t* psrc;
    uint32_t pbytes;
    if ((more_ahead = ahead.next(psrc, pbytes))) prefetch_l2(psrc, pbytes);
  }
  int slot_i = 0, tn = 0;

  uint32_t phase_bit = 0;
  int ph = next_gemv_phase(ctab, 0, nphases);
  ProdPhase cur, nxt;
  if (ph < nphases) prod_load(phases[ph], cur);
  while (ph < nphases) {
    const int phn = next_gemv_phase(ctab, ph + 1, nphases);
    if (phn < nphases) prod_load(phases[phn], nxt);  // in flight while this phase streams
    const CtlEntry& E = ctab[ph];
    const int nseg = E.nseg, nkb = cur.nkb;
#pragma unroll
    for (int i = 0; i < 2 * kMaxMat; ++i) s_base[i] = cur.t[i];
    const int bpt = nseg * nkb;
    int tile = E.g0 / bpt;
    int rem = E.g0 - tile * bpt;
    int seg = rem / nkb, kb = rem - seg * nkb;
    int left = E.g1 - E.g0;
    int mw = E.segmw[seg];
    while (left > 0) {
      const int w = mw & 1;
      const int bb = w == 0 ? kBlockBytes8 : kBlockBytes4;
      const int nb = min(min(w == 0 ? kStageBlocks8 : kStageBlocks4, nkb - kb), left);
      const uint8_t* src = s_base[mw] + (static_cast<int64_t>(tile) * nkb + kb) * bb;
      if (more_ahead) {
        const uint8_t* psrc;
        uint32_t pbytes;
        if ((more_ahead = ahead.next(psrc, pbytes))) prefetch_l2(psrc, pbytes);
      }
      const int s = slot_i;
      mbar_wait(&R.empty[s], phase_bit ^ 1u);
      if (tr && tn < kTraceStages) tr[3 * tn] = gtimer();
      ++tn;
      if (++slot_i == R.nstages) {
        slot_i = 0;
        phase_bit ^= 1u;
      }
      const uint32_t bytes = static_cast<uint32_t>(nb * bb);
      if (noload) {  // profiling: consumer-only timing, the ring keeps whatever it holds
        mbar_arrive(&R.full[s]);
      } else {
        mbar_expect_tx(&R.full[s], bytes);
        bulk_g2s(R.base + static_cast<size_t>(s) * kStageBytes, src, bytes, &R.full[s]);
      }
      left -= nb;
      kb += nb;
      if (kb == nkb) {
        kb = 0;
        if (++seg == nseg) {
          seg = 0;
          ++tile;
        }
        mw = E.segmw[seg];
      }
    }
    ph = phn;
    cur = nxt;
  }
}

// Per-phase control block, computed by consumer warp 1 (the lanes evaluate the range starts of
// this CTA and its followers in parallel) while warp 0 computes the RMSNorm factors.
template <bool LEAN = false>
__device__ void phase_setup(const Phase& P, PhaseCtl& C, int red_floats, int lane, unsigned long long* gpa,
                            const CtlEntry* E) {
  // LEAN: the partition table always covers the program and whole tiles never have followers
  if (LEAN || (E && E->valid && E->nfollow != 0xFF)) {
    // precomputed at kernel start: copy into the working control block
    if (lane == 0) {
      C.S.n = E->nseg;
      C.S.tile_bytes = 0;
      for (int s = 0; s < E->nseg; ++s) {
        C.S.m[s] = E->segmw[s] >> 1;
        C.S.w[s] = E->segmw[s] & 1;
        C.S.mask[s] = E->mask[s];
        C.zmagic[s] = 8388608.0f - static_cast<float>(P.mat[C.S.m[s]].zpbase[C.S.w[s]]);
      }
      C.g0 = E->g0;
      C.g1 = E->g1;
      C.tile0 = E->tile0;
      C.ntiles = E->ntiles;
      C.head_shared = E->head_shared;
      C.nfollow = E->nfollow;
      for (int f = 0; f < E->nfollow; ++f) C.follow[f] = E->follow[f];
      C.cap = E->nseg > 0 ? max(1, red_floats / (P.nmat * kNCW * 16 * P.B)) : 1;
    }
    __syncwarp();
    return;
  }
  if constexpr (!LEAN) {
  Segs S;
  phase_segs(P, S);

  int64_t g0 = 0, g1 = 0, tile0 = 0;
  int ntiles = 0, head_shared = 0, nfollow = 0;
  if (S.n > 0) {
    const int64_t bpt = static_cast<int64_t>(S.n) * P.nkb;
    const int64_t mine = cta_start_or_end(P, S, blockIdx.x + lane);
    g0 = __shfl_sync(0xffffffffu, mine, 0);
    g1 = __shfl_sync(0xffffffffu, mine, 1);
    if (g0 < g1) {
      tile0 = g0 / bpt;
      const int64_t tl = (g1 - 1) / bpt;
      ntiles = static_cast<int>(tl - tile0 + 1);
      head_shared = g0 > tile0 * bpt;
      const int64_t t1 = (tl + 1) * bpt;
      if (t1 > g1 && tl * bpt >= g0) {
        // we hold the head of our last tile and it continues: followers are the later CTAs with a
        // non-empty range starting inside it
        for (int base = 1;; base += 32) {
          const int c = blockIdx.x + base + lane;
          const int64_t cs = cta_start_or_end(P, S, c), cn = cta_start_or_end(P, S, c + 1);
          const bool ok = c < static_cast<int>(gridDim.x) && cs < t1 && cn > cs;
          const unsigned m = __ballot_sync(0xffffffffu, ok);
          if (lane == 0)
            for (unsigned mm = m; mm; mm &= mm - 1)
              if (nfollow < 512) C.follow[nfollow++] = static_cast<short>(blockIdx.x + base + __ffs(mm) - 1);
          const int64_t last = __shfl_sync(0xffffffffu, cn, 31);
          if (last >= t1 || blockIdx.x + base + 32 >= gridDim.x) break;
        }
      }
    }
  }
  if (lane == 0) {
    C.S = S;
    for (int s = 0; s < S.n; ++s) C.zmagic[s] = 8388608.0f - static_cast<float>(P.mat[S.m[s]].zpbase[S.w[s]]);
    C.g0 = g0;
    C.g1 = g1;
    C.tile0 = tile0;
    C.ntiles = ntiles;
    C.head_shared = head_shared;
    C.nfollow = nfollow;
    C.cap = S.n > 0 ? max(1, red_floats / (P.nmat * kNCW * 16 * P.B)) : 1;
  }
  __syncwarp();
  }
}

__device__ __forceinline__ void add_into(float (&y)[kMaxMat][4], int m, float (&yc)[4]) {
  switch (m) {
    case 0:
#pragma unroll
      for (int e = 0; e < 4; ++e) y[0][e] += yc[e];
      break;
    case 1:
#pragma unroll
      for (int e = 0; e < 4; ++e) y[1][e] += yc[e];
      break;
    default:
#pragma unroll
      for (int e = 0; e < 4; ++e) y[2][e] += yc[e];
      break;
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) yc[e] = 0.f;
}

template <bool LEAN>
__device__ void run_gemv_phase(const Phase& P, const Ring R, const GemvSmem& G, PhaseCtl& C, int red_floats,
                               int& slot_ref, uint32_t& phase_ref, int phase_idx, const CtlEntry* ctab, unsigned int tag,
                               unsigned long long* gprof) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long* gpa = (FQ_GEMV_HOOKS && gprof) ? gprof + (static_cast<size_t>(phase_idx) * gridDim.x + blockIdx.x) * 8
                                                      : nullptr;  // compiled out: every gp test folds away
  unsigned long long* gp = threadIdx.x == 0 ? gpa : nullptr;
  if (warp == 1) {
    phase_setup<LEAN>(P, C, red_floats, lane, gpa, ctab ? ctab + phase_idx : nullptr);  // warp 0: norm factors
    if (lane == 0) C.tag = tag;
    if (gpa && lane == 0) gpa[0] = gtimer();
  }
  stage_acts<LEAN>(P, G, gp, tag - 1);  // ends with a consumer barrier: C is visible (tag - 1: the previous phase)
  if (gp) gp[3] = gtimer();
  const int B = P.B, nmat = P.nmat;
  float sqb[kMaxB];
#pragma unroll
  for (int b = 0; b < kMaxB; ++b) sqb[b] = 0.f;
  StatPart st;
  stat_init(st);
  if (C.ntiles > 0) {
    int slot_i = slot_ref;
    uint32_t phase_bit = phase_ref;
    const int g = lane >> 2, tig = lane & 3;
    // lanes of batch columns past B read column B-1 (valid data; those MMA columns are ignored)
    const uint4* xl = G.xs + static_cast<size_t>(min(g, B - 1)) * P.nkb * 16 + tig;
    const bool ca0 = 2 * tig < B, cb0 = 2 * tig + 1 < B;
    float y[kMaxMat][4], yc[4];
#pragma unroll
    for (int m = 0; m < kMaxMat; ++m)
#pragma unroll
      for (int e = 0; e < 4; ++e) y[m][e] = 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e) yc[e] = 0.f;
    // incremental walk of the block sequence (no divisions per stage)
    const int nkb = P.nkb, nseg = C.S.n;
    const int64_t bpt = static_cast<int64_t>(nseg) * nkb;
    int rem = static_cast<int>(C.g0 - C.tile0 * bpt);
    int seg = rem / nkb, kb = rem - seg * nkb;
    int left = static_cast<int>(C.g1 - C.g0);
    int loc = 0, wlo = 0;
    const int cap = C.cap;
    // segment state (refreshed when the segment changes)
    int m = 0, w = 0, bsz = kBlockBytes8, capb = kStageBlocks8;
    bool ca = false, cb = false;
    float zm = 0.f;
    auto load_seg = [&]() {
      m = C.S.m[seg];
      w = C.S.w[seg];
      bsz = w == 0 ? kBlockBytes8 : kBlockBytes4;
      capb = w == 0 ? kStageBlocks8 : kStageBlocks4;
      const int cmask = C.S.mask[seg];
      ca = ca0 && ((cmask >> (2 * tig)) & 1);
      cb = cb0 && ((cmask >> (2 * tig + 1)) & 1);
      zm = C.zmagic[seg];
    };
    load_seg();
    while (left > 0) {
      const int nb = min(min(capb, nkb - kb), left);
#if FQ_RING_TRACE
      const bool stamp = G.tr != nullptr && warp == 0 && lane == 0 && *G.tn < kTraceStages;
      if (stamp) G.tr[3 * *G.tn + 1] = gtimer();
#endif
      mbar_wait(&R.full[slot_i], phase_bit);
#if FQ_RING_TRACE
      if (stamp) G.tr[3 * (*G.tn)++ + 2] = gtimer();
#endif
      const uint8_t* slot = R.base + static_cast<size_t>(slot_i) * kStageBytes;
      const float4* dxa = G.dx + static_cast<size_t>(kb) * B + 2 * tig;
      for (int j = warp; j < nb; j += 2 * kNCW) {
        const uint8_t* bk = slot + j * bsz;
        const uint4* xj = xl + (kb + j) * 16;
        const float4* dj = dxa + j * B;
        if (j + kNCW < nb) {
          if (w == 0) gemv_blocks<0, 2>(bk, xj, dj, kNCW * B, lane, ca, cb, zm, yc);
          else gemv_blocks<1, 2>(bk, xj, dj, kNCW * B, lane, ca, cb, zm, yc);
        } else {
          if (w == 0) gemv_blocks<0, 1>(bk, xj, dj, 0, lane, ca, cb, zm, yc);
          else gemv_blocks<1, 1>(bk, xj, dj, 0, lane, ca, cb, zm, yc);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&R.empty[slot_i]);
      if (++slot_i == R.nstages) {
        slot_i = 0;
        phase_bit ^= 1u;
      }
      left -= nb;
      kb += nb;
      if (kb == nkb) {  // segment finished
        kb = 0;
        add_into(y, m, yc);
        if (++seg == nseg) {
          seg = 0;
          // tile finished on this CTA: flush this warp's partial into the window
          flush_partial(G, loc - wlo, nmat, B, warp, lane, y);
#pragma unroll
          for (int mm = 0; mm < kMaxMat; ++mm)
#pragma unroll
            for (int e = 0; e < 4; ++e) y[mm][e] = 0.f;
          ++loc;
          if (left > 0 && (loc - wlo == cap || (!FQ_TILE_PART && loc == 1 && C.head_shared))) {
            reduce_window(P, C, G, wlo, loc, sqb, st);
            wlo = loc;
          }
        }
        load_seg();
      }
    }
    if (kb != 0 || seg != 0) {  // the range ended inside a tile
      add_into(y, m, yc);
      flush_partial(G, loc - wlo, nmat, B, warp, lane, y);
      ++loc;
    }
    if (gp) gp[4] = gtimer();
    reduce_window(P, C, G, wlo, loc, sqb, st, gp);
    if (gp) gp[5] = gtimer();
    slot_ref = slot_i;
    phase_ref = phase_bit;
  }
  if (P.stat_part) {
    // per-CTA softmax partial of each batch row over the logits this CTA finalised: thread t's
    // items belong to row t % B; fixed-order tree merge over j = t / B in shared memory
    named_sync(1, kNCW * 32);
    StatPart* sp = reinterpret_cast<StatPart*>(G.red);
    sp[threadIdx.x] = st;
    const int per = 16 * B;
    const int nb = ((kNCW * 32 / per) * per) / B;  // entries per row
    for (int len = nb; len > 1;) {
      const int up = (len + 1) >> 1;
      named_sync(1, kNCW * 32);
      const int j = threadIdx.x / B, b = threadIdx.x - j * B;
      if (j < len - up) sp[j * B + b] = stat_merge(sp[j * B + b], sp[(j + up) * B + b]);
      len = up;
    }
    named_sync(1, kNCW * 32);
    if (static_cast<int>(threadIdx.x) < B)
      reinterpret_cast<StatPart*>(P.stat_part)[threadIdx.x * gridDim.x + blockIdx.x] = sp[threadIdx.x];
  }
  if (P.epi == EPI_RESIDUAL) {
    // per-CTA sum of squares of the rows this CTA finalised (RMSNorm of the next phase)
#pragma unroll
    for (int b = 0; b < kMaxB; ++b) {
      if (FQ_SQ_B && b >= B) break;  // warp-uniform: no shuffles for absent batch rows
      float v = sqb[b];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) G.sq[b * kNCW + warp] = v;
    }
    named_sync(1, kNCW * 32);
    if (static_cast<int>(threadIdx.x) < B) {
      float s = 0.f;
      for (int w2 = 0; w2 < kNCW; ++w2) s += G.sq[threadIdx.x * kNCW + w2];
      P.out_partials[threadIdx.x * P.out_partials_stride + blockIdx.x] = s;
    }
  }
  named_sync(1, kNCW * 32);  // staging / reduction buffers and C are reused by the next phase
  if (gp) gp[6] = gtimer();
}

// ---------------------------------------------------------------- consumers: embedding
__device__ __forceinline__ void cta_rows(int64_t N, int64_t& r0, int& rows) {
  r0 = (N * blockIdx.x) / gridDim.x;
  rows = static_cast<int>((N * (blockIdx.x + 1)) / gridDim.x - r0);
}

FQ_ONCE void run_embed(const Phase& P, float (*sq_red)[kNCW]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t c0;
  int cnt;
  cta_rows(P.d, c0, cnt);
  // tok_emb null: residual add of an exchanged partial (tensor-parallel step, resid += x[b])
  const bool add = P.tok_emb == nullptr;
  for (int b = 0; b < P.B; ++b) {
    const float* e = add ? static_cast<const float*>(P.x) + b * P.d
                         : P.tok_emb + static_cast<int64_t>(P.tokens[b * max(1, P.token_stride)]) * P.d;
    float sq = 0.f;
    for (int i = threadIdx.x; i < cnt; i += kNCW * 32) {
      float* rp = P.resid + b * P.resid_stride + c0 + i;
      const float v = add ? *rp + e[c0 + i] : e[c0 + i];
      *rp = v;
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
// One (row, head, 64-key chunk) item per warp; lane l owns head dims [DPL*l, DPL*l + DPL) of q,
// the keys, the values and the output (coalesced fp16 rows of the cache).  Scores: per-lane
// partial dots for the chunk's 64 keys, then a transposing butterfly (62 shuffles) leaves lane l
// with the full scores of keys base(l), base(l)+1.  The chunk's (max, sum, o) partial goes to the
// workspace; the last chunk of a head (ticket) merges them.  RoPE pairs (i, i + hd/2) live on
// lanes l and l^16; cos/sin come from the model's table (double-computed angles).
constexpr int kMaxMetaRows = 64;
struct MetaSmem {
  const int32_t* pos;
  const int32_t* slots;
  int n;
  int p[kMaxMetaRows], s[kMaxMetaRows];
};
__device__ __forceinline__ int meta_pos(const MetaSmem& M, const int32_t* pos, int b) {
  return (pos == M.pos && b < M.n) ? M.p[b] : pos[b];
}
__device__ __forceinline__ int meta_slot(const MetaSmem& M, const int32_t* slots, int b) {
  return (slots == M.slots && b < M.n) ? M.s[b] : slots[b];
}

struct AttnSmem {
  float o[kNCW][128];
  float m[kNCW], l[kNCW];
};

template <int DPL>
__device__ __forceinline__ void rope_lane(float (&x)[DPL], const float2* __restrict__ cs, int lane) {
  // lane < 16 holds the first halves (dims i), lane >= 16 the second (i + hd/2), i = DPL*(lane&15)+e
#pragma unroll
  for (int e = 0; e < DPL; ++e) {
    const float other = __shfl_xor_sync(0xffffffffu, x[e], 16);
    const float2 t = cs[DPL * (lane & 15) + e];
    x[e] = lane < 16 ? x[e] * t.x - other * t.y : x[e] * t.x + other * t.y;
  }
}

template <int DPL>
__device__ __forceinline__ void load_lane(const void* src, int dtype, int64_t off, float (&x)[DPL]) {
  // activations of the attention phase are bf16 / fp16: DPL consecutive 16-bit values
  const unsigned short* h = static_cast<const unsigned short*>(src) + off;
  unsigned short u[DPL];
#pragma unroll
  for (int e = 0; e < DPL; ++e) u[e] = h[e];
#pragma unroll
  for (int e = 0; e < DPL; ++e)
    x[e] = dtype == FQ_DT_BF16 ? __uint_as_float(static_cast<uint32_t>(u[e]) << 16) : __half2float(__ushort_as_half(u[e]));
}

// One 16-key chunk of head (b, h) on one warp, in two parts so the K/V loads of a warp's first
// chunk go out before its query is loaded and rotated (one round trip for both).
template <int DPL>
struct AttnRaw {
  using Raw = typename std::conditional<DPL == 4, uint2, uint32_t>::type;
  Raw kr[kAttnChunk], vr[kAttnChunk];
};

template <int DPL>
__device__ __forceinline__ void attn_load(const Phase& P, int slot, int h, int chunk, int lane, AttnRaw<DPL>& R) {
  constexpr int hd = DPL * 32;
  using Raw = typename AttnRaw<DPL>::Raw;
  const int H = P.n_heads;
  const __half* kc = P.kv + slot * P.slot_stride + P.layer_off + static_cast<int64_t>(h) * P.max_seq * hd;
  const __half* vc = kc + static_cast<int64_t>(H) * P.max_seq * hd;
  const int j0 = chunk * kAttnChunk;
  const int last_row = static_cast<int>(P.max_seq) - 1;
#pragma unroll
  for (int t = 0; t < kAttnChunk; ++t) {
    const int64_t row = static_cast<int64_t>(min(j0 + t, last_row)) * hd + DPL * lane;
    R.kr[t] = *reinterpret_cast<const Raw*>(kc + row);
    R.vr[t] = *reinterpret_cast<const Raw*>(vc + row);
  }
}

// Returns the chunk's max score, exp-sum and the unnormalised P.V slice of this lane (dims
// DPL*lane ...).  The chunk holding the row's own position writes the RoPE'd key / value to the
// cache first (decode; prefill appended them in a phase of its own).
template <int DPL>
__device__ __forceinline__ void attn_compute(const Phase& P, int b, int h, int chunk, const float (&q)[DPL], int lane,
                                             AttnRaw<DPL>& R, float& mx, float& l, float (&o)[DPL], int pos, int slot) {
  constexpr int hd = DPL * 32;
  constexpr int CH = kAttnChunk;  // 16 keys
  using Raw = typename AttnRaw<DPL>::Raw;
  const int H = P.n_heads;
  const int j0 = chunk * CH;
  const int nk = min(CH, pos + 1 - j0);
  const bool owns_new = !P.appended && pos >= j0 && pos < j0 + CH;
  if (owns_new) {
    __half* kc = P.kv + slot * P.slot_stride + P.layer_off + static_cast<int64_t>(h) * P.max_seq * hd;
    __half* vc = kc + static_cast<int64_t>(H) * P.max_seq * hd;
    const int64_t off = static_cast<int64_t>(b) * H * hd + h * hd + DPL * lane;
    float kn[DPL], vn[DPL];
    load_lane<DPL>(P.k, P.act_dtype, off, kn);
    load_lane<DPL>(P.v, P.act_dtype, off, vn);
    rope_lane<DPL>(kn, P.rope_cs + static_cast<int64_t>(pos) * (hd / 2), lane);
    Raw kw, vw;
    __half* kh = reinterpret_cast<__half*>(&kw);
    __half* vh = reinterpret_cast<__half*>(&vw);
#pragma unroll
    for (int e = 0; e < DPL; ++e) {
      kh[e] = __float2half_rn(kn[e]);
      vh[e] = __float2half_rn(vn[e]);
    }
    *reinterpret_cast<Raw*>(kc + static_cast<int64_t>(pos) * hd + DPL * lane) = kw;
    *reinterpret_cast<Raw*>(vc + static_cast<int64_t>(pos) * hd + DPL * lane) = vw;
#pragma unroll
    for (int t = 0; t < CH; ++t)
      if (j0 + t == pos) {
        R.kr[t] = kw;
        R.vr[t] = vw;
      }
  }
  // per-lane partial dots, then a transposing butterfly over lane bits 4..1: lanes l and l^1 end
  // with the full score of key base(l) = 8*b4 + 4*b3 + 2*b2 + b1
  float part[CH];
#pragma unroll
  for (int t = 0; t < CH; ++t) {
    const __half2* hp = reinterpret_cast<const __half2*>(&R.kr[t]);
    float acc = 0.f;
#pragma unroll
    for (int e = 0; e < DPL / 2; ++e) {
      const float2 f = __half22float2(hp[e]);
      acc = fmaf(q[2 * e], f.x, acc);
      acc = fmaf(q[2 * e + 1], f.y, acc);
    }
    part[t] = acc;
  }
  int key = 0;
#pragma unroll
  for (int step = 0; step < 4; ++step) {
    const int m = 16 >> step;
    const int half = CH >> (step + 1);
    const bool up = lane & m;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const float keep = up ? part[i + half] : part[i];
      const float send = up ? part[i] : part[i + half];
      part[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
    }
    if (up) key += half;
  }
  const float pair = __shfl_xor_sync(0xffffffffu, part[0], 1);  // every lane takes part in the shuffle
  const float sc = key < nk ? part[0] + pair : -INFINITY;
  mx = sc;
#pragma unroll
  for (int off = 16; off > 1; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  const float p = key < nk ? expf(sc - mx) : 0.f;
  l = (lane & 1) ? 0.f : p;  // each key lives on two lanes
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
#pragma unroll
  for (int e = 0; e < DPL; ++e) o[e] = 0.f;
#pragma unroll
  for (int t = 0; t < CH; ++t) {
    const int owner = ((t >> 3) & 1) << 4 | ((t >> 2) & 1) << 3 | ((t >> 1) & 1) << 2 | (t & 1) << 1;
    const float pj = __shfl_sync(0xffffffffu, p, owner);
    const __half2* hp = reinterpret_cast<const __half2*>(&R.vr[t]);
#pragma unroll
    for (int e = 0; e < DPL / 2; ++e) {
      const float2 f = __half22float2(hp[e]);
      o[2 * e] = fmaf(pj, f.x, o[2 * e]);
      o[2 * e + 1] = fmaf(pj, f.y, o[2 * e + 1]);
    }
  }
}

// Attention of one (row, head) over split sp of ns contiguous chunk ranges on one CTA: warp w
// takes chunks c0 + w, c0 + w + 8, ... with an online softmax across its chunks; the eight warp
// states merge in shared memory (fixed order, no atomics).  ns == 1: the normalised output goes to
// attn_out; ns > 1: the CTA's unnormalised partial (O[hd], m, l) goes to attn_ws and the next GEMV
// phase (the O projection) merges the splits while staging its input.
template <int DPL>
__device__ void attn_head(const Phase& P, int b, int h, int sp, int ns, int lane, int warp, AttnSmem& S, int pos,
                          int slot, unsigned int tag) {
  constexpr int hd = DPL * 32;
  const int H = P.n_heads;
  const int nch = (pos + kAttnChunk) / kAttnChunk;
  const int c0 = (nch * sp) / ns, c1 = (nch * (sp + 1)) / ns;
  const int64_t qoff = static_cast<int64_t>(b) * H * hd + h * hd + DPL * lane;
  float q[DPL];
  float M = -INFINITY, L = 0.f, O[DPL];
#pragma unroll
  for (int e = 0; e < DPL; ++e) O[e] = 0.f;
#ifndef FQ_ATTN_L2PF
#define FQ_ATTN_L2PF 1
#endif
  if (FQ_ATTN_L2PF && (lane & 15) == 0) {
    // the warp's later chunks: L2 prefetch of their K / V rows (no registers), in flight with the
    // first chunk's loads, so the later rounds hit L2 instead of HBM
    const __half* kc = P.kv + slot * P.slot_stride + P.layer_off + static_cast<int64_t>(h) * P.max_seq * hd;
    const __half* vc = kc + static_cast<int64_t>(H) * P.max_seq * hd;
    const int half = (lane >> 4) * (hd / 2);
    for (int c = c0 + warp + kNCW; c < c1; c += kNCW) {
      const int r1 = min((c + 1) * kAttnChunk, pos + 1);
      for (int r = c * kAttnChunk; r < r1; ++r) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(kc + static_cast<int64_t>(r) * hd + half));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(vc + static_cast<int64_t>(r) * hd + half));
      }
    }
  }
  for (int c = c0 + warp; c < c1; c += kNCW) {
    AttnRaw<DPL> R;
    attn_load<DPL>(P, slot, h, c, lane, R);
    if (c == c0 + warp) {
      // first chunk: the query loads go out behind its K/V loads (one round trip for both)
      load_lane<DPL>(P.q, P.act_dtype, qoff, q);
      rope_lane<DPL>(q, P.rope_cs + static_cast<int64_t>(pos) * (hd / 2), lane);
      const float scale = 1.0f / sqrtf(static_cast<float>(hd));
#pragma unroll
      for (int e = 0; e < DPL; ++e) q[e] *= scale;
    }
    float mx, l, o[DPL];
    attn_compute<DPL>(P, b, h, c, q, lane, R, mx, l, o, pos, slot);
    const float Mn = fmaxf(M, mx);
    const float fa = M == -INFINITY ? 0.f : expf(M - Mn), fb = expf(mx - Mn);
    L = L * fa + l * fb;
#pragma unroll
    for (int e = 0; e < DPL; ++e) O[e] = O[e] * fa + o[e] * fb;
    M = Mn;
  }
#pragma unroll
  for (int e = 0; e < DPL; ++e) S.o[warp][DPL * lane + e] = O[e];
  if (lane == 0) {
    S.m[warp] = M;
    S.l[warp] = L;
  }
  named_sync(1, kNCW * 32);
  if (warp == 0) {
    float Mt = -INFINITY;
#pragma unroll
    for (int w = 0; w < kNCW; ++w) Mt = fmaxf(Mt, S.m[w]);
    float Lt = 0.f, Ot[DPL];
#pragma unroll
    for (int e = 0; e < DPL; ++e) Ot[e] = 0.f;
#pragma unroll
    for (int w = 0; w < kNCW; ++w) {
      const float f = S.m[w] == -INFINITY ? 0.f : expf(S.m[w] - Mt);
      Lt += S.l[w] * f;
#pragma unroll
      for (int e = 0; e < DPL; ++e) Ot[e] += S.o[w][DPL * lane + e] * f;
    }
    if (ns == 1) {
#pragma unroll
      for (int e = 0; e < DPL; ++e) {
        const float o = round_act(Ot[e] / Lt, P.act_dtype);
        store_out(P.attn_out, P.act_dtype, qoff + e, o);
        if (P.yfrag && P.yfrag_nkb > 0) frag_store(P.yfrag, P.yfrag_nkb, b, static_cast<int64_t>(h) * hd + DPL * lane + e, o);
      }
    } else {
      float* part = P.attn_ws + ((static_cast<int64_t>(b) * H + h) * ns + sp) * (hd + 4);
#pragma unroll
      for (int e = 0; e < DPL; ++e) part[DPL * lane + e] = Ot[e];
      if (lane == 0) *reinterpret_cast<float2*>(part + hd) = make_float2(Mt, Lt);
    }
  }
  named_sync(1, kNCW * 32);
}

// Prefill append: row b's RoPE'd key and value (fp16) go to its cache position before the
// attention phase (one (row, head) item per warp, lane-owned dims as in attn_item).
template <int DPL>
__device__ void append_item(const Phase& P, int b, int h, int lane) {
  constexpr int hd = DPL * 32;
  const int H = P.n_heads;
  const int pos = P.pos[b];
  __half* kc = P.kv + P.slots[b] * P.slot_stride + P.layer_off + static_cast<int64_t>(h) * P.max_seq * hd;
  __half* vc = kc + static_cast<int64_t>(H) * P.max_seq * hd;
  const int64_t off = static_cast<int64_t>(b) * H * hd + h * hd + DPL * lane;
  float kn[DPL], vn[DPL];
  load_lane<DPL>(P.k, P.act_dtype, off, kn);
  load_lane<DPL>(P.v, P.act_dtype, off, vn);
  rope_lane<DPL>(kn, P.rope_cs + static_cast<int64_t>(pos) * (hd / 2), lane);
#pragma unroll
  for (int e = 0; e < DPL; ++e) {
    kc[static_cast<int64_t>(pos) * hd + DPL * lane + e] = __float2half_rn(kn[e]);
    vc[static_cast<int64_t>(pos) * hd + DPL * lane + e] = __float2half_rn(vn[e]);
  }
}

FQ_ONCE void run_append(const Phase& P) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int total = P.B * P.n_heads;
  for (int item = warp * gridDim.x + blockIdx.x; item < total; item += gridDim.x * kNCW) {
    const int b = item / P.n_heads, h = item - b * P.n_heads;
    if (P.head_dim == 128) append_item<4>(P, b, h, lane);
    else append_item<2>(P, b, h, lane);
  }
}

#ifndef FQ_ATTN_INLINE
#define FQ_ATTN_INLINE 1  // measured -1.2% per step vs an out-of-line call
#endif
#if FQ_ATTN_INLINE
__device__ __forceinline__
#else
__device__ __noinline__
#endif
void run_attn(const Phase& P, AttnSmem& S, const MetaSmem& MS, unsigned int tag) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // one (row, head, split) per CTA at a time, spread over the grid
  const int ns = max(1, P.attn_splits);
  for (int item = blockIdx.x; item < P.B * P.n_heads * ns; item += gridDim.x) {
    const int bh = item / ns, sp = item - bh * ns;
    const int b = bh / P.n_heads, h = bh - b * P.n_heads;
    const int pos = meta_pos(MS, P.pos, b), slot = meta_slot(MS, P.slots, b);
    if (P.head_dim == 128) attn_head<4>(P, b, h, sp, ns, lane, warp, S, pos, slot, tag);
    else attn_head<2>(P, b, h, sp, ns, lane, warp, S, pos, slot, tag);
  }
}

// ---------------------------------------------------------------- consumers: row statistics
// Combines the head GEMV's per-CTA softmax partials of row b (warp b of CTA 0, fixed-order merge)
// into fq_row_stats: ppl_entropy / fault_tolerance / argmax_token (src/scheduler.cpp:13-49,
// src/engine.cpp:144-155) in double.
FQ_ONCE void run_stats(const Phase& P) {
  if (blockIdx.x != 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const StatPart* parts = static_cast<const StatPart*>(P.stat_part);
  const int n = gridDim.x;
  for (int b = warp; b < P.B; b += kNCW) {
    StatPart a;
    stat_init(a);
    for (int c = lane; c < n; c += 32) a = stat_merge(a, parts[b * n + c]);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const StatPart o2 = stat_shfl(a, o);
      a = (lane & o) ? stat_merge(o2, a) : stat_merge(a, o2);
    }
    if (lane == 0 && P.y) {
      // tensor-parallel head (vocab slice): the mergeable partial itself, merged across ranks
      // by the host (fq_tp_merge_stats)
      static_cast<StatPart*>(P.y)[b] = a;
    } else if (lane == 0) {
      fq_row_stats r;
      const double H = log(a.S) - a.T / a.S;
      r.entropy = H;
      r.ppl_entropy = exp(H);
      r.p1 = exp(static_cast<double>(a.v1) - a.m) / a.S;
      r.p2 = a.v2 == -INFINITY ? -1.0 : exp(static_cast<double>(a.v2) - a.m) / a.S;
      r.fault_tolerance = r.p1 - r.p2;
      r.max_logit = a.m;
      r.argmax = a.arg == 0x7fffffff ? 0 : a.arg;
      P.stats[b] = r;
    }
  }
}

// ---------------------------------------------------------------- grid barrier (consumers)
// Grid barrier (consumer threads): arrival counter in global memory, reset before every launch.
// Arrival is one release reduction (no returned value to wait for); the poll is relaxed (an
// acquire load per iteration would invalidate L1 each time) and one acquire fence follows it.
__device__ __forceinline__ unsigned int ld_relaxed(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ void grid_barrier(unsigned int* counter, unsigned int& epoch) {
  named_sync(1, kNCW * 32);
  if (threadIdx.x == 0) {
    const unsigned int target = (++epoch) * gridDim.x;
    const unsigned long long t0 = gtimer_now();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
    for (uint32_t spins = 0; ld_relaxed(counter) < target; ++spins)
      if ((spins & 255u) == 255u && gtimer_now() - t0 > kWatchdogNs)
        watchdog_fire("grid barrier", static_cast<int>(target), static_cast<int>(ld_relaxed(counter)));
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  } else {
    ++epoch;
  }
  named_sync(1, kNCW * 32);
}

// ---------------------------------------------------------------- the program kernel
// Dynamic shared memory: ring stages | full/empty mbarriers | xs | dx | red | sq | rstd.
struct SmemLayout {
  int nstages, xs_bytes, dx_bytes, red_bytes;
  int ctl_phases;  // phases with a precomputed partition table in shared memory (0 = none)
  unsigned int* lctr;  // [launch epoch, CTAs done]: the epoch tags this launch's stream-K parts
  int prefetch;  // L2 prefetch distance of the weight stream, in stages
  const int32_t* pos;    // per-row positions / cache slots of the step (shared-memory copies)
  const int32_t* slots;
  int nrows;
};

template <bool LEAN>
__device__ void run_program(const Phase* phases, int nphases, unsigned int* barrier, SmemLayout L) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ float sq_red[kMaxB][kNCW];
  __shared__ AttnSmem attn_smem;
  __shared__ PhaseCtl ctl;
  __shared__ int trace_n;
  __shared__ Phase pbuf[2];
  Ring R;
  R.base = smem;
  R.nstages = L.nstages;
  R.full = reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(L.nstages) * kStageBytes);
  R.empty = R.full + kMaxStages;
  GemvSmem G;
  uint8_t* p = reinterpret_cast<uint8_t*>(R.empty + kMaxStages);
  G.xs = reinterpret_cast<uint4*>(p);
  p += L.xs_bytes;
  G.dx = reinterpret_cast<float4*>(p);
  p += L.dx_bytes;
  G.red = reinterpret_cast<float*>(p);
  p += L.red_bytes;
  G.sq = reinterpret_cast<float*>(p);
  p += kNCW * 32 * sizeof(float);
  G.rstd = reinterpret_cast<float*>(p);
  p += kMaxB * sizeof(float);
  G.mbuf = reinterpret_cast<float*>(p);
  p += kMaxMat * 16 * kMaxB * sizeof(float);
  CtlEntry* ctab = L.ctl_phases > 0 ? reinterpret_cast<CtlEntry*>(p) : nullptr;
  G.tr = blockIdx.x == static_cast<unsigned>(g_trace_cta) ? g_ring_trace : nullptr;
  G.tn = &trace_n;
  if (threadIdx.x == 0) trace_n = 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < L.nstages; ++s) {
      mbar_init(&R.full[s], 1);
      mbar_init(&R.empty[s], kNCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  __shared__ const uint8_t* s_pbase[2][2 * kMaxMat];
  if (warp == kNCW) {
    unsigned long long* tr = blockIdx.x == static_cast<unsigned>(g_trace_cta) ? g_ring_trace : nullptr;
    if (LEAN || ctab != nullptr) {
      // the weight stream depends on nothing produced at run time, only on the partition table
      // the consumers compute first (named barrier 2)
      named_sync(2, kThreads);
      if (lane == 0) produce_table(phases, nphases, ctab, R, tr, s_pbase[0], L.prefetch < 0, L.prefetch, s_pbase[1]);
    } else if (lane == 0) {
      produce_all(phases, nphases, R, tr, L.prefetch);
    }
    return;
  }
  pdl_wait();
  __shared__ MetaSmem meta_smem;
  if (threadIdx.x == 0) {
    meta_smem.pos = L.pos;
    meta_smem.slots = L.slots;
    meta_smem.n = min(L.nrows, kMaxMetaRows);
  }
  for (int b = threadIdx.x; b < min(L.nrows, kMaxMetaRows); b += kNCW * 32) {
    meta_smem.p[b] = L.pos[b];
    meta_smem.s[b] = L.slots[b];
  }
  __shared__ unsigned int s_lepoch;
  if (threadIdx.x == 0) s_lepoch = *reinterpret_cast<volatile unsigned int*>(L.lctr);
  int slot_i = 0;
  uint32_t phase_bit = 0;
  unsigned int epoch = 0;
  unsigned long long* prof = threadIdx.x == 0 ? g_phase_prof : nullptr;
  unsigned long long* const gprof = g_gemv_prof;  // read once: a per-phase load would sit on the critical path
  if (prof) prof[static_cast<size_t>(nphases) * gridDim.x * 2 + blockIdx.x] = gtimer();
  // Phase descriptors live in shared memory: warp 0 loads descriptor i+1 into registers during
  // phase i (one 16-byte load per lane, latency hidden by the phase) and stores it at the end.
  if (ctab) {
    for (int t = threadIdx.x; t < nphases; t += kNCW * 32) compute_ctl(phases[t], ctab[t]);
    asm volatile("bar.arrive 2, %0;" ::"r"(kThreads) : "memory");  // table ready: producer starts
  }
  constexpr int kPW = static_cast<int>(sizeof(Phase) / 16);
  uint4 next_desc = make_uint4(0u, 0u, 0u, 0u);
  if (warp == 0) {
    if (lane < kPW) reinterpret_cast<uint4*>(&pbuf[0])[lane] = reinterpret_cast<const uint4*>(&phases[0])[lane];
    if (nphases > 1 && lane < kPW) next_desc = reinterpret_cast<const uint4*>(&phases[1])[lane];
  }
  named_sync(1, kNCW * 32);
  for (int i = 0; i < nphases; ++i) {
    const Phase& P = pbuf[i & 1];
    if (P.type == PH_GEMV)
      run_gemv_phase<LEAN>(P, R, G, ctl, L.red_bytes / 4, slot_i, phase_bit, i, ctab, s_lepoch * 1024u + i, gprof);
    else if (P.type == PH_EMBED) run_embed(P, sq_red);
    else if (P.type == PH_ATTN) run_attn(P, attn_smem, meta_smem, s_lepoch * 1024u + i);
    else if (P.type == PH_APPEND) run_append(P);
    else run_stats(P);
    if (prof) prof[(static_cast<size_t>(i) * gridDim.x + blockIdx.x) * 2] = gtimer();
    const bool bar = P.barrier_after && i + 1 < nphases;
    named_sync(1, kNCW * 32);  // everyone is done with descriptor i
    if (warp == 0 && i + 1 < nphases) {
      if (lane < kPW) reinterpret_cast<uint4*>(&pbuf[(i + 1) & 1])[lane] = next_desc;
      if (i + 2 < nphases && lane < kPW) next_desc = reinterpret_cast<const uint4*>(&phases[i + 2])[lane];
    }
    if (bar) grid_barrier(barrier, epoch);
    else named_sync(1, kNCW * 32);
    if (prof) prof[(static_cast<size_t>(i) * gridDim.x + blockIdx.x) * 2 + 1] = gtimer();
  }
  // the last CTA to finish advances the launch epoch (every CTA read it at its start)
  if (threadIdx.x == 0 && atomicAdd(&L.lctr[1], 1u) == gridDim.x - 1) {
    L.lctr[1] = 0u;
    __threadfence();
    atomicAdd(&L.lctr[0], 1u);
  }
}

__global__ void __launch_bounds__(kThreads, 1) program_kernel(const Phase* phases, int nphases, unsigned int* barrier,
                                                              SmemLayout L) {
  run_program<false>(phases, nphases, barrier, L);
}

__global__ void __launch_bounds__(kThreads, 1) program_kernel_inline(const __grid_constant__ InlineProgram prog,
                                                                     int nphases, unsigned int* barrier, SmemLayout L) {
  run_program<false>(prog.phases, nphases, barrier, L);
}

__global__ void __launch_bounds__(kThreads, 1) program_kernel_lean(const Phase* phases, int nphases, unsigned int* barrier,
                                                                   SmemLayout L) {
  run_program<true>(phases, nphases, barrier, L);
}

int max_dynamic_smem() {
  static int v = -1;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (v < 0) {
    int dev = 0, optin = 0;
    FQ_CUDA(cudaGetDevice(&dev));
    FQ_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes a1{}, a2{}, a3{};
    FQ_CUDA(cudaFuncGetAttributes(&a1, program_kernel));
    FQ_CUDA(cudaFuncGetAttributes(&a2, program_kernel_inline));
    FQ_CUDA(cudaFuncGetAttributes(&a3, program_kernel_lean));
    v = optin - static_cast<int>(std::max({a1.sharedSizeBytes, a2.sharedSizeBytes, a3.sharedSizeBytes})) - 1024;
    FQ_CUDA(cudaFuncSetAttribute(program_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, v));
    FQ_CUDA(cudaFuncSetAttribute(program_kernel_inline, cudaFuncAttributeMaxDynamicSharedMemorySize, v));
    FQ_CUDA(cudaFuncSetAttribute(program_kernel_lean, cudaFuncAttributeMaxDynamicSharedMemorySize, v));
  }
  return v;
}

constexpr int kMaxCtlPhases = 512;
static_assert(sizeof(CtlEntry) == 32 || !FQ_TILE_PART, "partition table entry grew: it costs ring stages");  // longer programs compute their partitions per phase

SmemLayout layout_for(int64_t kpad, int bb, int nphases, int& nstages_out, size_t& total_out, int64_t xs_bytes = -1) {
  SmemLayout L{};
  L.xs_bytes = static_cast<int>(xs_bytes >= 0 ? xs_bytes : kpad * 2 * bb);
  L.dx_bytes = static_cast<int>(L.xs_bytes / 256 * 16);  // one float4 per (block, row)
  // >= 8 KB: the fused softmax statistics use it as kNCW * 32 StatPart scratch; every byte saved
  // here goes to the weight ring (a 5th stage at the 7B shape)
  L.red_bytes = std::max(kNCW * 32 * 32, 2 * kMaxMat * kNCW * 16 * bb * 4);
  L.ctl_phases = nphases <= kMaxCtlPhases ? nphases : 0;
  const int fixed = 2 * kMaxStages * 8 + L.xs_bytes + L.dx_bytes + L.red_bytes + kNCW * 32 * 4 + kMaxB * 4 +
                    kMaxMat * 16 * kMaxB * 4 + L.ctl_phases * static_cast<int>(sizeof(CtlEntry));
  const int budget = max_dynamic_smem();
  L.nstages = std::min(kMaxStages, (budget - fixed) / kStageBytes);
  nstages_out = L.nstages;
  total_out = static_cast<size_t>(L.nstages) * kStageBytes + fixed;
  return L;
}

}  // namespace

int gemv_batch_chunk(int64_t K) {
  const int64_t kpad = (K + kBlockK - 1) / kBlockK * kBlockK;
  for (int bb = kMaxB; bb > 1; --bb) {
    int ns = 0;
    size_t tot = 0;
    layout_for(kpad, bb, 200, ns, tot);
    if (ns >= 3) return bb;
  }
  return 1;
}

ProgramRun upload_program(fq_ctx* ctx, ProgramBuilder& pb, bool transient) {
  ProgramRun r;
  r.nphases = static_cast<int>(pb.phases.size());
  r.grid = pb.grid;
  r.bb = pb.max_bb;
  int ns = 0;
  size_t tot = 0;
  const SmemLayout L = layout_for(pb.max_kpad, pb.max_bb, r.nphases, ns, tot, std::max<int64_t>(pb.max_xs, 256));
  if (ns < 2) fail(FQ_E_CONFIG, "gemv: activations of this width do not fit in shared memory");
  r.nstages = ns;
  // the lean kernel when every GEMV phase stages through one of its two paths
  r.lean = !transient && std::getenv("FQ_NO_LEAN") == nullptr && L.ctl_phases > 0 && FQ_TILE_PART;
  for (const Phase& P : pb.phases) {
    if (P.type != PH_GEMV || P.xfrag != nullptr) continue;
    const bool ok = P.x_dtype == FQ_DT_F32 && P.norm_gain != nullptr && P.attn_splits <= 1 &&
                    (reinterpret_cast<uintptr_t>(P.x) & 15) == 0 && ((P.x_stride * 4) & 15) == 0 && (P.K & 7) == 0 &&
                    (reinterpret_cast<uintptr_t>(P.norm_gain) & 15) == 0;
    if (!ok) r.lean = false;
  }
  if (std::getenv("FQ_DEBUG_LAYOUT"))
    std::fprintf(stderr, "fq program: %d phases, ring %d x %d B, xs %d, red %d, ctl %d, smem %zu B\n", r.nphases, ns,
                 kStageBytes, L.xs_bytes, L.red_bytes, L.ctl_phases, tot);
  r.smem = tot;
  r.xs_bytes = L.xs_bytes;
  r.dx_bytes = L.dx_bytes;
  r.red_bytes = L.red_bytes;
  r.ctl_phases = L.ctl_phases;
  if (const char* e = std::getenv("FQ_PREFETCH")) r.prefetch = std::atoi(e);
  const size_t fstride = static_cast<size_t>(kMaxMat) * 16 * pb.max_bb;
  const bool inl = r.nphases <= kInlinePhases && transient;
  // stream-K fix-up parts (only the byte-balanced partition, -DFQ_TILE_PART=0, writes them)
  float* fix;
  if (inl) {
    if (ctx->gemv_fix == nullptr) {
      ctx->gemv_fix = static_cast<float*>(dmalloc(sizeof(float2) * kInlinePhases * 1024 * kMaxMat * 16 * kMaxB));
      FQ_CUDA(cudaMemset(ctx->gemv_fix, 0, sizeof(float2) * kInlinePhases * 1024 * kMaxMat * 16 * kMaxB));
    }
    if (r.grid > 1024) fail(FQ_E_CONFIG, "gemv: grid too large");
    fix = ctx->gemv_fix;
  } else {
    r.fix = static_cast<float*>(dmalloc(sizeof(float2) * r.nphases * r.grid * fstride));
    FQ_CUDA(cudaMemset(r.fix, 0, sizeof(float2) * r.nphases * r.grid * fstride));
    fix = r.fix;
  }
  for (int i = 0; i < r.nphases; ++i) {
    Phase& P = pb.phases[i];
    if (P.type != PH_GEMV) continue;
    P.fix = fix + 2 * static_cast<size_t>(i) * r.grid * (inl ? kMaxMat * 16 * kMaxB : fstride);  // float2 parts
  }
  if (inl) {
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
  SmemLayout L{};
  L.nstages = run.nstages;
  L.xs_bytes = run.xs_bytes;
  L.dx_bytes = run.dx_bytes;
  L.red_bytes = run.red_bytes;
  L.prefetch = run.prefetch;
  L.ctl_phases = run.ctl_phases;
  L.pos = run.pos;
  L.slots = run.slots;
  L.nrows = run.pos && run.slots ? run.nrows : 0;
  if (ctx->launch_ctr == nullptr) {
    ctx->launch_ctr = static_cast<unsigned int*>(dmalloc(2 * sizeof(unsigned int)));
    const unsigned int init[2] = {1u, 0u};  // epoch 0 never tags anything (fresh memory is zero)
    FQ_CUDA(cudaMemcpy(ctx->launch_ctr, init, sizeof(init), cudaMemcpyHostToDevice));
  }
  L.lctr = ctx->launch_ctr;
  max_dynamic_smem();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(run.grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = run.smem;
  cfg.stream = ctx->stream;
  // cooperative: the grid barriers need every CTA resident at once -- the launch fails cleanly
  // (instead of spinning into the watchdog) when another stream's kernel holds SMs
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  if (run.dev_phases && run.lean)
    FQ_CUDA(cudaLaunchKernelEx(&cfg, program_kernel_lean, static_cast<const Phase*>(run.dev_phases), run.nphases, barrier,
                               L));
  else if (run.dev_phases)
    FQ_CUDA(cudaLaunchKernelEx(&cfg, program_kernel, static_cast<const Phase*>(run.dev_phases), run.nphases, barrier, L));
  else
    FQ_CUDA(cudaLaunchKernelEx(&cfg, program_kernel_inline, run.inl, run.nphases, barrier, L));
  ctx->launches += 1;
}

}  // namespace fqc
