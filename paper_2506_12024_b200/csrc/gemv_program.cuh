// The TMA-fed streaming program: phase descriptors, the persistent program kernel and its
// host-side builder.  Shared by the stand-alone GEMV entry point (gemv.cu) and the decode step
// (model.cu).  See gemv.cu for the design notes and fq_internal.cuh for the tiled weight layout.
#pragma once

#include "fq_internal.cuh"

#include <vector>

namespace fqc {

constexpr int kMaxB = 8;          // batch rows per GEMV phase (the MMA's n = 8 columns)
constexpr int kMaxMat = 3;        // matrices sharing one input (QKV)
constexpr int kMaxStages = 8;
#ifndef FQ_NCW
#define FQ_NCW 11  // 12 warps = 3 per SM sub-partition: same 168-register cap as 9 warps, 37% more consumers
#endif
constexpr int kNCW = FQ_NCW;      // consumer warps (2 blocks in flight each)
constexpr int kThreads = (kNCW + 1) * 32;  // + one producer warp
constexpr int kAttnChunk = 16;    // keys per attention work item (one warp)
#ifndef FQ_STAGE8
#define FQ_STAGE8 16
#endif
constexpr int kStageBlocks8 = FQ_STAGE8;       // W8 blocks per ring stage (2 per consumer warp)
#ifndef FQ_STAGE4
#define FQ_STAGE4 (2 * FQ_STAGE8)
#endif
constexpr int kStageBlocks4 = FQ_STAGE4;       // W4 blocks per ring stage
constexpr int kStageBytes = kStageBlocks8 * (2048 + 80) > kStageBlocks4 * (1024 + 80) ? kStageBlocks8 * (2048 + 80)
                                                                                      : kStageBlocks4 * (1024 + 80);
constexpr int kSmemBudget = 220 * 1024;

enum PhaseType : int { PH_GEMV = 0, PH_EMBED = 1, PH_ATTN = 2, PH_STATS = 3, PH_APPEND = 4 };

struct DevMat {
  const uint8_t* tiles[2];    // [0] = W8, [1] = W4 tiled copies (fq_rung_store::tiles)
  int32_t zpbase[2];
  const uint8_t* rung_table;  // per batch row, or null
  int64_t rung_stride;
  int rung;                   // when no table
  void* y;
};

// One phase of a program.  GEMV fields follow GemvLaunch; EMBED / ATTN / STATS use the extra
// fields at the end.  At most 512 bytes: one warp moves it into shared memory with one 16-byte
// load per lane.
struct alignas(16) Phase {
  int type;
  int barrier_after;  // grid barrier between this phase and the next
  // ---- GEMV
  DevMat mat[kMaxMat];
  int nmat;
  int B;
  int64_t N, K;
  int n_tiles, nkb;   // 16-row tiles, 128-code blocks per row
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
  int out_partials_stride;
  void* stat_part;        // GEMV: per-(row, CTA) softmax partials of the stored outputs (fused
                          // entropy, head only); STATS: their input [B][grid]
  const uint4* xfrag;     // GEMV: input already in B-fragment order (fp16, batch-major, the smem
                          // xs layout) written by the producing phase's epilogue: staging is a copy
  __half* yfrag;          // GEMV (SwiGLU epilogue) / ATTN: also write the output in that order; as
                          // (half2, tag) words when the next phase has no barrier (yfrag_tagged)
  int yfrag_nkb;          // 128-blocks per batch row of yfrag; < 0: tagged words, nkb = -yfrag_nkb
  float* fix;             // stream-K fix-up partials [grid][kMaxMat * 16 * kMaxB]
  // ---- EMBED / ATTN / STATS (decode step)
  union {
    const float* tok_emb;     // EMBED
    unsigned int* tile_flags; // QKV GEMV: stamps each finished 16-row tile with the phase tag;
                              // ATTN: polls its head's tiles instead of a grid barrier (decode)
  };
  const int32_t* tokens;
  const int32_t* pos;
  const int32_t* slots;
  int64_t d;
  const void* q;
  const void* k;
  const void* v;
  __half* kv;
  int64_t slot_stride, layer_off, max_seq;
  int n_heads, head_dim;
  union {
    int appended;         // ATTN: the rows' keys / values are already in the cache (prefill)
    int xfrag_tagged;     // GEMV: xfrag holds (half2, tag) 8-byte words written by the previous
                          // phase (no grid barrier before this phase: staging polls the tags)
    int token_stride;     // EMBED: row b's token is tokens[b * token_stride] (0 = 1); a chained
                          // decode step points tokens at the previous step's fq_row_stats argmax
  };
  int attn_splits;        // ATTN: CTAs per (row, head), each over a contiguous chunk range; > 1:
                          // unnormalised partials (O[hd], m, l) in attn_ws, merged by the next
                          // GEMV phase's staging (the O projection reads them as its input)
  const float2* rope_cs;  // [max_seq][head_dim / 2] (cos, sin) of pos * theta^(-2i/hd)
  float* attn_ws;
  void* attn_out;
  fq_row_stats* stats;
};

static_assert(sizeof(Phase) <= 512, "Phase must fit one warp-wide 16-byte load");

constexpr int kInlinePhases = 4;
struct InlineProgram {
  Phase phases[kInlinePhases];
};

struct ProgramBuilder {
  std::vector<Phase> phases;
  int grid = 148;
  int max_bb = 1;          // largest GEMV batch chunk
  int64_t max_kpad = 128;  // largest K rounded up to a block
  int64_t max_xs = 0;      // largest activation staging (K_pad * 2 * chunk) of a GEMV phase
  void add_gemv(const GemvLaunch& g, int64_t b0, int bb);
  void add(const Phase& p);
};

struct ProgramRun {
  Phase* dev_phases = nullptr;  // device copy (long programs); null -> inline
  InlineProgram inl;
  int nphases = 0;
  int grid = 0;
  int nstages = 0;
  size_t smem = 0;
  int bb = 1;
  int xs_bytes = 0;   // activation fragments
  int dx_bytes = 0;   // per-block activation sums
  int red_bytes = 0;  // per-warp tile partials (reduction window)
  int prefetch = 0;   // L2 prefetch distance in stages (env FQ_PREFETCH overrides; -1 = no loads)
  int ctl_phases = 0; // phases with a precomputed partition table in shared memory
  bool lean = false;  // decode / prefill step program: launch the lean kernel (program.cu)
  const int32_t* pos = nullptr;   // decode step: per-row positions / cache slots, copied into shared
  const int32_t* slots = nullptr; // memory at kernel start (the attention phases read them there)
  int nrows = 0;
  const void* tp_in = nullptr;    // tensor-parallel segment: the exchange buffers baked in
  const void* tp_out = nullptr;
  float* fix = nullptr;           // owned stream-K scratch (device programs)
  unsigned int* flags = nullptr;
};

// Sizes the ring and the staging buffers for a program; long programs are copied to device
// memory owned by the caller (dev_phases / fix / flags must be freed with dfree), short ones
// go inline and use the context's workspace.
ProgramRun upload_program(fq_ctx* ctx, ProgramBuilder& pb, bool transient);
void launch_program(fq_ctx* ctx, const ProgramRun& run, unsigned int* barrier, bool pdl);
int gemv_batch_chunk(int64_t K);
// Profiling hook: device buffer receiving per-phase timestamps of the next programs (null = off).
void set_phase_profile(unsigned long long* dev);
// Profiling hook: ring trace of one CTA (3 stamps per stage, see program.cu); null = off.
void set_ring_trace(unsigned long long* dev, int cta);
void set_gemv_profile(unsigned long long* dev);

}  // namespace fqc
