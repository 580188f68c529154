// The TMA-fed streaming program: phase descriptors, the persistent program kernel and its
// host-side builder.  Shared by the stand-alone GEMV entry point (gemv.cu) and the decode step
// (model.cu).  See gemv.cu for the design notes.
#pragma once

#include "fq_internal.cuh"

#include <vector>

namespace fqc {

constexpr int kStepCodes = 512;  // codes per row per warp step (32 lanes x 16)
constexpr int kSegCodes = 16;    // codes per lane per step
constexpr int kMaxB = 4;         // batch rows per phase
constexpr int kMaxStages = 8;
constexpr int kSplit = 8;        // consumer warps splitting the K-steps of a row
#ifndef FQ_RG
#define FQ_RG 2
#endif
constexpr int kRG = FQ_RG;       // row groups of consumer warps
constexpr int kNCW = kSplit * kRG;
constexpr int kThreads = (kNCW + 1) * 32;  // + one producer warp
constexpr int kMaxSW = 4;        // K-steps per warp (K <= 16384)
constexpr int kAttnChunk = 64;   // keys per attention work item
constexpr float kTwo109 = 649037107316853453566312041152512.0f;  // 2^109
constexpr float kTwo40 = 1099511627776.0f;                        // 2^40
constexpr float kTwoM40 = 9.094947017729282379150390625e-13f;     // 2^-40

enum PhaseType : int { PH_GEMV = 0, PH_EMBED = 1, PH_ATTN = 2, PH_STATS = 3 };

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

// One phase of a program.  GEMV fields follow GemvLaunch; EMBED / ATTN / STATS use the extra
// fields at the end.
struct Phase {
  int type;
  int barrier_after;  // grid barrier between this phase and the next
  // ---- GEMV
  DevMat mat[3];
  int nmat;
  int B;
  int64_t N, K, G, ng_pad, zp_pad;
  int nsteps, sw;
  int rows_per_stage[2];
  int sc_off[2], zp_off[2];
  int sc_row, zp_row;
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
  // ---- EMBED / ATTN / STATS (decode step)
  const float* tok_emb;
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
  float rope_theta;
  float* attn_ws;
  unsigned int* tickets;
  void* attn_out;
  const float* logits;
  int64_t vocab;
  fq_row_stats* stats;
};

constexpr int kInlinePhases = 4;
struct InlineProgram {
  Phase phases[kInlinePhases];
};

struct ProgramBuilder {
  std::vector<Phase> phases;
  int grid = 148;
  int64_t stage_bytes = 0;
  int64_t red_floats = 0;
  int max_sw = 1;
  int max_bb = 1;
  int max_nsteps = 1;
  void add_gemv(const GemvLaunch& g, int64_t b0, int bb);
  void add(const Phase& p);
};

struct ProgramRun {
  Phase* dev_phases = nullptr;  // device copy (long programs); null -> inline
  InlineProgram inl;
  int nphases = 0;
  int grid = 0;
  int stage_bytes = 0;
  int nstages = 0;
  size_t smem = 0;
  int bb = 1;
  int red_floats = 0;
  int xs_floats = 0;
  unsigned int* barrier = nullptr;  // grid-barrier counter (reset before every launch)
};

// Sizes the ring and the reduction buffer for a program; long programs are copied to device
// memory owned by the caller (dev_phases must be freed with dfree), short ones go inline.
ProgramRun upload_program(fq_ctx* ctx, const ProgramBuilder& pb, bool transient);
void launch_program(fq_ctx* ctx, const ProgramRun& run, unsigned int* barrier, bool pdl);
int gemv_batch_chunk(int64_t K);

}  // namespace fqc
