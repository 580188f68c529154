// Device-resident decoder: precision table, KV cache, and the graph-captured decode step.
//
// Two block families behind one object (include/fq_cuda.h):
//  * FQ_ARCH_LLAMA (BASELINE configs): RMSNorm (fused into the next GEMV's prologue through
//    per-CTA sum-of-squares partials), fused QKV GEMV, RoPE + fp16 KV append + attention in one
//    kernel, residual-add epilogues, gate/up GEMV with a SwiGLU epilogue, head GEMV, fused
//    softmax statistics.  bf16 (or fp16) activations, fp32 residual stream, fp32 logits.
//  * FQ_ARCH_REFERENCE: the reference's own model (/root/reference/proj/src/model.cpp:193-266):
//    learned positions, LayerNorm + biases, GELU FFN, fp32 activations, every reduction done
//    sequentially in double in the reference's order, so logits are bit-identical to the CPU
//    reference (the golden-trace mode).
//
// A rung switch (Model::set_precision, src/model.cpp:268-278) is a one-byte write into the
// host precision table; the per-step table for the batch rows is copied to the device by the
// captured graph, and the GEMVs select the W8 or W4 copy from it, so no weights move and the
// graph is never re-captured.
#include "fq_internal.cuh"
#include "gemv_program.cuh"

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <set>
#include <string>

namespace fqc {
namespace {

constexpr int kPartStride = 1024;
constexpr int kMaxChain = 64;  // decode steps per fq_model_decode_chain call
constexpr int kPrefillRows = 8;  // prompt positions per prefill step (llama): the GEMV's MMA n

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Step metadata staged by the host each step: tokens[B], pos[B], slots[B], then the per-row
// precision table [B][n_lin] (bytes).
struct StepMeta {
  const int32_t* tokens;
  const int32_t* pos;
  const int32_t* slots;
};

// Fused softmax statistics of B logits rows (double), one CTA per row; writes fq_row_stats.
// (Same arithmetic as stats.cu, kept local so the step graph has no cross-TU dependency.)
__global__ void __launch_bounds__(1024) row_stats_kernel(const float* __restrict__ logits, int64_t vocab,
                                                         fq_row_stats* __restrict__ out) {
  pdl_wait();
  __shared__ double shd[33];
  __shared__ float shv[33];
  __shared__ int shi[33];
  __shared__ double sha[33], shb[33];
  const float* l = logits + blockIdx.x * vocab;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int64_t i = threadIdx.x; i < vocab; i += blockDim.x) {
    const float x = l[i];
    if (x > bv || (x == bv && i < bi)) { bv = x; bi = static_cast<int>(i); }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
  }
  if (lane == 0) { shv[warp] = bv; shi[warp] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < nw; ++w)
      if (shv[w] > shv[0] || (shv[w] == shv[0] && shi[w] < shi[0])) { shv[0] = shv[w]; shi[0] = shi[w]; }
  }
  __syncthreads();
  const double mx = shv[0];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < vocab; i += blockDim.x) s += exp(static_cast<double>(l[i]) - mx);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) shd[warp] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t += shd[w];
    shd[32] = t;
  }
  __syncthreads();
  const double sum = shd[32];
  double h = 0.0, t1 = -1.0, t2 = -1.0;
  for (int64_t i = threadIdx.x; i < vocab; i += blockDim.x) {
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
  __syncthreads();
  if (lane == 0) { shd[warp] = h; sha[warp] = t1; shb[warp] = t2; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double H = 0.0, a1 = -1.0, a2 = -1.0;
    for (int w = 0; w < nw; ++w) {
      H += shd[w];
      const double n1 = fmax(a1, sha[w]), n2 = fmax(fmin(a1, sha[w]), fmax(a2, shb[w]));
      a1 = n1;
      a2 = n2;
    }
    fq_row_stats st;
    st.entropy = H;
    st.ppl_entropy = exp(H);
    st.p1 = a1;
    st.p2 = a2;
    st.fault_tolerance = a1 - a2;
    st.max_logit = shv[0];
    st.argmax = shi[0];
    out[blockIdx.x] = st;
  }
}

// ------------------------------------------------------------------ reference-arch kernels
// x = tok_emb[token] + pos_emb[pos] in float (src/model.cpp:245-252, 261-264)
__global__ void embed_ref_kernel(const float* __restrict__ tok, const float* __restrict__ posemb, StepMeta meta,
                                 int64_t d, float* __restrict__ x) {
  const int b = blockIdx.x;
  const float* e = tok + static_cast<int64_t>(meta.tokens[b]) * d;
  const float* p = posemb + static_cast<int64_t>(meta.pos[b]) * d;
  for (int64_t c = threadIdx.x; c < d; c += blockDim.x) x[b * d + c] = e[c] + p[c];
}

// layer_norm (src/tensor.cpp:124-145): sequential double mean / variance, then per element
// (in - mean) * inv * gamma + beta in double, stored as float.
__global__ void layernorm_ref_kernel(const float* __restrict__ x, int64_t d, const float* __restrict__ g,
                                     const float* __restrict__ be, float eps, float* __restrict__ y) {
  const int b = blockIdx.x;
  const float* in = x + b * d;
  __shared__ double mean_s, inv_s;
  if (threadIdx.x == 0) {
    double mean = 0.0;
    for (int64_t c = 0; c < d; ++c) mean += in[c];
    mean /= static_cast<double>(d);
    double var = 0.0;
    for (int64_t c = 0; c < d; ++c) {
      const double dv = in[c] - mean;
      var += dv * dv;
    }
    var /= static_cast<double>(d);
    mean_s = mean;
    inv_s = 1.0 / sqrt(var + static_cast<double>(eps));
  }
  __syncthreads();
  for (int64_t c = threadIdx.x; c < d; c += blockDim.x)
    y[b * d + c] = static_cast<float>((in[c] - mean_s) * inv_s * g[c] + be[c]);
}

// gelu, erf form, in double (src/tensor.cpp:154-161)
__global__ void gelu_ref_kernel(float* __restrict__ x, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) {
    const double v = x[i];
    x[i] = static_cast<float>(0.5 * v * (1.0 + erf(v / sqrt(2.0))));
  }
}

// add (src/tensor.cpp:147-152): float + float
__global__ void add_kernel(float* __restrict__ x, const float* __restrict__ y, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) x[i] = x[i] + y[i];
}

// Appends k/v rows (fp32) to the reference-arch cache at each row's position.
__global__ void append_ref_kernel(const float* __restrict__ k, const float* __restrict__ v, StepMeta meta, int64_t d,
                                  float* __restrict__ kv, int64_t slot_stride, int64_t layer_off, int64_t max_seq) {
  const int b = blockIdx.x;
  float* kc = kv + meta.slots[b] * slot_stride + layer_off;
  float* vc = kc + max_seq * d;
  const int64_t p = meta.pos[b];
  for (int64_t c = threadIdx.x; c < d; c += blockDim.x) {
    kc[p * d + c] = k[b * d + c];
    vc[p * d + c] = v[b * d + c];
  }
}

// attention (src/model.cpp:100-140) for one (row, head): keys 0..pos of the slot, sequential
// double arithmetic in the reference's loop order.  One CTA per (head, row); scores by thread 0.
__global__ void attn_ref_kernel(const float* __restrict__ q, StepMeta meta, const float* __restrict__ kv,
                                int64_t slot_stride, int64_t layer_off, int64_t max_seq, int n_heads, int hd,
                                double* __restrict__ scratch, float* __restrict__ out) {
  const int h = blockIdx.x, b = blockIdx.y;
  const int64_t d = static_cast<int64_t>(n_heads) * hd;
  const int pos = meta.pos[b];
  const float* kc = kv + meta.slots[b] * slot_stride + layer_off;
  const float* vc = kc + max_seq * d;
  double* probs = scratch + (static_cast<int64_t>(b) * n_heads + h) * max_seq;
  __shared__ double sum_s;
  const float* qi = q + b * d + h * hd;
  const int visible = pos + 1;
  if (threadIdx.x == 0) {
    const double scale = 1.0 / sqrt(static_cast<double>(hd));
    double mx = -INFINITY;
    for (int j = 0; j < visible; ++j) {
      const float* kj = kc + static_cast<int64_t>(j) * d + h * hd;
      double dot = 0.0;
      for (int p = 0; p < hd; ++p) dot += static_cast<double>(qi[p]) * static_cast<double>(kj[p]);
      probs[j] = dot * scale;
      mx = fmax(mx, probs[j]);
    }
    double sum = 0.0;
    for (int j = 0; j < visible; ++j) {
      probs[j] = exp(probs[j] - mx);
      sum += probs[j];
    }
    sum_s = sum;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < hd; c += blockDim.x) {
    double acc = 0.0;
    for (int j = 0; j < visible; ++j)
      acc += (probs[j] / sum_s) * static_cast<double>(vc[static_cast<int64_t>(j) * d + h * hd + c]);
    out[b * d + h * hd + c] = static_cast<float>(acc);
  }
}

// Sequential statistics (exact order of softmax_double / ppl_entropy / fault_tolerance /
// argmax_token) for small vocabularies: one thread per row.
__global__ void row_stats_seq_kernel(const float* __restrict__ logits, int64_t V, double* scratch,
                                     fq_row_stats* __restrict__ out) {
  const int b = blockIdx.x;
  if (threadIdx.x != 0) return;
  const float* l = logits + b * V;
  double* p = scratch + b * V;
  double mx = l[0];
  for (int64_t i = 1; i < V; ++i) mx = fmax(mx, static_cast<double>(l[i]));
  double sum = 0.0;
  for (int64_t i = 0; i < V; ++i) {
    p[i] = exp(static_cast<double>(l[i]) - mx);
    sum += p[i];
  }
  for (int64_t i = 0; i < V; ++i) p[i] /= sum;
  double h = 0.0;
  for (int64_t i = 0; i < V; ++i)
    if (p[i] > 0.0) h -= p[i] * log(p[i]);
  double t1 = -1.0, t2 = -1.0;
  for (int64_t i = 0; i < V; ++i) {
    if (p[i] > t1) { t2 = t1; t1 = p[i]; } else if (p[i] > t2) { t2 = p[i]; }
  }
  int best = 0;
  float bv = l[0];
  for (int64_t i = 1; i < V; ++i)
    if (l[i] > bv) { bv = l[i]; best = static_cast<int>(i); }
  fq_row_stats st;
  st.entropy = h;
  st.ppl_entropy = exp(h);
  st.p1 = t1;
  st.p2 = t2;
  st.fault_tolerance = t1 - t2;
  st.max_logit = bv;
  st.argmax = best;
  out[b] = st;
}

}  // namespace
}  // namespace fqc

using namespace fqc;

struct fq_model {
  fq_ctx* ctx = nullptr;
  fq_model_config cfg{};
  bool llama = true;
  int n_lin = 0;
  std::vector<std::string> ids;
  std::vector<fq_layer*> lin;
  // non-switchable parameters (device fp32)
  float* tok_emb = nullptr;
  float* pos_emb = nullptr;
  std::vector<float*> n1g, n1b, n2g, n2b;  // ln1/ln2 (reference) or attn_norm/ffn_norm (llama: g only)
  float* fng = nullptr;
  float* fnb = nullptr;
  fq_layer tied_head;  // reference arch with tied embeddings
  // per-slot state
  std::vector<int64_t> slot_len;
  std::vector<uint8_t> rungs;  // [max_batch][n_lin]
  void* kv = nullptr;
  int64_t slot_stride = 0;     // elements per slot
  int64_t layer_stride = 0;    // elements per layer within a slot
  // activations / workspace (max_batch rows)
  float* resid = nullptr;      // [B, d]
  float* hbuf = nullptr;       // [B, d] (reference: normalized activations)
  void* q = nullptr;           // [B, d]
  void* k = nullptr;
  void* v = nullptr;
  void* attn = nullptr;        // [B, d]
  void* mid = nullptr;         // [B, ffn]
  void* attn_frag = nullptr;   // [B][d/128][16] uint4: attention output in B-fragment order (fp16)
  void* mid_frag = nullptr;    // [B][ffn/128][16] uint4: SwiGLU output in B-fragment order
  float* tmp = nullptr;        // [B, max(d, ffn)] fp32 (reference)
  float* partials[2] = {nullptr, nullptr};  // ping-pong sum-of-squares partials [B][kPartStride]
  float* logits = nullptr;     // [max_batch, V]
  fq_row_stats* stats_dev = nullptr;
  void* stat_part = nullptr;  // llama step: [max_batch][grid] softmax partials of the head GEMV
  float* attn_ws = nullptr;
  float2* rope_cs = nullptr;  // llama: [max_seq][head_dim/2] (cos, sin)
  unsigned int* tickets = nullptr;
  double* dscratch = nullptr;
  int n_chunks = 1;
  // step staging
  uint8_t* meta_dev = nullptr;
  uint8_t* meta_host = nullptr;  // pinned
  size_t meta_bytes = 0;
  fq_row_stats* stats_host = nullptr;  // pinned [max_batch]
  std::map<int, cudaGraphExec_t> graphs;
  std::map<int, int64_t> graph_kernels;  // kernels inside each captured step graph
  std::map<std::pair<int, int>, ProgramRun> programs;  // (batch, StepMode) -> uploaded program
  unsigned int* grid_barrier = nullptr;
  bool use_graphs = std::getenv("FQ_NO_GRAPHS") == nullptr;  // FQ_NO_GRAPHS: plain launches (the tests' control)
  uint64_t built_epoch = 0;  // ctx->weight_epoch the cached programs / graphs were built at
  // batched tensor-core steps: captured graphs per (copies per linear, B) signature
  std::map<std::string, std::pair<cudaGraphExec_t, int64_t>> batch_graphs;
  std::set<std::string> batch_seen;
  // device-timed latency buckets (fq_model_decode_timed): phase clock buffer and phase -> linears
  unsigned long long* timed_ticks = nullptr;
  int64_t timed_ticks_n = 0;
  std::vector<std::vector<int>> timed_roles;
  // device time of the step program kernels (events around the launch, captured into the graph)
  cudaEvent_t ev_prog[2] = {nullptr, nullptr};
  double prog_ms = 0.0;
  int64_t prog_steps = 0;
  // tensor-core prefill workspace (llama; grown to the longest prompt seen, prefill_gemm)
  struct PrefillWs {
    int64_t cap = 0;
    float *x = nullptr, *q = nullptr, *k = nullptr, *v = nullptr, *qr = nullptr, *g = nullptr, *u = nullptr,
          *logits = nullptr;
    void *h = nullptr, *a = nullptr, *m = nullptr;
    fq_row_stats* stats = nullptr;
    int32_t* tok = nullptr;
  } pw;
  int rows = 1;  // activation rows: max(max_batch, prefill chunk) (llama); max_batch (reference)
  // tensor-parallel rank (fq_model_create_tp): this model holds heads [sh.head0, +heads), ffn
  // columns [sh.ffn0, +ffn) and vocab rows [sh.vocab0, +vocab) of the full config `cfg`; without
  // TP the shard is the whole model.  q_dim = local attention width (heads * head_dim).
  fq_tp_shard sh{};
  int64_t q_dim = 0;
  int tp_batch = 0;     // rows of the step begun by fq_model_tp_begin (0: none)
  int tp_next_seg = 0;  // next segment the step expects
  std::vector<int32_t> tp_slots_step = std::vector<int32_t>(256);
  bool tp() const { return sh.size > 1; }
  // chained decode (fq_model_decode_chain): the slot whose single-row decode step ran last (its
  // argmax is stats_dev[0]), -1 when another step / prefill ran since; pinned stats ring, events
  int chain_slot = -1;
  fq_row_stats* chain_ring = nullptr;      // pinned [kMaxChain]
  fq_row_stats* chain_ring_dev = nullptr;  // [kMaxChain], filled by the chained steps in order
  unsigned int* chain_count = nullptr;     // device write index into chain_ring_dev
  cudaGraphExec_t chain_graph = nullptr;   // one chained step: advance pos | step program | collect

  int lin_index(int layer, int j) const { return layer * (llama ? 7 : 6) + j; }
  int head_index() const { return static_cast<int>(cfg.n_layers) * (llama ? 7 : 6); }
  size_t act_size() const { return cfg.act_dtype == FQ_DT_F32 ? 4 : 2; }
  StepMeta meta(int B) const {
    StepMeta m;
    m.tokens = reinterpret_cast<const int32_t*>(meta_dev);
    m.pos = m.tokens + rows;
    m.slots = m.pos + rows;
    (void)B;
    return m;
  }
  const uint8_t* table_dev() const { return meta_dev + 3 * sizeof(int32_t) * rows; }
  uint8_t* table_host() const { return meta_host + 3 * sizeof(int32_t) * rows; }
};

namespace fqc {
namespace mdl {

void require(bool c, fq_status code, const std::string& msg) {
  if (!c) fail(code, msg);
}

void launch_dev(fq_model* M) { M->ctx->launches += 1; }

// Adds a GEMV for B batch rows as independent phases of at most gemv_batch_chunk(K) rows.
void add_chunked(ProgramBuilder& pb, const GemvLaunch& g, int B) {
  const int chunk = gemv_batch_chunk(g.mat[0].layer->K);
  for (int b0 = 0; b0 < B; b0 += chunk) {
    pb.add_gemv(g, b0, std::min(chunk, B - b0));
    pb.phases.back().barrier_after = b0 + chunk >= B ? 1 : 0;
  }
}

bool capturing(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  return cs != cudaStreamCaptureStatusNone;
}

// Enqueues one decode step for B rows (metadata already staged in meta_dev).  gemv_only keeps
// just the GEMV launches (kernel-level profiling; activations are whatever the buffers hold).
// STEP_CHAIN: a decode step whose token is the previous step's argmax, read on the device
// (fq_model_decode_chain)
enum StepMode : int { STEP_DECODE = 0, STEP_GEMV_ONLY = 1, STEP_PREFILL = 2, STEP_CHAIN = 3 };

// Prefill steps (STEP_PREFILL) take B consecutive positions of one sequence as their rows: an
// append phase writes every row's RoPE'd key / value to the cache before the attention phase, so
// row b attends to the rows before it in the same step.
// Step programs and captured graphs bake in the tiled weight pointers: after any layer's resident
// copies change (ctx->weight_epoch), drop them so the next step rebuilds against the new pointers.
void sync_weight_epoch(fq_model* M) {
  if (M->built_epoch == M->ctx->weight_epoch) return;
  if (!M->graphs.empty() || !M->programs.empty()) {
    FQ_CUDA(cudaStreamSynchronize(M->ctx->stream));
    for (auto& kv : M->graphs) cudaGraphExecDestroy(kv.second);
    for (auto& kv : M->programs) dfree(kv.second.dev_phases);
    for (auto& kv : M->batch_graphs) cudaGraphExecDestroy(kv.second.first);
    M->graphs.clear();
    M->graph_kernels.clear();
    M->programs.clear();
    M->batch_graphs.clear();
    M->batch_seen.clear();
    M->timed_roles.clear();
  }
  if (M->chain_graph) {
    FQ_CUDA(cudaStreamSynchronize(M->ctx->stream));
    cudaGraphExecDestroy(M->chain_graph);
    M->chain_graph = nullptr;
  }
  M->built_epoch = M->ctx->weight_epoch;
}

void enqueue_step(fq_model* M, int B, int mode = STEP_DECODE) {
  if (!capturing(M->ctx->stream)) sync_weight_epoch(M);
  const bool gemv_only = mode == STEP_GEMV_ONLY;
  const bool prefill = mode == STEP_PREFILL;
  fq_ctx* ctx = M->ctx;
  const fq_model_config& c = M->cfg;
  cudaStream_t st = ctx->stream;
  const int64_t d = c.d_model, V = c.vocab_size;
  const StepMeta meta = M->meta(B);
  const uint8_t* table = M->table_dev();
  if (M->llama) {
    // The whole llama step is one persistent program (program.cu): embedding, then per layer
    // QKV GEMV (fused RMSNorm) | attention | WO (+residual) | gate/up (+SwiGLU) | down
    // (+residual), then the head and the row statistics, with a grid barrier between
    // dependent phases while the weight stream runs ahead.
    auto key = std::make_pair(B, mode);
    auto it = M->programs.find(key);
    if (it == M->programs.end()) {
      if (capturing(st)) fail(FQ_E_STATE, "step program must be built before graph capture");
      ProgramBuilder pb;
      pb.grid = ctx->num_sms;
      const int G = pb.grid;
      if (!gemv_only) {
        Phase e{};
        e.type = PH_EMBED;
        e.barrier_after = 1;
        e.B = B;
        e.tok_emb = M->tok_emb;
        e.tokens = meta.tokens;
        if (mode == STEP_CHAIN) {
          e.tokens = &M->stats_dev[0].argmax;
          e.token_stride = static_cast<int>(sizeof(fq_row_stats) / sizeof(int32_t));
        }
        e.d = d;
        e.resid = M->resid;
        e.resid_stride = d;
        e.out_partials = M->partials[0];
        e.out_partials_stride = kPartStride;
        pb.add(e);
      }
      int cur = 0;
      // the O and down projections read their inputs pre-staged in B-fragment order (written by the
      // attention / SwiGLU epilogues); FQ_NO_FRAG=1 stages them from the plain activations
      const bool use_frag = std::getenv("FQ_NO_FRAG") == nullptr && B <= kMaxB;
      // (measured alternatives to the grid barriers -- tagged activation words, per-head QKV tile
      // flags, attention split over CTAs with the O staging merging the partials -- were all
      // slower at the 7B shape and are not built: DESIGN.md §4)
      const int frag_nkb_d = static_cast<int>((d + kBlockK - 1) / kBlockK);
      const int attn_splits = 1;
      for (int64_t l = 0; l < c.n_layers; ++l) {
        GemvLaunch g;
        g.nmat = 3;
        for (int j = 0; j < 3; ++j) {
          g.mat[j].layer = M->lin[M->lin_index(static_cast<int>(l), j)];
          g.mat[j].rung_table = table + M->lin_index(static_cast<int>(l), j);
          g.mat[j].rung_stride = M->n_lin;
        }
        g.mat[0].y = M->q;
        g.mat[1].y = M->k;
        g.mat[2].y = M->v;
        g.x = M->resid;
        g.x_dtype = FQ_DT_F32;
        g.x_stride = d;
        g.norm_gain = M->n1g[l];
        g.norm_partials = M->partials[cur];
        g.n_partials = G;
        g.partials_stride = kPartStride;
        g.norm_eps = c.norm_eps;
        g.act_dtype = c.act_dtype;
        g.epi = EPI_SPLIT3;
        g.y_dtype = c.act_dtype;
        g.y_stride = d;
        add_chunked(pb, g, B);
        if (prefill) {
          Phase ap{};
          ap.type = PH_APPEND;
          ap.barrier_after = 1;
          ap.B = B;
          ap.k = M->k;
          ap.v = M->v;
          ap.act_dtype = c.act_dtype;
          ap.pos = meta.pos;
          ap.slots = meta.slots;
          ap.kv = static_cast<__half*>(M->kv);
          ap.slot_stride = M->slot_stride;
          ap.layer_off = l * M->layer_stride;
          ap.max_seq = c.max_seq_len;
          ap.n_heads = static_cast<int>(c.n_heads);
          ap.head_dim = static_cast<int>(c.head_dim);
          ap.rope_cs = M->rope_cs;
          pb.add(ap);
        }
        if (!gemv_only) {
          Phase a{};
          a.type = PH_ATTN;
          a.appended = prefill ? 1 : 0;
          a.barrier_after = 1;
          a.B = B;
          a.q = M->q;
          a.k = M->k;
          a.v = M->v;
          a.act_dtype = c.act_dtype;
          a.pos = meta.pos;
          a.slots = meta.slots;
          a.kv = static_cast<__half*>(M->kv);
          a.slot_stride = M->slot_stride;
          a.layer_off = l * M->layer_stride;
          a.max_seq = c.max_seq_len;
          a.n_heads = static_cast<int>(c.n_heads);
          a.head_dim = static_cast<int>(c.head_dim);
          a.rope_cs = M->rope_cs;
          a.attn_ws = M->attn_ws;
          a.attn_out = M->attn;
          a.attn_splits = attn_splits;
          if (use_frag && attn_splits == 1) {
            a.yfrag = static_cast<__half*>(M->attn_frag);
            a.yfrag_nkb = frag_nkb_d;
          }
          pb.add(a);
        }
        GemvLaunch o;
        o.nmat = 1;
        o.mat[0].layer = M->lin[M->lin_index(static_cast<int>(l), 3)];
        o.mat[0].rung_table = table + M->lin_index(static_cast<int>(l), 3);
        o.mat[0].rung_stride = M->n_lin;
        o.x = M->attn;
        if (use_frag && attn_splits == 1 && !gemv_only) o.xfrag = M->attn_frag;
        o.x_dtype = c.act_dtype;
        o.x_stride = d;
        o.epi = EPI_RESIDUAL;
        o.resid = M->resid;
        o.resid_stride = d;
        o.out_partials = M->partials[cur ^ 1];
        o.out_n_partials = kPartStride;
        const size_t o_first = pb.phases.size();
        add_chunked(pb, o, B);
        if (attn_splits > 1) {
          if (pb.phases.size() != o_first + 1) fail(FQ_E_STATE, "split attention needs one O-projection phase");
          Phase& op = pb.phases.back();
          op.attn_splits = attn_splits;
          op.attn_ws = M->attn_ws;
          op.n_heads = static_cast<int>(c.n_heads);
          op.head_dim = static_cast<int>(c.head_dim);
        }
        cur ^= 1;
        GemvLaunch gu;
        gu.nmat = 2;
        for (int j = 0; j < 2; ++j) {
          gu.mat[j].layer = M->lin[M->lin_index(static_cast<int>(l), 4 + j)];
          gu.mat[j].rung_table = table + M->lin_index(static_cast<int>(l), 4 + j);
          gu.mat[j].rung_stride = M->n_lin;
        }
        gu.x = M->resid;
        gu.x_dtype = FQ_DT_F32;
        gu.x_stride = d;
        gu.norm_gain = M->n2g[l];
        gu.norm_partials = M->partials[cur];
        gu.n_partials = G;
        gu.partials_stride = kPartStride;
        gu.norm_eps = c.norm_eps;
        gu.act_dtype = c.act_dtype;
        gu.epi = EPI_SWIGLU;
        gu.y = M->mid;
        if (use_frag) gu.yfrag = M->mid_frag;
        gu.y_dtype = c.act_dtype;
        gu.y_stride = c.ffn_dim;
        add_chunked(pb, gu, B);
        GemvLaunch dn;
        dn.nmat = 1;
        dn.mat[0].layer = M->lin[M->lin_index(static_cast<int>(l), 6)];
        dn.mat[0].rung_table = table + M->lin_index(static_cast<int>(l), 6);
        dn.mat[0].rung_stride = M->n_lin;
        dn.x = M->mid;
        if (use_frag) dn.xfrag = M->mid_frag;
        dn.x_dtype = c.act_dtype;
        dn.x_stride = c.ffn_dim;
        dn.epi = EPI_RESIDUAL;
        dn.resid = M->resid;
        dn.resid_stride = d;
        dn.out_partials = M->partials[cur ^ 1];
        dn.out_n_partials = kPartStride;
        add_chunked(pb, dn, B);
        cur ^= 1;
      }
      GemvLaunch hd;
      hd.nmat = 1;
      hd.mat[0].layer = M->lin[M->head_index()];
      hd.mat[0].rung_table = table + M->head_index();
      hd.mat[0].rung_stride = M->n_lin;
      hd.x = M->resid;
      hd.x_dtype = FQ_DT_F32;
      hd.x_stride = d;
      hd.norm_gain = M->fng;
      hd.norm_partials = M->partials[cur];
      hd.n_partials = G;
      hd.partials_stride = kPartStride;
      hd.norm_eps = c.norm_eps;
      hd.act_dtype = c.act_dtype;
      hd.epi = EPI_STORE;
      hd.y = M->logits;
      hd.y_dtype = FQ_DT_F32;
      hd.y_stride = V;
      if (!gemv_only) hd.stat_part = M->stat_part;  // fused softmax partials (entropy / top-2 / argmax)
      add_chunked(pb, hd, B);
      if (!gemv_only) {
        Phase sp{};
        sp.type = PH_STATS;
        sp.B = B;
        sp.stats = M->stats_dev;
        sp.stat_part = M->stat_part;
        pb.add(sp);
      }
      ProgramRun run = upload_program(ctx, pb, false);
      run.pos = meta.pos;  // constant per (batch, mode): the step's row metadata lives in fixed buffers
      run.slots = meta.slots;
      run.nrows = B;
      it = M->programs.emplace(key, run).first;
    }
    FQ_CUDA(cudaMemsetAsync(M->grid_barrier, 0, sizeof(unsigned int), st));
    const bool timed = mode == STEP_DECODE && M->ev_prog[0] != nullptr;
    // inside a capture the records must be external nodes to record at replay
    const unsigned int ev_flags = capturing(st) ? cudaEventRecordExternal : cudaEventRecordDefault;
    if (timed) FQ_CUDA(cudaEventRecordWithFlags(M->ev_prog[0], st, ev_flags));
    launch_program(ctx, it->second, M->grid_barrier, false);
    if (timed) FQ_CUDA(cudaEventRecordWithFlags(M->ev_prog[1], st, ev_flags));
    return;
  }
  // ---------------- reference architecture (exact numerics)
  const int64_t ffn = c.ffn_dim;
  float* x = M->resid;
  float* h = M->hbuf;
  float* qf = static_cast<float*>(M->q);
  float* kf = static_cast<float*>(M->k);
  float* vf = static_cast<float*>(M->v);
  float* af = static_cast<float*>(M->attn);
  float* mid = static_cast<float*>(M->mid);
  float* tmp = M->tmp;
  auto gemv = [&](int li, const float* in, float* out) {
    // the rung of row b comes from the host table; exact launches are per distinct rung
    const fq_layer* L = M->lin[li];
    // all rows of a reference-arch step share the slot rung of row 0 when B == 1; for B > 1
    // rows are launched individually so each uses its own rung.
    for (int b = 0; b < B; ++b) {
      const int rung = M->table_host()[b * M->n_lin + li];
      launch_gemv_exact(ctx, L, rung, 1, in + b * L->K, FQ_DT_F32, out + b * L->N, FQ_DT_F32);
    }
  };
  embed_ref_kernel<<<B, 128, 0, st>>>(M->tok_emb, M->pos_emb, meta, d, x);
  launch_dev(M);
  const int n1 = static_cast<int>((B * d + 255) / 256), nf = static_cast<int>((B * ffn + 255) / 256);
  for (int64_t l = 0; l < c.n_layers; ++l) {
    const int base = M->lin_index(static_cast<int>(l), 0);
    layernorm_ref_kernel<<<B, 128, 0, st>>>(x, d, M->n1g[l], M->n1b[l], c.norm_eps, h);
    launch_dev(M);
    gemv(base + 0, h, qf);
    gemv(base + 1, h, kf);
    gemv(base + 2, h, vf);
    append_ref_kernel<<<B, 128, 0, st>>>(kf, vf, meta, d, static_cast<float*>(M->kv), M->slot_stride,
                                         l * M->layer_stride, c.max_seq_len);
    launch_dev(M);
    attn_ref_kernel<<<dim3(static_cast<unsigned>(c.n_heads), static_cast<unsigned>(B)), 32, 0, st>>>(
        qf, meta, static_cast<float*>(M->kv), M->slot_stride, l * M->layer_stride, c.max_seq_len,
        static_cast<int>(c.n_heads), static_cast<int>(c.head_dim), M->dscratch, af);
    launch_dev(M);
    gemv(base + 3, af, tmp);
    add_kernel<<<n1, 256, 0, st>>>(x, tmp, B * d);
    launch_dev(M);
    layernorm_ref_kernel<<<B, 128, 0, st>>>(x, d, M->n2g[l], M->n2b[l], c.norm_eps, h);
    launch_dev(M);
    gemv(base + 4, h, mid);
    gelu_ref_kernel<<<nf, 256, 0, st>>>(mid, B * ffn);
    launch_dev(M);
    gemv(base + 5, mid, tmp);
    add_kernel<<<n1, 256, 0, st>>>(x, tmp, B * d);
    launch_dev(M);
  }
  layernorm_ref_kernel<<<B, 128, 0, st>>>(x, d, M->fng, M->fnb, c.norm_eps, h);
  launch_dev(M);
  if (c.tie_embeddings) {
    for (int b = 0; b < B; ++b)
      launch_gemv_exact(ctx, &M->tied_head, FQ_RUNG_FP, 1, h + b * d, FQ_DT_F32, M->logits + b * V, FQ_DT_F32);
  } else {
    gemv(M->head_index(), h, M->logits);
  }
  if (V <= 4096) {
    row_stats_seq_kernel<<<B, 32, 0, st>>>(M->logits, V, M->dscratch, M->stats_dev);
  } else {
    row_stats_kernel<<<B, 1024, 0, st>>>(M->logits, V, M->stats_dev);
  }
  FQ_CUDA(cudaGetLastError());
  launch_dev(M);
}

// Runs one step for B rows whose metadata is staged in meta_host; results in stats_host.
void run_step(fq_model* M, int B) {
  fq_ctx* ctx = M->ctx;
  cudaStream_t st = ctx->stream;
  // reference-arch steps launch per-row exact GEMVs whose rung is read on the host: no graph
  const bool graphable = M->llama && M->use_graphs;
  if (!graphable) {
    FQ_CUDA(cudaMemcpyAsync(M->meta_dev, M->meta_host, M->meta_bytes, cudaMemcpyHostToDevice, st));
    enqueue_step(M, B);
    FQ_CUDA(cudaMemcpyAsync(M->stats_host, M->stats_dev, sizeof(fq_row_stats) * B, cudaMemcpyDeviceToHost, st));
    FQ_CUDA(cudaStreamSynchronize(st));
    return;
  }
  sync_weight_epoch(M);
  auto it = M->graphs.find(B);
  if (it == M->graphs.end()) {
    if (M->programs.find(std::make_pair(B, 0)) == M->programs.end()) {
      // first use: build + upload the step program (allocates) and run the step un-captured
      FQ_CUDA(cudaMemcpyAsync(M->meta_dev, M->meta_host, M->meta_bytes, cudaMemcpyHostToDevice, st));
      enqueue_step(M, B);
      FQ_CUDA(cudaMemcpyAsync(M->stats_host, M->stats_dev, sizeof(fq_row_stats) * B, cudaMemcpyDeviceToHost, st));
      FQ_CUDA(cudaStreamSynchronize(st));
      return;
    }
    cudaGraph_t graph;
    const int64_t l0 = ctx->launches;
    FQ_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    try {
      FQ_CUDA(cudaMemcpyAsync(M->meta_dev, M->meta_host, M->meta_bytes, cudaMemcpyHostToDevice, st));
      enqueue_step(M, B);
      FQ_CUDA(cudaMemcpyAsync(M->stats_host, M->stats_dev, sizeof(fq_row_stats) * B, cudaMemcpyDeviceToHost, st));
    } catch (...) {
      cudaStreamEndCapture(st, &graph);
      throw;
    }
    FQ_CUDA(cudaStreamEndCapture(st, &graph));
    cudaGraphExec_t exec;
    FQ_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    FQ_CUDA(cudaGraphDestroy(graph));
    it = M->graphs.emplace(B, exec).first;
    M->graph_kernels[B] = ctx->launches - l0;
    ctx->launches = l0;  // counted when replayed
  }
  FQ_CUDA(cudaGraphLaunch(it->second, st));
  ctx->launches += M->graph_kernels[B];
  FQ_CUDA(cudaStreamSynchronize(st));
  if (M->ev_prog[0]) {
    float ms = 0.f;
    const cudaError_t e = cudaEventElapsedTime(&ms, M->ev_prog[0], M->ev_prog[1]);
    if (e == cudaSuccess) {
      M->prog_ms += ms;
      M->prog_steps += 1;
    } else {
      cudaGetLastError();  // not sticky: keep it out of the next launch check
      static bool once = false;
      if (!once && std::getenv("FQ_DEBUG_TIMING")) {
        std::fprintf(stderr, "fq: step timing unavailable: %s\n", cudaGetErrorString(e));
        once = true;
      }
    }
  }
}

int64_t ffn_or_d(const fq_model_config& c) { return std::max(c.d_model, c.ffn_dim); }

void stage_rows(fq_model* M, int B, const int32_t* slots, const int32_t* tokens) {
  const fq_model_config& c = M->cfg;
  int32_t* tok = reinterpret_cast<int32_t*>(M->meta_host);
  int32_t* pos = tok + M->rows;
  int32_t* sl = pos + M->rows;
  uint8_t* tab = M->table_host();
  for (int b = 0; b < B; ++b) {
    const int s = slots[b];
    require(s >= 0 && s < c.max_batch, FQ_E_INPUT, "decode: slot out of range");
    require(tokens[b] >= 0 && tokens[b] < c.vocab_size, FQ_E_INPUT, "decode: token id out of vocabulary");
    if (M->slot_len[s] >= c.max_seq_len) fail(FQ_E_CAPACITY, "decode: cache is full");
    for (int b2 = 0; b2 < b; ++b2) require(slots[b2] != s, FQ_E_INPUT, "decode: duplicate slot in a batch");
    tok[b] = tokens[b];
    pos[b] = static_cast<int32_t>(M->slot_len[s]);
    sl[b] = s;
    std::memcpy(tab + b * M->n_lin, &M->rungs[static_cast<size_t>(s) * M->n_lin], M->n_lin);
    for (int i = 0; i < M->n_lin; ++i)
      if (!M->lin[i]->has(tab[b * M->n_lin + i]))
        fail(FQ_E_STATE, "layer " + M->ids[i] + ": active precision has no payload");
  }
}

void ensure_prefill_ws(fq_model* M, int64_t T);

// ---------------------------------------------------------------- batched decode (tensor cores)
// B >= batch_gemm_min() rows of a llama model (BASELINE C5): the step runs as row-parallel kernels
// and one tcgen05 GEMM per (linear, precision copy present in the batch) -- every resident copy is
// streamed at most once per step, however the rows' precision tables mix (batched.cu).
int batch_gemm_min() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("FQ_BATCH_GEMM_MIN");
    v = e ? std::max(1, std::atoi(e)) : 16;
  }
  return v;
}

bool batched_gemm_usable(const fq_model* M, int B) {
  if (!M->llama || B < batch_gemm_min()) return false;
  const fq_model_config& c = M->cfg;
  if (c.head_dim != 64 && c.head_dim != 128) return false;
  if (c.d_model % 8 != 0 || c.ffn_dim % 8 != 0) return false;
  return true;
}

// Enqueues one batched step for the B rows staged in meta_dev (tokens / pos / slots / rung table);
// `present[i]` = bit r set when some row runs linear i at rung r.
void batched_step_enqueue(fq_model* M, int B, const std::vector<uint8_t>& present) {
  fq_ctx* ctx = M->ctx;
  const fq_model_config& c = M->cfg;
  auto& w = M->pw;
  const int64_t d = c.d_model, f = c.ffn_dim, V = c.vocab_size;
  const int H = static_cast<int>(c.n_heads), hd = static_cast<int>(c.head_dim);
  const int ad = c.act_dtype;
  const StepMeta mt = M->meta(B);
  const uint8_t* table = M->table_dev();
  const int64_t nl = M->n_lin;
  // one product per copy present among the rows of linear i, each writing only its rows; the
  // products of linears that read the same activations go to one grouped launch (gemm_tc.cu)
  std::vector<GemmJob> jobs;
  auto add = [&](int i, float* y, int64_t ys, bool acc) {
    for (int r = FQ_RUNG_INT8; r <= FQ_RUNG_INT4; ++r)
      if (present[static_cast<size_t>(i)] & (1u << r)) jobs.push_back(GemmJob{M->lin[i], r, y, ys, acc, table + i, nl});
  };
  auto run = [&](const void* xt) {
    for (size_t j = 0; j < jobs.size(); j += 8)
      launch_gemm_group(ctx, jobs.data() + j, static_cast<int>(std::min<size_t>(8, jobs.size() - j)), B, xt);
    jobs.clear();
  };
  auto linear = [&](int i, const void* xt, float* y, int64_t ys, bool acc) {
    add(i, y, ys, acc);
    run(xt);
  };
  prefill_embed(ctx, M->tok_emb, mt.tokens, B, d, w.x);
  for (int l = 0; l < c.n_layers; ++l) {
    const int b0 = M->lin_index(l, 0);
    const int64_t lo = static_cast<int64_t>(l) * M->layer_stride;
    prefill_rmsnorm(ctx, w.x, B, d, M->n1g[l], c.norm_eps, w.h, ad);
    add(b0 + 0, w.q, d, false);
    add(b0 + 1, w.k, d, false);
    add(b0 + 2, w.v, d, false);
    run(w.h);
    batched_rope_append(ctx, w.q, w.k, w.v, B, H, hd, M->rope_cs, mt.pos, mt.slots, static_cast<__half*>(M->kv),
                        M->slot_stride, lo, c.max_seq_len, w.qr, ad);
    batched_attention(ctx, w.qr, static_cast<const __half*>(M->kv), B, H, hd, mt.pos, mt.slots, M->slot_stride, lo,
                      c.max_seq_len, w.a, ad);
    linear(b0 + 3, w.a, w.x, d, true);  // x += attn . Wo^T
    prefill_rmsnorm(ctx, w.x, B, d, M->n2g[l], c.norm_eps, w.h, ad);
    add(b0 + 4, w.g, f, false);
    add(b0 + 5, w.u, f, false);
    run(w.h);
    prefill_swiglu(ctx, w.g, w.u, static_cast<int64_t>(B) * f, f, w.m, ad);
    linear(b0 + 6, w.m, w.x, d, true);  // x += mid . Wdown^T
  }
  prefill_rmsnorm(ctx, w.x, B, d, M->fng, c.norm_eps, w.h, ad);
  linear(M->head_index(), w.h, M->logits, V, false);
  launch_softmax_stats(ctx, M->logits, B, V, V, M->stats_dev);
}

// One batched step.  The launch sequence depends only on B and on which copies each linear needs
// (it changes at switch events), so it is captured once per such signature into a CUDA graph and
// replayed; the first step of a signature runs uncaptured (it sizes the workspaces).
void batched_step(fq_model* M, int B) {
  fq_ctx* ctx = M->ctx;
  cudaStream_t st = ctx->stream;
  sync_weight_epoch(M);
  ensure_prefill_ws(M, B);
  std::string sig(static_cast<size_t>(M->n_lin), '\0');
  const uint8_t* tab = M->table_host();
  for (int b = 0; b < B; ++b)
    for (int i = 0; i < M->n_lin; ++i) sig[static_cast<size_t>(i)] |= static_cast<char>(1u << tab[b * M->n_lin + i]);
  const std::vector<uint8_t> present(sig.begin(), sig.end());
  sig += "|" + std::to_string(B);
  auto enqueue = [&] {
    FQ_CUDA(cudaMemcpyAsync(M->meta_dev, M->meta_host, M->meta_bytes, cudaMemcpyHostToDevice, st));
    batched_step_enqueue(M, B, present);
    FQ_CUDA(cudaMemcpyAsync(M->stats_host, M->stats_dev, sizeof(fq_row_stats) * B, cudaMemcpyDeviceToHost, st));
  };
  auto it = M->batch_graphs.find(sig);
  if (!M->use_graphs || (it == M->batch_graphs.end() && !M->batch_seen.count(sig))) {
    M->batch_seen.insert(sig);
    enqueue();
  } else {
    if (it == M->batch_graphs.end()) {
      if (M->batch_graphs.size() >= 8) {  // a few live signatures at a time
        cudaGraphExecDestroy(M->batch_graphs.begin()->second.first);
        M->batch_graphs.erase(M->batch_graphs.begin());
      }
      cudaGraph_t graph;
      const int64_t l0 = ctx->launches;
      FQ_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      try {
        enqueue();
      } catch (...) {
        cudaStreamEndCapture(st, &graph);
        throw;
      }
      FQ_CUDA(cudaStreamEndCapture(st, &graph));
      cudaGraphExec_t exec;
      FQ_CUDA(cudaGraphInstantiate(&exec, graph, 0));
      FQ_CUDA(cudaGraphDestroy(graph));
      it = M->batch_graphs.emplace(sig, std::make_pair(exec, ctx->launches - l0)).first;
      ctx->launches = l0;
    }
    FQ_CUDA(cudaGraphLaunch(it->second.first, st));
    ctx->launches += it->second.second;
  }
  FQ_CUDA(cudaStreamSynchronize(st));
  if (prefill_overflow_take(ctx)) fail(FQ_E_INPUT, "decode: an activation exceeds fp16's range (GEMM operand format)");
}

void model_step(fq_model* M, int B, const int32_t* slots, const int32_t* tokens, float* logits_dev,
                fq_row_stats* stats_host) {
  require(B >= 1 && B <= M->cfg.max_batch, FQ_E_INPUT, "decode: batch out of range");
  require(!M->tp(), FQ_E_STATE, "tensor-parallel rank: decode through fq_model_tp_begin / fq_model_tp_segment");
  if (M->llama) {
    for (int i = 0; i < M->n_lin; ++i) {
      require(gemv_fast_supported(M->lin[i], FQ_RUNG_INT8) || !M->lin[i]->has(FQ_RUNG_INT8), FQ_E_STATE,
              "layer " + M->ids[i] + ": W8 copy not usable by the fast kernel");
      require(gemv_fast_supported(M->lin[i], FQ_RUNG_INT4) || !M->lin[i]->has(FQ_RUNG_INT4), FQ_E_STATE,
              "layer " + M->ids[i] + ": W4 copy not usable by the fast kernel");
    }
  }
  stage_rows(M, B, slots, tokens);
  M->chain_slot = -1;
  if (batched_gemm_usable(M, B)) batched_step(M, B);
  else run_step(M, B);
  for (int b = 0; b < B; ++b) M->slot_len[slots[b]] += 1;
  if (B == 1 && M->llama) M->chain_slot = slots[0];
  if (stats_host) std::memcpy(stats_host, M->stats_host, sizeof(fq_row_stats) * B);
  if (logits_dev)
    FQ_CUDA(cudaMemcpyAsync(logits_dev, M->logits, sizeof(float) * B * M->cfg.vocab_size, cudaMemcpyDeviceToDevice,
                            M->ctx->stream));
}

// One llama prefill step: R consecutive prompt positions of `slot` as the rows of a prefill
// program (append phase, then causal attention over the cache).
void prefill_step(fq_model* M, int slot, const int32_t* tokens, int R, float* logits_dev, fq_row_stats* stats_host) {
  const fq_model_config& c = M->cfg;
  M->chain_slot = -1;
  int32_t* tok = reinterpret_cast<int32_t*>(M->meta_host);
  int32_t* pos = tok + M->rows;
  int32_t* sl = pos + M->rows;
  uint8_t* tab = M->table_host();
  if (M->slot_len[slot] + R > c.max_seq_len) fail(FQ_E_CAPACITY, "prefill: cache is full");
  for (int b = 0; b < R; ++b) {
    tok[b] = tokens[b];
    pos[b] = static_cast<int32_t>(M->slot_len[slot] + b);
    sl[b] = slot;
    std::memcpy(tab + b * M->n_lin, &M->rungs[static_cast<size_t>(slot) * M->n_lin], M->n_lin);
  }
  for (int i = 0; i < M->n_lin; ++i)
    if (!M->lin[i]->has(tab[i])) fail(FQ_E_STATE, "layer " + M->ids[i] + ": active precision has no payload");
  fq_ctx* ctx = M->ctx;
  cudaStream_t st = ctx->stream;
  FQ_CUDA(cudaMemcpyAsync(M->meta_dev, M->meta_host, M->meta_bytes, cudaMemcpyHostToDevice, st));
  enqueue_step(M, R, STEP_PREFILL);
  FQ_CUDA(cudaMemcpyAsync(M->stats_host, M->stats_dev, sizeof(fq_row_stats) * R, cudaMemcpyDeviceToHost, st));
  FQ_CUDA(cudaStreamSynchronize(st));
  M->slot_len[slot] += R;
  if (stats_host) std::memcpy(stats_host, M->stats_host, sizeof(fq_row_stats) * R);
  if (logits_dev)
    FQ_CUDA(cudaMemcpyAsync(logits_dev, M->logits, sizeof(float) * R * c.vocab_size, cudaMemcpyDeviceToDevice, st));
}

// ---------------------------------------------------------------- tensor-core prefill (llama)
// A prompt of T tokens goes through each block as T rows at once: the seven linears and the head
// on the tcgen05 dequant-GEMM (gemm_tc.cu, weights read once per 256 rows instead of once per
// 8), norms / RoPE + cache append / causal attention / SwiGLU on the row kernels of prefill.cu.
// Same arithmetic contract as the decode program; used for prompts of at least
// gemm_prefill_min() tokens (env FQ_GEMM_PREFILL_MIN, 0 = off) when every linear's active rung
// is W8/W4 in the tiled layout and activations are bf16.

int64_t gemm_prefill_min() {
  static const int64_t v = [] {
    const char* e = std::getenv("FQ_GEMM_PREFILL_MIN");
    return e ? static_cast<int64_t>(std::atoll(e)) : static_cast<int64_t>(16);
  }();
  return v;
}

bool gemm_prefill_usable(const fq_model* M, int slot, int64_t T) {
  const fq_model_config& c = M->cfg;
  const int64_t lo = gemm_prefill_min();
  if (!M->llama || lo <= 0 || T < lo || (c.act_dtype != FQ_DT_BF16 && c.act_dtype != FQ_DT_F16)) return false;
  if (c.d_model % 8 != 0 || c.ffn_dim % 8 != 0) return false;
  for (int i = 0; i < M->n_lin; ++i) {
    const int r = M->rungs[static_cast<size_t>(slot) * M->n_lin + i];
    if (r != FQ_RUNG_INT8 && r != FQ_RUNG_INT4) return false;
    const fq_rung_store& st = M->lin[i]->store(r);
    if (!st.present || st.tiles == nullptr) return false;
  }
  return true;
}

void free_prefill_ws(fq_model* M) {
  auto& w = M->pw;
  for (void* p : {static_cast<void*>(w.x), static_cast<void*>(w.q), static_cast<void*>(w.k), static_cast<void*>(w.v),
                  static_cast<void*>(w.qr), static_cast<void*>(w.g), static_cast<void*>(w.u),
                  static_cast<void*>(w.logits), w.h, w.a, w.m, static_cast<void*>(w.stats), static_cast<void*>(w.tok)})
    dfree(p);
  w = fq_model::PrefillWs{};
}

void ensure_prefill_ws(fq_model* M, int64_t T) {
  auto& w = M->pw;
  if (T <= w.cap) return;
  // the batched decode step's captured graphs run on these buffers: drop them with the buffers
  if (!M->batch_graphs.empty()) {
    FQ_CUDA(cudaStreamSynchronize(M->ctx->stream));
    for (auto& kv : M->batch_graphs) cudaGraphExecDestroy(kv.second.first);
    M->batch_graphs.clear();
    M->batch_seen.clear();
  }
  free_prefill_ws(M);
  const fq_model_config& c = M->cfg;
  const int64_t cap = std::min<int64_t>(c.max_seq_len, (T + 63) / 64 * 64);
  const int64_t d = c.d_model, f = c.ffn_dim, V = c.vocab_size;
  auto f32 = [&](int64_t n) { return static_cast<float*>(dmalloc(sizeof(float) * n)); };
  w.x = f32(cap * d);
  w.q = f32(cap * d);
  w.k = f32(cap * d);
  w.v = f32(cap * d);
  w.qr = f32(cap * d);
  w.g = f32(cap * f);
  w.u = f32(cap * f);
  w.logits = f32(cap * V);
  // GEMM inputs: tiled bf16 (tiled_act_offset), zero-filled so the padding rows / columns are 0
  auto tiled = [&](int64_t K) {
    const size_t bytes = 2 * static_cast<size_t>(tiled_act_elems(cap, K));
    void* p = dmalloc(bytes);
    FQ_CUDA(cudaMemset(p, 0, bytes));
    return p;
  };
  w.h = tiled(d);
  w.a = tiled(d);
  w.m = tiled(f);
  w.stats = static_cast<fq_row_stats*>(dmalloc(sizeof(fq_row_stats) * cap));
  w.tok = static_cast<int32_t*>(dmalloc(sizeof(int32_t) * cap));
  w.cap = cap;
}

// Enqueues the whole prefill of `slot` (cache rows 0..T-1).  logits_out: [T, V] fp32 (null = the
// workspace); stats_dev: [T] row statistics (null = none).  Does not synchronise.
// first_layer / snap (the calibration's block reuse): with snap, record = true copies the residual
// stream entering every block into snap[l] ([n_layers][T][d] fp32); first_layer > 0 resumes from
// snap[first_layer] -- the blocks below it are bit-identical to the recorded forward's
void prefill_gemm_enqueue(fq_model* M, int slot, const int32_t* tokens_host, int64_t T, float* logits_out,
                          fq_row_stats* stats_dev, int first_layer = 0, float* snap = nullptr, bool record = false) {
  fq_ctx* ctx = M->ctx;
  const fq_model_config& c = M->cfg;
  cudaStream_t st = ctx->stream;
  ensure_prefill_ws(M, T);
  auto& w = M->pw;
  const int64_t d = c.d_model, f = c.ffn_dim, V = c.vocab_size;
  const int H = static_cast<int>(c.n_heads), hd = static_cast<int>(c.head_dim);
  const int Ti = static_cast<int>(T);
  const uint8_t* r = &M->rungs[static_cast<size_t>(slot) * M->n_lin];
  const int ad = c.act_dtype;  // bf16 or fp16 roundings; the GEMM operands are stored fp16 (exact)
  const size_t xbytes = sizeof(float) * static_cast<size_t>(T) * d;
  if (first_layer > 0) {
    FQ_CUDA(cudaMemcpyAsync(w.x, snap + static_cast<size_t>(first_layer) * T * d, xbytes, cudaMemcpyDeviceToDevice, st));
  } else {
    FQ_CUDA(cudaMemcpyAsync(w.tok, tokens_host, sizeof(int32_t) * T, cudaMemcpyHostToDevice, st));
    prefill_embed(ctx, M->tok_emb, w.tok, Ti, d, w.x);
  }
  __half* kv_slot = static_cast<__half*>(M->kv) + static_cast<int64_t>(slot) * M->slot_stride;
  for (int l = first_layer; l < c.n_layers; ++l) {
    if (record && snap != nullptr)
      FQ_CUDA(cudaMemcpyAsync(snap + static_cast<size_t>(l) * T * d, w.x, xbytes, cudaMemcpyDeviceToDevice, st));
    const int b = M->lin_index(l, 0);
    __half* kvl = kv_slot + static_cast<int64_t>(l) * M->layer_stride;
    prefill_rmsnorm(ctx, w.x, Ti, d, M->n1g[l], c.norm_eps, w.h, ad);
    {  // q, k, v read the same activations: one grouped launch (gemm_tc.cu)
      const GemmJob qkv[3] = {{M->lin[b + 0], r[b + 0], w.q, d, false, nullptr, 0},
                              {M->lin[b + 1], r[b + 1], w.k, d, false, nullptr, 0},
                              {M->lin[b + 2], r[b + 2], w.v, d, false, nullptr, 0}};
      launch_gemm_group(ctx, qkv, 3, T, w.h);
    }
    prefill_rope_kv(ctx, w.q, w.k, w.v, Ti, H, hd, M->rope_cs, w.qr, kvl, c.max_seq_len, ad);
    // causal attention of the prompt rows: 32 keys per warp round (batched.cu)
    batched_attention(ctx, w.qr, static_cast<const __half*>(M->kv), Ti, H, hd, nullptr, nullptr, M->slot_stride,
                      static_cast<int64_t>(l) * M->layer_stride, c.max_seq_len, w.a, ad, slot);
    launch_gemm_dq(ctx, M->lin[b + 3], r[b + 3], T, w.a, FQ_DT_F16, w.x, d, true);  // x += attn . Wo^T
    prefill_rmsnorm(ctx, w.x, Ti, d, M->n2g[l], c.norm_eps, w.h, ad);
    {
      const GemmJob gu[2] = {{M->lin[b + 4], r[b + 4], w.g, f, false, nullptr, 0},
                             {M->lin[b + 5], r[b + 5], w.u, f, false, nullptr, 0}};
      launch_gemm_group(ctx, gu, 2, T, w.h);
    }
    prefill_swiglu(ctx, w.g, w.u, T * f, f, w.m, ad);
    launch_gemm_dq(ctx, M->lin[b + 6], r[b + 6], T, w.m, FQ_DT_F16, w.x, d, true);  // x += mid . Wdown^T
  }
  prefill_rmsnorm(ctx, w.x, Ti, d, M->fng, c.norm_eps, w.h, ad);
  float* lg = logits_out ? logits_out : w.logits;
  const int hi = M->head_index();
  launch_gemm_dq(ctx, M->lin[hi], r[hi], T, w.h, FQ_DT_F16, lg, V);
  if (stats_dev) launch_softmax_stats(ctx, lg, T, V, V, stats_dev);
}

void prefill_gemm(fq_model* M, int slot, const int32_t* tokens, int64_t T, float* logits_dev, fq_row_stats* stats_host) {
  if (T > M->cfg.max_seq_len) fail(FQ_E_CAPACITY, "prefill: cache is full");
  ensure_prefill_ws(M, T);
  prefill_gemm_enqueue(M, slot, tokens, T, logits_dev, stats_host ? M->pw.stats : nullptr);
  if (stats_host)
    FQ_CUDA(cudaMemcpyAsync(stats_host, M->pw.stats, sizeof(fq_row_stats) * T, cudaMemcpyDeviceToHost, M->ctx->stream));
  FQ_CUDA(cudaStreamSynchronize(M->ctx->stream));
  if (prefill_overflow_take(M->ctx))
    fail(FQ_E_INPUT, "prefill: an activation exceeds fp16's range (the tcgen05 GEMM operand format)");
  M->slot_len[slot] = T;
}

// ---------------------------------------------------------------- tensor-parallel step (variant)
// A TP rank's decode step is 2L + 1 segments, each one step-program launch; between segments the
// caller sums the ranks' fp32 partials (NCCL all-reduce over NVLink) and hands the sum to the next
// segment, which adds it to the replicated residual:
//   segment 2l     : [embed | resid += sum] -> RMSNorm + q/k/v of the rank's heads -> RoPE +
//                    KV append + attention of those heads -> O projection (its input columns) ->
//                    fp32 partial [B, d]
//   segment 2l + 1 : resid += sum -> RMSNorm + gate/up of the rank's ffn columns -> SwiGLU -> down
//                    projection (its input columns) -> fp32 partial [B, d]
//   segment 2L     : resid += sum -> final RMSNorm + head rows of the rank's vocab slice -> fused
//                    softmax partials merged over the grid -> fq_stat_part [B] (the host merges the
//                    ranks' partials: fq_tp_merge_stats)
// The unsplit block is src/model.cpp:201-233; the statistics src/scheduler.cpp:13-49.
void add_resid_phase(ProgramBuilder& pb, fq_model* M, int B, const float* reduced, const StepMeta& meta) {
  Phase e{};
  e.type = PH_EMBED;
  e.barrier_after = 1;
  e.B = B;
  e.tok_emb = reduced ? nullptr : M->tok_emb;
  e.x = reduced;
  e.tokens = meta.tokens;
  e.d = M->cfg.d_model;
  e.resid = M->resid;
  e.resid_stride = M->cfg.d_model;
  e.out_partials = M->partials[0];
  e.out_partials_stride = kPartStride;
  pb.add(e);
}

ProgramRun& tp_program(fq_model* M, int B, int seg, const float* reduced, void* out) {
  // programs bake the exchange buffers in: cached per (batch, segment, buffers)
  const int key_mode = 1000 + seg;
  auto key = std::make_pair(B, key_mode);
  auto it = M->programs.find(key);
  if (it != M->programs.end() && it->second.tp_in == reduced && it->second.tp_out == out) return it->second;
  if (it != M->programs.end()) {
    FQ_CUDA(cudaStreamSynchronize(M->ctx->stream));
    dfree(it->second.dev_phases);
    M->programs.erase(it);
  }
  fq_ctx* ctx = M->ctx;
  const fq_model_config& c = M->cfg;
  const int64_t d = c.d_model, L = c.n_layers;
  const StepMeta meta = M->meta(B);
  const uint8_t* table = M->table_dev();
  ProgramBuilder pb;
  pb.grid = ctx->num_sms;
  const int G = pb.grid;
  add_resid_phase(pb, M, B, seg == 0 ? nullptr : reduced, meta);
  const int frag_nkb_q = static_cast<int>((M->q_dim + kBlockK - 1) / kBlockK);
  auto norm_in = [&](GemvLaunch& g, const float* gain) {
    g.x = M->resid;
    g.x_dtype = FQ_DT_F32;
    g.x_stride = d;
    g.norm_gain = gain;
    g.norm_partials = M->partials[0];
    g.n_partials = G;
    g.partials_stride = kPartStride;
    g.norm_eps = c.norm_eps;
    g.act_dtype = c.act_dtype;
  };
  auto lin = [&](GemvLaunch& g, int m, int index) {
    g.mat[m].layer = M->lin[index];
    g.mat[m].rung_table = table + index;
    g.mat[m].rung_stride = M->n_lin;
  };
  if (seg < 2 * L && seg % 2 == 0) {
    const int l = seg / 2;
    GemvLaunch g;
    g.nmat = 3;
    for (int j = 0; j < 3; ++j) lin(g, j, M->lin_index(l, j));
    g.mat[0].y = M->q;
    g.mat[1].y = M->k;
    g.mat[2].y = M->v;
    norm_in(g, M->n1g[l]);
    g.epi = EPI_SPLIT3;
    g.y_dtype = c.act_dtype;
    g.y_stride = M->q_dim;
    add_chunked(pb, g, B);
    Phase a{};
    a.type = PH_ATTN;
    a.barrier_after = 1;
    a.B = B;
    a.q = M->q;
    a.k = M->k;
    a.v = M->v;
    a.act_dtype = c.act_dtype;
    a.pos = meta.pos;
    a.slots = meta.slots;
    a.kv = static_cast<__half*>(M->kv);
    a.slot_stride = M->slot_stride;
    a.layer_off = l * M->layer_stride;
    a.max_seq = c.max_seq_len;
    a.n_heads = static_cast<int>(M->sh.heads);
    a.head_dim = static_cast<int>(c.head_dim);
    a.rope_cs = M->rope_cs;
    a.attn_ws = M->attn_ws;
    a.attn_out = M->attn;
    a.attn_splits = 1;
    if (B <= kMaxB) {
      a.yfrag = static_cast<__half*>(M->attn_frag);
      a.yfrag_nkb = frag_nkb_q;
    }
    pb.add(a);
    GemvLaunch o;
    o.nmat = 1;
    lin(o, 0, M->lin_index(l, 3));
    o.x = M->attn;
    if (B <= kMaxB) o.xfrag = M->attn_frag;
    o.x_dtype = c.act_dtype;
    o.x_stride = M->q_dim;
    o.epi = EPI_STORE;
    o.y = out;
    o.y_dtype = FQ_DT_F32;
    o.y_stride = d;
    add_chunked(pb, o, B);
  } else if (seg < 2 * L) {
    const int l = seg / 2;
    GemvLaunch gu;
    gu.nmat = 2;
    for (int j = 0; j < 2; ++j) lin(gu, j, M->lin_index(l, 4 + j));
    norm_in(gu, M->n2g[l]);
    gu.epi = EPI_SWIGLU;
    gu.y = M->mid;
    if (B <= kMaxB) gu.yfrag = M->mid_frag;
    gu.y_dtype = c.act_dtype;
    gu.y_stride = M->sh.ffn;
    add_chunked(pb, gu, B);
    GemvLaunch dn;
    dn.nmat = 1;
    lin(dn, 0, M->lin_index(l, 6));
    dn.x = M->mid;
    if (B <= kMaxB) dn.xfrag = M->mid_frag;
    dn.x_dtype = c.act_dtype;
    dn.x_stride = M->sh.ffn;
    dn.epi = EPI_STORE;
    dn.y = out;
    dn.y_dtype = FQ_DT_F32;
    dn.y_stride = d;
    add_chunked(pb, dn, B);
  } else {
    GemvLaunch hd;
    hd.nmat = 1;
    lin(hd, 0, M->head_index());
    norm_in(hd, M->fng);
    hd.epi = EPI_STORE;
    hd.y = M->logits;
    hd.y_dtype = FQ_DT_F32;
    hd.y_stride = M->sh.vocab;
    hd.stat_part = M->stat_part;
    add_chunked(pb, hd, B);
    Phase sp{};
    sp.type = PH_STATS;
    sp.B = B;
    sp.stats = M->stats_dev;
    sp.stat_part = M->stat_part;
    sp.y = out;  // merged partial per row (fq_stat_part), not the final statistics
    pb.add(sp);
  }
  pb.phases.back().barrier_after = 0;
  ProgramRun run = upload_program(ctx, pb, false);
  run.pos = meta.pos;
  run.slots = meta.slots;
  run.nrows = B;
  run.tp_in = reduced;
  run.tp_out = out;
  return M->programs.emplace(key, run).first->second;
}

__global__ void advance_pos_kernel(int32_t* pos) { pos[0] += 1; }
__global__ void collect_stats_kernel(const fq_row_stats* stats, fq_row_stats* ring, unsigned int* count) {
  ring[*count] = stats[0];
  *count += 1;
}

float* param_slot(fq_model* M, const std::string& name, int64_t& expect) {
  const fq_model_config& c = M->cfg;
  const int64_t d = c.d_model;
  if (name == "tok_emb") { expect = c.vocab_size * d; return M->tok_emb; }
  if (!M->llama && name == "pos_emb") { expect = c.max_seq_len * d; return M->pos_emb; }
  if (M->llama && name == "final_norm") { expect = d; return M->fng; }
  if (!M->llama && name == "final_norm.gamma") { expect = d; return M->fng; }
  if (!M->llama && name == "final_norm.beta") { expect = d; return M->fnb; }
  if (name.rfind("blocks.", 0) == 0) {
    const size_t dot = name.find('.', 7);
    if (dot == std::string::npos) return nullptr;
    const int64_t i = std::stoll(name.substr(7, dot - 7));
    if (i < 0 || i >= c.n_layers) return nullptr;
    const std::string rest = name.substr(dot + 1);
    expect = d;
    if (M->llama) {
      if (rest == "attn_norm") return M->n1g[i];
      if (rest == "ffn_norm") return M->n2g[i];
    } else {
      if (rest == "ln1.gamma") return M->n1g[i];
      if (rest == "ln1.beta") return M->n1b[i];
      if (rest == "ln2.gamma") return M->n2g[i];
      if (rest == "ln2.beta") return M->n2b[i];
    }
  }
  return nullptr;
}

__global__ void fill_kernel(float* p, int64_t n, float v) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

}  // namespace mdl
}  // namespace fqc

using namespace fqc::mdl;

extern "C" {

fq_status fq_model_create(fq_ctx* ctx, const fq_model_config* cfg, fq_model** out) {
  return fq_model_create_tp(ctx, cfg, 0, 1, out);
}

fq_status fq_model_create_tp(fq_ctx* ctx, const fq_model_config* cfg, int32_t tp_rank, int32_t tp_size, fq_model** out) {
  return guarded([&] {
    require(ctx && cfg && out, FQ_E_INPUT, "null argument");
    const fq_model_config& c = *cfg;
    if (c.vocab_size < 1 || c.d_model < 1 || c.n_heads < 1 || c.head_dim < 1 || c.n_layers < 1 || c.ffn_dim < 1 ||
        c.max_seq_len < 1)
      fail(FQ_E_CONFIG, "model config: all dimensions must be >= 1");
    if (c.d_model != c.n_heads * c.head_dim) fail(FQ_E_CONFIG, "model config: d_model must equal n_heads * head_dim");
    fq_tp_shard sh{};
    if (fq_tp_shard_spec(cfg, tp_rank, tp_size, &sh) != FQ_OK) fail(FQ_E_CONFIG, fq_last_error());
    require(tp_size == 1 || c.arch == FQ_ARCH_LLAMA, FQ_E_CONFIG, "tensor parallel: llama arch only");
    require(c.arch == FQ_ARCH_LLAMA || c.arch == FQ_ARCH_REFERENCE, FQ_E_CONFIG, "model config: unknown arch");
    require(c.max_batch >= 1 && c.max_batch <= 256, FQ_E_CONFIG, "model config: max_batch must be in [1, 256]");
    if (c.arch == FQ_ARCH_LLAMA) {
      require(c.act_dtype == FQ_DT_BF16 || c.act_dtype == FQ_DT_F16, FQ_E_CONFIG, "llama arch: activations must be bf16/fp16");
      require(c.head_dim == 64 || c.head_dim == 128, FQ_E_CONFIG, "llama arch: head_dim must be 64 or 128");
      require(!c.tie_embeddings, FQ_E_CONFIG, "llama arch: tied embeddings not supported");
    } else {
      require(c.act_dtype == FQ_DT_F32, FQ_E_CONFIG, "reference arch: activations are fp32");
    }
    auto* M = new fq_model();
    M->ctx = ctx;
    M->cfg = c;
    M->llama = c.arch == FQ_ARCH_LLAMA;
    M->sh = sh;
    M->q_dim = sh.heads * c.head_dim;
    const int64_t d = c.d_model, ffn = c.ffn_dim, V = c.vocab_size, L = c.n_layers;
    const int64_t qd = M->q_dim, fl = sh.ffn, vl = sh.vocab;  // this rank's shard (== full without TP)
    const int per = M->llama ? 7 : 6;
    for (int64_t i = 0; i < L; ++i) {
      const std::string p = "blocks." + std::to_string(i) + ".";
      std::vector<std::pair<std::string, std::pair<int64_t, int64_t>>> specs;
      // column split: q/k/v/gate/up keep their rows of the rank's heads / ffn columns; row split:
      // o/down keep the matching input columns (model.cpp:201-233 is the unsplit block)
      specs.push_back({p + "attn.wq", {qd, d}});
      specs.push_back({p + "attn.wk", {qd, d}});
      specs.push_back({p + "attn.wv", {qd, d}});
      specs.push_back({p + "attn.wo", {d, qd}});
      if (M->llama) {
        specs.push_back({p + "ffn.w_gate", {fl, d}});
        specs.push_back({p + "ffn.w_up", {fl, d}});
        specs.push_back({p + "ffn.w_down", {d, fl}});
      } else {
        specs.push_back({p + "ffn.w1", {ffn, d}});
        specs.push_back({p + "ffn.w2", {d, ffn}});
      }
      for (auto& sp : specs) {
        fq_layer* lay = nullptr;
        FQ_CUDA(cudaSuccess);
        if (fq_layer_create(ctx, sp.second.first, sp.second.second, c.group_size, &lay) != FQ_OK)
          fail(FQ_E_CONFIG, fq_last_error());
        lay->borrowed = true;
        M->ids.push_back(sp.first);
        M->lin.push_back(lay);
      }
    }
    (void)per;
    if (!(c.arch == FQ_ARCH_REFERENCE && c.tie_embeddings)) {
      fq_layer* lay = nullptr;
      if (fq_layer_create(ctx, vl, d, c.group_size, &lay) != FQ_OK) fail(FQ_E_CONFIG, fq_last_error());
      lay->borrowed = true;
      M->ids.push_back("head");
      M->lin.push_back(lay);
    }
    M->n_lin = static_cast<int>(M->lin.size());
    cudaStream_t st = ctx->stream;
    auto zeros = [&](int64_t n) {
      float* p = static_cast<float*>(dmalloc(sizeof(float) * n));
      FQ_CUDA(cudaMemsetAsync(p, 0, sizeof(float) * n, st));
      return p;
    };
    auto ones = [&](int64_t n) {
      float* p = static_cast<float*>(dmalloc(sizeof(float) * n));
      fill_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(p, n, 1.0f);
      return p;
    };
    M->tok_emb = zeros(V * d);
    if (!M->llama) M->pos_emb = zeros(c.max_seq_len * d);
    for (int64_t i = 0; i < L; ++i) {
      M->n1g.push_back(ones(d));
      M->n2g.push_back(ones(d));
      M->n1b.push_back(M->llama ? nullptr : zeros(d));
      M->n2b.push_back(M->llama ? nullptr : zeros(d));
    }
    M->fng = ones(d);
    M->fnb = M->llama ? nullptr : zeros(d);
    if (!M->llama && c.tie_embeddings) {
      M->tied_head.ctx = ctx;
      M->tied_head.N = V;
      M->tied_head.K = d;
      M->tied_head.G = d;
      M->tied_head.ng = 1;
      M->tied_head.ng_pad = 4;
      M->tied_head.zp_pad = 16;
      M->tied_head.fp = M->tok_emb;
      M->tied_head.borrowed = true;
    }
    const int B = c.max_batch;
    M->slot_len.assign(B, 0);
    M->rungs.assign(static_cast<size_t>(B) * M->n_lin, static_cast<uint8_t>(M->llama ? FQ_RUNG_INT8 : FQ_RUNG_FP));
    // KV cache
    const size_t kv_elem = M->llama ? 2 : 4;
    M->layer_stride = 2 * c.max_seq_len * qd;
    M->slot_stride = L * M->layer_stride;
    M->kv = dmalloc(kv_elem * M->slot_stride * B);
    FQ_CUDA(cudaMemsetAsync(M->kv, 0, kv_elem * M->slot_stride * B, st));
    const size_t as = M->act_size();
    M->rows = M->llama ? std::max(B, kPrefillRows) : B;
    {
      const int B = M->rows;  // activation buffers hold a prefill chunk too
    M->resid = zeros(B * d);
    M->hbuf = zeros(B * d);
    M->q = dmalloc(as * B * d);
    M->k = dmalloc(as * B * d);
    M->v = dmalloc(as * B * d);
    M->attn = dmalloc(as * B * d);
    M->mid = dmalloc(as * B * ffn);
    {
      const int64_t fd = (d + kBlockK - 1) / kBlockK * kBlockK, ff = (ffn + kBlockK - 1) / kBlockK * kBlockK;
      M->attn_frag = dmalloc(4 * B * fd);
      M->mid_frag = dmalloc(4 * B * ff);
      FQ_CUDA(cudaMemsetAsync(M->attn_frag, 0, 4 * B * fd, st));  // padding past K stays zero
      FQ_CUDA(cudaMemsetAsync(M->mid_frag, 0, 4 * B * ff, st));
    }
    M->tmp = zeros(B * ffn_or_d(c));
    M->partials[0] = zeros(static_cast<int64_t>(B) * kPartStride);
    M->partials[1] = zeros(static_cast<int64_t>(B) * kPartStride);
    M->logits = zeros(B * V);
    M->stat_part = dmalloc(static_cast<size_t>(B) * 1024 * 32);  // [B][grid <= 1024] StatPart
    M->stats_dev = static_cast<fq_row_stats*>(dmalloc(sizeof(fq_row_stats) * B));
    M->n_chunks = static_cast<int>((c.max_seq_len + kAttnChunk - 1) / kAttnChunk);
    M->attn_ws = zeros(static_cast<int64_t>(B) * c.n_heads * M->n_chunks * (c.head_dim + 4));
    M->tickets = static_cast<unsigned int*>(dmalloc(sizeof(unsigned int) * B * c.n_heads));
    FQ_CUDA(cudaMemsetAsync(M->tickets, 0, sizeof(unsigned int) * B * c.n_heads, st));
    const int64_t dsz = std::max<int64_t>(static_cast<int64_t>(B) * c.n_heads * c.max_seq_len, B * V);
    M->dscratch = static_cast<double*>(dmalloc(sizeof(double) * dsz));
    M->meta_bytes = 3 * sizeof(int32_t) * B + static_cast<size_t>(B) * M->n_lin;
    M->meta_dev = static_cast<uint8_t*>(dmalloc(M->meta_bytes));
    FQ_CUDA(cudaMallocHost(&M->meta_host, M->meta_bytes));
    std::memset(M->meta_host, 0, M->meta_bytes);
    FQ_CUDA(cudaMallocHost(&M->stats_host, sizeof(fq_row_stats) * B));
    }
    if (M->llama) {
      // RoPE table: angle pos * theta^(-2i/hd) in double, cos/sin rounded to fp32
      const int64_t half = c.head_dim / 2;
      std::vector<float2> cs(static_cast<size_t>(c.max_seq_len * half));
      for (int64_t p = 0; p < c.max_seq_len; ++p)
        for (int64_t i = 0; i < half; ++i) {
          const double inv = std::pow(static_cast<double>(c.rope_theta), -2.0 * static_cast<double>(i) / c.head_dim);
          const double a = static_cast<double>(p) * inv;
          cs[p * half + i] = make_float2(static_cast<float>(std::cos(a)), static_cast<float>(std::sin(a)));
        }
      M->rope_cs = static_cast<float2*>(dmalloc(sizeof(float2) * cs.size()));
      FQ_CUDA(cudaMemcpy(M->rope_cs, cs.data(), sizeof(float2) * cs.size(), cudaMemcpyHostToDevice));
    }
    M->grid_barrier = static_cast<unsigned int*>(dmalloc(sizeof(unsigned int) * 4));
    if (M->llama) {
      FQ_CUDA(cudaEventCreate(&M->ev_prog[0]));
      FQ_CUDA(cudaEventCreate(&M->ev_prog[1]));
    }
    FQ_CUDA(cudaStreamSynchronize(st));
    *out = M;
  });
}

fq_status fq_model_decode_chain(fq_model* M, int32_t slot, int32_t n, fq_row_stats* stats_host) {
  return guarded([&] {
    require(M && stats_host, FQ_E_INPUT, "null argument");
    require(!M->tp(), FQ_E_STATE, "tensor-parallel rank: only fq_model_tp_begin / fq_model_tp_segment run it");
    require(M->llama, FQ_E_CONFIG, "decode chain: llama arch only");
    require(n >= 1 && n <= kMaxChain, FQ_E_INPUT, "decode chain: 1..64 steps");
    require(slot >= 0 && slot < M->cfg.max_batch, FQ_E_INPUT, "slot out of range");
    require(M->chain_slot == slot, FQ_E_STATE,
            "decode chain: the slot's previous operation must be a single-row decode step (its argmax feeds the chain)");
    if (M->slot_len[slot] + n > M->cfg.max_seq_len) fail(FQ_E_CAPACITY, "decode: cache is full");
    fq_ctx* ctx = M->ctx;
    cudaStream_t st = ctx->stream;
    sync_weight_epoch(M);
    if (M->chain_ring == nullptr) {
      FQ_CUDA(cudaMallocHost(&M->chain_ring, sizeof(fq_row_stats) * kMaxChain));
      M->chain_ring_dev = static_cast<fq_row_stats*>(dmalloc(sizeof(fq_row_stats) * kMaxChain));
      M->chain_count = static_cast<unsigned int*>(dmalloc(sizeof(unsigned int)));
    }
    // rows of the step: this slot with its current precision row, staged one position back --
    // every chained step first advances the position on the device; the token slot of the
    // staging is unused (the embedding reads the previous step's argmax on the device)
    const int32_t tok0 = M->stats_host[0].argmax;
    stage_rows(M, 1, &slot, &tok0);
    reinterpret_cast<int32_t*>(M->meta_host)[M->rows] -= 1;
    FQ_CUDA(cudaMemcpyAsync(M->meta_dev, M->meta_host, M->meta_bytes, cudaMemcpyHostToDevice, st));
    FQ_CUDA(cudaMemsetAsync(M->chain_count, 0, sizeof(unsigned int), st));
    int32_t* pos_dev = reinterpret_cast<int32_t*>(M->meta_dev) + M->rows;
    auto one_step = [&]() {
      advance_pos_kernel<<<1, 1, 0, st>>>(pos_dev);
      enqueue_step(M, 1, STEP_CHAIN);
      collect_stats_kernel<<<1, 1, 0, st>>>(M->stats_dev, M->chain_ring_dev, M->chain_count);
      ctx->launches += 2;
    };
    int i = 0;
    if (M->chain_graph == nullptr) {
      one_step();  // builds the chained-step program on first use, then captures one step
      FQ_CUDA(cudaGetLastError());
      ++i;
      if (M->use_graphs) {
        cudaGraph_t graph;
        const int64_t l0 = ctx->launches;
        FQ_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        try {
          one_step();
        } catch (...) {
          cudaStreamEndCapture(st, &graph);
          throw;
        }
        FQ_CUDA(cudaStreamEndCapture(st, &graph));
        FQ_CUDA(cudaGraphInstantiate(&M->chain_graph, graph, 0));
        FQ_CUDA(cudaGraphDestroy(graph));
        ctx->launches = l0;
      }
    }
    for (; i < n; ++i) {
      if (M->chain_graph) {
        FQ_CUDA(cudaGraphLaunch(M->chain_graph, st));
        ctx->launches += 3;
      } else {
        one_step();
      }
    }
    FQ_CUDA(cudaMemcpyAsync(M->chain_ring, M->chain_ring_dev, sizeof(fq_row_stats) * n, cudaMemcpyDeviceToHost, st));
    FQ_CUDA(cudaStreamSynchronize(st));
    FQ_CUDA(cudaGetLastError());
    std::memcpy(stats_host, M->chain_ring, sizeof(fq_row_stats) * n);
    std::memcpy(M->stats_host, M->chain_ring + (n - 1), sizeof(fq_row_stats));
    M->slot_len[slot] += n;
  });
}

fq_status fq_model_tp_shard(const fq_model* M, fq_tp_shard* out) {
  return guarded([&] {
    require(M && out, FQ_E_INPUT, "null argument");
    *out = M->sh;
  });
}

fq_status fq_model_tp_begin(fq_model* M, int32_t batch, const int32_t* slots, const int32_t* tokens) {
  return guarded([&] {
    require(M && slots && tokens, FQ_E_INPUT, "null argument");
    require(M->llama, FQ_E_CONFIG, "tensor parallel: llama arch only");
    require(batch >= 1 && batch <= M->cfg.max_batch, FQ_E_INPUT, "tp step: batch out of range");
    // a step abandoned mid-way (a failed segment) is dropped: its slots' lengths did not advance,
    // so the next step rewrites the same cache positions
    sync_weight_epoch(M);
    for (int i = 0; i < M->n_lin; ++i)
      for (int r : {FQ_RUNG_INT8, FQ_RUNG_INT4})
        require(gemv_fast_supported(M->lin[i], r) || !M->lin[i]->has(r), FQ_E_STATE,
                "layer " + M->ids[i] + ": copy not usable by the fast kernel");
    // the pinned staging buffer may still feed the previous step's copy
    FQ_CUDA(cudaStreamSynchronize(M->ctx->stream));
    stage_rows(M, batch, slots, tokens);
    FQ_CUDA(cudaMemcpyAsync(M->meta_dev, M->meta_host, M->meta_bytes, cudaMemcpyHostToDevice, M->ctx->stream));
    M->tp_batch = batch;
    M->tp_next_seg = 0;
    for (int b = 0; b < batch; ++b) M->tp_slots_step[b] = slots[b];
  });
}

fq_status fq_model_tp_segment(fq_model* M, int32_t seg, const float* reduced_dev, void* out_dev) {
  return guarded([&] {
    require(M && out_dev, FQ_E_INPUT, "null argument");
    require(M->tp_batch > 0, FQ_E_STATE, "tp step: fq_model_tp_begin first");
    require(seg == M->tp_next_seg, FQ_E_STATE, "tp step: segments must run in order");
    require(seg == 0 || reduced_dev, FQ_E_INPUT, "tp step: segment > 0 needs the reduced partial");
    const int B = M->tp_batch;
    ProgramRun& run = tp_program(M, B, seg, seg == 0 ? nullptr : reduced_dev, out_dev);
    FQ_CUDA(cudaMemsetAsync(M->grid_barrier, 0, sizeof(unsigned int), M->ctx->stream));
    launch_program(M->ctx, run, M->grid_barrier, false);
    M->tp_next_seg = seg + 1;
  });
}

fq_status fq_model_tp_end(fq_model* M) {
  return guarded([&] {
    require(M != nullptr, FQ_E_INPUT, "null model");
    require(M->tp_batch > 0, FQ_E_STATE, "tp step: no step begun");
    for (int b = 0; b < M->tp_batch; ++b) M->slot_len[M->tp_slots_step[b]] += 1;
    M->tp_batch = 0;
  });
}

fq_status fq_model_destroy(fq_model* M) {
  return guarded([&] {
    if (!M) return;
    cudaStreamSynchronize(M->ctx->stream);
    if (M->chain_ring) cudaFreeHost(M->chain_ring);
    dfree(M->chain_ring_dev);
    dfree(M->chain_count);
    if (M->chain_graph) cudaGraphExecDestroy(M->chain_graph);
    for (auto& kv : M->graphs) cudaGraphExecDestroy(kv.second);
    for (auto& kv : M->programs) dfree(kv.second.dev_phases);
    for (auto& kv : M->batch_graphs) cudaGraphExecDestroy(kv.second.first);
    dfree(M->grid_barrier);
    dfree(M->timed_ticks);
    free_prefill_ws(M);
    for (cudaEvent_t e : M->ev_prog)
      if (e) cudaEventDestroy(e);
    for (fq_layer* L : M->lin) {
      L->borrowed = false;
      fq_layer_destroy(L);
    }
    dfree(M->tok_emb);
    dfree(M->pos_emb);
    for (auto* p : M->n1g) dfree(p);
    for (auto* p : M->n2g) dfree(p);
    for (auto* p : M->n1b) dfree(p);
    for (auto* p : M->n2b) dfree(p);
    dfree(M->fng);
    dfree(M->fnb);
    dfree(M->kv);
    dfree(M->resid);
    dfree(M->hbuf);
    dfree(M->q);
    dfree(M->k);
    dfree(M->v);
    dfree(M->attn);
    dfree(M->mid);
    dfree(M->attn_frag);
    dfree(M->mid_frag);
    dfree(M->tmp);
    dfree(M->partials[0]);
    dfree(M->partials[1]);
    dfree(M->logits);
    dfree(M->stats_dev);
    dfree(M->attn_ws);
    dfree(M->tickets);
    dfree(M->stat_part);
    dfree(M->rope_cs);
    dfree(M->dscratch);
    dfree(M->meta_dev);
    if (M->meta_host) cudaFreeHost(M->meta_host);
    if (M->stats_host) cudaFreeHost(M->stats_host);
    delete M;
  });
}

fq_status fq_model_num_linears(const fq_model* M, int32_t* out) {
  return guarded([&] {
    require(M && out, FQ_E_INPUT, "null argument");
    *out = M->n_lin;
  });
}

fq_status fq_model_linear_id(const fq_model* M, int32_t index, char* buf, int32_t buflen) {
  return guarded([&] {
    require(M && buf && buflen > 0, FQ_E_INPUT, "null argument");
    require(index >= 0 && index < M->n_lin, FQ_E_INPUT, "linear index out of range");
    const std::string& s = M->ids[index];
    require(static_cast<int32_t>(s.size()) < buflen, FQ_E_INPUT, "buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

fq_status fq_model_linear_index(const fq_model* M, const char* id, int32_t* out) {
  return guarded([&] {
    require(M && id && out, FQ_E_INPUT, "null argument");
    for (int i = 0; i < M->n_lin; ++i)
      if (M->ids[i] == id) {
        *out = i;
        return;
      }
    fail(FQ_E_STATE, std::string("set_precision: unknown layer '") + id + "'");
  });
}

fq_status fq_model_linear(fq_model* M, int32_t index, fq_layer** out) {
  return guarded([&] {
    require(M && out, FQ_E_INPUT, "null argument");
    require(index >= 0 && index < M->n_lin, FQ_E_INPUT, "linear index out of range");
    *out = M->lin[index];
  });
}

fq_status fq_model_set_param(fq_model* M, const char* name, const float* host, int64_t numel) {
  return guarded([&] {
    require(M && name && host, FQ_E_INPUT, "null argument");
    int64_t expect = 0;
    float* dst = param_slot(M, name, expect);
    if (!dst) fail(FQ_E_FORMAT, std::string("weights: unknown parameter '") + name + "'");
    if (numel != expect) fail(FQ_E_DIMENSION, std::string("weights: parameter '") + name + "' has the wrong size");
    FQ_CUDA(cudaMemcpyAsync(dst, host, sizeof(float) * numel, cudaMemcpyHostToDevice, M->ctx->stream));
    FQ_CUDA(cudaStreamSynchronize(M->ctx->stream));
  });
}

fq_status fq_model_get_param(fq_model* M, const char* name, float* host, int64_t numel) {
  return guarded([&] {
    require(M && name && host, FQ_E_INPUT, "null argument");
    int64_t expect = 0;
    const float* src = param_slot(M, name, expect);
    if (!src) fail(FQ_E_FORMAT, std::string("weights: unknown parameter '") + name + "'");
    if (numel != expect) fail(FQ_E_DIMENSION, std::string("weights: parameter '") + name + "' has the wrong size");
    FQ_CUDA(cudaMemcpyAsync(host, src, sizeof(float) * numel, cudaMemcpyDeviceToHost, M->ctx->stream));
    FQ_CUDA(cudaStreamSynchronize(M->ctx->stream));
  });
}

fq_status fq_model_param_size(fq_model* M, const char* name, int64_t* numel) {
  return guarded([&] {
    require(M && name && numel, FQ_E_INPUT, "null argument");
    int64_t expect = 0;
    if (!param_slot(M, name, expect)) fail(FQ_E_FORMAT, std::string("weights: unknown parameter '") + name + "'");
    *numel = expect;
  });
}

fq_status fq_model_init_random_kl(fq_model* M, uint64_t seed, float std, int32_t bins, double* kl8, double* kl4) {
  return guarded([&] {
    require(M != nullptr, FQ_E_INPUT, "null model");
    fq_ctx* ctx = M->ctx;
    const fq_model_config& c = M->cfg;
    int64_t maxn = c.vocab_size * c.d_model;
    for (fq_layer* L : M->lin) maxn = std::max(maxn, L->N * L->K);
    float* w = static_cast<float*>(dmalloc(sizeof(float) * maxn));
    fill_normal(ctx, M->tok_emb, c.vocab_size * c.d_model, seed, 0, std);
    if (M->pos_emb) fill_normal(ctx, M->pos_emb, c.max_seq_len * c.d_model, seed, 1, std);
    for (int i = 0; i < M->n_lin; ++i) {
      fq_layer* L = M->lin[i];
      fill_normal(ctx, w, L->N * L->K, seed, 100 + i, std);
      quantize_device(ctx, L, FQ_RUNG_INT8, FQ_MODE_ASYM, w);
      quantize_device(ctx, L, FQ_RUNG_INT4, FQ_MODE_ASYM, w);
      if (kl8 || kl4) {
        float* keep = L->fp;
        L->fp = w;  // borrowed for the histogram pass only
        try {
          if (kl8) kl8[i] = hist_kl(ctx, L, FQ_RUNG_INT8, bins);
          if (kl4) kl4[i] = hist_kl(ctx, L, FQ_RUNG_INT4, bins);
        } catch (...) {
          L->fp = keep;
          throw;
        }
        L->fp = keep;
      }
      if (!M->llama) {
        if (!L->fp) L->fp = static_cast<float*>(dmalloc(sizeof(float) * L->N * L->K));
        FQ_CUDA(cudaMemcpyAsync(L->fp, w, sizeof(float) * L->N * L->K, cudaMemcpyDeviceToDevice, ctx->stream));
      }
    }
    FQ_CUDA(cudaStreamSynchronize(ctx->stream));
    dfree(w);
  });
}

fq_status fq_model_init_random(fq_model* M, uint64_t seed, float std) {
  return fq_model_init_random_kl(M, seed, std, 0, nullptr, nullptr);
}

fq_status fq_model_set_rung(fq_model* M, int32_t slot, int32_t li, int32_t rung) {
  return guarded([&] {
    require(M != nullptr, FQ_E_INPUT, "null model");
    require(slot >= 0 && slot < M->cfg.max_batch, FQ_E_INPUT, "slot out of range");
    require(li >= 0 && li < M->n_lin, FQ_E_INPUT, "linear index out of range");
    require(rung >= FQ_RUNG_FP && rung <= FQ_RUNG_INT4, FQ_E_CONFIG, "unknown precision rung");
    if (!M->lin[li]->has(rung))
      fail(FQ_E_STATE, "set_precision: layer '" + M->ids[li] + "' has no rung '" +
                           (rung == FQ_RUNG_FP ? "fp" : rung == FQ_RUNG_INT8 ? "8" : "4") + "'");
    if (M->llama && rung == FQ_RUNG_FP) fail(FQ_E_STATE, "llama arch: the fp rung is not resident on the device");
    if (M->llama && !gemv_fast_supported(M->lin[li], rung))
      fail(FQ_E_STATE, "set_precision: layer '" + M->ids[li] + "' has no tiled copy of that rung (zero points span > 255)");
    M->rungs[static_cast<size_t>(slot) * M->n_lin + li] = static_cast<uint8_t>(rung);
  });
}

fq_status fq_model_get_rung(const fq_model* M, int32_t slot, int32_t li, int32_t* out) {
  return guarded([&] {
    require(M && out, FQ_E_INPUT, "null argument");
    require(slot >= 0 && slot < M->cfg.max_batch && li >= 0 && li < M->n_lin, FQ_E_INPUT, "index out of range");
    *out = M->rungs[static_cast<size_t>(slot) * M->n_lin + li];
  });
}

fq_status fq_model_get_rungs(const fq_model* M, int32_t slot, int32_t* out, int32_t n) {
  return guarded([&] {
    require(M != nullptr && out != nullptr, FQ_E_INPUT, "null argument");
    require(slot >= 0 && slot < M->cfg.max_batch, FQ_E_INPUT, "slot out of range");
    require(n == M->n_lin, FQ_E_DIMENSION, "get_rungs: n must equal the number of linears");
    const uint8_t* row = &M->rungs[static_cast<size_t>(slot) * M->n_lin];
    for (int i = 0; i < n; ++i) out[i] = row[i];
  });
}

fq_status fq_model_set_all_rungs(fq_model* M, int32_t slot, int32_t rung) {
  return guarded([&] {
    require(M != nullptr, FQ_E_INPUT, "null model");
    for (int i = 0; i < M->n_lin; ++i)
      if (fq_model_set_rung(M, slot, i, rung) != FQ_OK) fail(FQ_E_STATE, fq_last_error());
  });
}

fq_status fq_model_reset_slot(fq_model* M, int32_t slot) {
  return guarded([&] {
    if (M && M->chain_slot == slot) M->chain_slot = -1;
    require(M != nullptr, FQ_E_INPUT, "null model");
    require(slot >= 0 && slot < M->cfg.max_batch, FQ_E_INPUT, "slot out of range");
    M->slot_len[slot] = 0;
  });
}

fq_status fq_model_slot_length(const fq_model* M, int32_t slot, int64_t* out) {
  return guarded([&] {
    require(M && out, FQ_E_INPUT, "null argument");
    require(slot >= 0 && slot < M->cfg.max_batch, FQ_E_INPUT, "slot out of range");
    *out = M->slot_len[slot];
  });
}

fq_status fq_model_prefill(fq_model* M, int32_t slot, const int32_t* tokens, int64_t n, float* logits_dev,
                           fq_row_stats* stats_host) {
  return guarded([&] {
    require(M && tokens, FQ_E_INPUT, "null argument");
    M->chain_slot = -1;  // stats_dev no longer holds a single decode row
    require(!M->tp(), FQ_E_STATE, "tensor-parallel rank: only fq_model_tp_begin / fq_model_tp_segment run it");
    if (n < 1) fail(FQ_E_INPUT, "prefill: empty prompt");
    require(slot >= 0 && slot < M->cfg.max_batch, FQ_E_INPUT, "slot out of range");
    if (M->slot_len[slot] != 0) fail(FQ_E_STATE, "prefill: cache already populated");
    if (n > M->cfg.max_seq_len) fail(FQ_E_CAPACITY, "prefill: prompt longer than max sequence length");
    for (int64_t i = 0; i < n; ++i)
      if (tokens[i] < 0 || tokens[i] >= M->cfg.vocab_size) fail(FQ_E_INPUT, "prefill: token id out of vocabulary");
    if (!M->llama) {
      // reference architecture: row i of a prefill equals a decode step at position i (causal
      // attention over 0..i with the same per-row arithmetic)
      for (int64_t i = 0; i < n; ++i) {
        const int32_t s = slot, t = tokens[i];
        model_step(M, 1, &s, &t, logits_dev ? logits_dev + i * M->cfg.vocab_size : nullptr,
                   stats_host ? stats_host + i : nullptr);
      }
      return;
    }
    if (gemm_prefill_usable(M, slot, n)) {
      prefill_gemm(M, slot, tokens, n, logits_dev, stats_host);
      return;
    }
    // llama: kPrefillRows consecutive positions per step (rows of one program launch)
    for (int64_t p0 = 0; p0 < n; p0 += kPrefillRows) {
      const int R = static_cast<int>(std::min<int64_t>(kPrefillRows, n - p0));
      prefill_step(M, slot, tokens + p0, R, logits_dev ? logits_dev + p0 * M->cfg.vocab_size : nullptr,
                   stats_host ? stats_host + p0 : nullptr);
    }
  });
}

fq_status fq_model_decode(fq_model* M, int32_t batch, const int32_t* slots, const int32_t* tokens, float* logits_dev,
                          fq_row_stats* stats_host) {
  return guarded([&] {
    require(M && slots && tokens, FQ_E_INPUT, "null argument");
    model_step(M, batch, slots, tokens, logits_dev, stats_host);
  });
}

fq_status fq_model_step_kernel_time(fq_model* M, int32_t reset, double* ms_total, int64_t* steps) {
  return guarded([&] {
    require(M != nullptr, FQ_E_INPUT, "null model");
    if (ms_total) *ms_total = M->prog_ms;
    if (steps) *steps = M->prog_steps;
    if (reset) {
      M->prog_ms = 0.0;
      M->prog_steps = 0;
    }
  });
}

fq_status fq_model_logits(fq_model* M, float** out) {
  return guarded([&] {
    require(M && out, FQ_E_INPUT, "null argument");
    *out = M->logits;
  });
}

fq_status fq_model_step_bytes(const fq_model* M, int32_t batch, const int32_t* slots, int64_t* weight_bytes,
                              int64_t* kv_bytes) {
  return guarded([&] {
    require(M && slots, FQ_E_INPUT, "null argument");
    int64_t wb = 0, kb = 0;
    for (int i = 0; i < M->n_lin; ++i) {
      bool w8 = false, w4 = false, fp = false;
      for (int b = 0; b < batch; ++b) {
        const int r = M->rungs[static_cast<size_t>(slots[b]) * M->n_lin + i];
        w8 |= r == FQ_RUNG_INT8;
        w4 |= r == FQ_RUNG_INT4;
        fp |= r == FQ_RUNG_FP;
      }
      const fq_layer* L = M->lin[i];
      if (w8) wb += L->N * L->K + L->N * L->ng * 5;
      if (w4) wb += (L->N * L->K + 1) / 2 + L->N * L->ng * 5;
      if (fp) wb += L->N * L->K * 4;
    }
    const int64_t es = M->llama ? 2 : 4;
    for (int b = 0; b < batch; ++b) {
      const int64_t ctxlen = M->slot_len[slots[b]] + 1;
      kb += M->cfg.n_layers * 2 * ctxlen * M->cfg.d_model * es;  // read incl. the new position
    }
    if (weight_bytes) *weight_bytes = wb;
    if (kv_bytes) *kv_bytes = kb;
  });
}

fq_status fq_model_profile_step(fq_model* M, int32_t slot, int32_t token, uint64_t* ticks_host, int64_t capacity,
                                int32_t* nphases_out, int32_t* grid_out, int32_t* phase_types_host) {
  return guarded([&] {
    require(M && ticks_host && nphases_out && grid_out, FQ_E_INPUT, "null argument");
    M->chain_slot = -1;  // stats_dev no longer holds a single decode row
    require(!M->tp(), FQ_E_STATE, "tensor-parallel rank: only fq_model_tp_begin / fq_model_tp_segment run it");
    require(M->llama, FQ_E_CONFIG, "profile_step: llama arch only");
    fq_ctx* ctx = M->ctx;
    cudaStream_t st = ctx->stream;
    stage_rows(M, 1, &slot, &token);
    FQ_CUDA(cudaMemcpyAsync(M->meta_dev, M->meta_host, M->meta_bytes, cudaMemcpyHostToDevice, st));
    if (M->programs.find(std::make_pair(1, 0)) == M->programs.end()) {
      enqueue_step(M, 1);  // builds the program; this run is not profiled
      FQ_CUDA(cudaStreamSynchronize(st));
      stage_rows(M, 1, &slot, &token);
      FQ_CUDA(cudaMemcpyAsync(M->meta_dev, M->meta_host, M->meta_bytes, cudaMemcpyHostToDevice, st));
    }
    const ProgramRun& run = M->programs.at(std::make_pair(1, 0));
    const int64_t ring = 3 * 16384;  // ring trace of CTA 0 (program.cu kTraceStages)
    const int64_t gdet = static_cast<int64_t>(run.nphases) * run.grid * 8;  // GEMV phase detail
    const int64_t need = (static_cast<int64_t>(run.nphases) * 2 + 1) * run.grid + ring + gdet;
    *nphases_out = run.nphases;
    *grid_out = run.grid;
    require(capacity >= need, FQ_E_CAPACITY, "profile_step: tick buffer too small");
    auto* dev = static_cast<unsigned long long*>(dmalloc(sizeof(uint64_t) * need));
    FQ_CUDA(cudaStreamSynchronize(st));
    FQ_CUDA(cudaMemset(dev, 0, sizeof(uint64_t) * need));
    set_phase_profile(dev);
    set_ring_trace(dev + (need - ring - gdet), 0);
    set_gemv_profile(dev + (need - gdet));
    try {
      enqueue_step(M, 1);
      FQ_CUDA(cudaStreamSynchronize(st));
    } catch (...) {
      set_phase_profile(nullptr);
      set_ring_trace(nullptr, 0);
      set_gemv_profile(nullptr);
      dfree(dev);
      throw;
    }
    set_phase_profile(nullptr);
    set_ring_trace(nullptr, 0);
    set_gemv_profile(nullptr);
    FQ_CUDA(cudaMemcpy(ticks_host, dev, sizeof(uint64_t) * need, cudaMemcpyDeviceToHost));
    dfree(dev);
    if (phase_types_host) {
      std::vector<Phase> ph(run.nphases);
      if (run.dev_phases)
        FQ_CUDA(cudaMemcpy(ph.data(), run.dev_phases, sizeof(Phase) * run.nphases, cudaMemcpyDeviceToHost));
      else
        for (int i = 0; i < run.nphases; ++i) ph[i] = run.inl.phases[i];
      for (int i = 0; i < run.nphases; ++i) phase_types_host[i] = ph[i].type;
    }
    M->slot_len[slot] += 1;
  });
}

// One B = 1 decode step with the per-phase device clock on (the program's phase hooks): the step's
// device time split into the linears' precision buckets -- each GEMV phase's duration (barrier
// release to barrier release, max over CTAs) shared among its linears by their bytes at the
// slot's rungs -- and the rest (embedding, attention over the cache, statistics).  The trace's
// latency breakdown in device time instead of a byte-proportional split (src/engine.cpp:214-233).
fq_status fq_model_decode_timed(fq_model* M, int32_t slot, int32_t token, float* logits_dev, fq_row_stats* stats_host,
                                uint64_t* ns_by_rung, uint64_t* ns_step) {
  return guarded([&] {
    require(M && stats_host && ns_by_rung && ns_step, FQ_E_INPUT, "null argument");
    M->chain_slot = -1;  // stats_dev no longer holds a single decode row
    require(!M->tp(), FQ_E_STATE, "tensor-parallel rank: only fq_model_tp_begin / fq_model_tp_segment run it");
    require(M->llama, FQ_E_CONFIG, "decode_timed: llama arch only");
    fq_ctx* ctx = M->ctx;
    cudaStream_t st = ctx->stream;
    sync_weight_epoch(M);
    if (M->programs.find(std::make_pair(1, 0)) == M->programs.end()) {
      // first use builds the program: run this step unprofiled, then account it byte-proportionally
      model_step(M, 1, &slot, &token, logits_dev, stats_host);
      ns_by_rung[0] = ns_by_rung[1] = ns_by_rung[2] = 0;
      *ns_step = 0;
      return;
    }
    stage_rows(M, 1, &slot, &token);
    const ProgramRun& run = M->programs.at(std::make_pair(1, 0));
    const int64_t n = (static_cast<int64_t>(run.nphases) * 2 + 1) * run.grid;
    if (M->timed_ticks_n < n) {
      dfree(M->timed_ticks);
      M->timed_ticks = static_cast<unsigned long long*>(dmalloc(sizeof(uint64_t) * n));
      M->timed_ticks_n = n;
    }
    if (M->timed_roles.size() != static_cast<size_t>(run.nphases)) {
      // per phase: the linears of a GEMV phase (matched by their W8 tile pointers), or none
      std::vector<Phase> ph(run.nphases);
      if (run.dev_phases)
        FQ_CUDA(cudaMemcpy(ph.data(), run.dev_phases, sizeof(Phase) * run.nphases, cudaMemcpyDeviceToHost));
      else
        for (int i = 0; i < run.nphases; ++i) ph[i] = run.inl.phases[i];
      M->timed_roles.assign(run.nphases, {});
      for (int i = 0; i < run.nphases; ++i) {
        if (ph[i].type != PH_GEMV) continue;
        for (int m = 0; m < ph[i].nmat; ++m)
          for (int li = 0; li < M->n_lin; ++li)
            if (M->lin[li]->r8.tiles != nullptr && M->lin[li]->r8.tiles == ph[i].mat[m].tiles[0])
              M->timed_roles[i].push_back(li);
      }
    }
    FQ_CUDA(cudaMemcpyAsync(M->meta_dev, M->meta_host, M->meta_bytes, cudaMemcpyHostToDevice, st));
    FQ_CUDA(cudaMemsetAsync(M->timed_ticks, 0, sizeof(uint64_t) * n, st));
    FQ_CUDA(cudaStreamSynchronize(st));
    set_phase_profile(M->timed_ticks);
    try {
      enqueue_step(M, 1);
      FQ_CUDA(cudaStreamSynchronize(st));
    } catch (...) {
      set_phase_profile(nullptr);
      throw;
    }
    set_phase_profile(nullptr);
    std::vector<uint64_t> t(static_cast<size_t>(n));
    FQ_CUDA(cudaMemcpy(t.data(), M->timed_ticks, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost));
    FQ_CUDA(cudaMemcpy(stats_host, M->stats_dev, sizeof(fq_row_stats), cudaMemcpyDeviceToHost));
    if (logits_dev)
      FQ_CUDA(cudaMemcpy(logits_dev, M->logits, sizeof(float) * M->cfg.vocab_size, cudaMemcpyDeviceToDevice));
    const int G = run.grid;
    uint64_t prev = ~0ull;
    for (int c = 0; c < G; ++c) prev = std::min<uint64_t>(prev, t[static_cast<size_t>(run.nphases) * G * 2 + c]);
    const uint64_t t0 = prev;
    double acc[3] = {0, 0, 0}, other = 0;
    const uint8_t* rung = &M->rungs[static_cast<size_t>(slot) * M->n_lin];
    for (int i = 0; i < run.nphases; ++i) {
      uint64_t rel = 0;
      for (int c = 0; c < G; ++c) rel = std::max<uint64_t>(rel, t[(static_cast<size_t>(i) * G + c) * 2 + 1]);
      const double dur = rel > prev ? static_cast<double>(rel - prev) : 0.0;
      prev = std::max(prev, rel);
      const std::vector<int>& ls = M->timed_roles[static_cast<size_t>(i)];
      if (ls.empty()) {
        other += dur;
        continue;
      }
      double tot = 0;
      for (int li : ls) tot += static_cast<double>(M->lin[li]->N * M->lin[li]->K) * (rung[li] == FQ_RUNG_INT4 ? 4 : 8);
      for (int li : ls)
        acc[rung[li]] += dur * static_cast<double>(M->lin[li]->N * M->lin[li]->K) * (rung[li] == FQ_RUNG_INT4 ? 4 : 8) / tot;
    }
    for (int r = 0; r < 3; ++r) ns_by_rung[r] = static_cast<uint64_t>(acc[r]);
    *ns_step = prev > t0 ? prev - t0 : 0;
    M->slot_len[slot] += 1;
  });
}

fq_status fq_model_profile_gemvs(fq_model* M, int32_t slot, int32_t reps, double* ms_per_launch,
                                 int64_t* launches_per_pass, int64_t* bytes_per_pass) {
  return guarded([&] {
    require(M && ms_per_launch, FQ_E_INPUT, "null argument");
    M->chain_slot = -1;  // stats_dev no longer holds a single decode row
    require(!M->tp(), FQ_E_STATE, "tensor-parallel rank: only fq_model_tp_begin / fq_model_tp_segment run it");
    require(M->llama, FQ_E_CONFIG, "profile_gemvs: llama arch only");
    require(reps >= 1, FQ_E_INPUT, "profile_gemvs: reps must be >= 1");
    const int32_t tok = 0;
    if (M->slot_len[slot] >= M->cfg.max_seq_len) fail(FQ_E_CAPACITY, "profile_gemvs: slot is full");
    stage_rows(M, 1, &slot, &tok);
    fq_ctx* ctx = M->ctx;
    cudaStream_t st = ctx->stream;
    FQ_CUDA(cudaMemcpyAsync(M->meta_dev, M->meta_host, M->meta_bytes, cudaMemcpyHostToDevice, st));
    if (M->programs.find(std::make_pair(1, 1)) == M->programs.end()) {
      enqueue_step(M, 1, STEP_GEMV_ONLY);  // builds + uploads the GEMV-only program (un-captured run)
      FQ_CUDA(cudaStreamSynchronize(st));
    }
    const int64_t l0 = ctx->launches;
    cudaGraph_t graph;
    FQ_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    enqueue_step(M, 1, STEP_GEMV_ONLY);
    FQ_CUDA(cudaStreamEndCapture(st, &graph));
    const int64_t per_pass = ctx->launches - l0;
    cudaGraphExec_t exec;
    FQ_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    FQ_CUDA(cudaGraphDestroy(graph));
    cudaEvent_t e0, e1;
    FQ_CUDA(cudaEventCreate(&e0));
    FQ_CUDA(cudaEventCreate(&e1));
    for (int i = 0; i < 2; ++i) FQ_CUDA(cudaGraphLaunch(exec, st));
    FQ_CUDA(cudaEventRecord(e0, st));
    for (int i = 0; i < reps; ++i) FQ_CUDA(cudaGraphLaunch(exec, st));
    FQ_CUDA(cudaEventRecord(e1, st));
    FQ_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    FQ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaGraphExecDestroy(exec);
    ctx->launches += per_pass * (reps + 1);
    *ms_per_launch = static_cast<double>(ms) / reps / static_cast<double>(per_pass);
    if (launches_per_pass) *launches_per_pass = per_pass;
    if (bytes_per_pass) {
      int64_t b = 0;
      for (int i = 0; i < M->n_lin; ++i) {
        const fq_layer* L = M->lin[i];
        const int r = M->rungs[static_cast<size_t>(slot) * M->n_lin + i];
        b += (r == FQ_RUNG_INT8 ? L->N * L->K : (L->N * L->K + 1) / 2) + L->N * L->ng * 5 + L->K * 2 + L->N * 2;
      }
      *bytes_per_pass = b;
    }
  });
}

fq_status fq_model_calibrate_logit_kl(fq_model* M, const int32_t* tokens, int64_t n_seqs, int64_t len,
                                      int32_t base_rung, int32_t flip_rung, double* kl_host, double* entropy_host) {
  return guarded([&] {
    require(M && tokens && kl_host, FQ_E_INPUT, "null argument");
    M->chain_slot = -1;  // stats_dev no longer holds a single decode row
    require(!M->tp(), FQ_E_STATE, "tensor-parallel rank: only fq_model_tp_begin / fq_model_tp_segment run it");
    require(n_seqs >= 1 && len >= 1, FQ_E_INPUT, "calibrate: empty token set");
    require(len <= M->cfg.max_seq_len, FQ_E_CAPACITY, "calibrate: sequence longer than max_seq_len");
    const fq_model_config& c = M->cfg;
    const int per = M->llama ? 7 : 6;
    const int B = static_cast<int>(std::min<int64_t>(n_seqs, c.max_batch));
    const int64_t V = c.vocab_size;
    const int64_t rows = n_seqs * len;
    float* base_logits = static_cast<float*>(dmalloc(sizeof(float) * rows * V));
    float* flip_logits = static_cast<float*>(dmalloc(sizeof(float) * B * V));
    double* kl_dev = static_cast<double*>(dmalloc(sizeof(double) * B * 2));
    std::vector<double> klsum(c.n_layers, 0.0), entsum(c.n_layers, 0.0);
    std::vector<uint8_t> saved(M->rungs);
    // llama with W8/W4 rungs: every sequence is one tensor-core prefill (all len rows at once)
    // and the KL of all its rows one launch
    auto gemm_path = [&](int flip_layer) {
      for (int i = 0; i < M->n_lin; ++i) {
        const bool in_block = flip_layer >= 0 && i / per == flip_layer && i < M->head_index();
        M->rungs[i] = static_cast<uint8_t>(in_block ? flip_rung : base_rung);
      }
      return gemm_prefill_usable(M, 0, len);
    };
    if (gemm_path(-1) && gemm_path(0)) {
      try {
        double* kl_rows = static_cast<double*>(dmalloc(sizeof(double) * 2 * len));
        float* flip_all = static_cast<float*>(dmalloc(sizeof(float) * len * V));
        // residual stream entering each block of the sequence's base forward: a forward with block
        // fl flipped starts at fl (blocks below it are bit-identical to the base forward's), ~half
        // the work of 33 full forwards per sequence
        float* snap = nullptr;
        // FQ_CALIB_FULL=1: every flipped forward from the embedding (the check that the reuse is exact)
        const bool full = std::getenv("FQ_CALIB_FULL") != nullptr;
        try {
          snap = static_cast<float*>(dmalloc(sizeof(float) * static_cast<size_t>(c.n_layers) * len * c.d_model));
          std::vector<double> h(2 * len);
          for (int64_t s = 0; s < n_seqs; ++s) {
            float* base = base_logits + s * len * V;
            gemm_path(-1);
            prefill_gemm_enqueue(M, 0, tokens + s * len, len, base, nullptr, 0, snap, true);
            for (int fl = 0; fl < c.n_layers; ++fl) {
              gemm_path(fl);
              prefill_gemm_enqueue(M, 0, tokens + s * len, len, flip_all, nullptr, full ? 0 : fl, snap, false);
              launch_kl_rows(M->ctx, flip_all, base, FQ_DT_F32, len, V, kl_rows, kl_rows + len);
              FQ_CUDA(cudaMemcpyAsync(h.data(), kl_rows, sizeof(double) * 2 * len, cudaMemcpyDeviceToHost, M->ctx->stream));
              FQ_CUDA(cudaStreamSynchronize(M->ctx->stream));
              for (int64_t t = 0; t < len; ++t) {  // per block, sequences in order: the sums of the
                klsum[fl] += h[t];                 // block-major loop, bit for bit
                entsum[fl] += h[len + t];
              }
            }
          }
        } catch (...) {
          dfree(snap);
          dfree(kl_rows);
          dfree(flip_all);
          throw;
        }
        dfree(snap);
        dfree(kl_rows);
        dfree(flip_all);
      } catch (...) {
        M->rungs = saved;
        dfree(base_logits);
        dfree(flip_logits);
        dfree(kl_dev);
        throw;
      }
      M->rungs = saved;
      M->slot_len[0] = 0;
      for (int l = 0; l < c.n_layers; ++l) {
        kl_host[l] = klsum[l] / static_cast<double>(rows);
        if (entropy_host) entropy_host[l] = entsum[l] / static_cast<double>(rows);
      }
      dfree(base_logits);
      dfree(flip_logits);
      dfree(kl_dev);
      return;
    }
    M->rungs = saved;
    auto run = [&](int flip_layer) {
      for (int64_t s0 = 0; s0 < n_seqs; s0 += B) {
        const int nb = static_cast<int>(std::min<int64_t>(B, n_seqs - s0));
        std::vector<int32_t> slots(nb);
        for (int b = 0; b < nb; ++b) {
          slots[b] = b;
          M->slot_len[b] = 0;
          for (int i = 0; i < M->n_lin; ++i) {
            const bool in_block = flip_layer >= 0 && i / per == flip_layer && i < M->head_index();
            M->rungs[static_cast<size_t>(b) * M->n_lin + i] = static_cast<uint8_t>(in_block ? flip_rung : base_rung);
          }
        }
        for (int64_t t = 0; t < len; ++t) {
          std::vector<int32_t> tk(nb);
          for (int b = 0; b < nb; ++b) tk[b] = tokens[(s0 + b) * len + t];
          if (flip_layer < 0) {
            stage_rows(M, nb, slots.data(), tk.data());
            run_step(M, nb);
            for (int b = 0; b < nb; ++b) {
              M->slot_len[b] += 1;
              FQ_CUDA(cudaMemcpyAsync(base_logits + ((s0 + b) * len + t) * V, M->logits + b * V, sizeof(float) * V,
                                      cudaMemcpyDeviceToDevice, M->ctx->stream));
            }
          } else {
            stage_rows(M, nb, slots.data(), tk.data());
            run_step(M, nb);
            for (int b = 0; b < nb; ++b) M->slot_len[b] += 1;
            // KL of each row against the stored baseline row (rows of different sequences are
            // not contiguous in the baseline buffer: one launch per row)
            for (int b = 0; b < nb; ++b)
              launch_kl_rows(M->ctx, M->logits + b * V, base_logits + ((s0 + b) * len + t) * V, FQ_DT_F32, 1, V,
                             kl_dev + 2 * b, kl_dev + 2 * b + 1);
            std::vector<double> h(2 * nb);
            FQ_CUDA(cudaMemcpyAsync(h.data(), kl_dev, sizeof(double) * 2 * nb, cudaMemcpyDeviceToHost, M->ctx->stream));
            FQ_CUDA(cudaStreamSynchronize(M->ctx->stream));
            for (int b = 0; b < nb; ++b) {
              klsum[flip_layer] += h[2 * b];
              entsum[flip_layer] += h[2 * b + 1];
            }
          }
        }
      }
    };
    try {
      run(-1);
      for (int l = 0; l < c.n_layers; ++l) run(l);
    } catch (...) {
      M->rungs = saved;
      dfree(base_logits);
      dfree(flip_logits);
      dfree(kl_dev);
      throw;
    }
    M->rungs = saved;
    for (int b = 0; b < B; ++b) M->slot_len[b] = 0;
    for (int l = 0; l < c.n_layers; ++l) {
      kl_host[l] = klsum[l] / static_cast<double>(rows);
      if (entropy_host) entropy_host[l] = entsum[l] / static_cast<double>(rows);
    }
    dfree(base_logits);
    dfree(flip_logits);
    dfree(kl_dev);
  });
}

}  // extern "C"
