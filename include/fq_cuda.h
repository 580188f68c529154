/*
 * fq_cuda.h — the C-ABI boundary of the B200 FlexQuant decode engine.
 *
 * Everything the reference's hot path computes on the CPU is reachable through
 * these entry points: plain pointers, sizes and opaque handles, no C++ or torch
 * types, no exceptions.  Every function returns an fq_status; on failure the
 * message is available from fq_last_error() (thread-local).  Status codes map
 * one-to-one onto the reference's exception hierarchy
 * (/root/reference/proj/include/flexquant/error.hpp:10-49) so the C++ wrapper
 * (the headers under include/flexquant) can rethrow the matching flexquant::Error subclass.
 *
 * Pointer convention: arguments named *_host are host memory, *_dev are device
 * (cudaMalloc / torch CUDA) memory.  All device work is ordered on the stream
 * bound to the fq_ctx (fq_ctx_set_stream).
 *
 * Which reference interface each entry point replaces is cited next to it as
 * file:line under /root/reference/proj.
 */
#ifndef FQ_CUDA_H
#define FQ_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FQ_ABI_VERSION 1

typedef int32_t fq_status;
enum {
  FQ_OK = 0,
  FQ_E_DIMENSION = 1, /* flexquant::DimensionError */
  FQ_E_CONFIG = 2,    /* flexquant::ConfigError    */
  FQ_E_INPUT = 3,     /* flexquant::InputError     */
  FQ_E_STATE = 4,     /* flexquant::StateError     */
  FQ_E_FORMAT = 5,    /* flexquant::FormatError    */
  FQ_E_CAPACITY = 6,  /* flexquant::CapacityError  */
  FQ_E_CUDA = 7       /* device / driver failure (no reference analogue) */
};

/* Precision rungs: include/flexquant/rung.hpp:13 (Rung{Fp,Int8,Int4}). */
enum { FQ_RUNG_FP = 0, FQ_RUNG_INT8 = 1, FQ_RUNG_INT4 = 2 };
/* Quantization modes: include/flexquant/quantizer.hpp:12 (QuantMode). */
enum { FQ_MODE_ASYM = 0, FQ_MODE_SYM = 1 };
/* Element types of activations / logits. */
enum { FQ_DT_F32 = 0, FQ_DT_F16 = 1, FQ_DT_BF16 = 2 };
/* Decoder block families. */
enum {
  FQ_ARCH_REFERENCE = 0, /* LayerNorm+bias, GELU w1/w2, learned positions, fp32 activations,
                            double accumulation: the reference's own model (src/model.cpp:193-266) */
  FQ_ARCH_LLAMA = 1      /* RMSNorm, SwiGLU gate/up/down, RoPE, no biases, bf16/fp16 activations,
                            fp16 KV cache (BASELINE configs) */
};
/* GEMV numerics. */
enum {
  FQ_NUMERICS_FAST = 0, /* fp32 accumulation, per-group Σx zero-point folding (decode hot path) */
  FQ_NUMERICS_EXACT = 1 /* dequantize-on-use in fp32 then double accumulation, as
                           MultiPrecisionLayer::forward (src/model.cpp:77-98) + linear (src/tensor.cpp:83-101) */
};

typedef struct fq_ctx fq_ctx;
typedef struct fq_layer fq_layer;
typedef struct fq_model fq_model;

/* Per-logits-row statistics, all in double (src/scheduler.cpp:13-49, src/engine.cpp:144-155). */
typedef struct fq_row_stats {
  double ppl_entropy;     /* exp(H), ppl_entropy()            scheduler.cpp:29-35 */
  double entropy;         /* H = -sum p ln p                                      */
  double p1;              /* largest softmax probability                          */
  double p2;              /* second largest (duplicates count)                    */
  double fault_tolerance; /* p1 - p2, fault_tolerance()       scheduler.cpp:37-49 */
  float max_logit;        /* max over the float logits                            */
  int32_t argmax;         /* argmax_token(): strict >, lowest index  engine.cpp:144-155 */
} fq_row_stats;

/* ---------------------------------------------------------------- context */
const char* fq_last_error(void);
int32_t fq_abi_version(void);
fq_status fq_ctx_create(int32_t device, fq_ctx** out);
fq_status fq_ctx_destroy(fq_ctx* ctx);
/* Binds a cudaStream_t (passed as void*); NULL selects the context's own stream. */
fq_status fq_ctx_set_stream(fq_ctx* ctx, void* stream);
fq_status fq_ctx_get_stream(fq_ctx* ctx, void** stream_out);
fq_status fq_ctx_synchronize(fq_ctx* ctx);
/* Number of kernels this context has launched (evidence counter for the bench). */
fq_status fq_ctx_launch_count(fq_ctx* ctx, int64_t* out);

/* ------------------------------------------------------ weight store (a1-a4, a6) */
/* One linear layer [out_features x in_features] with resident per-precision copies.
 * group_size: quantization group along in_features (0 or >= in_features = per row,
 * the reference's granularity, src/quantizer.cpp:128-185).  Replaces
 * MultiPrecisionLayer (include/flexquant/model.hpp:45-92). */
fq_status fq_layer_create(fq_ctx* ctx, int64_t out_features, int64_t in_features,
                          int64_t group_size, fq_layer** out);
fq_status fq_layer_destroy(fq_layer* layer);
/* Uploads one quantized rung from the canonical QuantizedTensor layout
 * (include/flexquant/quantizer.hpp:24-44 applied to the [N*ceil(K/G), G] group view):
 * payload = packed codes of the row-major stream (4-bit: low nibble = even index),
 * scale/zero_point = one per group in (row, group) order. */
fq_status fq_layer_upload_quantized(fq_layer* layer, int32_t rung, int32_t mode,
                                    const uint8_t* payload_host, int64_t payload_bytes,
                                    const float* scale_host, const int32_t* zero_point_host,
                                    int64_t n_groups);
/* Reads a rung back in the canonical layout (round trip of the device layout). */
fq_status fq_layer_download_quantized(const fq_layer* layer, int32_t rung, uint8_t* payload_host,
                                      float* scale_host, int32_t* zero_point_host);
/* Full-precision rung (fp32 [N,K]) and optional bias [N]. */
fq_status fq_layer_upload_fp(fq_layer* layer, const float* weight_host);
fq_status fq_layer_upload_bias(fq_layer* layer, const float* bias_host);
/* Copies the fp weights / bias back to the host (the weights container writer, MultiPrecisionLayer::
 * fp_weight / bias); *present = 0 (and nothing copied) when the layer holds none. */
fq_status fq_layer_download_fp(const fq_layer* layer, float* weight_host, int32_t* present);
fq_status fq_layer_download_bias(const fq_layer* layer, float* bias_host, int32_t* present);
/* Device-side RTN quantizer (K9): quantizes fp32 weights already on the device with the
 * reference rules (src/quantizer.cpp:111-189, round-half-even in double). */
fq_status fq_layer_quantize_device(fq_layer* layer, int32_t rung, int32_t mode, const float* weight_dev);
fq_status fq_layer_has(const fq_layer* layer, int32_t rung, int32_t* out);
fq_status fq_layer_shape(const fq_layer* layer, int64_t* out_features, int64_t* in_features,
                         int64_t* group_size);
/* Algorithmic bytes one B-row GEMV over `rung` touches (payload + 5 B/group + activations). */
fq_status fq_layer_bytes(const fq_layer* layer, int32_t rung, int64_t batch, int64_t* out);

/* y[B,N] = x[B,K] * dequant(W_rung)^T (+ bias).  Replaces MultiPrecisionLayer::forward
 * (src/model.cpp:77-98): dequantize (src/quantizer.cpp:205-219) + linear (src/tensor.cpp:83-101).
 * x_dev / y_dev are device buffers of the given dtypes. */
fq_status fq_gemv(fq_ctx* ctx, const fq_layer* layer, int32_t rung, int64_t batch,
                  const void* x_dev, int32_t x_dtype, void* y_dev, int32_t y_dtype,
                  int32_t numerics);

/* Benchmark form of fq_gemv (BASELINE config 2): n independent GEMVs y_i = x . dequant(W_i)^T
 * (same x, fast numerics) as ONE persistent step-program launch with no grid barrier between
 * them, so the TMA weight stream runs across layer boundaries as it does inside a decode step.
 * Launched `reps` times on the context stream; *ms_per_launch = mean device time of one launch
 * (CUDA events around the launches).  The outputs are those of n fq_gemv calls. */
fq_status fq_gemv_chain_time(fq_ctx* ctx, const fq_layer* const* layers, int32_t n, int32_t rung, int64_t batch,
                             const void* x_dev, int32_t x_dtype, void* const* y_devs, int32_t y_dtype,
                             int32_t reps, double* ms_per_launch);

/* Prefill / calibration contraction on the tcgen05 tensor cores (BASELINE config 4):
 * y[rows, N] (fp32, row stride y_stride) = x[rows, K] (bf16, row stride x_stride) . dequant(W_rung)^T.
 * MultiPrecisionLayer::forward (src/model.cpp:77-98) on many rows at once.  The tensor cores
 * multiply the exact integer codes (q - z) by the activations, each 128-code quantization group
 * accumulates alone in fp32 in tensor memory and its fp32 scale is applied in the epilogue, so
 * no weight is rounded (the decode GEMV's precision contract).  x is re-laid into the GEMM's
 * tiled operand format in context scratch first (fq_tile_activations). */
fq_status fq_gemm(fq_ctx* ctx, const fq_layer* layer, int32_t rung, int64_t rows, const void* x_dev,
                  int64_t x_stride, float* y_dev, int64_t y_stride);
/* The GEMM's activation operand format: 16-bit [ceil(rows/128)][ceil(K/128)][128 x 128] tiles in
 * the UMMA canonical K-major layout, rows past `rows` / columns past K zero.  Bytes needed: */
int64_t fq_tiled_activation_bytes(int64_t rows, int64_t K);
/* x (x_dtype f32 / f16 / bf16, row stride x_stride) -> tiled fp16 (out_dtype must be FQ_DT_F16:
 * bf16 values are exact in fp16's normal range); xt_dev must hold fq_tiled_activation_bytes and be
 * zeroed once by the caller. */
fq_status fq_tile_activations(fq_ctx* ctx, const void* x_dev, int32_t x_dtype, int64_t x_stride, int64_t rows,
                              int64_t K, int32_t out_dtype, void* xt_dev);
/* fq_gemm on pre-tiled fp16 activations (x_dtype FQ_DT_F16): the prefill's own call. */
fq_status fq_gemm_tiled(fq_ctx* ctx, const fq_layer* layer, int32_t rung, int64_t rows, const void* xt_dev,
                        int32_t x_dtype, float* y_dev, int64_t y_stride, int32_t accumulate);

/* ------------------------------------------------------- statistics (a10, a11, a18) */
/* One fq_row_stats per logits row (fp32 [rows, vocab] on device); stats_dev on device. */
fq_status fq_softmax_stats(fq_ctx* ctx, const float* logits_dev, int64_t rows, int64_t vocab,
                           fq_row_stats* stats_dev);
/* Per row r: kl[r] = KL(softmax(lq_r) || softmax(lp_r)) = sum p_q ln(p_q/p_p),
 * entropy[r] = H(softmax(lq_r)).  Logit-mode calibration (BASELINE config 4); the
 * divergence follows kl_divergence (src/analyzer.cpp:65-79). Logits fp32 or bf16. */
fq_status fq_kl_rows(fq_ctx* ctx, const void* logits_q_dev, const void* logits_p_dev, int32_t dtype,
                     int64_t rows, int64_t vocab, double* kl_dev, double* entropy_dev);
/* Weight-histogram KL of one layer's rung against its fp weights (src/analyzer.cpp:83-94:
 * uniform_edges over [min,max], weight_histogram with +1e-10 smoothing, kl_divergence). */
fq_status fq_hist_kl(fq_ctx* ctx, const fq_layer* layer, int32_t rung, int32_t bins, double* kl_host);

/* Deterministic N(0, std) generator keyed by (seed, stream_id, element index); the same
 * values are produced by the host generator in the C++ library and the oracle. */
fq_status fq_fill_normal(fq_ctx* ctx, float* dst_dev, int64_t n, uint64_t seed, uint64_t stream_id,
                         float std);

/* ------------------------------------------------------------ device decoder (a7-a9, a14) */
typedef struct fq_model_config {
  int32_t arch;          /* FQ_ARCH_*                                   */
  int32_t act_dtype;     /* llama: FQ_DT_BF16 / FQ_DT_F16; reference: FQ_DT_F32 */
  int64_t vocab_size;
  int64_t d_model;
  int64_t n_heads;
  int64_t head_dim;
  int64_t n_layers;
  int64_t ffn_dim;
  int64_t max_seq_len;
  int32_t tie_embeddings; /* reference arch only */
  int32_t max_batch;      /* resident sequence slots (KV caches, precision-table rows) */
  int64_t group_size;     /* quantization group (0 = per row) */
  float norm_eps;         /* LayerNorm / RMSNorm epsilon */
  float rope_theta;       /* llama only */
} fq_model_config;

fq_status fq_model_create(fq_ctx* ctx, const fq_model_config* cfg, fq_model** out);
fq_status fq_model_destroy(fq_model* model);
/* Switchable linears in the reference's accounting order (src/model.cpp:304-330):
 * reference arch: blocks.i.attn.{wq,wk,wv,wo}, blocks.i.ffn.{w1,w2}, head;
 * llama arch:     blocks.i.attn.{wq,wk,wv,wo}, blocks.i.ffn.{w_gate,w_up,w_down}, head. */
fq_status fq_model_num_linears(const fq_model* model, int32_t* out);
fq_status fq_model_linear_id(const fq_model* model, int32_t index, char* buf, int32_t buflen);
fq_status fq_model_linear_index(const fq_model* model, const char* layer_id, int32_t* out);
fq_status fq_model_linear(fq_model* model, int32_t index, fq_layer** out); /* borrowed */
/* Non-switchable parameters by name: tok_emb, pos_emb, blocks.i.ln1.gamma/beta,
 * blocks.i.ln2.gamma/beta (reference), blocks.i.attn_norm / blocks.i.ffn_norm (llama),
 * final_norm(.gamma/.beta).  fp32 host data. */
fq_status fq_model_set_param(fq_model* model, const char* name, const float* host, int64_t numel);
/* The reverse of fq_model_set_param (save_model_file), and a parameter's element count. */
fq_status fq_model_get_param(fq_model* model, const char* name, float* host, int64_t numel);
fq_status fq_model_param_size(fq_model* model, const char* name, int64_t* numel);
/* Fills every parameter / rung from the deterministic generator on the device (bench). */
fq_status fq_model_init_random(fq_model* model, uint64_t seed, float std);
/* Same, and while each linear's fp32 weights are on the device computes the reference analyzer's
 * weight-histogram KL of its W8 and W4 rungs (src/analyzer.cpp:83-94, `bins` bins) into
 * kl8_host / kl4_host [num_linears] (either may be NULL). */
fq_status fq_model_init_random_kl(fq_model* model, uint64_t seed, float std, int32_t bins, double* kl8_host,
                                  double* kl4_host);
/* Precision table: rung of (sequence slot, linear).  A pointer-of-record write, no payload
 * touched (Model::set_precision, src/model.cpp:268-278).  Takes effect at the next step. */
fq_status fq_model_set_rung(fq_model* model, int32_t slot, int32_t linear_index, int32_t rung);
fq_status fq_model_get_rung(const fq_model* model, int32_t slot, int32_t linear_index, int32_t* out);
fq_status fq_model_set_all_rungs(fq_model* model, int32_t slot, int32_t rung);
/* The whole precision row of a slot (n = number of linears) in one call (host bookkeeping:
 * effective bits, bytes per pass, latency buckets per token). */
fq_status fq_model_get_rungs(const fq_model* model, int32_t slot, int32_t* out, int32_t n);
/* KV cache of a slot (KvCache, src/model.cpp:142-171). */
fq_status fq_model_reset_slot(fq_model* model, int32_t slot);
fq_status fq_model_slot_length(const fq_model* model, int32_t slot, int64_t* out);
/* Prefill n prompt tokens into an empty slot (Model::forward_prefill, src/model.cpp:239-255).
 * logits_dev: optional device buffer [n, V] fp32 receiving every row; stats_host: n rows. */
fq_status fq_model_prefill(fq_model* model, int32_t slot, const int32_t* tokens_host, int64_t n,
                           float* logits_dev, fq_row_stats* stats_host);
/* One decode step for `batch` slots (Model::forward_decode, src/model.cpp:257-266, batched):
 * appends one position per slot and writes per-row stats to stats_host.  The step is
 * replayed from a captured CUDA graph. logits_dev optional [batch, V] copy-out. */
fq_status fq_model_decode(fq_model* model, int32_t batch, const int32_t* slots_host,
                          const int32_t* tokens_host, float* logits_dev, fq_row_stats* stats_host);
/* n (<= 64) further decode steps of `slot`, each fed on the device with the previous step's
 * argmax (argmax_token, src/engine.cpp:144-155) and run at the slot's current precision row, with
 * no host round trip between them; stats_host receives the n rows.  For a decode loop whose
 * scheduler provably cannot switch during those tokens (SchedulerState::observe, src/scheduler.cpp:
 * 85-104: window still filling or cooldown running); the slot's previous operation must be a
 * single-row fq_model_decode (or chain) step. */
fq_status fq_model_decode_chain(fq_model* model, int32_t slot, int32_t n, fq_row_stats* stats_host);
/* fq_model_decode for one slot with the device phase clock on: also returns the step's device
 * time split by precision (ns_by_rung[FQ_RUNG_*]: each GEMV phase's time shared among its
 * linears by bytes) and the whole step (*ns_step); the remainder is embedding, attention over the
 * cache and the statistics.  The trace's latency breakdown (src/engine.cpp:214-233) in device time. */
fq_status fq_model_decode_timed(fq_model* model, int32_t slot, int32_t token, float* logits_dev,
                                fq_row_stats* stats_host, uint64_t* ns_by_rung, uint64_t* ns_step);
/* Device time of the decode-step program kernels (CUDA events recorded around the launch inside
 * the step graph): total ms and number of steps since the last reset (reset != 0 clears after
 * reading).  bench.py's roofline divides the step's algorithmic bytes by this per-launch time. */
fq_status fq_model_step_kernel_time(fq_model* model, int32_t reset, double* ms_total, int64_t* steps);
/* Device pointer of the model's internal logits buffer [max_batch, V] (valid after a step). */
fq_status fq_model_logits(fq_model* model, float** logits_dev);
/* Algorithmic bytes of one decode step for `batch` slots at their current rungs/lengths. */
fq_status fq_model_step_bytes(const fq_model* model, int32_t batch, const int32_t* slots_host,
                              int64_t* weight_bytes, int64_t* kv_bytes);
/* Kernel-level measurement: captures the decode step's GEMV launches alone (same layers, the
 * slot's current rungs, same launch parameters) into a graph, replays it `reps` times between
 * CUDA events on the context stream and reports the mean time of one GEMV launch (ms) and the
 * algorithmic bytes of one pass over the step's GEMVs. */
fq_status fq_model_profile_gemvs(fq_model* model, int32_t slot, int32_t reps, double* ms_per_launch,
                                 int64_t* launches_per_pass, int64_t* bytes_per_pass);
/* Profiling: runs one decode step of `slot` (appending `token`) with per-phase timestamps.
 * ticks_host receives (nphases * 2 + 1) * grid %globaltimer values: [(phase * grid + cta) * 2]
 * = end of the phase's work on that CTA, [... + 1] = after the grid barrier that follows, and
 * [nphases * grid * 2 + cta] = the CTA's start; then 3 * 16384 ring-trace stamps of CTA 0 (per
 * weight stage: producer got the slot, consumers saw the data, consumers released it; 0 = unused);
 * then nphases * grid * 8 GEMV-phase stamps [(phase * grid + cta) * 8 + k] (k = 0 partition set
 * up, 1 norm factors, 2 first barrier, 3 activations staged, 4 weight loop done, 5 final reduction
 * done, 6 phase done).
 * phase_types_host (optional, nphases entries)
 * receives the phase kinds (0 GEMV, 1 embedding, 2 attention, 3 row statistics). */
fq_status fq_model_profile_step(fq_model* model, int32_t slot, int32_t token, uint64_t* ticks_host,
                                int64_t capacity, int32_t* nphases_out, int32_t* grid_out,
                                int32_t* phase_types_host);
/* Logit-mode calibration (BASELINE config 4): teacher-forced prefill of `n_seqs` token rows
 * of length `len`, all linears at `base_rung`, then for every block b the block's linears at
 * `flip_rung`; kl_host[b] = mean KL(softmax(l_flip) || softmax(l_base)), entropy_host[b] =
 * mean entropy of the flipped distribution. */
fq_status fq_model_calibrate_logit_kl(fq_model* model, const int32_t* tokens_host, int64_t n_seqs,
                                      int64_t len, int32_t base_rung, int32_t flip_rung,
                                      double* kl_host, double* entropy_host);

/* ------------------------------------------- tensor-parallel variant (north_star)
 * The reference has no distribution (its block is src/model.cpp:201-233 on one core); this is
 * the variant north_star names: column-split q/k/v/gate/up, row-split o/down and a vocab-split
 * head, with one all-reduce (sum) of an fp32 [batch, d_model] partial after each row-split
 * projection and one all-gather of the head's softmax partials.  The collectives are the
 * caller's (NCCL over NVLink through torch.distributed in paper_2506_12024_b200/tp.py). */
typedef struct fq_tp_shard {
  int32_t rank, size;
  int64_t head0, heads;  /* attention heads [head0, head0 + heads) */
  int64_t ffn0, ffn;     /* SwiGLU columns [ffn0, ffn0 + ffn), whole quantization groups */
  int64_t vocab0, vocab; /* head rows [vocab0, vocab0 + vocab) */
  int32_t n_segments;    /* 2 * n_layers + 1 */
} fq_tp_shard;
/* Mergeable softmax partial of one logits row (max m, S = sum e^(l-m), T = sum e^(l-m)(l-m) in
 * double, the two largest logits, the lowest index of the largest); 32 bytes. */
typedef struct fq_stat_part {
  double S, T;
  float m, v1, v2;
  int32_t arg;
} fq_stat_part;
/* Host only: the shard of rank `rank` of `size` (heads split evenly -- n_heads % size == 0 and
 * each rank's heads * head_dim a multiple of group_size; ffn split in whole groups, the ragged
 * tail group on the last rank; vocab rows split evenly). */
fq_status fq_tp_shard_spec(const fq_model_config* cfg, int32_t rank, int32_t size, fq_tp_shard* out);
/* Host only: the quantized sub-matrix rows [row0, row1) x columns [col0, col1) of a g-grouped
 * QuantizedTensor of an [N, K] weight (quantizer.hpp:24-44 in the g128 view: codes row-major,
 * one scale / zero point per (row, group)); col0 a multiple of `group`, col1 a multiple of
 * `group` or K.  Bit-identical to quantizing the sliced fp32 weights (groups are independent). */
fq_status fq_shard_quantized(int32_t bits, int64_t N, int64_t K, int64_t group, const uint8_t* payload,
                             const float* scale, const int32_t* zp, int64_t row0, int64_t row1, int64_t col0,
                             int64_t col1, uint8_t* payload_out, float* scale_out, int32_t* zp_out);
/* Host only: merges the ranks' head partials parts[rank * batch + b] (argmax indices local to the
 * rank's vocab slice, offset by vocab0[rank]) into the row statistics of softmax_double /
 * ppl_entropy / fault_tolerance / argmax_token (src/scheduler.cpp:13-49, src/engine.cpp:144-155). */
fq_status fq_tp_merge_stats(const fq_stat_part* parts, int32_t nranks, int32_t batch, const int64_t* vocab0,
                            fq_row_stats* out);
/* A TP rank of the llama config `cfg` (the FULL model's config): its linears have the shard's
 * shapes (upload the fq_shard_quantized slices), the embedding and norms are full. */
fq_status fq_model_create_tp(fq_ctx* ctx, const fq_model_config* cfg, int32_t tp_rank, int32_t tp_size,
                             fq_model** out);
fq_status fq_model_tp_shard(const fq_model* model, fq_tp_shard* out);
/* Starts one TP decode step for `batch` slots (stages tokens, positions and precision rows). */
fq_status fq_model_tp_begin(fq_model* model, int32_t batch, const int32_t* slots_host,
                            const int32_t* tokens_host);
/* Enqueues segment `seg` (0 .. n_segments-1, in order) on the context stream.  reduced_dev: the
 * sum over ranks of the previous segment's partials (fp32 [batch, d_model]; NULL for seg 0).
 * out_dev: seg < n_segments-1 -> this rank's fp32 [batch, d_model] partial of the O / down
 * projection; the last segment -> fq_stat_part [batch] of the rank's vocab slice (its logits
 * stay in fq_model_logits, [batch, shard.vocab]).  Segments only enqueue work, so the sequence
 * (with the caller's collectives) can be captured into a CUDA graph and replayed. */
fq_status fq_model_tp_segment(fq_model* model, int32_t seg, const float* reduced_dev, void* out_dev);
/* Completes the step begun by fq_model_tp_begin after its segments were enqueued (or a captured
 * sequence of them replayed): every slot of the step advances by one position. */
fq_status fq_model_tp_end(fq_model* model);

#ifdef __cplusplus
}
#endif
#endif /* FQ_CUDA_H */
