// Internal declarations shared by the CUDA translation units of libfq_cuda.so.
// Nothing here crosses the C-ABI; see include/fq_cuda.h for the boundary.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>
#include <string>
#include <vector>

#include "fq_cuda.h"

namespace fqc {

// Error carried from the implementation to the ABI wrapper (status + message).
struct Failure {
  fq_status code;
  std::string msg;
};

[[noreturn]] void fail(fq_status code, const std::string& msg);
void check_cuda(cudaError_t e, const char* what);
void set_last_error(const std::string& msg);

#define FQ_CUDA(call) ::fqc::check_cuda((call), #call)

// Runs `body` and converts a Failure (or any exception) into a status + fq_last_error().
template <class F>
fq_status guarded(F&& body) {
  try {
    body();
    return FQ_OK;
  } catch (const Failure& f) {
    set_last_error(f.msg);
    return f.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return FQ_E_CUDA;
  }
}

}  // namespace fqc

// ------------------------------------------------------------------ context
struct fq_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  int64_t launches = 0;
  // scratch: grows on demand, never shrinks
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  void* ensure_scratch(size_t bytes);
  // stream-K fix-up workspace of transient (stand-alone) GEMV programs
  float* gemv_fix = nullptr;
  unsigned int* gemv_flags = nullptr;
  unsigned int* launch_ctr = nullptr;  // [epoch, done] of the program kernels on this context
  float* gemm_ws = nullptr;  // split-K partial sums of the tensor-core GEMM (grown on demand)
  float* direct_ws = nullptr;     // split-K partials of the stand-alone GEMV (gemv_direct.cu)
  size_t direct_ws_bytes = 0;
  unsigned* direct_cnt = nullptr; // its per-tile arrival counters (self-resetting)
  size_t direct_cnt_n = 0;
  size_t gemm_ws_bytes = 0;
  std::vector<void*> retired;  // outgrown workspaces captured graphs may still point at (freed at destroy)
  // bumped whenever a layer's resident copies change (upload, device quantization): models
  // drop step programs and captured graphs built against older weight pointers
  uint64_t weight_epoch = 0;
};

// ------------------------------------------------------------------ tiled fast-path layout
// Each rung of a linear keeps, next to its canonical QuantizedTensor arrays, a tiled copy the
// decode GEMV streams: blocks of 16 rows x 128 codes, tile-major ([tile][k-block]), each block
// self-contained:
//   codes  W8: 2048 B = [i 0..3][lane 0..31] 16-byte words; word i of lane t feeds the m16n8k16
//              MMAs 2i and 2i+1 of the block: per MMA j two u32
//              {q(r,k0), q(r,k0+1), q(r+8,k0), q(r+8,k0+1)}, {same at k0+8}
//              with r = t/4, k0 = 16j + 2(t%4) (the A-fragment order of mma.sync m16n8k16).
//          W4: 1024 B = [i 0..1][lane] 16-byte words; u32 u of word i feeds MMA 4i+u with nibbles
//              (low to high) q(r,k0), q(r,k0+8), q(r+8,k0), q(r+8,k0+8), q(r,k0+1), q(r,k0+9),
//              q(r+8,k0+1), q(r+8,k0+9).
//   meta   16 f32 scales (rows 0..15) + 16 u8 zero points (z - zp_base).
// Rows past N and codes past K are zero (scale 0); a block lies in one quantization group, so
// the layout exists when G % 128 == 0 or G >= K and the zero points span <= 255.
constexpr int kTileRows = 16;
constexpr int kBlockK = 128;
constexpr int kBlockBytes8 = 2048 + 80;
constexpr int kBlockBytes4 = 1024 + 80;

// One resident precision copy of a linear layer.
struct fq_rung_store {
  bool present = false;
  int bits = 8;            // 8 or 4
  int mode = FQ_MODE_ASYM;
  uint8_t* payload = nullptr;   // canonical row-major packed codes (device)
  int64_t payload_bytes = 0;
  float* scale = nullptr;       // [N, ng_pad]
  int32_t* zp32 = nullptr;      // [N, ng] effective zero point (z + stored offset), always kept
  uint8_t* tiles = nullptr;     // tiled fast-path copy (see above), or null
  int64_t tiles_bytes = 0;
  int32_t zp_base = 0;          // tiles hold z - zp_base in one byte
  bool zp_fits_u8 = false;      // fast kernel usable
};

struct fq_layer {
  fq_ctx* ctx = nullptr;
  int64_t N = 0, K = 0, G = 0;  // out, in, group (G == K for per-row)
  int64_t ng = 0;               // groups per row = ceil(K / G)
  int64_t ng_pad = 0;           // scale row stride (multiple of 4 floats = 16 B)
  int64_t zp_pad = 0;           // u8 zero-point row stride (multiple of 16 B)
  float* fp = nullptr;          // fp32 [N, K] (optional)
  float* bias = nullptr;        // fp32 [N] (optional)
  fq_rung_store r8, r4;
  bool borrowed = false;        // owned by a model

  const fq_rung_store& store(int rung) const { return rung == FQ_RUNG_INT4 ? r4 : r8; }
  fq_rung_store& store(int rung) { return rung == FQ_RUNG_INT4 ? r4 : r8; }
  bool has(int rung) const {
    if (rung == FQ_RUNG_FP) return fp != nullptr;
    if (rung == FQ_RUNG_INT8) return r8.present;
    if (rung == FQ_RUNG_INT4) return r4.present;
    return false;
  }
};

namespace fqc {

// ---------------------------------------------------------------- GEMV launch API
// A multi-matrix GEMV: up to 3 matrices with identical [N, K] shapes sharing one input
// (QKV, gate/up).  Each CTA owns the same row range of every matrix.
enum Epilogue : int {
  EPI_STORE = 0,     // y[b][m*N + row] = acc (+bias), dtype y_dtype
  EPI_RESIDUAL = 1,  // resid[b][row] += acc (fp32), per-CTA sum of squares -> partials
  EPI_SWIGLU = 2,    // y[b][row] = silu(acc_gate) * acc_up   (2 matrices)
  EPI_SPLIT3 = 3     // y_m[b][row] = acc_m for 3 matrices (q, k, v outputs)
};

struct GemvMatrix {
  const fq_layer* layer = nullptr;
  const uint8_t* rung_table = nullptr;  // device: rung per batch row (stride below) or null
  int64_t rung_stride = 0;              // bytes between batch rows in rung_table
  int rung = FQ_RUNG_INT8;              // used when rung_table == null
  void* y = nullptr;                    // per-matrix output (EPI_SPLIT3)
};

struct GemvLaunch {
  GemvMatrix mat[3];
  int nmat = 1;
  int64_t batch = 1;
  // input activations [batch, K]
  const void* x = nullptr;
  int x_dtype = FQ_DT_F32;
  int64_t x_stride = 0;  // elements
  // optional fused RMSNorm prologue: x is the fp32 residual; h = round_act(x*rstd*gain)
  const float* norm_gain = nullptr;
  const float* norm_partials = nullptr;  // [batch][partials_stride] sums of squares
  int n_partials = 0;
  int partials_stride = 0;               // 0 = n_partials
  float norm_eps = 1e-5f;
  int act_dtype = FQ_DT_BF16;  // rounding applied to the normalized activations
  // output
  int epi = EPI_STORE;
  void* y = nullptr;
  int y_dtype = FQ_DT_F32;
  int64_t y_stride = 0;        // elements between batch rows of y
  float* resid = nullptr;      // EPI_RESIDUAL
  int64_t resid_stride = 0;
  float* out_partials = nullptr;  // EPI_RESIDUAL: [batch, out_n_partials]
  int out_n_partials = 0;
  bool pdl = false;            // launch with programmatic stream serialization
  void* stat_part = nullptr;   // EPI_STORE: fused softmax partials [batch][grid] (StatPart)
  const void* xfrag = nullptr; // input in B-fragment order (see Phase::xfrag), or null
  void* yfrag = nullptr;       // EPI_SWIGLU: also write the output in B-fragment order
};

bool gemv_fast_supported(const fq_layer* L, int rung);
int gemv_fast_grid(const fq_ctx* ctx, int64_t N);
// Returns the grid size used (the residual epilogue writes one sum-of-squares partial per CTA;
// out_n_partials must be >= #SM x 4).
int launch_gemv_fast(fq_ctx* ctx, const GemvLaunch& g);
// Stand-alone dequant-GEMV of one linear at one precision (fq_gemv FAST; gemv_direct.cu).
void launch_gemv_direct(fq_ctx* ctx, const fq_layer* L, int rung, int64_t batch, const void* x, int x_dtype, void* y,
                        int y_dtype);
double time_gemv_chain(fq_ctx* ctx, const GemvLaunch* gs, int n, int reps);
void launch_gemv_exact(fq_ctx* ctx, const fq_layer* L, int rung, int64_t batch, const void* x,
                       int x_dtype, void* y, int y_dtype);

// Activations of the tcgen05 GEMM are stored pre-tiled: bf16 [T/128][K/128][128 x 128] with each
// 32 KB tile in the UMMA canonical K-major layout (8 rows x 16 B core matrices, K-adjacent core
// matrices 128 B apart, 8-row groups 2 KB apart), so one 1-D bulk copy moves a tile.  Rows past T
// and columns past K stay zero (buffers are cleared at allocation).  Element offset of (t, k):
__host__ __device__ inline int64_t tiled_act_offset(int t, int64_t k, int nkb) {
  return ((static_cast<int64_t>(t >> 7) * nkb + (k >> 7)) << 14) + (((t & 127) >> 3) << 10) + (((k & 127) >> 3) << 6) +
         ((t & 7) << 3) + (k & 7);
}
int64_t tiled_act_elems(int64_t T, int64_t K);  // buffer size (elements) for T rows of K features
void launch_tile_acts(fq_ctx* ctx, const void* x, int x_dtype, int64_t x_stride, int64_t T, int64_t K, void* xt,
                      int out_dtype = FQ_DT_BF16);

// tcgen05 dequant-GEMM: y[T, N] (fp32, row stride y_stride) = x[T, K] . dequant(W_rung)^T with x the
// tiled bf16 (x_dtype FQ_DT_BF16) or fp16 (FQ_DT_F16) activations above; the tensor cores multiply the exact integer codes (q - z) and the
// per-group fp32 scale is applied per 128-code k-block in the epilogue (no weight rounding);
// accumulate: y += instead (the residual add of the O / down projections)
// row_rung (device, optional): rung of each row at stride rr_stride; only rows at `rung` are
// written (a batch whose rows decode at different precisions runs one launch per copy)
void launch_gemm_dq(fq_ctx* ctx, const fq_layer* L, int rung, int64_t T, const void* xt, int x_dtype, float* y,
                    int64_t y_stride, bool accumulate = false, const uint8_t* row_rung = nullptr,
                    int64_t rr_stride = 0);
// One launch for several (linear, rung) products of the SAME tiled activations (equal K): q/k/v,
// gate/up, the copies of one linear in a mixed batch.  Work is split evenly over all SMs.
struct GemmJob {
  const fq_layer* L;
  int rung;
  float* y;
  int64_t y_stride;
  bool accumulate;
  const uint8_t* row_rung;  // optional, as in launch_gemm_dq
  int64_t rr_stride;
};
void launch_gemm_group(fq_ctx* ctx, const GemmJob* jobs, int n_jobs, int64_t T, const void* xt);

// row-parallel prefill kernels (prefill.cu; llama arch; GEMM operands bf16, stored tiled)
// true (and cleared) when a prefill GEMM operand exceeded fp16's range since the last call
bool prefill_overflow_take(fq_ctx* ctx);
void prefill_embed(fq_ctx* ctx, const float* tok_emb, const int32_t* tokens_dev, int T, int64_t d, float* x);
void prefill_rmsnorm(fq_ctx* ctx, const float* x, int T, int64_t d, const float* g, float eps, void* h16, int act_dtype);
void prefill_rope_kv(fq_ctx* ctx, const float* q, const float* k, const float* v, int T, int H, int hd,
                     const float2* cs, float* qr, __half* kv_layer, int64_t max_seq, int act_dtype);
void prefill_swiglu(fq_ctx* ctx, const float* g, const float* u, int64_t n, int64_t f, void* out16, int act_dtype);

// batched decode on the tensor-core path (batched.cu): per-row positions / slots
void batched_rope_append(fq_ctx* ctx, const float* q, const float* k, const float* v, int B, int H, int hd,
                         const float2* cs, const int32_t* pos, const int32_t* slots, __half* kv, int64_t slot_stride,
                         int64_t layer_off, int64_t max_seq, float* qr, int act_dtype);
// pos / slots null: the T rows of one prompt in slot slot0 (row t attends keys 0..t)
void batched_attention(fq_ctx* ctx, const float* qr, const __half* kv, int B, int H, int hd, const int32_t* pos,
                       const int32_t* slots, int64_t slot_stride, int64_t layer_off, int64_t max_seq, void* out16,
                       int act_dtype, int slot0 = 0);

// statistics
void launch_softmax_stats(fq_ctx* ctx, const float* logits, int64_t rows, int64_t vocab,
                          int64_t row_stride, fq_row_stats* out);
void launch_kl_rows(fq_ctx* ctx, const void* lq, const void* lp, int dtype, int64_t rows,
                    int64_t vocab, double* kl, double* ent);
double hist_kl(fq_ctx* ctx, const fq_layer* L, int rung, int bins);

// quantization / generation
void quantize_device(fq_ctx* ctx, fq_layer* L, int rung, int mode, const float* w_dev);
void fill_normal(fq_ctx* ctx, float* dst, int64_t n, uint64_t seed, uint64_t stream, float std);
void finalize_rung_meta(fq_ctx* ctx, fq_layer* L, int rung);  // zp32 -> zp8/zp_base

// allocation helpers
void* dmalloc(size_t bytes);
void dfree(void* p);

inline int ceil_div_i(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

}  // namespace fqc
