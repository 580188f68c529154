// C-ABI implementation: contexts, the resident weight store and the stateless kernels.
// Every entry point converts internal failures into an fq_status + fq_last_error().
#include <vector>
#include "fq_internal.cuh"

#include <cstdlib>
#include <cstring>
#include <string>

namespace fqc {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }

void fail(fq_status code, const std::string& msg) { throw Failure{code, msg}; }

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(FQ_E_CUDA, std::string("CUDA error ") + cudaGetErrorString(e) + " in " + what);
}

void* dmalloc(size_t bytes) {
  void* p = nullptr;
  if (bytes == 0) bytes = 16;
  check_cuda(cudaMalloc(&p, bytes), "cudaMalloc");
  return p;
}

void dfree(void* p) {
  if (p) cudaFree(p);
}

}  // namespace fqc

using namespace fqc;

void* fq_ctx::ensure_scratch(size_t bytes) {
  if (bytes > scratch_bytes) {
    FQ_CUDA(cudaStreamSynchronize(stream));
    dfree(scratch);
    scratch = dmalloc(bytes);
    scratch_bytes = bytes;
  }
  return scratch;
}

namespace {

void require(bool cond, fq_status code, const char* msg) {
  if (!cond) fail(code, msg);
}

void free_store(fq_rung_store& s) {
  dfree(s.payload);
  dfree(s.scale);
  dfree(s.tiles);
  dfree(s.zp32);
  s = fq_rung_store{};
}

}  // namespace

extern "C" {

const char* fq_last_error(void) { return g_last_error.c_str(); }

int32_t fq_abi_version(void) { return FQ_ABI_VERSION; }

fq_status fq_ctx_create(int32_t device, fq_ctx** out) {
  return guarded([&] {
    require(out != nullptr, FQ_E_INPUT, "fq_ctx_create: null out");
    int n = 0;
    FQ_CUDA(cudaGetDeviceCount(&n));
    require(device >= 0 && device < n, FQ_E_CONFIG, "fq_ctx_create: no such CUDA device");
    FQ_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    FQ_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) fail(FQ_E_CONFIG, "fq_ctx_create: this library is built for sm_100a (B200)");
    auto* c = new fq_ctx();
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    FQ_CUDA(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
    c->stream = c->own_stream;
    *out = c;
  });
}

fq_status fq_ctx_destroy(fq_ctx* ctx) {
  return guarded([&] {
    if (!ctx) return;
    cudaStreamSynchronize(ctx->stream);
    dfree(ctx->scratch);
    dfree(ctx->gemv_fix);
    dfree(ctx->gemv_flags);
    dfree(ctx->launch_ctr);
    dfree(ctx->gemm_ws);
    dfree(ctx->direct_ws);
    dfree(ctx->direct_cnt);
    for (void* r : ctx->retired) dfree(r);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    delete ctx;
  });
}

fq_status fq_ctx_set_stream(fq_ctx* ctx, void* stream) {
  return guarded([&] {
    require(ctx != nullptr, FQ_E_INPUT, "null ctx");
    ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
  });
}

fq_status fq_ctx_get_stream(fq_ctx* ctx, void** stream_out) {
  return guarded([&] {
    require(ctx != nullptr && stream_out != nullptr, FQ_E_INPUT, "null argument");
    *stream_out = ctx->stream;
  });
}

fq_status fq_ctx_synchronize(fq_ctx* ctx) {
  return guarded([&] {
    require(ctx != nullptr, FQ_E_INPUT, "null ctx");
    FQ_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

fq_status fq_ctx_launch_count(fq_ctx* ctx, int64_t* out) {
  return guarded([&] {
    require(ctx != nullptr && out != nullptr, FQ_E_INPUT, "null argument");
    *out = ctx->launches;
  });
}

// ------------------------------------------------------------------ layers
fq_status fq_layer_create(fq_ctx* ctx, int64_t out_features, int64_t in_features, int64_t group_size,
                          fq_layer** out) {
  return guarded([&] {
    require(ctx != nullptr && out != nullptr, FQ_E_INPUT, "null argument");
    require(out_features >= 1 && in_features >= 1, FQ_E_DIMENSION, "layer: dimensions must be >= 1");
    require(group_size >= 0, FQ_E_CONFIG, "layer: negative group size");
    auto* L = new fq_layer();
    L->ctx = ctx;
    L->N = out_features;
    L->K = in_features;
    L->G = (group_size == 0 || group_size >= in_features) ? in_features : group_size;
    L->ng = (L->K + L->G - 1) / L->G;
    L->ng_pad = (L->ng + 3) / 4 * 4;
    L->zp_pad = (L->ng + 15) / 16 * 16;
    *out = L;
  });
}

fq_status fq_layer_destroy(fq_layer* L) {
  return guarded([&] {
    if (!L) return;
    require(!L->borrowed, FQ_E_STATE, "layer is owned by a model");
    dfree(L->fp);
    dfree(L->bias);
    free_store(L->r8);
    free_store(L->r4);
    delete L;
  });
}

fq_status fq_layer_upload_quantized(fq_layer* L, int32_t rung, int32_t mode, const uint8_t* payload_host,
                                    int64_t payload_bytes, const float* scale_host, const int32_t* zero_point_host,
                                    int64_t n_groups) {
  return guarded([&] {
    require(L != nullptr && payload_host && scale_host && zero_point_host, FQ_E_INPUT, "null argument");
    require(rung == FQ_RUNG_INT8 || rung == FQ_RUNG_INT4, FQ_E_CONFIG, "upload: rung must be 8 or 4");
    require(mode == FQ_MODE_ASYM || mode == FQ_MODE_SYM, FQ_E_CONFIG, "upload: bad quantization mode");
    const int bits = rung == FQ_RUNG_INT8 ? 8 : 4;
    const int64_t expect = (L->N * L->K * bits + 7) / 8;
    if (payload_bytes != expect)
      fail(FQ_E_FORMAT, "quantized tensor payload length " + std::to_string(payload_bytes) +
                            " does not match expected " + std::to_string(expect));
    require(n_groups == L->N * L->ng, FQ_E_FORMAT, "quantized tensor scale/zero-point length mismatch");
    for (int64_t i = 0; i < n_groups; ++i)
      if (!(scale_host[i] > 0.0f) || !std::isfinite(scale_host[i]))
        fail(FQ_E_FORMAT, "quantized tensor scale must be positive and finite");
    fq_rung_store& st = L->store(rung);
    if (st.present && st.bits != bits) free_store(st);
    if (!st.present) {
      st.payload = static_cast<uint8_t*>(dmalloc(payload_bytes));
      st.scale = static_cast<float*>(dmalloc(sizeof(float) * L->N * L->ng_pad));
      st.zp32 = static_cast<int32_t*>(dmalloc(sizeof(int32_t) * n_groups));
    }
    st.bits = bits;
    st.mode = mode;
    st.payload_bytes = payload_bytes;
    cudaStream_t s = L->ctx->stream;
    FQ_CUDA(cudaMemcpyAsync(st.payload, payload_host, payload_bytes, cudaMemcpyHostToDevice, s));
    // device layout: scale rows padded to ng_pad (a fixed, invertible re-layout)
    std::vector<float> spad(static_cast<size_t>(L->N * L->ng_pad), 0.0f);
    for (int64_t r = 0; r < L->N; ++r)
      std::memcpy(&spad[r * L->ng_pad], scale_host + r * L->ng, sizeof(float) * L->ng);
    FQ_CUDA(cudaMemcpyAsync(st.scale, spad.data(), sizeof(float) * spad.size(), cudaMemcpyHostToDevice, s));
    // effective zero point = z + stored offset (symmetric codes are stored offset by 2^(n-1)-1)
    std::vector<int32_t> zeff(zero_point_host, zero_point_host + n_groups);
    const int32_t off = mode == FQ_MODE_SYM ? (1 << (bits - 1)) - 1 : 0;
    for (auto& z : zeff) z += off;
    FQ_CUDA(cudaMemcpyAsync(st.zp32, zeff.data(), sizeof(int32_t) * n_groups, cudaMemcpyHostToDevice, s));
    FQ_CUDA(cudaStreamSynchronize(s));
    st.present = true;
    finalize_rung_meta(L->ctx, L, rung);
  });
}

fq_status fq_layer_download_quantized(const fq_layer* L, int32_t rung, uint8_t* payload_host, float* scale_host,
                                      int32_t* zero_point_host) {
  return guarded([&] {
    require(L != nullptr, FQ_E_INPUT, "null layer");
    require(rung == FQ_RUNG_INT8 || rung == FQ_RUNG_INT4, FQ_E_CONFIG, "download: rung must be 8 or 4");
    const fq_rung_store& st = L->store(rung);
    require(st.present, FQ_E_STATE, "download: rung not resident");
    const int64_t ngr = L->N * L->ng;
    cudaStream_t s = L->ctx->stream;
    if (payload_host) FQ_CUDA(cudaMemcpyAsync(payload_host, st.payload, st.payload_bytes, cudaMemcpyDeviceToHost, s));
    std::vector<float> spad(static_cast<size_t>(L->N * L->ng_pad));
    if (scale_host) FQ_CUDA(cudaMemcpyAsync(spad.data(), st.scale, sizeof(float) * spad.size(), cudaMemcpyDeviceToHost, s));
    if (zero_point_host) {
      FQ_CUDA(cudaMemcpyAsync(zero_point_host, st.zp32, sizeof(int32_t) * ngr, cudaMemcpyDeviceToHost, s));
    }
    FQ_CUDA(cudaStreamSynchronize(s));
    if (scale_host)
      for (int64_t r = 0; r < L->N; ++r) std::memcpy(scale_host + r * L->ng, &spad[r * L->ng_pad], sizeof(float) * L->ng);
    if (zero_point_host && st.mode == FQ_MODE_SYM) {
      const int32_t off = (1 << (st.bits - 1)) - 1;
      for (int64_t i = 0; i < ngr; ++i) zero_point_host[i] -= off;
    }
  });
}

fq_status fq_layer_upload_fp(fq_layer* L, const float* w) {
  return guarded([&] {
    require(L != nullptr && w != nullptr, FQ_E_INPUT, "null argument");
    if (!L->fp) L->fp = static_cast<float*>(dmalloc(sizeof(float) * L->N * L->K));
    FQ_CUDA(cudaMemcpyAsync(L->fp, w, sizeof(float) * L->N * L->K, cudaMemcpyHostToDevice, L->ctx->stream));
    FQ_CUDA(cudaStreamSynchronize(L->ctx->stream));
  });
}

fq_status fq_layer_upload_bias(fq_layer* L, const float* b) {
  return guarded([&] {
    require(L != nullptr && b != nullptr, FQ_E_INPUT, "null argument");
    if (!L->bias) L->bias = static_cast<float*>(dmalloc(sizeof(float) * L->N));
    FQ_CUDA(cudaMemcpyAsync(L->bias, b, sizeof(float) * L->N, cudaMemcpyHostToDevice, L->ctx->stream));
    FQ_CUDA(cudaStreamSynchronize(L->ctx->stream));
  });
}

fq_status fq_layer_download_fp(const fq_layer* L, float* w_host, int32_t* present) {
  return guarded([&] {
    require(L != nullptr && present != nullptr, FQ_E_INPUT, "null argument");
    *present = L->fp != nullptr ? 1 : 0;
    if (L->fp && w_host) {
      FQ_CUDA(cudaMemcpyAsync(w_host, L->fp, sizeof(float) * L->N * L->K, cudaMemcpyDeviceToHost, L->ctx->stream));
      FQ_CUDA(cudaStreamSynchronize(L->ctx->stream));
    }
  });
}

fq_status fq_layer_download_bias(const fq_layer* L, float* b_host, int32_t* present) {
  return guarded([&] {
    require(L != nullptr && present != nullptr, FQ_E_INPUT, "null argument");
    *present = L->bias != nullptr ? 1 : 0;
    if (L->bias && b_host) {
      FQ_CUDA(cudaMemcpyAsync(b_host, L->bias, sizeof(float) * L->N, cudaMemcpyDeviceToHost, L->ctx->stream));
      FQ_CUDA(cudaStreamSynchronize(L->ctx->stream));
    }
  });
}

fq_status fq_layer_quantize_device(fq_layer* L, int32_t rung, int32_t mode, const float* w_dev) {
  return guarded([&] {
    require(L != nullptr && w_dev != nullptr, FQ_E_INPUT, "null argument");
    quantize_device(L->ctx, L, rung, mode, w_dev);
  });
}

fq_status fq_layer_has(const fq_layer* L, int32_t rung, int32_t* out) {
  return guarded([&] {
    require(L != nullptr && out != nullptr, FQ_E_INPUT, "null argument");
    *out = L->has(rung) ? 1 : 0;
  });
}

fq_status fq_layer_shape(const fq_layer* L, int64_t* n, int64_t* k, int64_t* g) {
  return guarded([&] {
    require(L != nullptr, FQ_E_INPUT, "null layer");
    if (n) *n = L->N;
    if (k) *k = L->K;
    if (g) *g = L->G;
  });
}

fq_status fq_layer_bytes(const fq_layer* L, int32_t rung, int64_t batch, int64_t* out) {
  return guarded([&] {
    require(L != nullptr && out != nullptr, FQ_E_INPUT, "null argument");
    int64_t w;
    if (rung == FQ_RUNG_FP) w = L->N * L->K * 4;
    else w = (L->N * L->K * (rung == FQ_RUNG_INT8 ? 8 : 4) + 7) / 8 + L->N * L->ng * 5;
    *out = w + batch * L->K * 2 + batch * L->N * 2;
  });
}

fq_status fq_gemv(fq_ctx* ctx, const fq_layer* L, int32_t rung, int64_t batch, const void* x_dev, int32_t x_dtype,
                  void* y_dev, int32_t y_dtype, int32_t numerics) {
  return guarded([&] {
    require(ctx != nullptr && L != nullptr && x_dev != nullptr && y_dev != nullptr, FQ_E_INPUT, "null argument");
    require(batch >= 1, FQ_E_DIMENSION, "gemv: batch must be >= 1");
    require(x_dtype >= FQ_DT_F32 && x_dtype <= FQ_DT_BF16 && y_dtype >= FQ_DT_F32 && y_dtype <= FQ_DT_BF16,
            FQ_E_CONFIG, "gemv: bad dtype");
    if (!L->has(rung)) fail(FQ_E_STATE, std::string("layer: precision '") +
                                            (rung == FQ_RUNG_FP ? "fp" : rung == FQ_RUNG_INT8 ? "8" : "4") +
                                            "' not available");
    const bool fast = numerics == FQ_NUMERICS_FAST && gemv_fast_supported(L, rung) && L->bias == nullptr;
    if (!fast) {
      launch_gemv_exact(ctx, L, rung, batch, x_dev, x_dtype, y_dev, y_dtype);
      return;
    }
    // kernel choice by shape (measured, profiles/r03_gemv_sweep_c2.jsonl): the direct kernel
    // (gemv_direct.cu) starts streaming at once and keeps every batch row of a > 8-row batch in
    // one pass; the step-program form (a one-phase persistent program) sustains more bandwidth
    // on long layers (N >= 16384, the 32000-row head) at up to 8 rows
    static const bool all_direct = std::getenv("FQ_GEMV_DIRECT_ALL") != nullptr;  // A/B measurement
    if (L->N >= 16384 && batch <= 8 && !all_direct) {
      GemvLaunch g;
      g.mat[0].layer = L;
      g.mat[0].rung = rung;
      g.nmat = 1;
      g.batch = batch;
      g.x = x_dev;
      g.x_dtype = x_dtype;
      g.x_stride = L->K;
      g.epi = EPI_STORE;
      g.y = y_dev;
      g.y_dtype = y_dtype;
      g.y_stride = L->N;
      launch_gemv_fast(ctx, g);
      return;
    }
    launch_gemv_direct(ctx, L, rung, batch, x_dev, x_dtype, y_dev, y_dtype);
  });
}

fq_status fq_gemv_chain_time(fq_ctx* ctx, const fq_layer* const* layers, int32_t n, int32_t rung, int64_t batch,
                             const void* x_dev, int32_t x_dtype, void* const* y_devs, int32_t y_dtype, int32_t reps,
                             double* ms_per_launch) {
  return guarded([&] {
    require(ctx != nullptr && layers != nullptr && x_dev != nullptr && y_devs != nullptr && ms_per_launch != nullptr,
            FQ_E_INPUT, "null argument");
    require(n >= 1 && batch >= 1 && reps >= 1, FQ_E_DIMENSION, "gemv chain: n, batch and reps must be >= 1");
    require(x_dtype >= FQ_DT_F32 && x_dtype <= FQ_DT_BF16 && y_dtype >= FQ_DT_F32 && y_dtype <= FQ_DT_BF16,
            FQ_E_CONFIG, "gemv: bad dtype");
    std::vector<GemvLaunch> gs(n);
    for (int i = 0; i < n; ++i) {
      const fq_layer* L = layers[i];
      require(L != nullptr && y_devs[i] != nullptr, FQ_E_INPUT, "null argument");
      require(L->K == layers[0]->K && L->N == layers[0]->N, FQ_E_DIMENSION, "gemv chain: layers differ in shape");
      require(gemv_fast_supported(L, rung) && L->bias == nullptr, FQ_E_STATE, "gemv chain: rung not on the fast path");
      GemvLaunch& g = gs[i];
      g.mat[0].layer = L;
      g.mat[0].rung = rung;
      g.nmat = 1;
      g.batch = batch;
      g.x = x_dev;
      g.x_dtype = x_dtype;
      g.x_stride = L->K;
      g.epi = EPI_STORE;
      g.y = y_devs[i];
      g.y_dtype = y_dtype;
      g.y_stride = L->N;
    }
    *ms_per_launch = time_gemv_chain(ctx, gs.data(), n, reps);
  });
}

fq_status fq_gemm(fq_ctx* ctx, const fq_layer* L, int32_t rung, int64_t rows, const void* x_dev, int64_t x_stride,
                  float* y_dev, int64_t y_stride) {
  return guarded([&] {
    require(ctx != nullptr && L != nullptr && x_dev != nullptr && y_dev != nullptr, FQ_E_INPUT, "null argument");
    require(rows >= 1, FQ_E_DIMENSION, "gemm: rows must be >= 1");
    require(x_stride >= L->K && y_stride >= L->N, FQ_E_DIMENSION, "gemm: row stride smaller than the row");
    // row-major bf16 -> the GEMM's tiled operand layout (scratch), then the tcgen05 GEMM
    const size_t bytes = 2 * static_cast<size_t>(tiled_act_elems(rows, L->K));
    void* xt = ctx->ensure_scratch(bytes);
    FQ_CUDA(cudaMemsetAsync(xt, 0, bytes, ctx->stream));
    launch_tile_acts(ctx, x_dev, FQ_DT_BF16, x_stride, rows, L->K, xt, FQ_DT_F16);  // bf16 -> fp16: exact in range
    launch_gemm_dq(ctx, L, rung, rows, xt, FQ_DT_F16, y_dev, y_stride);
  });
}

int64_t fq_tiled_activation_bytes(int64_t rows, int64_t K) {
  return rows < 1 || K < 1 ? 0 : 2 * tiled_act_elems(rows, K);
}

fq_status fq_tile_activations(fq_ctx* ctx, const void* x_dev, int32_t x_dtype, int64_t x_stride, int64_t rows,
                              int64_t K, int32_t out_dtype, void* xt_dev) {
  return guarded([&] {
    require(ctx != nullptr && x_dev != nullptr && xt_dev != nullptr, FQ_E_INPUT, "null argument");
    require(rows >= 1 && K >= 1 && x_stride >= K, FQ_E_DIMENSION, "tile_activations: bad shape");
    require(x_dtype >= FQ_DT_F32 && x_dtype <= FQ_DT_BF16, FQ_E_CONFIG, "tile_activations: bad input dtype");
    require(out_dtype == FQ_DT_F16, FQ_E_CONFIG, "tile_activations: the GEMM operand format is fp16");
    launch_tile_acts(ctx, x_dev, x_dtype, x_stride, rows, K, xt_dev, out_dtype);
  });
}

fq_status fq_gemm_tiled(fq_ctx* ctx, const fq_layer* L, int32_t rung, int64_t rows, const void* xt_dev, int32_t x_dtype,
                        float* y_dev, int64_t y_stride, int32_t accumulate) {
  return guarded([&] {
    require(ctx != nullptr && L != nullptr && xt_dev != nullptr && y_dev != nullptr, FQ_E_INPUT, "null argument");
    require(rows >= 1, FQ_E_DIMENSION, "gemm: rows must be >= 1");
    require(y_stride >= L->N, FQ_E_DIMENSION, "gemm: row stride smaller than the row");
    launch_gemm_dq(ctx, L, rung, rows, xt_dev, x_dtype, y_dev, y_stride, accumulate != 0);
  });
}

fq_status fq_softmax_stats(fq_ctx* ctx, const float* logits_dev, int64_t rows, int64_t vocab, fq_row_stats* stats_dev) {
  return guarded([&] {
    require(ctx != nullptr && logits_dev != nullptr && stats_dev != nullptr, FQ_E_INPUT, "null argument");
    if (vocab < 1) fail(FQ_E_DIMENSION, "ppl_entropy: empty logits");
    launch_softmax_stats(ctx, logits_dev, rows, vocab, vocab, stats_dev);
  });
}

fq_status fq_kl_rows(fq_ctx* ctx, const void* lq, const void* lp, int32_t dtype, int64_t rows, int64_t vocab,
                     double* kl_dev, double* entropy_dev) {
  return guarded([&] {
    require(ctx != nullptr && lq && lp && kl_dev, FQ_E_INPUT, "null argument");
    require(vocab >= 1, FQ_E_DIMENSION, "kl_rows: empty rows");
    launch_kl_rows(ctx, lq, lp, dtype, rows, vocab, kl_dev, entropy_dev);
  });
}

fq_status fq_hist_kl(fq_ctx* ctx, const fq_layer* L, int32_t rung, int32_t bins, double* kl_host) {
  return guarded([&] {
    require(ctx != nullptr && L != nullptr && kl_host != nullptr, FQ_E_INPUT, "null argument");
    *kl_host = hist_kl(ctx, L, rung, bins);
  });
}

fq_status fq_fill_normal(fq_ctx* ctx, float* dst_dev, int64_t n, uint64_t seed, uint64_t stream_id, float std) {
  return guarded([&] {
    require(ctx != nullptr && (dst_dev != nullptr || n == 0), FQ_E_INPUT, "null argument");
    fill_normal(ctx, dst_dev, n, seed, stream_id, std);
  });
}

}  // extern "C"
