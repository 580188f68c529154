// Vocab-row statistics and KL reductions (K4, K5 of SURVEY §2.1).
//
//  * softmax_stats_kernel — ppl_entropy / fault_tolerance / argmax_token of a logits row
//    (/root/reference/proj/src/scheduler.cpp:13-49, src/engine.cpp:144-155).  Same
//    arithmetic as softmax_double: max in double, e_i = exp(l_i - max), p_i = e_i / sum,
//    H = -sum_{p>0} p ln p, PPLE = exp(H); only the summation order differs (tree).
//  * kl_rows_kernel — logit-mode calibration: KL(softmax(l_q) || softmax(l_p)) and H(p_q)
//    per row, double accumulation of fp32 exponentials (BASELINE config 4).
//  * hist kernels — weight_histogram counts (src/analyzer.cpp:31-63) of the fp weights and of
//    the dequantized rung over shared edges; the smoothing/normalisation/KL (a few thousand
//    doubles) is finished on the host in the reference's sequential order so the switch-plan
//    ordering matches the reference exactly.
#include "fq_internal.cuh"

#include <cfloat>
#include <cmath>

namespace fqc {
namespace {

constexpr int kStatThreads = 1024;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum (thread-strided partials -> warp butterfly -> warps in order).
__device__ double block_sum(double v, double* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0) {
    for (int w = 0; w < nw; ++w) t += sh[w];
    sh[32] = t;
  }
  __syncthreads();
  return sh[32];
}

struct MaxArg {
  float v;
  int i;
};
__device__ __forceinline__ MaxArg better(MaxArg a, MaxArg b) {
  // strict > with lowest index on ties (argmax_token, engine.cpp:144-155)
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}

__device__ MaxArg block_argmax(MaxArg m, MaxArg* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    MaxArg other{__shfl_xor_sync(0xffffffffu, m.v, o), __shfl_xor_sync(0xffffffffu, m.i, o)};
    m = better(m, other);
  }
  __syncthreads();
  if (lane == 0) sh[warp] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    MaxArg t = sh[0];
    for (int w = 1; w < nw; ++w) t = better(t, sh[w]);
    sh[32] = t;
  }
  __syncthreads();
  return sh[32];
}

struct Top2 {
  double a, b;  // a >= b, duplicates kept
};
__device__ __forceinline__ Top2 merge2(Top2 x, Top2 y) {
  Top2 r;
  r.a = fmax(x.a, y.a);
  r.b = fmax(fmin(x.a, y.a), fmax(x.b, y.b));
  return r;
}

__global__ void __launch_bounds__(kStatThreads) softmax_stats_kernel(const float* __restrict__ logits,
                                                                     int64_t vocab, int64_t stride,
                                                                     fq_row_stats* __restrict__ out) {
  __shared__ double shd[33];
  __shared__ MaxArg shm[33];
  __shared__ Top2 sht[33];
  const float* l = logits + blockIdx.x * stride;
  MaxArg m{-FLT_MAX, 0x7fffffff};
  bool first = true;
  for (int64_t i = threadIdx.x; i < vocab; i += blockDim.x) {
    MaxArg c{l[i], static_cast<int>(i)};
    if (first) { m = c; first = false; }
    else m = better(m, c);
  }
  if (first) m = MaxArg{-INFINITY, 0x7fffffff};
  const MaxArg mx = block_argmax(m, shm);
  const double dmax = static_cast<double>(mx.v);
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < vocab; i += blockDim.x) s += exp(static_cast<double>(l[i]) - dmax);
  const double sum = block_sum(s, shd);
  double h = 0.0;
  Top2 t{-1.0, -1.0};
  for (int64_t i = threadIdx.x; i < vocab; i += blockDim.x) {
    const double p = exp(static_cast<double>(l[i]) - dmax) / sum;
    if (p > 0.0) h -= p * log(p);
    t = merge2(t, Top2{p, -1.0});
  }
  const double H = block_sum(h, shd);
  // top-2 reduction
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Top2 o2{__shfl_xor_sync(0xffffffffu, t.a, o), __shfl_xor_sync(0xffffffffu, t.b, o)};
    t = merge2(t, o2);
  }
  if (lane == 0) sht[warp] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    Top2 r = sht[0];
    for (int w = 1; w < nw; ++w) r = merge2(r, sht[w]);
    fq_row_stats st;
    st.entropy = H;
    st.ppl_entropy = exp(H);
    st.p1 = r.a;
    st.p2 = r.b;
    st.fault_tolerance = r.a - r.b;
    st.max_logit = mx.v;
    st.argmax = mx.i;
    out[blockIdx.x] = st;
  }
}

template <typename T>
__device__ __forceinline__ float ld(const T* p, int64_t i);
template <>
__device__ __forceinline__ float ld<float>(const float* p, int64_t i) { return p[i]; }
template <>
__device__ __forceinline__ float ld<__nv_bfloat16>(const __nv_bfloat16* p, int64_t i) { return __bfloat162float(p[i]); }

template <typename T>
__global__ void __launch_bounds__(kStatThreads) kl_rows_kernel(const T* __restrict__ lq, const T* __restrict__ lp,
                                                               int64_t vocab, double* kl, double* ent) {
  __shared__ double shd[33];
  __shared__ MaxArg shm[33];
  const T* q = lq + blockIdx.x * vocab;
  const T* p = lp + blockIdx.x * vocab;
  MaxArg a{-FLT_MAX, 0}, b{-FLT_MAX, 0};
  for (int64_t i = threadIdx.x; i < vocab; i += blockDim.x) {
    a = better(a, MaxArg{ld(q, i), 0});
    b = better(b, MaxArg{ld(p, i), 0});
  }
  const float mq = block_argmax(a, shm).v;
  const float mp = block_argmax(b, shm).v;
  double sq = 0.0, sp = 0.0, wq = 0.0, wd = 0.0;
  for (int64_t i = threadIdx.x; i < vocab; i += blockDim.x) {
    const float xq = ld(q, i), xp = ld(p, i);
    const double eq = static_cast<double>(expf(xq - mq));
    sq += eq;
    sp += static_cast<double>(expf(xp - mp));
    wq += eq * static_cast<double>(xq - mq);
    wd += eq * (static_cast<double>(xq) - static_cast<double>(xp));
  }
  const double Sq = block_sum(sq, shd);
  const double Sp = block_sum(sp, shd);
  const double Wq = block_sum(wq, shd);
  const double Wd = block_sum(wd, shd);
  if (threadIdx.x == 0) {
    const double lse_q = static_cast<double>(mq) + log(Sq);
    const double lse_p = static_cast<double>(mp) + log(Sp);
    kl[blockIdx.x] = Wd / Sq - lse_q + lse_p;
    if (ent) ent[blockIdx.x] = log(Sq) - Wq / Sq;
  }
}

// ---- histogram (analyzer) ----
__global__ void minmax_kernel(const float* __restrict__ w, int64_t n, float* out /*[2*blocks]*/) {
  __shared__ float smin[32], smax[32];
  float lo = FLT_MAX, hi = -FLT_MAX;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    lo = fminf(lo, w[i]);
    hi = fmaxf(hi, w[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { smin[warp] = lo; smax[warp] = hi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < static_cast<int>(blockDim.x >> 5); ++i) { lo = fminf(lo, smin[i]); hi = fmaxf(hi, smax[i]); }
    lo = fminf(lo, smin[0]);
    hi = fmaxf(hi, smax[0]);
    out[2 * blockIdx.x] = lo;
    out[2 * blockIdx.x + 1] = hi;
  }
}

// counts[0..bins) for the fp weights, counts[bins..2bins) for the dequantized rung
__global__ void hist_kernel(const float* __restrict__ fpw, const uint8_t* __restrict__ payload, int bits,
                            const float* __restrict__ scale, const int32_t* __restrict__ zp, int64_t N,
                            int64_t K, int64_t G, int64_t ng, int64_t ng_pad, const double* __restrict__ edges_g, int bins,
                            unsigned long long* counts) {
  extern __shared__ unsigned char smem_raw[];
  double* edges = reinterpret_cast<double*>(smem_raw);
  unsigned int* c = reinterpret_cast<unsigned int*>(edges + bins + 1);
  for (int i = threadIdx.x; i <= bins; i += blockDim.x) edges[i] = edges_g[i];
  for (int i = threadIdx.x; i < 2 * bins; i += blockDim.x) c[i] = 0u;
  __syncthreads();
  const double lo = edges[0];
  const double width = (edges[bins] - edges[0]) / bins;
  auto bin_of = [&](double v) {
    int b;
    if (v < edges[1]) return 0;
    if (v >= edges[bins - 1]) return bins - 1;
    b = static_cast<int>(floor((v - lo) / width));
    b = max(0, min(bins - 1, b));
    while (b > 0 && v < edges[b]) --b;
    while (b < bins - 1 && v >= edges[b + 1]) ++b;
    return b;
  };
  const int64_t n = N * K;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    atomicAdd(&c[bin_of(static_cast<double>(fpw[i]))], 1u);
    const int64_t row = i / K, k = i % K;
    uint32_t code;
    if (bits == 8) code = payload[i];
    else code = (i & 1) ? (payload[i >> 1] >> 4) : (payload[i >> 1] & 0xFu);
    const int64_t g = k / G;
    const float dq = static_cast<float>(static_cast<int32_t>(code) - zp[row * ng + g]) * scale[row * ng_pad + g];
    atomicAdd(&c[bins + bin_of(static_cast<double>(dq))], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * bins; i += blockDim.x)
    if (c[i]) atomicAdd(&counts[i], static_cast<unsigned long long>(c[i]));
}

}  // namespace

void launch_softmax_stats(fq_ctx* ctx, const float* logits, int64_t rows, int64_t vocab, int64_t row_stride,
                          fq_row_stats* out) {
  if (rows <= 0) return;
  if (vocab < 1) fail(FQ_E_DIMENSION, "softmax_stats: empty logits");
  softmax_stats_kernel<<<static_cast<unsigned>(rows), kStatThreads, 0, ctx->stream>>>(logits, vocab, row_stride, out);
  FQ_CUDA(cudaGetLastError());
  ctx->launches += 1;
}

void launch_kl_rows(fq_ctx* ctx, const void* lq, const void* lp, int dtype, int64_t rows, int64_t vocab,
                    double* kl, double* ent) {
  if (rows <= 0) return;
  if (dtype == FQ_DT_F32)
    kl_rows_kernel<float><<<static_cast<unsigned>(rows), kStatThreads, 0, ctx->stream>>>(
        static_cast<const float*>(lq), static_cast<const float*>(lp), vocab, kl, ent);
  else if (dtype == FQ_DT_BF16)
    kl_rows_kernel<__nv_bfloat16><<<static_cast<unsigned>(rows), kStatThreads, 0, ctx->stream>>>(
        static_cast<const __nv_bfloat16*>(lq), static_cast<const __nv_bfloat16*>(lp), vocab, kl, ent);
  else
    fail(FQ_E_CONFIG, "kl_rows: logits must be f32 or bf16");
  FQ_CUDA(cudaGetLastError());
  ctx->launches += 1;
}

double hist_kl(fq_ctx* ctx, const fq_layer* L, int rung, int bins) {
  if (bins < 2) fail(FQ_E_INPUT, "analyze_model: need at least two bins");
  if (L->fp == nullptr) fail(FQ_E_STATE, "hist_kl: layer has no fp weights on the device");
  if (rung != FQ_RUNG_INT8 && rung != FQ_RUNG_INT4) fail(FQ_E_CONFIG, "analyze_model: target must be a quantized rung");
  const fq_rung_store& st = L->store(rung);
  if (!st.present) fail(FQ_E_STATE, "hist_kl: rung not resident");
  const int64_t n = L->N * L->K;
  if (n == 0) fail(FQ_E_INPUT, "weight_histogram: empty tensor");
  // 1) range of the fp weights
  const int mm_blocks = 256;
  float* d_mm = static_cast<float*>(ctx->ensure_scratch(sizeof(float) * 2 * mm_blocks + 64));
  minmax_kernel<<<mm_blocks, 256, 0, ctx->stream>>>(L->fp, n, d_mm);
  FQ_CUDA(cudaGetLastError());
  std::vector<float> mm(2 * mm_blocks);
  FQ_CUDA(cudaMemcpyAsync(mm.data(), d_mm, sizeof(float) * 2 * mm_blocks, cudaMemcpyDeviceToHost, ctx->stream));
  FQ_CUDA(cudaStreamSynchronize(ctx->stream));
  float lo = mm[0], hi = mm[1];
  for (int i = 1; i < mm_blocks; ++i) { lo = std::fmin(lo, mm[2 * i]); hi = std::fmax(hi, mm[2 * i + 1]); }
  // 2) edges exactly as uniform_edges (src/analyzer.cpp:17-29)
  double dlo = lo, dhi = hi;
  if (!(dhi > dlo)) { dlo -= 0.5; dhi += 0.5; }
  std::vector<double> edges(bins + 1);
  const double width = (dhi - dlo) / static_cast<double>(bins);
  for (int i = 0; i <= bins; ++i) edges[i] = dlo + width * i;
  edges[bins] = dhi;
  for (int i = 1; i <= bins; ++i)
    if (!(edges[i] > edges[i - 1])) fail(FQ_E_INPUT, "weight_histogram: edges must be strictly increasing");
  // 3) counts on the device
  const size_t edge_bytes = sizeof(double) * (bins + 1);
  const size_t cnt_bytes = sizeof(unsigned long long) * 2 * bins;
  char* scratch = static_cast<char*>(ctx->ensure_scratch(edge_bytes + cnt_bytes + 256));
  double* d_edges = reinterpret_cast<double*>(scratch);
  unsigned long long* d_counts = reinterpret_cast<unsigned long long*>(scratch + ((edge_bytes + 255) & ~size_t(255)));
  FQ_CUDA(cudaMemcpyAsync(d_edges, edges.data(), edge_bytes, cudaMemcpyHostToDevice, ctx->stream));
  FQ_CUDA(cudaMemsetAsync(d_counts, 0, cnt_bytes, ctx->stream));
  const size_t smem = edge_bytes + sizeof(unsigned int) * 2 * bins;
  if (smem > 200 * 1024) fail(FQ_E_CONFIG, "hist_kl: too many bins for shared memory");
  if (smem > 48 * 1024) FQ_CUDA(cudaFuncSetAttribute(hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const int blocks = static_cast<int>(std::min<int64_t>(ctx->num_sms * 2, (n + 1023) / 1024));
  hist_kernel<<<std::max(blocks, 1), 512, smem, ctx->stream>>>(L->fp, st.payload, st.bits, st.scale, st.zp32, L->N, L->K,
                                                              L->G, L->ng, L->ng_pad, d_edges, bins, d_counts);
  FQ_CUDA(cudaGetLastError());
  ctx->launches += 3;
  std::vector<unsigned long long> counts(2 * bins);
  FQ_CUDA(cudaMemcpyAsync(counts.data(), d_counts, cnt_bytes, cudaMemcpyDeviceToHost, ctx->stream));
  FQ_CUDA(cudaStreamSynchronize(ctx->stream));
  // 4) smoothing, normalisation and KL in the reference's sequential order
  auto normalise = [&](const unsigned long long* c) {
    std::vector<double> p(bins);
    double total = 0.0;
    for (int i = 0; i < bins; ++i) {
      p[i] = static_cast<double>(c[i]) + 1e-10;
      total += p[i];
    }
    for (int i = 0; i < bins; ++i) p[i] /= total;
    return p;
  };
  const std::vector<double> p = normalise(counts.data());
  const std::vector<double> q = normalise(counts.data() + bins);
  double sp = 0.0, sq = 0.0;
  for (int i = 0; i < bins; ++i) {
    if (!(p[i] > 0.0) || !(q[i] > 0.0)) fail(FQ_E_INPUT, "kl_divergence: entries must be strictly positive");
    sp += p[i];
    sq += q[i];
  }
  if (std::fabs(sp - 1.0) > 1e-6 || std::fabs(sq - 1.0) > 1e-6) fail(FQ_E_INPUT, "kl_divergence: inputs must sum to 1");
  double kl = 0.0;
  for (int i = 0; i < bins; ++i) kl += p[i] * std::log(p[i] / q[i]);
  return kl;
}

}  // namespace fqc
