// Dequant-fused weight-only GEMV over resident W8/W4 copies (K1/K2 of SURVEY §2.1) and the
// persistent decode-step program built from it.
//
// Replaces MultiPrecisionLayer::forward (/root/reference/proj/src/model.cpp:77-98), which
// dequantizes the active rung (src/quantizer.cpp:205-219) and runs a double-accumulated
// linear (src/tensor.cpp:83-101).
//
// Fast numerics — a TMA-fed streaming program (program.cu):
//  * the work is a list of phases (GEMVs, and for the decode step also the token embedding, the
//    attention of every layer and the row statistics).  One CTA per SM runs the whole list.
//  * weights are streamed from the tiled copy of each rung (fq_internal.cuh): self-contained
//    16-row x 128-code blocks (codes in MMA-fragment order + 16 scales + 16 u8 zero points).
//    A GEMV phase is the sequence of its blocks; CTA c owns a byte-balanced contiguous slice of
//    it (stream-K: a 16-row tile may be shared by neighbouring CTAs; the CTA holding the tile's
//    first block adds the later parts, published through flags, in CTA order).
//  * a producer warp streams the CTA's slices, phase after phase, through a shared-memory ring
//    with 1-D TMA bulk copies (cp.async.bulk + mbarrier complete_tx).  It never waits for
//    activations, so the HBM stream keeps running across phase boundaries while the consumer
//    warps synchronise on a grid barrier between dependent phases.
//  * 16 consumer warps take whole blocks.  Unpacking is a byte permute (W8: PRMT with 0x64 gives
//    the fp16 1024+q) or a masked OR (W4: 1024+q for the low nibbles, 64+q for the high ones), so
//    the dot products run on the tensor cores (mma.sync m16n8k16, fp32 accumulate) with the
//    batch rows as the MMA's n columns.  Offsets and zero points fold per block:
//    sum (q-z) x = acc - (D + z * X), D / X from the staged activations.  Fixed reduction order
//    (deterministic, no float atomics).
// Exact numerics — golden/parity mode: one thread per output, w = float(code - z) * s in fp32 as
// dequantize() does, then a sequential double accumulation in k order as linear() does:
// bit-identical to the reference.  Any group size, fp rung, bias.
#include "gemv_program.cuh"

#include <algorithm>

namespace fqc {
namespace {

// Exact kernel: one thread per (row, batch row); sequential k, double accumulation.
__global__ void gemv_exact_kernel(const int64_t N, const int64_t K, const int64_t G, const int64_t ng,
                                  const int64_t ng_pad, const int bits, const uint8_t* payload, const float* scale,
                                  const int32_t* zp, const float* fpw, const float* bias, const int B, const void* x,
                                  const int x_dtype, void* y, const int y_dtype) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= N * B) return;
  const int64_t row = t % N;
  const int b = static_cast<int>(t / N);
  auto act = [&](int64_t i) -> float {
    if (x_dtype == FQ_DT_F32) return static_cast<const float*>(x)[i];
    if (x_dtype == FQ_DT_BF16) return __bfloat162float(static_cast<const __nv_bfloat16*>(x)[i]);
    return __half2float(static_cast<const __half*>(x)[i]);
  };
  double acc = bias ? static_cast<double>(bias[row]) : 0.0;
  for (int64_t k = 0; k < K; ++k) {
    float w;
    if (bits == 0) {
      w = fpw[row * K + k];
    } else {
      const int64_t idx = row * K + k;
      uint32_t code;
      if (bits == 8) code = payload[idx];
      else code = (idx & 1) ? (payload[idx >> 1] >> 4) : (payload[idx >> 1] & 0xFu);
      const int64_t g = k / G;
      w = static_cast<float>(static_cast<int32_t>(code) - zp[row * ng + g]) * scale[row * ng_pad + g];
    }
    acc += static_cast<double>(act(b * K + k)) * static_cast<double>(w);
  }
  const float out = static_cast<float>(acc);
  if (y_dtype == FQ_DT_F32) static_cast<float*>(y)[b * N + row] = out;
  else if (y_dtype == FQ_DT_BF16) static_cast<__nv_bfloat16*>(y)[b * N + row] = __float2bfloat16_rn(out);
  else static_cast<__half*>(y)[b * N + row] = __float2half_rn(out);
}

}  // namespace

// ------------------------------------------------------------------ host-side program builder
void ProgramBuilder::add_gemv(const GemvLaunch& g, int64_t b0, int bb) {
  const fq_layer* L0 = g.mat[0].layer;
  Phase P{};
  P.type = PH_GEMV;
  P.barrier_after = 1;
  P.nmat = g.nmat;
  P.B = bb;
  P.N = L0->N;
  P.K = L0->K;
  P.n_tiles = ceil_div_i(L0->N, kTileRows);
  P.nkb = ceil_div_i(L0->K, kBlockK);
  const size_t xsz = g.x_dtype == FQ_DT_F32 ? 4 : 2;
  const int64_t xs = g.x_stride ? g.x_stride : L0->K;
  P.x = static_cast<const char*>(g.x) + b0 * xs * xsz;
  P.x_dtype = g.x_dtype;
  P.x_stride = xs;
  P.norm_gain = g.norm_gain;
  P.partials_stride = g.partials_stride ? g.partials_stride : g.n_partials;
  P.norm_partials = g.norm_partials ? g.norm_partials + b0 * P.partials_stride : nullptr;
  P.n_partials = g.n_partials;
  P.norm_eps = g.norm_eps;
  P.act_dtype = g.act_dtype;
  P.epi = g.epi;
  const size_t ysz = g.y_dtype == FQ_DT_F32 ? 4 : 2;
  P.y = g.y ? static_cast<char*>(g.y) + b0 * g.y_stride * ysz : nullptr;
  P.y_dtype = g.y_dtype;
  P.y_stride = g.y_stride;
  P.resid = g.resid ? g.resid + b0 * g.resid_stride : nullptr;
  P.resid_stride = g.resid_stride;
  P.out_partials = g.out_partials ? g.out_partials + b0 * g.out_n_partials : nullptr;
  P.out_partials_stride = g.out_n_partials;
  P.stat_part = g.stat_part ? static_cast<char*>(g.stat_part) + b0 * grid * 32 : nullptr;  // sizeof(StatPart)
  P.xfrag = g.xfrag ? static_cast<const uint4*>(g.xfrag) + b0 * P.nkb * 16 : nullptr;
  P.yfrag_nkb = static_cast<int>(ceil_div_i(P.N, kBlockK));
  P.yfrag = g.yfrag ? static_cast<__half*>(g.yfrag) + b0 * P.yfrag_nkb * 128 : nullptr;
  if (g.nmat < 1 || g.nmat > kMaxMat) fail(FQ_E_CONFIG, "multi-gemv: 1..3 matrices");
  if (bb < 1 || bb > kMaxB) fail(FQ_E_CONFIG, "gemv: batch chunk out of range");
  if (static_cast<double>(P.n_tiles) * P.nkb * (kBlockBytes8 + kBlockBytes4) * g.nmat >= 4294967296.0)
    fail(FQ_E_CONFIG, "gemv: layer too large for one phase (> 4 GiB of blocks)");
  for (int m = 0; m < g.nmat; ++m) {
    const fq_layer* L = g.mat[m].layer;
    if (L->N != P.N || L->K != P.K) fail(FQ_E_DIMENSION, "multi-gemv: matrices differ in shape");
    DevMat& M = P.mat[m];
    const fq_rung_store* st[2] = {&L->r8, &L->r4};
    for (int w = 0; w < 2; ++w) {
      M.tiles[w] = st[w]->present ? st[w]->tiles : nullptr;
      M.zpbase[w] = st[w]->zp_base;
    }
    M.rung_table = g.mat[m].rung_table ? g.mat[m].rung_table + b0 * g.mat[m].rung_stride : nullptr;
    M.rung_stride = g.mat[m].rung_stride;
    M.rung = g.mat[m].rung;
    M.y = g.mat[m].y ? static_cast<char*>(g.mat[m].y) + b0 * g.y_stride * ysz : nullptr;
  }
  max_kpad = std::max<int64_t>(max_kpad, static_cast<int64_t>(P.nkb) * kBlockK);
  max_xs = std::max<int64_t>(max_xs, static_cast<int64_t>(P.nkb) * kBlockK * 2 * bb);
  max_bb = std::max(max_bb, bb);
  phases.push_back(P);
}

void ProgramBuilder::add(const Phase& p) { phases.push_back(p); }

bool gemv_fast_supported(const fq_layer* L, int rung) {
  if (rung != FQ_RUNG_INT8 && rung != FQ_RUNG_INT4) return false;
  const fq_rung_store& s = L->store(rung);
  return s.present && s.tiles != nullptr;
}

int gemv_fast_grid(const fq_ctx* ctx, int64_t blocks) { return static_cast<int>(std::min<int64_t>(ctx->num_sms, blocks)); }

int launch_gemv_fast(fq_ctx* ctx, const GemvLaunch& g) {
  // A stand-alone GEMV is a program of independent phases, one per batch chunk.
  const fq_layer* L = g.mat[0].layer;
  const int64_t bchunk = gemv_batch_chunk(L->K);
  ProgramBuilder pb;
  pb.grid = gemv_fast_grid(ctx, static_cast<int64_t>(ceil_div_i(L->N, kTileRows)) * ceil_div_i(L->K, kBlockK));
  for (int64_t b0 = 0; b0 < g.batch; b0 += bchunk)
    pb.add_gemv(g, b0, static_cast<int>(std::min<int64_t>(bchunk, g.batch - b0)));
  if (g.epi == EPI_RESIDUAL && g.out_n_partials < pb.grid) fail(FQ_E_STATE, "gemv: residual partial buffer too small");
  for (auto& P : pb.phases) P.barrier_after = 0;
  for (size_t i = 0; i < pb.phases.size(); i += kInlinePhases) {
    ProgramBuilder part = pb;
    part.phases.assign(pb.phases.begin() + i, pb.phases.begin() + std::min(pb.phases.size(), i + kInlinePhases));
    const ProgramRun run = upload_program(ctx, part, true);
    launch_program(ctx, run, nullptr, g.pdl);
  }
  return pb.grid;
}

double time_gemv_chain(fq_ctx* ctx, const GemvLaunch* gs, int n, int reps) {
  // one device program of n independent GEMV phases (no barriers), launched reps times
  ProgramBuilder pb;
  const fq_layer* L0 = gs[0].mat[0].layer;
  pb.grid = gemv_fast_grid(ctx, static_cast<int64_t>(ceil_div_i(L0->N, kTileRows)) * ceil_div_i(L0->K, kBlockK));
  for (int i = 0; i < n; ++i) {
    const int64_t bchunk = gemv_batch_chunk(gs[i].mat[0].layer->K);
    for (int64_t b0 = 0; b0 < gs[i].batch; b0 += bchunk)
      pb.add_gemv(gs[i], b0, static_cast<int>(std::min<int64_t>(bchunk, gs[i].batch - b0)));
  }
  for (auto& P : pb.phases) P.barrier_after = 0;
  ProgramRun run = upload_program(ctx, pb, false);
  cudaEvent_t e0, e1;
  FQ_CUDA(cudaEventCreate(&e0));
  FQ_CUDA(cudaEventCreate(&e1));
  launch_program(ctx, run, nullptr, false);  // warm-up
  FQ_CUDA(cudaEventRecord(e0, ctx->stream));
  for (int r = 0; r < reps; ++r) launch_program(ctx, run, nullptr, false);
  FQ_CUDA(cudaEventRecord(e1, ctx->stream));
  FQ_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  FQ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  FQ_CUDA(cudaEventDestroy(e0));
  FQ_CUDA(cudaEventDestroy(e1));
  dfree(run.dev_phases);
  dfree(run.fix);
  dfree(run.flags);
  return static_cast<double>(ms) / std::max(reps, 1);
}

void launch_gemv_exact(fq_ctx* ctx, const fq_layer* L, int rung, int64_t batch, const void* x, int x_dtype, void* y,
                       int y_dtype) {
  if (!L->has(rung)) fail(FQ_E_STATE, "gemv: rung not resident on the device");
  const int threads = 128;
  const int64_t n = L->N * batch;
  const fq_rung_store* s = rung == FQ_RUNG_FP ? nullptr : &L->store(rung);
  gemv_exact_kernel<<<ceil_div_i(n, threads), threads, 0, ctx->stream>>>(
      L->N, L->K, L->G, L->ng, L->ng_pad, s ? s->bits : 0, s ? s->payload : nullptr, s ? s->scale : nullptr,
      s ? s->zp32 : nullptr, L->fp, L->bias, static_cast<int>(batch), x, x_dtype, y, y_dtype);
  FQ_CUDA(cudaGetLastError());
  ctx->launches += 1;
}

}  // namespace fqc
