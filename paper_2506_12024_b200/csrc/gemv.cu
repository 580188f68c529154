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
//  * each CTA owns a balanced contiguous row range of every matrix of a GEMV phase; that range
//    is one contiguous byte range of the row-major payload (plus its padded scale / zero-point
//    rows).  A producer warp streams all of the CTA's ranges, phase after phase, through a
//    shared-memory ring with 1-D TMA bulk copies (cp.async.bulk + mbarrier complete_tx).  It
//    never waits for activations, so the HBM stream keeps running across phase boundaries while
//    the consumer warps synchronise on a grid barrier between dependent phases.
//  * consumer warps split the K-steps of a row (512 codes per step, 16 per lane) and keep their
//    activations in registers for the phase.  Unpacking is one LOP/SHF per code: the masked
//    code bits (q << s), s < 24, reinterpreted as fp32 are exactly q * 2^(s-149) (subnormal /
//    first binade), so an FFMA2 with x * 2^(109-s) accumulates q*x*2^-40 with no int->float
//    conversion.  The zero point is folded per group: sum_j (q_j - z) x_j = sum_j q_j x_j -
//    z * sum_j x_j.  fp32 accumulation; fixed reduction order (deterministic, no atomics).
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
  P.G = L0->G;
  P.ng_pad = L0->ng_pad;
  P.zp_pad = L0->zp_pad;
  P.nsteps = ceil_div_i(L0->K, kStepCodes);
  P.sw = (P.nsteps + kSplit - 1) / kSplit;
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
  for (int m = 0; m < g.nmat; ++m) {
    const fq_layer* L = g.mat[m].layer;
    if (L->N != P.N || L->K != P.K || L->G != P.G) fail(FQ_E_DIMENSION, "multi-gemv: matrices differ in shape");
    DevMat& M = P.mat[m];
    const fq_rung_store* st[2] = {&L->r8, &L->r4};
    for (int w = 0; w < 2; ++w) {
      M.payload[w] = st[w]->payload;
      M.scale[w] = st[w]->scale;
      M.zp[w] = st[w]->zp8;
      M.zpbase[w] = st[w]->zp_base;
    }
    M.rung_table = g.mat[m].rung_table ? g.mat[m].rung_table + b0 * g.mat[m].rung_stride : nullptr;
    M.rung_stride = g.mat[m].rung_stride;
    M.rung = g.mat[m].rung;
    M.y = g.mat[m].y ? static_cast<char*>(g.mat[m].y) + b0 * g.y_stride * ysz : nullptr;
  }
  // ring-slot layout of this phase (per bit-width)
  const int64_t target = 40 * 1024;
  for (int w = 0; w < 2; ++w) {
    const int64_t row_bytes = w == 0 ? P.K : P.K / 2;
    const int64_t per_row = row_bytes + P.ng_pad * 4 + P.zp_pad;
    int rps = static_cast<int>(std::max<int64_t>(1, target / per_row));
    rps = std::min(rps, 32);
    // row groups consume octets (1 step, B=1), quads (1 step) or pairs (several steps)
    const int quantum = (P.sw == 1 ? (bb == 1 ? 8 : 4) : 2) * kRG;
    rps = rps >= quantum ? rps / quantum * quantum : quantum;
    const int64_t pad = rps;  // a multiple of the row-group quantum: partial stages read stale rows only
    P.rows_per_stage[w] = rps;
    P.sc_off[w] = static_cast<int>(pad * row_bytes);
    P.zp_off[w] = static_cast<int>(pad * row_bytes + pad * P.ng_pad * 4);
    stage_bytes = std::max<int64_t>(stage_bytes, (pad * per_row + 127) / 128 * 128);
  }
  P.sc_row = static_cast<int>(P.ng_pad * 4);
  P.zp_row = static_cast<int>(P.zp_pad);
  const int64_t rows_max = (P.N + grid - 1) / grid;
  red_floats = std::max<int64_t>(red_floats, static_cast<int64_t>(g.nmat) * rows_max * kSplit * (bb == 3 ? 4 : bb));
  if (bb > 1 && P.sw > (bb <= 2 ? 2 : 1)) fail(FQ_E_CONFIG, "gemv: batch chunk too large for the K-steps per warp");
  max_sw = std::max(max_sw, P.sw);
  max_nsteps = std::max(max_nsteps, P.nsteps);
  max_bb = std::max(max_bb, bb);
  phases.push_back(P);
}

void ProgramBuilder::add(const Phase& p) {
  phases.push_back(p);
  max_bb = std::max(max_bb, p.B);
}

int gemv_batch_chunk(int64_t K) {
  const int sw = (ceil_div_i(K, kStepCodes) + kSplit - 1) / kSplit;
  return sw == 1 ? kMaxB : (sw == 2 ? 2 : 1);
}

bool gemv_fast_supported(const fq_layer* L, int rung) {
  if (rung != FQ_RUNG_INT8 && rung != FQ_RUNG_INT4) return false;
  const fq_rung_store& s = L->store(rung);
  const int nsteps = ceil_div_i(L->K, kStepCodes);
  return s.present && s.zp_fits_u8 && L->K % 32 == 0 && L->G % kSegCodes == 0 && L->G >= kSegCodes &&
         nsteps <= kMaxSW * kSplit;
}

int gemv_fast_grid(const fq_ctx* ctx, int64_t N) { return static_cast<int>(std::min<int64_t>(ctx->num_sms, N)); }

int launch_gemv_fast(fq_ctx* ctx, const GemvLaunch& g) {
  // A stand-alone GEMV is a program of independent phases, one per batch chunk.
  const int64_t bchunk = gemv_batch_chunk(g.mat[0].layer->K);
  ProgramBuilder pb;
  pb.grid = gemv_fast_grid(ctx, g.mat[0].layer->N);
  for (int64_t b0 = 0; b0 < g.batch; b0 += bchunk)
    pb.add_gemv(g, b0, static_cast<int>(std::min<int64_t>(bchunk, g.batch - b0)));
  if (g.epi == EPI_RESIDUAL && g.out_n_partials < pb.grid) fail(FQ_E_STATE, "gemv: residual partial buffer too small");
  for (auto& P : pb.phases) P.barrier_after = 0;
  if (pb.phases.size() > static_cast<size_t>(kInlinePhases)) {
    // very large batches: launch chunk groups separately
    ProgramBuilder part = pb;
    for (size_t i = 0; i < pb.phases.size(); i += kInlinePhases) {
      part.phases.assign(pb.phases.begin() + i, pb.phases.begin() + std::min(pb.phases.size(), i + kInlinePhases));
      const ProgramRun run = upload_program(ctx, part, true);
      launch_program(ctx, run, nullptr, g.pdl);
    }
    return pb.grid;
  }
  const ProgramRun run = upload_program(ctx, pb, true);
  launch_program(ctx, run, nullptr, g.pdl);
  return pb.grid;
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
