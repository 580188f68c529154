// Tensor-parallel variant: host-side shard bookkeeping (no device code).
//
// The reference runs one Llama-less block on one core (src/model.cpp:201-233) and has no
// distribution at all; north_star asks for a tensor-parallel variant next to the sequence-sharded
// decode: column-split q/k/v/gate/up, row-split o/down (one all-reduce of an fp32 [B, d] partial
// after each), and a vocab-split head whose statistics are merged from per-rank softmax partials.
// This file holds the parts that need no GPU: the shard layout, slicing a quantized tensor into a
// rank's shard, and the merge of the head partials.  The segment programs are in model.cu
// (tp_program), the collectives in paper_2506_12024_b200/tp.py.
#include <cmath>
#include <cstring>
#include <string>

#include "fq_internal.cuh"

namespace {

int64_t groups_of(int64_t K, int64_t group) { return group > 0 ? (K + group - 1) / group : 1; }

// fq_stat_part merge in double -- the same arithmetic as the device stat_merge (program.cu), so a
// tree of merges over ranks reproduces the single-device statistics up to the merge order.
fq_stat_part merge(const fq_stat_part& a, const fq_stat_part& b) {
  if (b.m == -INFINITY) return a;
  if (a.m == -INFINITY) return b;
  fq_stat_part r;
  r.m = std::fmax(a.m, b.m);
  const double da = static_cast<double>(a.m) - r.m, db = static_cast<double>(b.m) - r.m;
  const double ea = std::exp(da), eb = std::exp(db);
  r.S = a.S * ea + b.S * eb;
  r.T = ea * (a.T + da * a.S) + eb * (b.T + db * b.S);
  r.v1 = std::fmax(a.v1, b.v1);
  r.v2 = std::fmax(std::fmin(a.v1, b.v1), std::fmax(a.v2, b.v2));
  // argmax_token: strict >, the lowest index wins ties (src/engine.cpp:144-155)
  r.arg = a.v1 > b.v1 ? a.arg : (b.v1 > a.v1 ? b.arg : std::min(a.arg, b.arg));
  return r;
}

}  // namespace

using fqc::fail;
using fqc::guarded;

extern "C" {

fq_status fq_tp_shard_spec(const fq_model_config* cfg, int32_t rank, int32_t size, fq_tp_shard* out) {
  return guarded([&] {
    if (!cfg || !out) fail(FQ_E_INPUT, "null argument");
    const fq_model_config& c = *cfg;
    if (size < 1 || rank < 0 || rank >= size) fail(FQ_E_CONFIG, "tensor parallel: rank / size out of range");
    if (c.n_heads % size != 0) fail(FQ_E_CONFIG, "tensor parallel: n_heads must be a multiple of the TP size");
    const int64_t g = c.group_size > 0 ? c.group_size : c.d_model;
    fq_tp_shard s{};
    s.rank = rank;
    s.size = size;
    s.heads = c.n_heads / size;
    s.head0 = s.heads * rank;
    if (size > 1 && (s.heads * c.head_dim) % g != 0)
      fail(FQ_E_CONFIG, "tensor parallel: a rank's attention width (heads * head_dim) must be whole groups");
    if (size > 1 && c.group_size <= 0) fail(FQ_E_CONFIG, "tensor parallel: per-group quantization required");
    // ffn columns in whole groups (the O / down projections are split along their input, so a
    // group must not straddle two ranks); the ragged tail group stays with the last rank
    const int64_t ng = groups_of(c.ffn_dim, g);
    if (ng < size) fail(FQ_E_CONFIG, "tensor parallel: fewer ffn groups than ranks");
    const int64_t g0 = ng * rank / size, g1 = ng * (rank + 1) / size;
    s.ffn0 = g0 * g;
    s.ffn = std::min(g1 * g, c.ffn_dim) - s.ffn0;
    s.vocab0 = c.vocab_size * rank / size;
    s.vocab = c.vocab_size * (rank + 1) / size - s.vocab0;
    if (s.vocab < 1) fail(FQ_E_CONFIG, "tensor parallel: more ranks than vocabulary rows");
    s.n_segments = static_cast<int32_t>(2 * c.n_layers + 1);
    *out = s;
  });
}

fq_status fq_shard_quantized(int32_t bits, int64_t N, int64_t K, int64_t group, const uint8_t* payload,
                             const float* scale, const int32_t* zp, int64_t row0, int64_t row1, int64_t col0,
                             int64_t col1, uint8_t* payload_out, float* scale_out, int32_t* zp_out) {
  return guarded([&] {
    if (!payload || !scale || !zp || !payload_out || !scale_out || !zp_out) fail(FQ_E_INPUT, "null argument");
    if (bits != 8 && bits != 4) fail(FQ_E_CONFIG, "shard: bits must be 8 or 4");
    if (N < 1 || K < 1 || group < 1) fail(FQ_E_DIMENSION, "shard: bad shape");
    if (row0 < 0 || row1 > N || row0 >= row1 || col0 < 0 || col1 > K || col0 >= col1)
      fail(FQ_E_DIMENSION, "shard: range out of bounds");
    if (col0 % group != 0 || (col1 % group != 0 && col1 != K))
      fail(FQ_E_DIMENSION, "shard: column range must cover whole quantization groups");
    const int64_t ng = groups_of(K, group), gc0 = col0 / group, gc1 = groups_of(col1, group);
    const int64_t kl = col1 - col0, ngl = gc1 - gc0;
    if (bits == 4 && ((K & 1) || (col0 & 1) || (kl & 1)))
      fail(FQ_E_DIMENSION, "shard: 4-bit rows must stay byte aligned (even K and column range)");
    for (int64_t r = row0; r < row1; ++r) {
      const int64_t ro = r - row0;
      if (bits == 8) {
        std::memcpy(payload_out + ro * kl, payload + r * K + col0, static_cast<size_t>(kl));
      } else {
        // pack_codes: low nibble = even flat index (src/quantizer.cpp:60-92); rows stay aligned
        std::memcpy(payload_out + ro * kl / 2, payload + (r * K + col0) / 2, static_cast<size_t>(kl / 2));
      }
      std::memcpy(scale_out + ro * ngl, scale + r * ng + gc0, sizeof(float) * static_cast<size_t>(ngl));
      std::memcpy(zp_out + ro * ngl, zp + r * ng + gc0, sizeof(int32_t) * static_cast<size_t>(ngl));
    }
  });
}

fq_status fq_tp_merge_stats(const fq_stat_part* parts, int32_t nranks, int32_t batch, const int64_t* vocab0,
                            fq_row_stats* out) {
  return guarded([&] {
    if (!parts || !vocab0 || !out) fail(FQ_E_INPUT, "null argument");
    if (nranks < 1 || batch < 1) fail(FQ_E_INPUT, "merge: nranks / batch must be >= 1");
    for (int b = 0; b < batch; ++b) {
      fq_stat_part a{0.0, 0.0, -INFINITY, -INFINITY, -INFINITY, 0x7fffffff};
      for (int r = 0; r < nranks; ++r) {
        fq_stat_part p = parts[static_cast<int64_t>(r) * batch + b];
        if (p.m != -INFINITY) p.arg = static_cast<int32_t>(p.arg + vocab0[r]);
        a = merge(a, p);
      }
      if (a.m == -INFINITY) fail(FQ_E_STATE, "merge: no logits in any rank's partial");
      fq_row_stats s;
      const double H = std::log(a.S) - a.T / a.S;
      s.entropy = H;
      s.ppl_entropy = std::exp(H);
      s.p1 = std::exp(static_cast<double>(a.v1) - a.m) / a.S;
      s.p2 = a.v2 == -INFINITY ? -1.0 : std::exp(static_cast<double>(a.v2) - a.m) / a.S;
      s.fault_tolerance = s.p1 - s.p2;
      s.max_logit = a.m;
      s.argmax = a.arg;
      out[b] = s;
    }
  });
}

}  // extern "C"
