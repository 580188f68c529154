/*
 * fq_oracle.c — CPU restatement of the reference FlexQuant hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker the parity tests, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg compare the CUDA engine against; nothing in the product
 * (paper_2506_12024_b200/) links, loads or calls it.
 *
 * Every function restates the reference algorithm in plain C and cites the reference
 * file:line it follows (paths under /root/reference/proj).  The restatement is pinned against
 * the reference itself, compiled from its own sources into oracle/_ref/libfqref.so
 * (oracle/Makefile), and against the reference's golden artefacts (tests/golden/).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define FQO_OK 0
#define FQO_E_DIMENSION 1
#define FQO_E_CONFIG 2
#define FQO_E_INPUT 3
#define FQO_E_STATE 4
#define FQO_E_FORMAT 5

/* round_half_even: src/quantizer.cpp:28-31 (nearbyint under FE_TONEAREST). */
static int64_t rhe(double v) { return (int64_t)nearbyint(v); }

/* quant_code_max: src/quantizer.cpp:21-26. */
static int64_t code_max(int bits, int mode) {
  const int64_t full = (1LL << bits) - 1;
  return mode == 0 ? full : full - 1;
}

/* Quantize one "row" of the reference quantizer (one group here):
 * src/quantizer.cpp:111-189 (row_range :101-109, constant row :134-159, asym :161-170,
 * sym :171-182).  Writes unsigned stored codes. */
static int quantize_row(const float* x, int64_t n, int bits, int mode, uint32_t* codes, float* s_out,
                        int32_t* z_out) {
  float lo = x[0], hi = x[0];
  for (int64_t i = 0; i < n; ++i) {
    if (!isfinite(x[i])) return FQO_E_INPUT;
    if (x[i] < lo) lo = x[i];
    if (x[i] > hi) hi = x[i];
  }
  const int64_t qmax = code_max(bits, mode);
  const int64_t m = (1LL << (bits - 1)) - 1;
  float s;
  int32_t z = 0;
  if (lo == hi) {
    const float c = lo;
    if (mode == 0) {
      uint32_t code;
      if (c == 0.0f) { s = 1.0f; z = 0; }
      else if (c > 0.0f) { s = c; z = 0; }
      else { s = -c; z = 1; }
      code = c > 0.0f ? 1u : 0u;
      for (int64_t i = 0; i < n; ++i) codes[i] = code;
    } else {
      s = c == 0.0f ? 1.0f : fabsf(c);
      const int32_t sc = c > 0.0f ? 1 : (c < 0.0f ? -1 : 0);
      for (int64_t i = 0; i < n; ++i) codes[i] = (uint32_t)(sc + m);
    }
  } else if (mode == 0) {
    s = (float)(((double)hi - (double)lo) / (double)qmax);
    const double sd = s;
    z = (int32_t)rhe(0.0 - (double)lo / sd);
    for (int64_t i = 0; i < n; ++i) {
      int64_t c = rhe((double)x[i] / sd + (double)z);
      if (c < 0) c = 0;
      if (c > qmax) c = qmax;
      codes[i] = (uint32_t)c;
    }
  } else {
    const double amax = fmax(fabs((double)lo), fabs((double)hi));
    s = (float)(amax / (double)m);
    const double sd = s;
    for (int64_t i = 0; i < n; ++i) {
      int64_t c = rhe((double)x[i] / sd);
      if (c < -m) c = -m;
      if (c > m) c = m;
      codes[i] = (uint32_t)(c + m);
    }
  }
  *s_out = s;
  *z_out = z;
  return FQO_OK;
}

/* pack_codes: src/quantizer.cpp:60-76 (4-bit: low nibble = even flat index). */
void fqo_pack(const uint32_t* codes, int64_t count, int bits, uint8_t* out) {
  if (bits == 8) {
    for (int64_t i = 0; i < count; ++i) out[i] = (uint8_t)(codes[i] & 0xFFu);
    return;
  }
  memset(out, 0, (size_t)((count + 1) / 2));
  for (int64_t i = 0; i < count; ++i) {
    const uint8_t nib = (uint8_t)(codes[i] & 0xFu);
    out[i / 2] |= (i % 2 == 0) ? nib : (uint8_t)(nib << 4);
  }
}

/* unpack_codes: src/quantizer.cpp:78-92. */
void fqo_unpack(const uint8_t* payload, int64_t count, int bits, uint32_t* out) {
  for (int64_t i = 0; i < count; ++i) {
    if (bits == 8) out[i] = payload[i];
    else out[i] = (i % 2 == 0) ? (payload[i / 2] & 0xFu) : (uint32_t)(payload[i / 2] >> 4);
  }
}

/* Group-wise quantization of W[N,K]: the reference quantizer applied to each group
 * [row, g*G : min((g+1)*G, K)) as its own row.  G >= K gives the
 * reference's per-row granularity exactly.  Outputs: payload over the row-major stream,
 * scale/zp per (row, group). */
int fqo_quantize(const float* w, int64_t N, int64_t K, int64_t G, int bits, int mode, uint8_t* payload,
                 float* scale, int32_t* zp) {
  if (bits != 4 && bits != 8) return FQO_E_CONFIG;
  if (K == 0) return FQO_E_DIMENSION;
  if (G <= 0 || G > K) G = K;
  const int64_t ng = (K + G - 1) / G;
  uint32_t* codes = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(N * K));
  if (!codes) return FQO_E_STATE;
  for (int64_t r = 0; r < N; ++r) {
    for (int64_t g = 0; g < ng; ++g) {
      const int64_t k0 = g * G;
      const int64_t len = (k0 + G <= K) ? G : K - k0;
      const int st = quantize_row(w + r * K + k0, len, bits, mode, codes + r * K + k0, &scale[r * ng + g],
                                  &zp[r * ng + g]);
      if (st != FQO_OK) {
        free(codes);
        return st;
      }
    }
  }
  fqo_pack(codes, N * K, bits, payload);
  free(codes);
  return FQO_OK;
}

/* dequantize: src/quantizer.cpp:205-219 — x = float(int32(code) - (z + offset)) * s in fp32. */
int fqo_dequantize(const uint8_t* payload, int64_t N, int64_t K, int64_t G, int bits, int mode, const float* scale,
                   const int32_t* zp, float* out) {
  if (G <= 0 || G > K) G = K;
  const int64_t ng = (K + G - 1) / G;
  const int32_t off = mode == 1 ? (1 << (bits - 1)) - 1 : 0;
  for (int64_t r = 0; r < N; ++r) {
    for (int64_t k = 0; k < K; ++k) {
      const int64_t i = r * K + k;
      const uint32_t c = bits == 8 ? payload[i] : ((i % 2 == 0) ? (payload[i / 2] & 0xFu) : (uint32_t)(payload[i / 2] >> 4));
      const int64_t g = r * ng + k / G;
      out[i] = (float)((int32_t)c - (zp[g] + off)) * scale[g];
    }
  }
  return FQO_OK;
}

/* linear: src/tensor.cpp:83-101 — y[i,j] = float(bias_j + sum_p x_ip * W_jp), double
 * accumulator, p ascending. */
void fqo_linear(const float* x, int64_t B, int64_t K, const float* w, int64_t N, const float* bias, float* y) {
  for (int64_t i = 0; i < B; ++i) {
    for (int64_t j = 0; j < N; ++j) {
      double acc = bias ? (double)bias[j] : 0.0;
      const float* wj = w + j * K;
      const float* xi = x + i * K;
      for (int64_t p = 0; p < K; ++p) acc += (double)xi[p] * (double)wj[p];
      y[i * N + j] = (float)acc;
    }
  }
}

/* MultiPrecisionLayer::forward at an integer rung (src/model.cpp:77-98): dequantize then linear. */
int fqo_quant_linear(const float* x, int64_t B, const uint8_t* payload, int64_t N, int64_t K, int64_t G, int bits,
                     int mode, const float* scale, const int32_t* zp, const float* bias, float* y) {
  float* w = (float*)malloc(sizeof(float) * (size_t)(N * K));
  if (!w) return FQO_E_STATE;
  fqo_dequantize(payload, N, K, G, bits, mode, scale, zp, w);
  fqo_linear(x, B, K, w, N, bias, y);
  free(w);
  return FQO_OK;
}

/* softmax_double + ppl_entropy + fault_tolerance (src/scheduler.cpp:13-49) and argmax_token
 * (src/engine.cpp:144-155) of one logits row. */
int fqo_row_stats(const float* l, int64_t V, double* ppl, double* entropy, double* ft, double* p1_out,
                  double* p2_out, int32_t* argmax) {
  if (V < 1) return FQO_E_DIMENSION;
  double mx = l[0];
  for (int64_t i = 1; i < V; ++i)
    if ((double)l[i] > mx) mx = l[i];
  double* p = (double*)malloc(sizeof(double) * (size_t)V);
  if (!p) return FQO_E_STATE;
  double sum = 0.0;
  for (int64_t i = 0; i < V; ++i) {
    p[i] = exp((double)l[i] - mx);
    sum += p[i];
  }
  for (int64_t i = 0; i < V; ++i) p[i] /= sum;
  double h = 0.0;
  for (int64_t i = 0; i < V; ++i)
    if (p[i] > 0.0) h -= p[i] * log(p[i]);
  double t1 = -1.0, t2 = -1.0;
  for (int64_t i = 0; i < V; ++i) {
    if (p[i] > t1) { t2 = t1; t1 = p[i]; }
    else if (p[i] > t2) { t2 = p[i]; }
  }
  free(p);
  int32_t best = 0;
  float bv = l[0];
  for (int64_t i = 1; i < V; ++i)
    if (l[i] > bv) { bv = l[i]; best = (int32_t)i; }
  if (ppl) *ppl = exp(h);
  if (entropy) *entropy = h;
  if (ft) *ft = V >= 2 ? t1 - t2 : 0.0;
  if (p1_out) *p1_out = t1;
  if (p2_out) *p2_out = t2;
  if (argmax) *argmax = best;
  return FQO_OK;
}

/* derive_threshold: src/scheduler.cpp:51-60. */
int fqo_derive_threshold(const float* logits, int64_t n, int64_t V, int window_len, double theta, double* out) {
  if (n < 1 || V < 1) return FQO_E_STATE;
  if (window_len < 1) return FQO_E_CONFIG;
  const int64_t k = window_len < n ? window_len : n;
  double sum = 0.0;
  for (int64_t r = n - k; r < n; ++r) {
    double ppl;
    fqo_row_stats(logits + r * V, V, &ppl, NULL, NULL, NULL, NULL, NULL);
    sum += ppl;
  }
  *out = theta * (sum / (double)k);
  return FQO_OK;
}

/* SchedulerState::observe over a PPLE stream (src/scheduler.cpp:85-104), restated with a ring
 * of explicit counters.  For every observation t: fire_first[t], fire_count[t] (0 = no switch),
 * mavg[t] / mavg_valid[t] (window mean evaluated at t, pre-clear). */
int fqo_scheduler_replay(const double* ppl, int64_t n, int window_len, double thre, int layers_per_switch,
                         int64_t plan_len, int64_t* fire_first, int64_t* fire_count, double* mavg,
                         int32_t* mavg_valid) {
  if (window_len < 1 || layers_per_switch < 1) return FQO_E_CONFIG;
  double* win = (double*)malloc(sizeof(double) * (size_t)window_len);
  if (!win) return FQO_E_STATE;
  int64_t fill = 0, head = 0; /* ring of the last `fill` values starting at head */
  int cooldown = 0;
  int64_t cursor = 0;
  for (int64_t t = 0; t < n; ++t) {
    if (fill < window_len) {
      win[(head + fill) % window_len] = ppl[t];
      ++fill;
    } else {
      win[head] = ppl[t];
      head = (head + 1) % window_len;
    }
    if (cooldown > 0) --cooldown;
    fire_first[t] = 0;
    fire_count[t] = 0;
    mavg_valid[t] = 0;
    mavg[t] = 0.0;
    if (fill < window_len) continue;
    double s = 0.0;
    for (int64_t i = 0; i < fill; ++i) s += win[(head + i) % window_len];
    const double avg = s / (double)fill;
    mavg[t] = avg;
    mavg_valid[t] = 1;
    if (cooldown > 0 || !(avg < thre) || cursor >= plan_len) continue;
    const int64_t rem = plan_len - cursor;
    const int64_t cnt = layers_per_switch < rem ? layers_per_switch : rem;
    fire_first[t] = cursor;
    fire_count[t] = cnt;
    cursor += cnt;
    fill = 0;
    head = 0;
    cooldown = window_len;
  }
  free(win);
  return FQO_OK;
}

/* uniform_edges + weight_histogram + kl_divergence (src/analyzer.cpp:17-79) for one layer:
 * p = histogram of the fp weights, q = histogram of the dequantized weights, edges over the
 * fp range. */
int fqo_hist_kl(const float* w, const float* wq, int64_t n, int bins, double* kl_out) {
  if (n < 1 || bins < 1) return FQO_E_INPUT;
  float lo = w[0], hi = w[0];
  for (int64_t i = 1; i < n; ++i) {
    if (w[i] < lo) lo = w[i];
    if (w[i] > hi) hi = w[i];
  }
  double dlo = lo, dhi = hi;
  if (!(dhi > dlo)) { dlo -= 0.5; dhi += 0.5; }
  double* e = (double*)malloc(sizeof(double) * (size_t)(bins + 1));
  double* p = (double*)calloc((size_t)bins, sizeof(double));
  double* q = (double*)calloc((size_t)bins, sizeof(double));
  if (!e || !p || !q) return FQO_E_STATE;
  const double width = (dhi - dlo) / (double)bins;
  for (int i = 0; i <= bins; ++i) e[i] = dlo + width * i;
  e[bins] = dhi;
  for (int pass = 0; pass < 2; ++pass) {
    const float* src = pass == 0 ? w : wq;
    double* c = pass == 0 ? p : q;
    for (int64_t i = 0; i < n; ++i) {
      const double v = src[i];
      int b;
      if (v < e[1]) b = 0;
      else if (v >= e[bins - 1]) b = bins - 1;
      else {
        /* largest b with e[b] <= v (== upper_bound - 1), by bisection */
        int lo_i = 1, hi_i = bins - 1;
        while (hi_i - lo_i > 1) {
          const int mid = (lo_i + hi_i) / 2;
          if (e[mid] <= v) lo_i = mid;
          else hi_i = mid;
        }
        b = lo_i;
      }
      c[b] += 1.0;
    }
    double total = 0.0;
    for (int i = 0; i < bins; ++i) {
      c[i] += 1e-10;
      total += c[i];
    }
    for (int i = 0; i < bins; ++i) c[i] /= total;
  }
  double kl = 0.0;
  for (int i = 0; i < bins; ++i) kl += p[i] * log(p[i] / q[i]);
  free(e);
  free(p);
  free(q);
  *kl_out = kl;
  return FQO_OK;
}

/* Logit-mode KL (BASELINE config 4; no reference function): softmax_double of both rows then
 * kl_divergence's sum p ln(p/q) (src/analyzer.cpp:65-79). */
int fqo_kl_logits(const float* lq, const float* lp, int64_t V, double* kl_out, double* ent_out) {
  double mq = lq[0], mp = lp[0];
  for (int64_t i = 1; i < V; ++i) {
    if ((double)lq[i] > mq) mq = lq[i];
    if ((double)lp[i] > mp) mp = lp[i];
  }
  double sq = 0.0, sp = 0.0;
  for (int64_t i = 0; i < V; ++i) {
    sq += exp((double)lq[i] - mq);
    sp += exp((double)lp[i] - mp);
  }
  double kl = 0.0, h = 0.0;
  for (int64_t i = 0; i < V; ++i) {
    const double a = exp((double)lq[i] - mq) / sq;
    const double b = exp((double)lp[i] - mp) / sp;
    if (a > 0.0) {
      kl += a * log(a / b);
      h -= a * log(a);
    }
  }
  *kl_out = kl;
  if (ent_out) *ent_out = h;
  return FQO_OK;
}

/* Deterministic N(0,std) values keyed by (seed, stream, index); same definition as the
 * engine's generator so oracle and device see identical weights. */
static uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

void fqo_fill_normal(float* dst, int64_t n, uint64_t seed, uint64_t stream, float std) {
  const uint64_t key = mix64(seed ^ mix64(stream + 0x5851f42d4c957f2dULL));
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t r1 = mix64(key + 2 * (uint64_t)i);
    const uint64_t r2 = mix64(key + 2 * (uint64_t)i + 1);
    const double u1 = (double)((r1 >> 40) + 1) * (1.0 / 16777216.0);
    const double u2 = (double)(r2 >> 40) * (1.0 / 16777216.0);
    const double z = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
    dst[i] = (float)(z * (double)std);
  }
}

/* std::mt19937_64 (the engine behind uniform_signed / random_tokens, src/fixture.cpp:32-38,
 * 133-138), restated so seeded fixtures can be regenerated without the reference. */
typedef struct { uint64_t mt[312]; int idx; } fqo_mt64;

void fqo_mt64_seed(fqo_mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i) s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->idx = 312;
}

uint64_t fqo_mt64_next(fqo_mt64* s) {
  if (s->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (s->mt[i] & 0xFFFFFFFF80000000ULL) | (s->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
    }
    s->idx = 0;
  }
  uint64_t y = s->mt[s->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= (y >> 43);
  return y;
}

size_t fqo_mt64_size(void) { return sizeof(fqo_mt64); }

/* uniform_signed (src/fixture.cpp:32-38): a * (2u - 1), u = 24-bit mantissa draw. */
void fqo_uniform_signed(fqo_mt64* s, float a, float* dst, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t r = fqo_mt64_next(s) >> 40;
    const float u = (float)r * (1.0f / 16777216.0f);
    dst[i] = a * (2.0f * u - 1.0f);
  }
}

/* random_tokens (src/fixture.cpp:133-138). */
void fqo_random_tokens(int64_t n, int64_t vocab, uint64_t seed, int32_t* out) {
  fqo_mt64 s;
  fqo_mt64_seed(&s, seed);
  for (int64_t i = 0; i < n; ++i) out[i] = (int32_t)(fqo_mt64_next(&s) % (uint64_t)vocab);
}
