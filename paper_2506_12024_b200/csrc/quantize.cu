// Device-side RTN quantizer (K9) and the deterministic normal generator.
//
// quantize_group_kernel restates quantize_impl (/root/reference/proj/src/quantizer.cpp:111-189)
// per quantization group (one group = one "row" of the reference quantizer on the
// [N*ceil(K/G), G] view; a ragged tail group is its own row):
//   asym:  s = float((double(hi) - double(lo)) / qmax); z = rint(-lo / double(s)) (not clamped);
//          code = clamp(rint(x / double(s) + z), 0, qmax)
//   sym:   s = float(amax / m); code = clamp(rint(x / double(s)), -m, m) + m
//   constant groups: the exact-dequantization special cases (quantizer.cpp:134-159).
// rint() rounds half to even like nearbyint under FE_TONEAREST; double division is IEEE, so the
// codes/scales/zero points are bit-identical to the reference.
#include "fq_internal.cuh"

#include <cfloat>
#include <cmath>

namespace fqc {
namespace {

__global__ void quantize_group_kernel(const float* __restrict__ w, int64_t N, int64_t K, int64_t G, int64_t ng, int64_t ng_pad,
                                      int bits, int mode, uint8_t* __restrict__ payload, float* __restrict__ scale,
                                      int32_t* __restrict__ zp_eff, int* __restrict__ bad) {
  const int lane = threadIdx.x & 31;
  const int64_t gid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (gid >= N * ng) return;
  const int64_t row = gid / ng, g = gid % ng;
  const int64_t k0 = g * G;
  const int64_t len = (k0 + G <= K) ? G : (K - k0);
  const float* x = w + row * K + k0;
  float lo = x[0], hi = x[0];
  bool finite = true;
  for (int64_t i = lane; i < len; i += 32) {
    const float v = x[i];
    if (!isfinite(v)) finite = false;
    lo = fminf(lo, v);
    hi = fmaxf(hi, v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  finite = __all_sync(0xffffffffu, finite);
  if (!finite) {
    if (lane == 0) atomicExch(bad, 1);
    return;
  }
  const int64_t qmax = mode == FQ_MODE_ASYM ? (1 << bits) - 1 : (1 << bits) - 2;
  const int64_t m = (1 << (bits - 1)) - 1;  // symmetric magnitude / stored offset
  float s;
  int32_t z = 0;
  // codes are written per element: 8-bit one byte each; 4-bit nibble pairs (group starts are even)
  auto put = [&](int64_t i, uint32_t code0, uint32_t code1, bool pair) {
    const int64_t flat = row * K + k0 + i;
    if (bits == 8) {
      payload[flat] = static_cast<uint8_t>(code0);
    } else {
      payload[flat >> 1] = static_cast<uint8_t>((code0 & 0xFu) | (pair ? (code1 & 0xFu) << 4 : 0u));
    }
  };
  const int step = bits == 8 ? 1 : 2;
  if (lo == hi) {
    const float c = lo;
    uint32_t code;
    if (mode == FQ_MODE_ASYM) {
      if (c == 0.0f) { s = 1.0f; z = 0; }
      else if (c > 0.0f) { s = c; z = 0; }
      else { s = -c; z = 1; }
      code = c > 0.0f ? 1u : 0u;
    } else {
      s = c == 0.0f ? 1.0f : fabsf(c);
      const int sc = c > 0.0f ? 1 : (c < 0.0f ? -1 : 0);
      code = static_cast<uint32_t>(sc + m);
    }
    for (int64_t i = lane * step; i < len; i += 32 * step) put(i, code, code, i + 1 < len);
  } else if (mode == FQ_MODE_ASYM) {
    s = static_cast<float>((static_cast<double>(hi) - static_cast<double>(lo)) / static_cast<double>(qmax));
    const double sd = s;
    z = static_cast<int32_t>(rint(0.0 - static_cast<double>(lo) / sd));
    auto code_of = [&](float v) {
      int64_t c = static_cast<int64_t>(rint(static_cast<double>(v) / sd + static_cast<double>(z)));
      c = c < 0 ? 0 : (c > qmax ? qmax : c);
      return static_cast<uint32_t>(c);
    };
    for (int64_t i = lane * step; i < len; i += 32 * step)
      put(i, code_of(x[i]), i + 1 < len ? code_of(x[i + 1]) : 0u, i + 1 < len);
  } else {
    const double amax = fmax(fabs(static_cast<double>(lo)), fabs(static_cast<double>(hi)));
    s = static_cast<float>(amax / static_cast<double>(m));
    const double sd = s;
    auto code_of = [&](float v) {
      int64_t c = static_cast<int64_t>(rint(static_cast<double>(v) / sd));
      c = c < -m ? -m : (c > m ? m : c);
      return static_cast<uint32_t>(c + m);
    };
    for (int64_t i = lane * step; i < len; i += 32 * step)
      put(i, code_of(x[i]), i + 1 < len ? code_of(x[i + 1]) : 0u, i + 1 < len);
  }
  if (lane == 0) {
    scale[row * ng_pad + g] = s;
    zp_eff[gid] = z + (mode == FQ_MODE_SYM ? static_cast<int32_t>(m) : 0);
  }
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// N(0, std): Box-Muller on two 24-bit uniforms drawn from a counter-based splitmix64 stream.
__global__ void fill_normal_kernel(float* __restrict__ dst, int64_t n, uint64_t seed, uint64_t stream, float std) {
  const uint64_t key = mix64(seed ^ mix64(stream + 0x5851f42d4c957f2dull));
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t r1 = mix64(key + 2 * static_cast<uint64_t>(i));
    const uint64_t r2 = mix64(key + 2 * static_cast<uint64_t>(i) + 1);
    const double u1 = static_cast<double>((r1 >> 40) + 1) * (1.0 / 16777216.0);
    const double u2 = static_cast<double>(r2 >> 40) * (1.0 / 16777216.0);
    const double z = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
    dst[i] = static_cast<float>(z * static_cast<double>(std));
  }
}

__global__ void zp_range_kernel(const int32_t* __restrict__ zp, int64_t n, int* out /*[2]: min,max*/) {
  int lo = INT_MAX, hi = INT_MIN;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    lo = min(lo, zp[i]);
    hi = max(hi, zp[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&out[0], lo);
    atomicMax(&out[1], hi);
  }
}

// Builds the tiled fast-path copy (fq_internal.cuh) of one rung from its canonical arrays:
// one CTA per 16x128 block, 128 threads = (word i, lane t) of the code region, then the meta.
__device__ __forceinline__ uint32_t canon_code(const uint8_t* __restrict__ p, int bits, int64_t N, int64_t K,
                                               int64_t row, int64_t k) {
  if (row >= N || k >= K) return 0u;
  const int64_t idx = row * K + k;
  if (bits == 8) return p[idx];
  const uint32_t b = p[idx >> 1];
  return (idx & 1) ? (b >> 4) : (b & 0xFu);
}

__global__ void tile_pack_kernel(const uint8_t* __restrict__ payload, const float* __restrict__ scale,
                                 const int32_t* __restrict__ zp32, int64_t N, int64_t K, int64_t G, int64_t ng,
                                 int64_t ng_pad, int bits, int32_t zbase, int64_t nkb, uint8_t* __restrict__ out) {
  const int64_t blk = blockIdx.x;
  const int64_t tile = blk / nkb, kb = blk % nkb;
  const int bb = bits == 8 ? kBlockBytes8 : kBlockBytes4;
  uint8_t* dst = out + blk * bb;
  const int64_t row0 = tile * kTileRows;
  const int t = threadIdx.x & 31, i = threadIdx.x >> 5;
  const int r = t >> 2, c2 = 2 * (t & 3);
  if (bits == 8) {
    uint32_t u[4];
    for (int h = 0; h < 2; ++h) {
      const int64_t k0 = kb * kBlockK + 16 * (2 * i + h) + c2;
      for (int e = 0; e < 2; ++e) {
        const int64_t k = k0 + 8 * e;
        u[2 * h + e] = canon_code(payload, 8, N, K, row0 + r, k) | canon_code(payload, 8, N, K, row0 + r, k + 1) << 8 |
                       canon_code(payload, 8, N, K, row0 + r + 8, k) << 16 |
                       canon_code(payload, 8, N, K, row0 + r + 8, k + 1) << 24;
      }
    }
    reinterpret_cast<uint4*>(dst)[i * 32 + t] = make_uint4(u[0], u[1], u[2], u[3]);
  } else if (i < 2) {
    uint32_t u[4];
    for (int v = 0; v < 4; ++v) {
      const int64_t k0 = kb * kBlockK + 16 * (4 * i + v) + c2;
      const int64_t ra = row0 + r, rb = row0 + r + 8;
      const uint32_t n[8] = {canon_code(payload, 4, N, K, ra, k0),     canon_code(payload, 4, N, K, ra, k0 + 8),
                             canon_code(payload, 4, N, K, rb, k0),     canon_code(payload, 4, N, K, rb, k0 + 8),
                             canon_code(payload, 4, N, K, ra, k0 + 1), canon_code(payload, 4, N, K, ra, k0 + 9),
                             canon_code(payload, 4, N, K, rb, k0 + 1), canon_code(payload, 4, N, K, rb, k0 + 9)};
      uint32_t w = 0;
      for (int e = 0; e < 8; ++e) w |= n[e] << (4 * e);
      u[v] = w;
    }
    reinterpret_cast<uint4*>(dst)[i * 32 + t] = make_uint4(u[0], u[1], u[2], u[3]);
  }
  if (threadIdx.x < kTileRows) {
    const int64_t row = row0 + threadIdx.x;
    const int64_t g = (kb * kBlockK) / G;
    const int codes = bits == 8 ? 2048 : 1024;
    float sc = 0.f;
    uint8_t z = 0;
    if (row < N) {
      sc = scale[row * ng_pad + g];
      z = static_cast<uint8_t>(zp32[row * ng + g] - zbase);
    }
    reinterpret_cast<float*>(dst + codes)[threadIdx.x] = sc;
    dst[codes + 64 + threadIdx.x] = z;
  }
}

}  // namespace

void finalize_rung_meta(fq_ctx* ctx, fq_layer* L, int rung) {
  fq_rung_store& st = L->store(rung);
  const int64_t n = L->N * L->ng;
  int* d = static_cast<int*>(ctx->ensure_scratch(64));
  const int init[2] = {INT_MAX, INT_MIN};
  FQ_CUDA(cudaMemcpyAsync(d, init, sizeof(init), cudaMemcpyHostToDevice, ctx->stream));
  const int blocks = static_cast<int>(std::min<int64_t>(1024, (n + 255) / 256));
  zp_range_kernel<<<std::max(blocks, 1), 256, 0, ctx->stream>>>(st.zp32, n, d);
  FQ_CUDA(cudaGetLastError());
  int h[2];
  FQ_CUDA(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  FQ_CUDA(cudaStreamSynchronize(ctx->stream));
  st.zp_fits_u8 = (static_cast<int64_t>(h[1]) - h[0]) <= 255;
  st.zp_base = st.zp_fits_u8 ? h[0] : 0;
  const bool one_group_per_block = L->G % kBlockK == 0 || L->G >= L->K;
  ctx->weight_epoch += 1;  // cached step programs / graphs hold tile pointers: rebuild them
  const int64_t n_tiles = (L->N + kTileRows - 1) / kTileRows, nkb = (L->K + kBlockK - 1) / kBlockK;
  const int64_t want = (st.zp_fits_u8 && one_group_per_block) ? n_tiles * nkb * (st.bits == 8 ? kBlockBytes8 : kBlockBytes4) : 0;
  if (want != st.tiles_bytes) {  // same size: repack in place (the pointer stays valid)
    dfree(st.tiles);
    st.tiles = nullptr;
    st.tiles_bytes = 0;
  }
  if (want > 0) {
    if (st.tiles == nullptr) st.tiles = static_cast<uint8_t*>(dmalloc(static_cast<size_t>(want)));
    st.tiles_bytes = want;
    tile_pack_kernel<<<static_cast<unsigned>(n_tiles * nkb), 128, 0, ctx->stream>>>(
        st.payload, st.scale, st.zp32, L->N, L->K, L->G, L->ng, L->ng_pad, st.bits, st.zp_base, nkb, st.tiles);
    FQ_CUDA(cudaGetLastError());
    ctx->launches += 1;
  }
  ctx->launches += 1;
}

void quantize_device(fq_ctx* ctx, fq_layer* L, int rung, int mode, const float* w_dev) {
  if (rung != FQ_RUNG_INT8 && rung != FQ_RUNG_INT4) fail(FQ_E_CONFIG, "quantize: rung must be 8 or 4");
  if (mode != FQ_MODE_ASYM && mode != FQ_MODE_SYM) fail(FQ_E_CONFIG, "quantize: bad mode");
  if (L->K == 0) fail(FQ_E_DIMENSION, "cannot quantize a tensor with zero columns");
  const int bits = rung == FQ_RUNG_INT8 ? 8 : 4;
  if (bits == 4 && (L->G % 2 != 0 || L->K % 2 != 0))
    fail(FQ_E_CONFIG, "quantize: 4-bit device packing needs even group size and row length");
  fq_rung_store& st = L->store(rung);
  const int64_t n = L->N * L->K;
  const int64_t bytes = (n * bits + 7) / 8;
  const int64_t groups = L->N * L->ng;
  if (!st.present) {
    st.payload = static_cast<uint8_t*>(dmalloc(bytes));
    st.scale = static_cast<float*>(dmalloc(sizeof(float) * L->N * L->ng_pad));
    FQ_CUDA(cudaMemsetAsync(st.scale, 0, sizeof(float) * L->N * L->ng_pad, ctx->stream));
    st.zp32 = static_cast<int32_t*>(dmalloc(sizeof(int32_t) * groups));
  }
  st.bits = bits;
  st.mode = mode;
  st.payload_bytes = bytes;
  int* bad = static_cast<int*>(ctx->ensure_scratch(64));
  FQ_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), ctx->stream));
  const int64_t threads = groups * 32;
  quantize_group_kernel<<<ceil_div_i(threads, 256), 256, 0, ctx->stream>>>(w_dev, L->N, L->K, L->G, L->ng, L->ng_pad, bits, mode,
                                                                          st.payload, st.scale, st.zp32, bad);
  FQ_CUDA(cudaGetLastError());
  ctx->launches += 1;
  int hbad = 0;
  FQ_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  FQ_CUDA(cudaStreamSynchronize(ctx->stream));
  if (hbad) fail(FQ_E_INPUT, "quantize: non-finite input value");
  st.present = true;
  finalize_rung_meta(ctx, L, rung);
}

void fill_normal(fq_ctx* ctx, float* dst, int64_t n, uint64_t seed, uint64_t stream, float std) {
  if (n <= 0) return;
  const int blocks = static_cast<int>(std::min<int64_t>(ctx->num_sms * 8, (n + 255) / 256));
  fill_normal_kernel<<<blocks, 256, 0, ctx->stream>>>(dst, n, seed, stream, std);
  FQ_CUDA(cudaGetLastError());
  ctx->launches += 1;
}

}  // namespace fqc
