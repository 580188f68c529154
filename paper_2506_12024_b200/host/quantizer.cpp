// Quantizer of the C++ API (reference semantics: /root/reference/proj/src/quantizer.cpp).
//
// quantize() is the offline conversion a user runs once per checkpoint; it restates the
// reference rules per quantization group (round half to even in double, asymmetric zero point
// not clamped, exact constant groups).  quantize_device() produces the same bits with the
// device quantizer (K9) for large checkpoints.
#include <algorithm>
#include <cmath>
#include <string>

#include "device_buffer.hpp"
#include "flexquant/model.hpp"
#include "flexquant/quantizer.hpp"

namespace flexquant {

const char* to_string(QuantMode mode) { return mode == QuantMode::Asymmetric ? "asymmetric" : "symmetric"; }

namespace {

void require_bits(int bits) {
  if (bits != 4 && bits != 8) throw ConfigError("unsupported bit-width " + std::to_string(bits));
}

// One reference "row" (here: one group) -> codes, scale, zero point.
void quantize_group(const float* x, int64_t n, int bits, QuantMode mode, uint32_t* codes, float& s_out,
                    int32_t& z_out) {
  float lo = x[0], hi = x[0];
  for (int64_t i = 0; i < n; ++i) {
    if (!std::isfinite(x[i])) throw InputError("quantize: non-finite input value");
    lo = std::min(lo, x[i]);
    hi = std::max(hi, x[i]);
  }
  const int64_t qmax = quant_code_max(bits, mode);
  const int64_t half = (int64_t{1} << (bits - 1)) - 1;
  if (lo == hi) {  // exact constant groups (quantizer.cpp:134-159)
    const float c = lo;
    if (mode == QuantMode::Asymmetric) {
      s_out = c == 0.0f ? 1.0f : std::fabs(c);
      z_out = c < 0.0f ? 1 : 0;
      std::fill(codes, codes + n, c > 0.0f ? 1u : 0u);
    } else {
      s_out = c == 0.0f ? 1.0f : std::fabs(c);
      z_out = 0;
      const int64_t sc = c > 0.0f ? 1 : (c < 0.0f ? -1 : 0);
      std::fill(codes, codes + n, static_cast<uint32_t>(sc + half));
    }
    return;
  }
  if (mode == QuantMode::Asymmetric) {
    const float s = static_cast<float>((static_cast<double>(hi) - static_cast<double>(lo)) / static_cast<double>(qmax));
    const double sd = s;
    const int32_t z = static_cast<int32_t>(round_half_even(-static_cast<double>(lo) / sd));
    for (int64_t i = 0; i < n; ++i)
      codes[i] = static_cast<uint32_t>(std::clamp<int64_t>(round_half_even(x[i] / sd + z), 0, qmax));
    s_out = s;
    z_out = z;
  } else {
    const double amax = std::max(std::fabs(static_cast<double>(lo)), std::fabs(static_cast<double>(hi)));
    const float s = static_cast<float>(amax / static_cast<double>(half));
    const double sd = s;
    for (int64_t i = 0; i < n; ++i)
      codes[i] = static_cast<uint32_t>(std::clamp<int64_t>(round_half_even(x[i] / sd), -half, half) + half);
    s_out = s;
    z_out = 0;
  }
}

}  // namespace

uint32_t quant_code_max(int bits, QuantMode mode) {
  require_bits(bits);
  const uint32_t full = (1u << bits) - 1u;
  return mode == QuantMode::Asymmetric ? full : full - 1u;
}

int64_t round_half_even(double v) { return static_cast<int64_t>(std::nearbyint(v)); }

uint32_t QuantizedTensor::code_at(int64_t r, int64_t c) const {
  const int64_t i = r * cols + c;
  if (bits == 8) return payload[static_cast<size_t>(i)];
  const uint8_t b = payload[static_cast<size_t>(i >> 1)];
  return (i & 1) ? (b >> 4) : (b & 0x0Fu);
}

void QuantizedTensor::validate() const {
  require_bits(bits);
  if (rows < 0 || cols < 0) throw FormatError("quantized tensor has negative shape");
  if (payload.size() != expected_payload_bytes())
    throw FormatError("quantized tensor payload length " + std::to_string(payload.size()) + " does not match expected " +
                      std::to_string(expected_payload_bytes()));
  const size_t groups = static_cast<size_t>(rows * groups_per_row());
  if (scale.size() != groups || zero_point.size() != groups)
    throw FormatError("quantized tensor scale/zero-point length mismatch");
  for (float s : scale)
    if (!(s > 0.0f) || !std::isfinite(s)) throw FormatError("quantized tensor scale must be positive and finite");
}

std::vector<uint8_t> pack_codes(std::span<const uint32_t> codes, int bits) {
  require_bits(bits);
  if (bits == 8) {
    std::vector<uint8_t> out(codes.size());
    std::transform(codes.begin(), codes.end(), out.begin(), [](uint32_t c) { return static_cast<uint8_t>(c); });
    return out;
  }
  std::vector<uint8_t> out((codes.size() + 1) / 2, 0);
  for (size_t i = 0; i < codes.size(); ++i)
    out[i >> 1] |= static_cast<uint8_t>((codes[i] & 0xFu) << ((i & 1) ? 4 : 0));
  return out;
}

std::vector<uint32_t> unpack_codes(std::span<const uint8_t> payload, int64_t count, int bits) {
  require_bits(bits);
  if (payload.size() != static_cast<size_t>((count * bits + 7) / 8))
    throw FormatError("payload length does not match element count");
  std::vector<uint32_t> out(static_cast<size_t>(count));
  for (int64_t i = 0; i < count; ++i) {
    if (bits == 8) out[static_cast<size_t>(i)] = payload[static_cast<size_t>(i)];
    else out[static_cast<size_t>(i)] = (i & 1) ? (payload[static_cast<size_t>(i >> 1)] >> 4)
                                               : (payload[static_cast<size_t>(i >> 1)] & 0x0Fu);
  }
  return out;
}

QuantizedTensor quantize(const Tensor& x, int bits, QuantMode mode, int64_t group_size) {
  require_bits(bits);
  const int64_t rows = x.rows(), cols = x.cols();
  if (cols == 0) throw DimensionError("cannot quantize a tensor with zero columns");
  QuantizedTensor q;
  q.bits = bits;
  q.mode = mode;
  q.rows = rows;
  q.cols = cols;
  q.group_size = group_size >= cols ? 0 : std::max<int64_t>(0, group_size);
  const int64_t G = q.group(), ng = q.groups_per_row();
  q.scale.resize(static_cast<size_t>(rows * ng));
  q.zero_point.resize(static_cast<size_t>(rows * ng));
  std::vector<uint32_t> codes(static_cast<size_t>(rows * cols));
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t g = 0; g < ng; ++g) {
      const int64_t k0 = g * G, len = std::min(G, cols - k0);
      quantize_group(x.row(r) + k0, len, bits, mode, codes.data() + r * cols + k0, q.scale[r * ng + g],
                     q.zero_point[r * ng + g]);
    }
  q.payload = pack_codes(codes, bits);
  return q;
}

QuantizedTensor quantize_asymmetric(const Tensor& x, int bits, int64_t group_size) {
  return quantize(x, bits, QuantMode::Asymmetric, group_size);
}
QuantizedTensor quantize_symmetric(const Tensor& x, int bits, int64_t group_size) {
  return quantize(x, bits, QuantMode::Symmetric, group_size);
}

QuantizedTensor quantize_device(const Tensor& x, int bits, QuantMode mode, int64_t group_size) {
  require_bits(bits);
  const int64_t rows = x.rows(), cols = x.cols();
  if (cols == 0) throw DimensionError("cannot quantize a tensor with zero columns");
  fq_ctx* ctx = runtime();
  fq_layer* L = nullptr;
  detail::check(fq_layer_create(ctx, rows, cols, group_size, &L));
  QuantizedTensor q;
  try {
    DeviceBuffer w(sizeof(float) * x.numel());
    w.upload(x.data(), sizeof(float) * x.numel());
    const int rung = bits == 8 ? FQ_RUNG_INT8 : FQ_RUNG_INT4;
    detail::check(fq_layer_quantize_device(L, rung, static_cast<int32_t>(mode), static_cast<const float*>(w.get())));
    q.bits = bits;
    q.mode = mode;
    q.rows = rows;
    q.cols = cols;
    q.group_size = group_size >= cols ? 0 : group_size;
    q.payload.resize(q.expected_payload_bytes());
    q.scale.resize(static_cast<size_t>(rows * q.groups_per_row()));
    q.zero_point.resize(q.scale.size());
    detail::check(fq_layer_download_quantized(L, rung, q.payload.data(), q.scale.data(), q.zero_point.data()));
  } catch (...) {
    fq_layer_destroy(L);
    throw;
  }
  fq_layer_destroy(L);
  return q;
}

Tensor dequantize(const QuantizedTensor& q) {
  q.validate();
  const std::vector<uint32_t> codes = unpack_codes(q.payload, q.numel(), q.bits);
  const int32_t off = q.stored_offset();
  const int64_t G = q.group(), ng = q.groups_per_row();
  Tensor out({q.rows, q.cols});
  for (int64_t r = 0; r < q.rows; ++r)
    for (int64_t c = 0; c < q.cols; ++c) {
      const int64_t g = r * ng + c / G;
      out.at(r, c) = static_cast<float>(static_cast<int32_t>(codes[static_cast<size_t>(r * q.cols + c)]) -
                                        (q.zero_point[static_cast<size_t>(g)] + off)) *
                     q.scale[static_cast<size_t>(g)];
    }
  return out;
}

QuantErrorStats quant_error_stats(const Tensor& x, const QuantizedTensor& q) {
  if (x.rows() != q.rows || x.cols() != q.cols) throw DimensionError("quant_error_stats: shape mismatch");
  const Tensor back = dequantize(q);
  QuantErrorStats st;
  double sq = 0.0;
  for (int64_t i = 0; i < x.numel(); ++i) {
    const double e = static_cast<double>(x.flat(i)) - static_cast<double>(back.flat(i));
    st.max_abs_err = std::max(st.max_abs_err, std::fabs(e));
    sq += e * e;
  }
  st.mean_sq_err = x.numel() ? sq / static_cast<double>(x.numel()) : 0.0;
  return st;
}

}  // namespace flexquant
