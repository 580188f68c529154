// Integer weight quantization (reference: include/flexquant/quantizer.hpp:12-71,
// src/quantizer.cpp).  Extended with a quantization group along the row: group_size == 0 (or
// >= cols) is the reference's per-row scheme bit for bit; group_size == 128 is the
// BASELINE g128 scheme (each group quantized as one reference row; scale / zero point per
// (row, group) in row-major order; the payload is the same flat row-major code stream).
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "flexquant/tensor.hpp"

namespace flexquant {

enum class QuantMode : uint8_t { Asymmetric = FQ_MODE_ASYM, Symmetric = FQ_MODE_SYM };
const char* to_string(QuantMode mode);

struct QuantizedTensor {
  int bits = 8;
  QuantMode mode = QuantMode::Asymmetric;
  int64_t rows = 0;
  int64_t cols = 0;
  int64_t group_size = 0;            // 0 = one group per row
  std::vector<uint8_t> payload;      // packed codes; 4-bit: low nibble = even flat index
  std::vector<float> scale;          // rows * groups_per_row()
  std::vector<int32_t> zero_point;   // rows * groups_per_row(); 0 in symmetric mode

  int64_t numel() const { return rows * cols; }
  int64_t group() const { return (group_size <= 0 || group_size >= cols) ? cols : group_size; }
  int64_t groups_per_row() const { return cols == 0 ? 0 : (cols + group() - 1) / group(); }
  size_t expected_payload_bytes() const { return static_cast<size_t>((numel() * bits + 7) / 8); }
  uint32_t code_at(int64_t r, int64_t c) const;
  int32_t stored_offset() const { return mode == QuantMode::Symmetric ? (1 << (bits - 1)) - 1 : 0; }
  void validate() const;
};

uint32_t quant_code_max(int bits, QuantMode mode);
int64_t round_half_even(double v);
std::vector<uint8_t> pack_codes(std::span<const uint32_t> codes, int bits);
std::vector<uint32_t> unpack_codes(std::span<const uint8_t> payload, int64_t count, int bits);

QuantizedTensor quantize_asymmetric(const Tensor& x, int bits, int64_t group_size = 0);
QuantizedTensor quantize_symmetric(const Tensor& x, int bits, int64_t group_size = 0);
QuantizedTensor quantize(const Tensor& x, int bits, QuantMode mode, int64_t group_size = 0);
// Same result computed by the device quantizer (K9); requires even group / row lengths for 4-bit.
QuantizedTensor quantize_device(const Tensor& x, int bits, QuantMode mode, int64_t group_size = 0);
Tensor dequantize(const QuantizedTensor& q);

struct QuantErrorStats {
  double max_abs_err = 0.0;
  double mean_sq_err = 0.0;
};
QuantErrorStats quant_error_stats(const Tensor& x, const QuantizedTensor& q);

}  // namespace flexquant
