// Internal helpers shared by the host library's translation units.
#pragma once

#include <vector>

#include "flexquant/tensor.hpp"

namespace flexquant::detail {

// Softmax statistics of `rows` logits rows of a host tensor, computed by the device kernel.
std::vector<fq_row_stats> device_row_stats(const Tensor& logits, int64_t rows, int64_t vocab);

}  // namespace flexquant::detail
