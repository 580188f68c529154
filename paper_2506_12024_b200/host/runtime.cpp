// Host runtime of the C++ API: the process-wide device context, status -> exception mapping,
// and the Tensor value type.
#include <cstdlib>
#include <mutex>
#include <sstream>

#include "flexquant/tensor.hpp"
#include "flexquant/model.hpp"

namespace flexquant {

namespace detail {

void throw_status(fq_status st) {
  const std::string msg = fq_last_error();
  switch (st) {
    case FQ_E_DIMENSION: throw DimensionError(msg);
    case FQ_E_CONFIG: throw ConfigError(msg);
    case FQ_E_INPUT: throw InputError(msg);
    case FQ_E_STATE: throw StateError(msg);
    case FQ_E_FORMAT: throw FormatError(msg);
    case FQ_E_CAPACITY: throw CapacityError(msg);
    default: throw DeviceError(msg);
  }
}

}  // namespace detail

fq_ctx* runtime() {
  static std::once_flag once;
  static fq_ctx* ctx = nullptr;
  static fq_status status = FQ_OK;
  static std::string err;
  std::call_once(once, [] {
    int dev = 0;
    if (const char* e = std::getenv("FQ_DEVICE")) dev = std::atoi(e);
    else if (const char* l = std::getenv("LOCAL_RANK")) dev = std::atoi(l);
    status = fq_ctx_create(dev, &ctx);
    if (status != FQ_OK) err = fq_last_error();
  });
  if (status != FQ_OK) {
    // No silent CPU path: without a B200 the API is unusable.
    throw DeviceError("flexquant runtime: no usable B200 device: " + err);
  }
  return ctx;
}

namespace {
int64_t checked_numel(const std::vector<int64_t>& shape) {
  int64_t n = 1;
  for (int64_t d : shape) {
    if (d < 0) throw DimensionError("negative dimension in shape");
    n *= d;
  }
  return n;
}
}  // namespace

Tensor::Tensor(std::vector<int64_t> shape) : shape_(std::move(shape)) {
  data_.assign(static_cast<size_t>(checked_numel(shape_)), 0.0f);
}

Tensor Tensor::from_data(std::vector<int64_t> shape, std::vector<float> data) {
  if (checked_numel(shape) != static_cast<int64_t>(data.size())) throw DimensionError("data length does not match shape");
  Tensor t;
  t.shape_ = std::move(shape);
  t.data_ = std::move(data);
  return t;
}

int64_t Tensor::rows() const {
  if (ndim() != 2) throw DimensionError("rows() requires a 2-D tensor, got " + shape_str());
  return shape_[0];
}

int64_t Tensor::cols() const {
  if (ndim() != 2) throw DimensionError("cols() requires a 2-D tensor, got " + shape_str());
  return shape_[1];
}

Tensor Tensor::row_copy(int64_t r) const {
  Tensor out({1, cols()});
  std::copy(row(r), row(r) + cols(), out.data());
  return out;
}

std::string Tensor::shape_str() const {
  std::ostringstream os;
  os << '[';
  for (size_t i = 0; i < shape_.size(); ++i) os << (i ? "x" : "") << shape_[i];
  os << ']';
  return os.str();
}

}  // namespace flexquant
