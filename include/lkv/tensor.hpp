// lkv/tensor.hpp -- the reference's float64 value type (proj/include/lkv/tensor.hpp:35-71) for
// the declaration-compatible B200 API: a shape plus a shared host buffer; copies share storage.
// This build is inference-only: there is no tape, requires_grad is carried as a flag and an input
// that requires a gradient is rejected by the device operators with contract_error.
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

namespace lkv {

using TensorId = const void*;

class Tensor {
public:
    Tensor() = default;
    explicit Tensor(std::vector<int> shape, bool requires_grad = false);
    static Tensor scalar(double v, bool requires_grad = false);
    static Tensor full(std::vector<int> shape, double v, bool requires_grad = false);
    static Tensor from(std::vector<int> shape, std::vector<double> values, bool requires_grad = false);

    bool defined() const { return buf_ != nullptr; }
    const std::vector<int>& shape() const { return shape_; }
    int rank() const { return static_cast<int>(shape_.size()); }
    int dim(int i) const { return shape_[static_cast<size_t>(i)]; }
    size_t numel() const;
    bool requires_grad() const { return grad_; }
    void set_requires_grad(bool v) { grad_ = v; }
    double* data() { return buf_->data(); }
    const double* data() const { return buf_->data(); }
    const std::vector<double>& vec() const { return *buf_; }
    double value() const;  // the single element of a one-element tensor
    TensorId id() const { return static_cast<TensorId>(buf_.get()); }
    Tensor detached_clone() const;

private:
    std::vector<int> shape_;
    std::shared_ptr<std::vector<double>> buf_;
    bool grad_ = false;
};

// Inference-only build: recording is always off; the guard exists so reference call sites compile.
bool grad_enabled();
class NoGradGuard {
public:
    NoGradGuard() = default;
    ~NoGradGuard() = default;
    NoGradGuard(const NoGradGuard&) = delete;
    NoGradGuard& operator=(const NoGradGuard&) = delete;
};

// Same data, new shape (element count must match).
Tensor reshape(const Tensor& x, std::vector<int> shape);

}  // namespace lkv
