// Test infrastructure (oracle/_ref build only).
//
// The reference's proj/src/tensor.cpp needs Eigen3, which is not installed
// here and cannot be fetched.  This file supplies, in our own
// code, the inference-only subset of the reference's tensor API
// (proj/include/lkv/tensor.hpp:35-144) that the reference's soft_topk.cpp and
// policy.cpp link against, so those two files compile UNMODIFIED from
// /root/reference into oracle/_ref/liblkv_ref.so.  No tape/autodiff: every op is
// a plain forward evaluation with the same finiteness checks
// (tensor.cpp:34-40) and the same elementwise formulas (silu: tensor.cpp:371-378).
// matmul is a plain i-k-j triple loop (Eigen's blocked order is not reproducible
// without Eigen; scorer values are "parity unpinned").

#include <cmath>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "lkv/errors.hpp"
#include "lkv/model.hpp"
#include "lkv/tensor.hpp"

namespace lkv {

namespace {

size_t shape_numel(const std::vector<int>& shape) {
    size_t n = 1;
    for (int d : shape) {
        if (d < 0) throw contract_error("negative extent in shape");
        n *= static_cast<size_t>(d);
    }
    return n;
}

void check_finite(const Tensor& t, const char* op) {
    for (size_t i = 0; i < t.numel(); ++i) {
        if (!std::isfinite(t.data()[i])) throw numeric_error(std::string(op) + ": non-finite input");
    }
}

}  // namespace

Tensor::Tensor(std::vector<int> shape, bool requires_grad)
    : shape_(std::move(shape)), requires_grad_(requires_grad) {
    data_ = std::make_shared<std::vector<double>>(shape_numel(shape_), 0.0);
}

Tensor Tensor::scalar(double v, bool requires_grad) {
    Tensor t(std::vector<int>{}, requires_grad);
    t.data()[0] = v;
    return t;
}

Tensor Tensor::from(std::vector<int> shape, std::vector<double> values, bool requires_grad) {
    if (shape_numel(shape) != values.size()) throw contract_error("Tensor::from: size mismatch");
    Tensor t(std::move(shape), requires_grad);
    *t.data_ = std::move(values);
    return t;
}

size_t Tensor::numel() const { return data_ ? data_->size() : 0; }

double Tensor::value() const {
    if (numel() != 1) throw contract_error("value(): tensor is not a scalar");
    return (*data_)[0];
}

Tensor Tensor::detached_clone() const { return Tensor::from(shape_, *data_); }

Tensor add(const Tensor& a, const Tensor& b) {
    if (a.shape() != b.shape()) throw contract_error("add: shape mismatch");
    check_finite(a, "add");
    check_finite(b, "add");
    Tensor out(a.shape());
    for (size_t i = 0; i < a.numel(); ++i) out.data()[i] = a.data()[i] + b.data()[i];
    return out;
}

Tensor add_rowvec(const Tensor& x, const Tensor& bias) {
    const int cols = x.dim(x.rank() - 1);
    const int rows = static_cast<int>(x.numel() / static_cast<size_t>(cols));
    if (bias.rank() != 1 || bias.dim(0) != cols) throw contract_error("add_rowvec: bias length mismatch");
    check_finite(x, "add_rowvec");
    check_finite(bias, "add_rowvec");
    Tensor out(x.shape());
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c)
            out.data()[static_cast<size_t>(r) * cols + c] = x.data()[static_cast<size_t>(r) * cols + c] + bias.data()[c];
    return out;
}

Tensor matmul(const Tensor& a, const Tensor& b) {
    if (a.rank() != 2 || b.rank() != 2) throw contract_error("matmul: rank-2 operands required");
    if (a.dim(1) != b.dim(0)) throw contract_error("matmul: inner extents differ");
    check_finite(a, "matmul");
    check_finite(b, "matmul");
    const int m = a.dim(0), k = a.dim(1), n = b.dim(1);
    Tensor out({m, n});
    for (int i = 0; i < m; ++i) {
        double* c = out.data() + static_cast<size_t>(i) * n;
        for (int p = 0; p < k; ++p) {
            const double av = a.data()[static_cast<size_t>(i) * k + p];
            const double* br = b.data() + static_cast<size_t>(p) * n;
            for (int j = 0; j < n; ++j) c[j] += av * br[j];
        }
    }
    return out;
}

Tensor concat_lastdim(const std::vector<Tensor>& parts) {
    if (parts.empty()) throw contract_error("concat_lastdim: no inputs");
    const int rank = parts[0].rank();
    int total = 0;
    for (const auto& p : parts) {
        if (p.rank() != rank) throw contract_error("concat_lastdim: rank mismatch");
        check_finite(p, "concat_lastdim");
        total += p.dim(rank - 1);
    }
    std::vector<int> shape = parts[0].shape();
    shape.back() = total;
    Tensor out(shape);
    const int rows = static_cast<int>(out.numel() / static_cast<size_t>(total));
    int off = 0;
    for (const auto& p : parts) {
        const int w = p.dim(rank - 1);
        for (int r = 0; r < rows; ++r)
            for (int c = 0; c < w; ++c)
                out.data()[static_cast<size_t>(r) * total + off + c] = p.data()[static_cast<size_t>(r) * w + c];
        off += w;
    }
    return out;
}

Tensor silu(const Tensor& x) {
    check_finite(x, "silu");
    Tensor out(x.shape());
    for (size_t i = 0; i < out.numel(); ++i) {
        const double v = x.data()[i];
        out.data()[i] = v / (1.0 + std::exp(-v));
    }
    return out;
}

Tensor reshape(const Tensor& x, std::vector<int> shape) {
    if (shape_numel(shape) != x.numel()) throw contract_error("reshape: element count mismatch");
    return Tensor::from(std::move(shape), x.vec());
}

Tensor make_op_output(std::vector<int> shape, std::vector<double> values, std::vector<Tensor>,
                      std::function<std::vector<Tensor>(const Tensor&)>) {
    return Tensor::from(std::move(shape), std::move(values));
}

// checkpoint.cpp's model save/load is not on this path; link-time stubs only.
ModelWeights init_model(const ModelConfig&) { throw contract_error("init_model: not part of the oracle/_ref build"); }
std::vector<std::pair<std::string, Tensor*>> ModelWeights::named_params() {
    throw contract_error("ModelWeights::named_params: not part of the oracle/_ref build");
}

void ModelConfig::validate() const {
    if (n_layers < 1 || n_query_heads < 1 || n_kv_heads < 1 || head_dim < 1)
        throw contract_error("model config: extents must be positive");
}

}  // namespace lkv
