// C++ host mirror of the reference operator API for the quire hot path.
//
// Same function names, argument meaning and error behaviour as
// /root/reference/proj/include/pnn/tensor_ops.hpp:17-61 (use_quire = true
// path), over a Tensor with the reference's storage convention: one posit
// code per uint64_t slot, row-major (tensor.hpp:10-14, 35-75).  Each call is
// synchronous like the reference's: host codes are packed, copied to the
// B200, run through the sm_100a kernels behind include/pnn_b200.h, and copied
// back.  Errors: std::invalid_argument for shape/rank/dtype problems (as the
// reference, tensor_ops.cpp:17-27), std::runtime_error for device failures.
// There is no CPU fallback: without a working GPU every call throws.
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

namespace pnn_b200 {

struct PositConfig {
    int nbits = 16;
    int es = 1;
    friend bool operator==(const PositConfig& a, const PositConfig& b) {
        return a.nbits == b.nbits && a.es == b.es;
    }
};

class Tensor {
public:
    Tensor() = default;
    Tensor(PositConfig cfg, std::vector<int64_t> shape);

    const PositConfig& config() const { return cfg_; }
    const std::vector<int64_t>& shape() const { return shape_; }
    int rank() const { return int(shape_.size()); }
    int64_t dim(int i) const { return shape_[size_t(i)]; }
    int64_t numel() const { return numel_; }
    uint64_t* data() { return buf_->data(); }
    const uint64_t* data() const { return buf_->data(); }
    uint64_t bits_at(int64_t i) const { return (*buf_)[size_t(i)]; }
    void set_bits(int64_t i, uint64_t b) { (*buf_)[size_t(i)] = b; }

private:
    PositConfig cfg_;
    std::vector<int64_t> shape_;
    int64_t numel_ = 0;
    std::shared_ptr<std::vector<uint64_t>> buf_;
};

// `pool` is accepted for signature compatibility and ignored: the reference's
// results are worker-count invariant (tensor_ops.hpp:12-13).
Tensor matmul(const Tensor& a, const Tensor& b, bool use_quire, const void* pool = nullptr);
Tensor par_matmul(const Tensor& a, const Tensor& b, bool use_quire, int workers);
Tensor conv2d(const Tensor& x, const Tensor& w, const Tensor* bias, int stride, int pad,
              bool use_quire, const void* pool = nullptr);
Tensor conv2d_input_grad(const Tensor& dy, const Tensor& w, const std::vector<int64_t>& x_shape,
                         int stride, int pad, bool use_quire, const void* pool = nullptr);
Tensor conv2d_weight_grad(const Tensor& dy, const Tensor& x, const std::vector<int64_t>& w_shape,
                          int stride, int pad, bool use_quire, const void* pool = nullptr);
Tensor conv2d_bias_grad(const Tensor& dy, bool use_quire);
Tensor column_sum(const Tensor& x, bool use_quire);

struct MaxPoolResult {
    Tensor out;
    std::vector<int64_t> argmax;  // flat input index per output element
};
MaxPoolResult maxpool2d(const Tensor& x, int k, int stride, const void* pool = nullptr);
// Reference signature (tensor_ops.hpp:50-51): any argmax, outputs added per
// target in increasing output order; out-of-range indices throw.
Tensor maxpool2d_backward(const Tensor& dy, const std::vector<int64_t>& argmax,
                          const std::vector<int64_t>& x_shape);
// Window-specialised: dy must be the (N, C, OH, OW) output of maxpool2d(x, k,
// stride) and every argmax inside its window (else std::invalid_argument).
Tensor maxpool2d_backward(const Tensor& dy, const std::vector<int64_t>& argmax,
                          const std::vector<int64_t>& x_shape, int k, int stride);
Tensor convert_tensor(const Tensor& t, const PositConfig& target);

}  // namespace pnn_b200
