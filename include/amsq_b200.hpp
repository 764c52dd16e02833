/*
 * amsq_b200.hpp -- header-only C++ wrapper that restores the reference's call shapes
 * (/root/reference/proj/include/amsq, namespace amsq) on top of the C-ABI in
 * amsq_b200.h, so reference-style host code switches to the B200 kernels by changing a
 * namespace.
 *
 *   reference (kernels.hpp / quantize.hpp)                  this wrapper
 *   amsq::gemv(qt, x, batch, threads)            -> amsq_b200::gemv(qt, x, batch, threads)
 *   amsq::restore_matrix(qt, threads)            -> amsq_b200::restore_matrix<Matrix>(qt)
 *   amsq::restore_matrix_half(qt, threads)       -> amsq_b200::restore_matrix_half(qt)
 *   amsq::restore_block(words, layout, table, o) -> DeviceTensor::restore_grid()
 *   amsq::quantize_tensor(w, scheme, threads)    -> amsq_b200::quantize_tensor<QT>(w, scheme)
 *                                                   (on the GPU, bit-identical)
 *   (resident weights, the serving path)         -> amsq_b200::DeviceTensor
 *
 * `QT` is any type with the fields of amsq::QuantizedTensor (quantize.hpp:45-61):
 * `scheme->id`, `rows`, `cols`, `padded_cols`, `scales` and `payload` (contiguous u16).
 * The wrapper never includes the reference headers. Errors keep the reference's types:
 * AMSQ_EINVAL -> std::invalid_argument, every other failure -> std::runtime_error
 * (including "no CUDA device": there is no CPU fallback). `threads` is accepted for
 * signature parity and ignored by device calls.
 */
#ifndef AMSQ_B200_HPP_
#define AMSQ_B200_HPP_

#include <cstddef>
#include <cstdint>
#include <cstring>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "amsq_b200.h"

namespace amsq_b200 {

inline void check(int rc, const char* what) {
  if (rc == AMSQ_OK) return;
  const std::string msg = std::string(what) + ": " + amsq_last_error();
  if (rc == AMSQ_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

// A QuantizedTensor resident on one GPU in the sm_100a tile layout (immutable; move-only).
class DeviceTensor {
 public:
  template <class QT>
  explicit DeviceTensor(const QT& qt, int device = 0, void* stream = nullptr) {
    check(amsq_weight_upload(static_cast<int>(qt.scheme->id), qt.rows, qt.cols, qt.padded_cols, qt.scales.data(),
                             qt.payload.data(), qt.payload.size(), device, stream, &h_),
          "amsq_weight_upload");
  }
  // Column-parallel shard: rows [row0, row0 + nrows).
  template <class QT>
  DeviceTensor(const QT& qt, size_t row0, size_t nrows, int device, void* stream = nullptr) {
    check(amsq_weight_upload_rows(static_cast<int>(qt.scheme->id), qt.rows, qt.cols, qt.padded_cols,
                                  qt.scales.data(), qt.payload.data(), qt.payload.size(), row0,
                                  nrows, device, stream, &h_),
          "amsq_weight_upload_rows");
  }
  DeviceTensor(DeviceTensor&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
  DeviceTensor& operator=(DeviceTensor&& o) noexcept {
    if (this != &o) {
      if (h_) amsq_weight_free(h_);
      h_ = std::exchange(o.h_, nullptr);
    }
    return *this;
  }
  DeviceTensor(const DeviceTensor&) = delete;
  DeviceTensor& operator=(const DeviceTensor&) = delete;
  ~DeviceTensor() {
    if (h_) amsq_weight_free(h_);
  }

  amsq_weight_t handle() const { return h_; }
  amsq_weight_info_t info() const {
    amsq_weight_info_t i{};
    check(amsq_weight_info(h_, &i), "amsq_weight_info");
    return i;
  }

  // kernels.hpp:151-187 with host buffers: x is [batch][cols] fp16 bits, y [batch][rows].
  std::vector<uint16_t> gemv(std::span<const uint16_t> x, size_t batch,
                             void* stream = nullptr) const {
    const amsq_weight_info_t i = info();
    std::vector<uint16_t> y(batch * i.rows);
    check(amsq_gemv_host(h_, x.data(), x.size(), batch, y.data(), stream), "gemv");
    return y;
  }
  // Device buffers, stream-ordered (the serving path).
  void linear(const uint16_t* d_x, size_t batch, uint16_t* d_y, void* stream = nullptr) const {
    check(amsq_linear(h_, d_x, batch, d_y, stream), "amsq_linear");
  }
  // bf16 activations and output (amsq_linear_ex; ldy = 0 means rows).
  void linear_bf16(const uint16_t* d_x, size_t batch, uint16_t* d_y, size_t ldy = 0,
                   void* stream = nullptr) const {
    check(amsq_linear_ex(h_, d_x, AMSQ_DTYPE_BF16, batch, d_y, AMSQ_DTYPE_BF16, ldy, stream),
          "amsq_linear_ex");
  }
  // The reference payload words back (inverse repack: bit-exact).
  void download(std::vector<uint16_t>& scales, std::vector<uint16_t>& payload) const {
    const amsq_weight_info_t i = info();
    scales.resize(i.rows);
    payload.resize(i.payload_bytes / 2);
    check(amsq_weight_download(h_, scales.data(), scales.size(), payload.data(), payload.size()),
          "amsq_weight_download");
  }

 private:
  amsq_weight_t h_ = nullptr;
};

// ---- the reference free functions, synchronous, host in / host out ------------------

// kernels.hpp:151-153 gemv(qt, x, batch, threads). The reference call shape is stateless, so
// this uploads (repacks + H2D) the weight on EVERY call before the kernel runs -- tens of ms
// for an 8B gate_up. It exists so the reference's tests run unchanged; serving code uploads
// once into a DeviceTensor and calls DeviceTensor::gemv / linear.
template <class QT>
std::vector<uint16_t> gemv(const QT& qt, std::span<const uint16_t> x, size_t batch,
                           int /*threads*/ = 1) {
  if (batch == 0 || x.size() != batch * qt.cols) {  // check_gemv_shapes, kernels.hpp:137-143
    throw std::invalid_argument("gemv: activation shape mismatch");
  }
  return DeviceTensor(qt).gemv(x, batch);
}

namespace detail {
template <class QT>
std::vector<uint8_t> device_restore(const QT& qt, int what) {
  DeviceTensor t(qt);
  const size_t n = qt.rows * (what == AMSQ_RESTORE_GRID ? qt.padded_cols : qt.cols);
  std::vector<uint8_t> host(n * (what == AMSQ_RESTORE_F32 ? 4 : 2));
  check(amsq_restore_to_host(t.handle(), what, host.data(), host.size(), nullptr), "restore");
  return host;
}
}  // namespace detail

// kernels.hpp:100-124 restore_matrix: fp32 w*s, [rows][cols]. MatrixT is constructed as
// MatrixT(rows, cols, std::vector<float>) -- amsq::Matrix has that constructor.
template <class MatrixT, class QT>
MatrixT restore_matrix(const QT& qt, int /*threads*/ = 1) {
  const std::vector<uint8_t> b = detail::device_restore(qt, AMSQ_RESTORE_F32);
  std::vector<float> data(qt.rows * qt.cols);
  std::memcpy(data.data(), b.data(), b.size());
  return MatrixT(qt.rows, qt.cols, std::move(data));
}

// kernels.hpp:127-133 restore_matrix_half: fp16(w*s) bits, [rows][cols].
template <class QT>
std::vector<uint16_t> restore_matrix_half(const QT& qt, int /*threads*/ = 1) {
  const std::vector<uint8_t> b = detail::device_restore(qt, AMSQ_RESTORE_F16);
  std::vector<uint16_t> out(b.size() / 2);
  std::memcpy(out.data(), b.data(), b.size());
  return out;
}

// quantize.hpp:188-216 quantize_tensor(weights, scheme, threads), on the GPU
// (amsq_quantize_device_host): bit-identical scales and payload. MatrixT has the reference
// Matrix's `rows`, `cols` and contiguous fp32 `data`; QT is default-constructible with the
// QuantizedTensor fields, and `scheme` must outlive it (as scheme_by_id's static schemes do).
template <class QT, class MatrixT, class SchemeT>
QT quantize_tensor(const MatrixT& weights, const SchemeT& scheme, int /*threads*/ = 1, int device = 0) {
  const int id = static_cast<int>(scheme.id);
  size_t pc = 0, words = 0;
  check(amsq_quantize_device_host(id, weights.rows, weights.cols, nullptr, device, &pc, &words, nullptr,
                                  nullptr),
        "quantize_tensor");
  QT qt;
  qt.scheme = &scheme;
  qt.rows = weights.rows;
  qt.cols = weights.cols;
  qt.padded_cols = pc;
  qt.scales.assign(weights.rows, 0);
  qt.payload.assign(words, 0);
  check(amsq_quantize_device_host(id, weights.rows, weights.cols, weights.data.data(), device, &pc, &words,
                                  qt.scales.data(), qt.payload.data()),
        "quantize_tensor");
  return qt;
}

// restore_block over the whole tensor (kernels.hpp:55-63): grid bits, [rows][padded_cols].
template <class QT>
std::vector<uint16_t> restore_grid(const QT& qt) {
  const std::vector<uint8_t> b = detail::device_restore(qt, AMSQ_RESTORE_GRID);
  std::vector<uint16_t> out(b.size() / 2);
  std::memcpy(out.data(), b.data(), b.size());
  return out;
}

}  // namespace amsq_b200

#endif  // AMSQ_B200_HPP_
