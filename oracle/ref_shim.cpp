// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// A thin extern "C" shim over the UNMODIFIED reference library, whose headers are
// included in place from /root/reference/proj/include (see oracle/Makefile; nothing
// from the reference is copied into this repository). The resulting
// oracle/_ref/libamsq_ref.so is used (a) by tests/ to validate the plain-C
// restatement in oracle/amsq_oracle.c, (b) by tests/golden/make_golden.py to
// generate the committed golden fixtures, and (c) by bench.py as the
// `cpu_baseline` / `--impl reference` arm (the reference's own amsq::gemv timed
// on the host cores).
//
// Status codes: 0 ok, 1 std::invalid_argument, 2 std::runtime_error, 3 other.

#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <stdexcept>
#include <vector>

#include "amsq/kernels.hpp"
#include "amsq/packing.hpp"
#include "amsq/quantize.hpp"
#include "amsq/scheme.hpp"

namespace {

thread_local char g_err[512];

int fail(int code, const char* what) {
  std::strncpy(g_err, what, sizeof(g_err) - 1);
  g_err[sizeof(g_err) - 1] = 0;
  return code;
}

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(1, e.what());
  } catch (const std::runtime_error& e) {
    return fail(2, e.what());
  } catch (const std::exception& e) {
    return fail(3, e.what());
  }
}

amsq::QuantizedTensor make_qt(int scheme_id, size_t rows, size_t cols, size_t padded_cols,
                              const uint16_t* scales, const uint16_t* payload, size_t words) {
  amsq::QuantizedTensor qt;
  qt.scheme = &amsq::scheme_by_id(static_cast<uint8_t>(scheme_id));
  qt.rows = rows;
  qt.cols = cols;
  qt.padded_cols = padded_cols;
  qt.scales.assign(scales, scales + rows);
  qt.payload.assign(payload, payload + words);
  return qt;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err; }

uint16_t ref_float_to_half(float f) { return amsq::float_to_half(f); }
float ref_half_to_float(uint16_t h) { return amsq::half_to_float(h); }

int ref_scheme_info(int scheme_id, int* exp_bits, int* man_bits, int* bias, int* k,
                    size_t* block, size_t* words_per_block) {
  return guarded([&] {
    const auto& s = amsq::scheme_by_id(static_cast<uint8_t>(scheme_id));
    const auto& L = amsq::layout_of(s);
    *exp_bits = s.base_format.exp_bits();
    *man_bits = s.base_format.man_bits();
    *bias = s.base_format.bias();
    *k = s.k;
    *block = L.block;
    *words_per_block = L.words_per_block;
  });
}

// restore_table (format.hpp:196): out[code] for every code of the scheme's format.
int ref_restore_table(int scheme_id, uint16_t* out, size_t n) {
  return guarded([&] {
    const auto& s = amsq::scheme_by_id(static_cast<uint8_t>(scheme_id));
    const auto t = amsq::restore_table(s.base_format);
    if (n < t.size()) throw std::invalid_argument("table buffer too small");
    std::copy(t.begin(), t.end(), out);
  });
}

size_t ref_packed_payload_bytes(int scheme_id, size_t rows, size_t cols) {
  return amsq::packed_payload_bytes(amsq::scheme_by_id(static_cast<uint8_t>(scheme_id)), rows,
                                    cols);
}

int ref_pack_row(int scheme_id, const uint8_t* codes, size_t n, uint16_t* words, size_t nw) {
  return guarded([&] {
    const auto& L = amsq::layout_of(amsq::scheme_by_id(static_cast<uint8_t>(scheme_id)));
    amsq::pack_row(std::span<const uint8_t>(codes, n), L, std::span<uint16_t>(words, nw));
  });
}

int ref_unpack_row(int scheme_id, const uint16_t* words, size_t nw, uint8_t* codes, size_t n) {
  return guarded([&] {
    const auto& L = amsq::layout_of(amsq::scheme_by_id(static_cast<uint8_t>(scheme_id)));
    amsq::unpack_row(std::span<const uint16_t>(words, nw), L, std::span<uint8_t>(codes, n));
  });
}

int ref_restore_block(int scheme_id, const uint16_t* words, uint16_t* out, int bitops) {
  return guarded([&] {
    const auto& s = amsq::scheme_by_id(static_cast<uint8_t>(scheme_id));
    const auto& L = amsq::layout_of(s);
    std::span<const uint16_t> w(words, L.words_per_block);
    std::span<uint16_t> o(out, L.block);
    if (bitops) {
      amsq::restore_block_bitops(w, L, o);
    } else {
      amsq::restore_block(w, L, amsq::restore_table(s.base_format), o);
    }
  });
}

// quantize_tensor (quantize.hpp:188-216). Call with scales/payload == nullptr to
// query padded_cols and words first.
int ref_quantize_tensor(int scheme_id, size_t rows, size_t cols, const float* w, int threads,
                        size_t* padded_cols, size_t* words, uint16_t* scales, uint16_t* payload) {
  return guarded([&] {
    const auto& s = amsq::scheme_by_id(static_cast<uint8_t>(scheme_id));
    if (!scales || !payload) {
      const auto& L = amsq::layout_of(s);
      *padded_cols = amsq::round_up(cols, L.block);
      *words = amsq::packed_payload_bytes(s, rows, cols) / 2;
      return;
    }
    amsq::Matrix m(rows, cols, std::vector<float>(w, w + rows * cols));
    const auto qt = amsq::quantize_tensor(m, s, threads);
    *padded_cols = qt.padded_cols;
    *words = qt.payload.size();
    std::copy(qt.scales.begin(), qt.scales.end(), scales);
    std::copy(qt.payload.begin(), qt.payload.end(), payload);
  });
}

int ref_restore_matrix(int scheme_id, size_t rows, size_t cols, size_t padded_cols,
                       const uint16_t* scales, const uint16_t* payload, size_t words, int threads,
                       float* out) {
  return guarded([&] {
    const auto qt = make_qt(scheme_id, rows, cols, padded_cols, scales, payload, words);
    const auto m = amsq::restore_matrix(qt, threads);
    std::copy(m.data.begin(), m.data.end(), out);
  });
}

int ref_restore_matrix_half(int scheme_id, size_t rows, size_t cols, size_t padded_cols,
                            const uint16_t* scales, const uint16_t* payload, size_t words,
                            int threads, uint16_t* out) {
  return guarded([&] {
    const auto qt = make_qt(scheme_id, rows, cols, padded_cols, scales, payload, words);
    const auto m = amsq::restore_matrix_half(qt, threads);
    std::copy(m.begin(), m.end(), out);
  });
}

// gemv (kernels.hpp:151-187) / gemv_reference (191-222). x is [batch][cols], y [batch][rows].
int ref_gemv(int scheme_id, size_t rows, size_t cols, size_t padded_cols, const uint16_t* scales,
             const uint16_t* payload, size_t words, const uint16_t* x, size_t x_len, size_t batch,
             int threads, int use_reference, uint16_t* y) {
  return guarded([&] {
    const auto qt = make_qt(scheme_id, rows, cols, padded_cols, scales, payload, words);
    std::span<const uint16_t> xs(x, x_len);
    const auto out = use_reference ? amsq::gemv_reference(qt, xs, batch, threads)
                                   : amsq::gemv(qt, xs, batch, threads);
    std::copy(out.begin(), out.end(), y);
  });
}

// A persistent tensor for timing loops: avoids re-copying the payload per call.
void* ref_tensor_new(int scheme_id, size_t rows, size_t cols, size_t padded_cols,
                     const uint16_t* scales, const uint16_t* payload, size_t words) {
  try {
    return new amsq::QuantizedTensor(
        make_qt(scheme_id, rows, cols, padded_cols, scales, payload, words));
  } catch (const std::exception& e) {
    fail(3, e.what());
    return nullptr;
  }
}

void ref_tensor_free(void* t) { delete static_cast<amsq::QuantizedTensor*>(t); }

int ref_tensor_gemv(void* t, const uint16_t* x, size_t batch, int threads, uint16_t* y) {
  return guarded([&] {
    const auto& qt = *static_cast<const amsq::QuantizedTensor*>(t);
    const auto out =
        amsq::gemv(qt, std::span<const uint16_t>(x, batch * qt.cols), batch, threads);
    std::copy(out.begin(), out.end(), y);
  });
}

// detail::gaussian_matrix / gaussian_half (kernels.hpp:294-310): libstdc++-specific
// streams, so fixtures store the generated bytes rather than the seeds alone.
void ref_gaussian_matrix(size_t rows, size_t cols, uint64_t seed, float* out) {
  const auto m = amsq::detail::gaussian_matrix(rows, cols, seed);
  std::copy(m.data.begin(), m.data.end(), out);
}

void ref_gaussian_half(size_t n, uint64_t seed, uint16_t* out) {
  const auto v = amsq::detail::gaussian_half(n, seed);
  std::copy(v.begin(), v.end(), out);
}

int ref_resolve_threads(int threads) { return amsq::resolve_threads(threads); }

}  // extern "C"
