// tests/cpp/dropin_test.cpp -- TEST ONLY. The reference's own types and functions
// (/root/reference/proj/include/amsq, compiled in place) side by side with the B200
// drop-in (include/amsq_b200.hpp over libamsq_b200.so): the same QuantizedTensor goes
// through amsq::gemv / restore_matrix / restore_matrix_half and through
// amsq_b200::gemv / restore_matrix / restore_matrix_half, acceptance-suite style
// (PASS/FAIL lines, exit code = number of failures; acceptance_main.cc:416-450).
//
// Built by oracle/Makefile into oracle/_ref/dropin_test (it contains reference code).
//   dropin_test            -- on a B200: parity (restore bit-exact, gemv within the bar)
//   dropin_test --no-gpu   -- without a GPU: device calls must throw std::runtime_error
//                             (no CPU fallback) and shape errors std::invalid_argument
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "amsq/amsq.hpp"
#include "amsq_b200.hpp"

namespace {

int g_fail = 0;

void report(const std::string& name, bool ok, const std::string& detail = "") {
  std::printf("%s %s%s%s\n", ok ? "PASS" : "FAIL", name.c_str(), detail.empty() ? "" : ": ",
              detail.c_str());
  if (!ok) ++g_fail;
}

template <class E>
bool throws(const std::function<void()>& fn) {
  try {
    fn();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

// SURVEY.md §8(d) bar: norm-wise rel <= 1e-3 and per element
// |y - y_ref| <= 1e-3 * sum_i |w_i s x_i| + ulp_fp16(y_ref).
bool within_bar(const amsq::QuantizedTensor& qt, const std::vector<uint16_t>& x, size_t batch,
                const std::vector<uint16_t>& y, const std::vector<uint16_t>& yref,
                std::string* why) {
  const amsq::Matrix w = amsq::restore_matrix(qt);
  double num = 0, den = 0;
  for (size_t b = 0; b < batch; ++b) {
    for (size_t r = 0; r < qt.rows; ++r) {
      double absum = 0;
      for (size_t i = 0; i < qt.cols; ++i) {
        absum += std::fabs(double(w.at(r, i)) * amsq::half_to_float(x[b * qt.cols + i]));
      }
      const double a = amsq::half_to_float(y[b * qt.rows + r]);
      const double e = amsq::half_to_float(yref[b * qt.rows + r]);
      const uint16_t eb = yref[b * qt.rows + r];
      const double ulp = std::fabs(double(amsq::half_to_float(uint16_t((eb & 0x7FFF) + 1))) -
                                   std::fabs(e));
      if (!std::isfinite(a) || std::fabs(a - e) > 1e-3 * absum + ulp) {
        char buf[160];
        std::snprintf(buf, sizeof buf, "b=%zu r=%zu got %.6g want %.6g (bound %.3g)", b, r, a, e,
                      1e-3 * absum + ulp);
        *why = buf;
        return false;
      }
      num += (a - e) * (a - e);
      den += e * e;
    }
  }
  const double rel = den > 0 ? std::sqrt(num / den) : std::sqrt(num);
  if (rel > 1e-3) {
    *why = "norm-wise rel " + std::to_string(rel);
    return false;
  }
  return true;
}

void gpu_suite() {
  for (const char* name : {"fp5.33-e2m3", "fp4.25-e2m2"}) {
    const amsq::QuantScheme& s = amsq::scheme_by_name(name);
    for (auto [rows, cols] : {std::pair<size_t, size_t>{32, 96}, {64, 192}, {128, 512},
                              {300, 1000}, {256, 4096}}) {
      const auto qt = amsq::quantize_tensor(amsq::detail::gaussian_matrix(rows, cols, rows + cols), s);
      const std::string tag = std::string(name) + " " + std::to_string(rows) + "x" +
                              std::to_string(cols);
      // bit-exact bar (kernels.hpp:100-133)
      const amsq::Matrix ref_m = amsq::restore_matrix(qt);
      const amsq::Matrix dev_m = amsq_b200::restore_matrix<amsq::Matrix>(qt);
      report("restore_matrix bit-exact " + tag,
             dev_m.rows == ref_m.rows && dev_m.cols == ref_m.cols &&
                 std::memcmp(dev_m.data.data(), ref_m.data.data(), ref_m.data.size() * 4) == 0);
      const auto ref_h = amsq::restore_matrix_half(qt);
      const auto dev_h = amsq_b200::restore_matrix_half(qt);
      report("restore_matrix_half bit-exact " + tag, dev_h == ref_h);
      // linear bar, acceptance criterion 6's batches (acceptance_main.cc:247-271)
      for (size_t batch : {1u, 2u, 4u, 8u, 16u, 32u}) {
        const auto x = amsq::detail::gaussian_half(batch * qt.cols, 7 ^ batch);
        const auto yref = amsq::gemv(qt, x, batch);
        const auto y = amsq_b200::gemv(qt, x, batch);
        std::string why;
        report("gemv " + tag + " M=" + std::to_string(batch),
               y.size() == yref.size() && within_bar(qt, x, batch, y, yref, &why), why);
      }
    }
  }
  // kernels_test.cc:165-173 error types
  const auto qt = amsq::quantize_tensor(amsq::detail::gaussian_matrix(4, 9, 1),
                                        amsq::scheme_by_name("fp5.33-e2m3"));
  report("gemv shape mismatch -> invalid_argument", throws<std::invalid_argument>([&] {
           amsq_b200::gemv(qt, std::vector<uint16_t>(7, 0), 1);
         }));
  report("gemv batch 0 -> invalid_argument", throws<std::invalid_argument>([&] {
           amsq_b200::gemv(qt, std::vector<uint16_t>(9, 0), 0);
         }));
  // quantize.hpp:188-216 on the GPU: the reference's own quantize_tensor, bit for bit
  for (const char* name : {"fp5.33-e2m3", "fp4.25-e2m2", "fp6-e3m2", "fp4-e2m1"}) {
    const amsq::QuantScheme& s = amsq::scheme_by_name(name);
    for (auto [rows, cols] : {std::pair<size_t, size_t>{7, 50}, {64, 192}, {300, 4098}}) {
      const amsq::Matrix w = amsq::detail::gaussian_matrix(rows, cols, 3 * rows + cols);
      const auto ref = amsq::quantize_tensor(w, s);
      const auto dev = amsq_b200::quantize_tensor<amsq::QuantizedTensor>(w, s);
      report(std::string("quantize_tensor on the GPU bit-exact ") + name + " " + std::to_string(rows) +
                 "x" + std::to_string(cols),
             dev.padded_cols == ref.padded_cols && dev.scales == ref.scales && dev.payload == ref.payload);
    }
  }
  {
    amsq::Matrix bad = amsq::detail::gaussian_matrix(3, 8, 2);
    bad.data[5] = std::nanf("");
    report("quantize_tensor non-finite -> runtime_error (quantize.hpp:77)",
           throws<std::runtime_error>([&] {
             amsq_b200::quantize_tensor<amsq::QuantizedTensor>(bad, amsq::scheme_by_name("fp5.33-e2m3"));
           }));
  }
  // resident weights: download is the reference stream, bit for bit
  amsq_b200::DeviceTensor t(qt);
  std::vector<uint16_t> sc, pl;
  t.download(sc, pl);
  report("DeviceTensor download round trip", sc == qt.scales && pl == qt.payload);
}

void no_gpu_suite() {
  const auto qt = amsq::quantize_tensor(amsq::detail::gaussian_matrix(4, 9, 1),
                                        amsq::scheme_by_name("fp5.33-e2m3"));
  const auto x = amsq::detail::gaussian_half(9, 3);
  report("gemv without a GPU -> runtime_error (no CPU fallback)",
         throws<std::runtime_error>([&] { amsq_b200::gemv(qt, x, 1); }));
  report("restore without a GPU -> runtime_error",
         throws<std::runtime_error>([&] { amsq_b200::restore_matrix_half(qt); }));
  report("gemv shape mismatch -> invalid_argument (before any device work)",
         throws<std::invalid_argument>([&] { amsq_b200::gemv(qt, x, 2); }));
  report("quantize_tensor without a GPU -> runtime_error (no CPU fallback)",
         throws<std::runtime_error>([&] {
           amsq_b200::quantize_tensor<amsq::QuantizedTensor>(amsq::detail::gaussian_matrix(4, 9, 1),
                                                             amsq::scheme_by_name("fp5.33-e2m3"));
         }));
}

}  // namespace

int main(int argc, char** argv) {
  const bool no_gpu = argc > 1 && std::strcmp(argv[1], "--no-gpu") == 0;
  if (no_gpu) {
    no_gpu_suite();
  } else {
    gpu_suite();
  }
  std::printf("%d failure(s)\n", g_fail);
  return g_fail;
}
