// host_core.cpp -- see host_core.hpp. Reference citations are file:line into
// /root/reference/proj/include/amsq.
#include "host_core.hpp"

#include <algorithm>
#include <array>
#include <bit>
#include <cmath>
#include <cstring>
#include <mutex>
#include <thread>

namespace amsqb {

// ============================================================== binary16
// half.hpp:16-47: round-to-nearest-even narrowing, overflow to inf, NaNs kept NaN.
uint16_t f32_to_f16(float f) {
  const uint32_t x = std::bit_cast<uint32_t>(f);
  const uint32_t sign = (x >> 16) & 0x8000u;
  const uint32_t ef = (x >> 23) & 0xFFu;
  const uint32_t mf = x & 0x7FFFFFu;
  if (ef == 0xFFu) {  // inf / nan
    const uint32_t p = mf >> 13;
    return static_cast<uint16_t>(sign | 0x7C00u | (mf && !p ? 1u : p));
  }
  const int e = static_cast<int>(ef) - 112;  // rebias 127 -> 15
  if (e >= 31) return static_cast<uint16_t>(sign | 0x7C00u);
  if (e <= 0) {
    if (e < -10) return static_cast<uint16_t>(sign);
    const uint32_t m = mf | 0x800000u;
    const int sh = 14 - e;
    const uint32_t q = m >> sh, r = m & ((1u << sh) - 1u), h = 1u << (sh - 1);
    return static_cast<uint16_t>(sign | (q + ((r > h || (r == h && (q & 1u))) ? 1u : 0u)));
  }
  const uint32_t q = sign | (static_cast<uint32_t>(e) << 10) | (mf >> 13);
  const uint32_t r = mf & 0x1FFFu;
  return static_cast<uint16_t>(q + ((r > 0x1000u || (r == 0x1000u && (q & 1u))) ? 1u : 0u));
}

// half.hpp:49-63: exact widening (subnormals normalised).
float f16_to_f32(uint16_t h) {
  const uint32_t sign = static_cast<uint32_t>(h & 0x8000u) << 16;
  const uint32_t e = (h >> 10) & 0x1Fu, m = h & 0x3FFu;
  uint32_t x;
  if (e == 0) {
    if (m == 0) {
      x = sign;
    } else {
      const int lead = std::bit_width(m) - 1;
      x = sign | (static_cast<uint32_t>(103 + lead) << 23) | ((m ^ (1u << lead)) << (23 - lead));
    }
  } else if (e == 31) {
    x = sign | 0x7F800000u | (m << 13);
  } else {
    x = sign | ((e + 112u) << 23) | (m << 13);
  }
  return std::bit_cast<float>(x);
}

// ============================================================== schemes
// scheme.hpp:59-74 (ids, formats, k) with packing.hpp:6-25 (block geometry).
static constexpr std::array<Scheme, kNumSchemes> kSchemes = {{
    {0, "fp4-e2m1", 2, 1, 1, 1, 16, 4, 1},
    {1, "fp5-e2m2", 2, 2, 1, 1, 16, 5, 2},
    {2, "fp6-e2m3", 2, 3, 1, 1, 16, 6, 2},
    {3, "fp6-e3m2", 3, 2, 3, 1, 16, 6, 2},
    {4, "fp4.25-e2m2", 2, 2, 1, 4, 64, 17, 1},
    {5, "fp4.33-e2m2", 2, 2, 1, 3, 48, 13, 1},
    {6, "fp4.5-e2m2", 2, 2, 1, 2, 32, 9, 1},
    {7, "fp5.33-e2m3", 2, 3, 1, 3, 3, 1, 1},
}};

const Scheme& scheme(int id) {
  if (id < 0 || id >= kNumSchemes) {
    throw InvalidArgument("unknown scheme id " + std::to_string(id));
  }
  return kSchemes[static_cast<size_t>(id)];
}

int scheme_id_by_name(const std::string& name) {
  for (const auto& s : kSchemes) {
    if (name == s.name) return s.id;
  }
  throw InvalidArgument("unknown scheme: " + name);
}

// packing.hpp:67-138 restated as closed forms.
Segment segment(const Scheme& s, int i, int j) {
  const auto u8 = [](int v) { return static_cast<uint8_t>(v); };
  switch (s.id) {
    case 0:
      return {u8(i / 4), u8(4 * (i % 4)), 4, 0};
    case 1:
      return j == 0 ? Segment{u8(i / 4), u8(4 * (i % 4)), 4, 1} : Segment{4, u8(i), 1, 0};
    case 2:
    case 3:
      return j == 0 ? Segment{u8(i / 4), u8(4 * (i % 4)), 4, 2}
                    : Segment{u8(4 + i / 8), u8(2 * (i % 8)), 2, 0};
    case 7:
      return {0, u8(5 * i), 5, 1};
    default:  // 4, 5, 6: top 4 bits as fp4 nibbles
      return {u8(i / 4), u8(4 * (i % 4)), 4, 1};
  }
}

int shared_groups(const Scheme& s) {
  if (s.k == 1) return 0;
  return s.id == 7 ? 1 : 16;
}

void shared_slot(const Scheme& s, int g, int* word, int* bit) {
  if (s.id == 7) {
    *word = 0, *bit = 15;
  } else {
    *word = s.block / 4, *bit = g;
  }
}

size_t padded_cols(const Scheme& s, size_t cols) {
  const size_t b = static_cast<size_t>(s.block);
  return (cols + b - 1) / b * b;
}

size_t words_per_row(const Scheme& s, size_t pc) {
  return pc / static_cast<size_t>(s.block) * static_cast<size_t>(s.words_per_block);
}

size_t packed_payload_bytes(const Scheme& s, size_t rows, size_t cols) {
  return rows * words_per_row(s, padded_cols(s, cols)) * 2;
}

// ============================================================== values
// format.hpp:82-93: zero exponent field selects the subnormal form.
float decode(const Scheme& s, unsigned code) {
  const int m = s.man_bits;
  const unsigned ex = (code >> m) & ((1u << s.exp_bits) - 1u);
  const unsigned man = code & ((1u << m) - 1u);
  const float mag = ex == 0 ? std::ldexp(static_cast<float>(man), 1 - s.bias - m)
                            : std::ldexp(static_cast<float>((1u << m) | man),
                                         static_cast<int>(ex) - s.bias - m);
  return (code & s.sign_mask()) ? -mag : mag;
}

namespace {

struct Tables {
  std::array<uint16_t, 256> f16{};
  std::array<float, 256> val{};
  std::vector<float> grid_v;  // strictly increasing (format.hpp:119-131)
  std::vector<uint8_t> grid_c;
};

const Tables& tables(const Scheme& s) {
  static std::array<Tables, kNumSchemes> t;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const auto& sc : kSchemes) {
      Tables& tb = t[static_cast<size_t>(sc.id)];
      for (unsigned c = 0; c < sc.code_count(); ++c) {
        tb.val[c] = decode(sc, c);
        tb.f16[c] = f32_to_f16(tb.val[c]);
      }
      const unsigned half_n = sc.code_count() / 2;
      for (unsigned mag = half_n - 1; mag >= 1; --mag) {
        tb.grid_v.push_back(tb.val[sc.sign_mask() | mag]);
        tb.grid_c.push_back(static_cast<uint8_t>(sc.sign_mask() | mag));
      }
      tb.grid_v.push_back(0.0f);
      tb.grid_c.push_back(0);
      for (unsigned mag = 1; mag < half_n; ++mag) {
        tb.grid_v.push_back(tb.val[mag]);
        tb.grid_c.push_back(static_cast<uint8_t>(mag));
      }
    }
  });
  return t[static_cast<size_t>(s.id)];
}

}  // namespace

uint16_t code_to_f16(const Scheme& s, unsigned code) { return tables(s).f16[code & 0xFFu]; }

float max_magnitude(const Scheme& s) { return tables(s).grid_v.back(); }

// format.hpp:165-182: nearest value; exact midpoints go to the even code, and to the
// smaller magnitude when both neighbours are even.
uint8_t round_to_nearest(const Scheme& s, float w) {
  const Tables& t = tables(s);
  const auto& v = t.grid_v;
  if (!(w > v.front())) return t.grid_c.front();
  if (w >= v.back()) return t.grid_c.back();
  const size_t hi = static_cast<size_t>(std::lower_bound(v.begin(), v.end(), w) - v.begin());
  const size_t lo = hi - 1;
  const double dlo = static_cast<double>(w) - static_cast<double>(v[lo]);
  const double dhi = static_cast<double>(v[hi]) - static_cast<double>(w);
  if (dlo != dhi) return dlo < dhi ? t.grid_c[lo] : t.grid_c[hi];
  const bool lo_even = (t.grid_c[lo] & 1u) == 0, hi_even = (t.grid_c[hi] & 1u) == 0;
  if (lo_even && hi_even) return std::fabs(v[lo]) <= std::fabs(v[hi]) ? t.grid_c[lo] : t.grid_c[hi];
  return lo_even ? t.grid_c[lo] : t.grid_c[hi];
}

// ============================================================== codec
void pack_block(const Scheme& s, const uint8_t* codes, uint16_t* words) {
  std::fill(words, words + s.words_per_block, uint16_t{0});
  for (int i = 0; i < s.block; ++i) {
    for (int j = 0; j < s.segs_per_weight; ++j) {
      const Segment g = segment(s, i, j);
      const unsigned bits = (static_cast<unsigned>(codes[i]) >> g.code_shift) & ((1u << g.width) - 1u);
      words[g.word] = static_cast<uint16_t>(words[g.word] | (bits << g.bit));
    }
  }
  const int groups = shared_groups(s);
  for (int g = 0; g < groups; ++g) {
    const unsigned bit = codes[g * s.k] & 1u;
    for (int j = 1; j < s.k; ++j) {
      if ((codes[g * s.k + j] & 1u) != bit) {  // packing.hpp:176-179
        throw Corrupt("pack_row: shared mantissa bit mismatch within a group");
      }
    }
    int w, b;
    shared_slot(s, g, &w, &b);
    words[w] = static_cast<uint16_t>(words[w] | (bit << b));
  }
}

void unpack_block(const Scheme& s, const uint16_t* words, uint8_t* codes) {
  for (int i = 0; i < s.block; ++i) {
    unsigned c = 0;
    for (int j = 0; j < s.segs_per_weight; ++j) {
      const Segment g = segment(s, i, j);
      c |= ((static_cast<unsigned>(words[g.word]) >> g.bit) & ((1u << g.width) - 1u)) << g.code_shift;
    }
    codes[i] = static_cast<uint8_t>(c);
  }
  const int groups = shared_groups(s);
  for (int g = 0; g < groups; ++g) {
    int w, b;
    shared_slot(s, g, &w, &b);
    const unsigned bit = (static_cast<unsigned>(words[w]) >> b) & 1u;
    for (int j = 0; j < s.k; ++j) codes[g * s.k + j] = static_cast<uint8_t>(codes[g * s.k + j] | bit);
  }
}

void pack_row(const Scheme& s, std::span<const uint8_t> codes, std::span<uint16_t> words) {
  const size_t b = static_cast<size_t>(s.block), wpb = static_cast<size_t>(s.words_per_block);
  if (codes.size() % b) throw InvalidArgument("pack_row: length is not a block multiple");
  if (words.size() != codes.size() / b * wpb) {
    throw InvalidArgument("pack_row: word buffer size mismatch");
  }
  for (size_t i = 0; i < codes.size() / b; ++i) pack_block(s, codes.data() + i * b, words.data() + i * wpb);
}

void unpack_row(const Scheme& s, std::span<const uint16_t> words, std::span<uint8_t> codes) {
  const size_t b = static_cast<size_t>(s.block), wpb = static_cast<size_t>(s.words_per_block);
  if (words.size() % wpb) throw InvalidArgument("unpack_row: length is not a block multiple");
  if (codes.size() != words.size() / wpb * b) {
    throw InvalidArgument("unpack_row: code buffer size mismatch");
  }
  for (size_t i = 0; i < words.size() / wpb; ++i) unpack_block(s, words.data() + i * wpb, codes.data() + i * b);
}

// ============================================================== quantizer
int resolve_threads(int threads) {
  if (threads > 0) return threads;
  const unsigned hw = std::thread::hardware_concurrency();
  return hw == 0 ? 1 : static_cast<int>(hw);
}

namespace {

// quantize.hpp:72-93: s = max|row| / M (1 for an all-zero row), rounded to binary16,
// forced positive, rejected on overflow.
uint16_t row_scale_bits(const Scheme& s, const float* row, size_t n) {
  float mx = 0.0f;
  for (size_t i = 0; i < n; ++i) {
    if (!std::isfinite(row[i])) throw Corrupt("non-finite weight");
    mx = std::max(mx, std::fabs(row[i]));
  }
  const float scale = mx == 0.0f ? 1.0f : mx / max_magnitude(s);
  uint16_t h = static_cast<uint16_t>(f32_to_f16(scale) & 0x7FFFu);
  if (h >= 0x7C00u) throw Corrupt("channel scale overflows half precision");
  return h == 0 ? uint16_t{1} : h;
}

// quantize.hpp:100-105: set the LSB, collapsing the -0 pattern to +0.
inline uint8_t with_lsb(const Scheme& s, uint8_t c, unsigned bit) {
  const uint8_t r = static_cast<uint8_t>((c & ~1u) | bit);
  return r == s.sign_mask() ? uint8_t{0} : r;
}

}  // namespace

Quantized quantize_tensor(const Scheme& s, size_t rows, size_t cols, const float* w,
                          int threads) {
  if (rows == 0 || cols == 0) throw InvalidArgument("quantize_tensor: empty matrix");
  Quantized q;
  q.rows = rows, q.cols = cols, q.padded_cols = padded_cols(s, cols);
  const size_t pc = q.padded_cols, wpr = words_per_row(s, pc);
  q.scales.assign(rows, 0);
  q.payload.assign(rows * wpr, 0);
  const Tables& tb = tables(s);
  parallel_rows(rows, threads, [&](size_t r0, size_t r1) {
    std::vector<float> row(pc, 0.0f);
    std::vector<uint8_t> codes(pc, 0);
    for (size_t r = r0; r < r1; ++r) {
      std::copy(w + r * cols, w + (r + 1) * cols, row.begin());  // pad_cols_to (matrix.hpp:47-56)
      const uint16_t s16 = row_scale_bits(s, row.data(), pc);
      q.scales[r] = s16;
      const float sc = f16_to_f32(s16);
      for (size_t c = 0; c < pc; ++c) codes[c] = round_to_nearest(s, row[c] / sc);  // rtn 112-131
      if (s.k > 1) {  // ams_share, quantize.hpp:138-184
        const size_t k = static_cast<size_t>(s.k);
        for (size_t b = 0; b < pc; b += k) {
          const size_t e = std::min(b + k, pc);
          unsigned bit = 0;
          if (e <= cols) {  // groups touching padding stay 0
            double err0 = 0.0, err1 = 0.0;
            for (size_t c = b; c < e; ++c) {
              const double d0 = static_cast<double>(tb.val[with_lsb(s, codes[c], 0)] * sc) - row[c];
              err0 += d0 * d0;
            }
            for (size_t c = b; c < e; ++c) {
              const double d1 = static_cast<double>(tb.val[with_lsb(s, codes[c], 1)] * sc) - row[c];
              err1 += d1 * d1;
            }
            bit = err1 < err0 ? 1u : 0u;  // ties keep 0
          }
          for (size_t c = b; c < e; ++c) codes[c] = with_lsb(s, codes[c], bit);
        }
      }
      pack_row(s, codes, std::span<uint16_t>(q.payload.data() + r * wpr, wpr));
    }
  });
  return q;
}

// ============================================================== container
namespace {
inline void put16(uint8_t*& p, uint16_t v) { *p++ = static_cast<uint8_t>(v), *p++ = static_cast<uint8_t>(v >> 8); }
inline void put32(uint8_t*& p, uint32_t v) { for (int i = 0; i < 4; ++i) *p++ = static_cast<uint8_t>(v >> (8 * i)); }
inline void put64(uint8_t*& p, uint64_t v) { for (int i = 0; i < 8; ++i) *p++ = static_cast<uint8_t>(v >> (8 * i)); }
template <typename T>
T get_le(const uint8_t*& p, const uint8_t* end) {
  if (static_cast<size_t>(end - p) < sizeof(T)) throw Corrupt("truncated container");
  uint64_t v = 0;
  for (size_t i = 0; i < sizeof(T); ++i) v |= static_cast<uint64_t>(p[i]) << (8 * i);
  p += sizeof(T);
  return static_cast<T>(v);
}
constexpr size_t kHeader = 4 + 2 + 1 + 1 + 4 + 4 + 4;
}  // namespace

size_t container_bytes(const Scheme& s, size_t rows, size_t cols) {
  return kHeader + 2 * rows + 8 + packed_payload_bytes(s, rows, cols);
}

// container.hpp:63-77.
void container_write(const Scheme& s, size_t rows, size_t cols, size_t pc, const uint16_t* scales,
                     const uint16_t* payload, size_t words, uint8_t* out, size_t out_bytes) {
  if (pc != padded_cols(s, cols) || words != rows * words_per_row(s, pc)) {
    throw InvalidArgument("container_write: shape mismatch");
  }
  if (out_bytes < container_bytes(s, rows, cols)) throw InvalidArgument("container_write: buffer too small");
  uint8_t* p = out;
  std::memcpy(p, "AMSQ", 4), p += 4;
  put16(p, 1);
  *p++ = static_cast<uint8_t>(s.id);
  *p++ = static_cast<uint8_t>(s.k);
  put32(p, static_cast<uint32_t>(rows));
  put32(p, static_cast<uint32_t>(cols));
  put32(p, static_cast<uint32_t>(pc));
  for (size_t r = 0; r < rows; ++r) put16(p, scales[r]);
  put64(p, static_cast<uint64_t>(words) * 2);
  for (size_t i = 0; i < words; ++i) put16(p, payload[i]);
}

// container.hpp:79-115: magic, version, scheme id (invalid_argument when unknown,
// scheme_by_id semantics), k, shape and payload length are all validated.
ContainerView container_parse(const uint8_t* in, size_t n) {
  const uint8_t* p = in;
  const uint8_t* end = in + n;
  if (n < 4 || std::memcmp(p, "AMSQ", 4) != 0) throw Corrupt("bad container magic");
  p += 4;
  if (get_le<uint16_t>(p, end) != 1) throw Corrupt("unsupported container version");
  const auto id = get_le<uint8_t>(p, end);
  const auto k = get_le<uint8_t>(p, end);
  const Scheme& s = scheme(id);
  if (k != s.k) throw Corrupt("container k/scheme mismatch");
  ContainerView v{};
  v.scheme_id = id;
  v.rows = get_le<uint32_t>(p, end);
  v.cols = get_le<uint32_t>(p, end);
  v.padded_cols = get_le<uint32_t>(p, end);
  if (v.rows == 0 || v.cols == 0 || v.padded_cols < v.cols ||
      v.padded_cols % static_cast<size_t>(s.block) != 0 || v.padded_cols != padded_cols(s, v.cols)) {
    throw Corrupt("container shape is invalid");
  }
  if (static_cast<size_t>(end - p) < 2 * v.rows) throw Corrupt("truncated container");
  v.scales = p;
  p += 2 * v.rows;
  const auto len = get_le<uint64_t>(p, end);
  if (len != static_cast<uint64_t>(v.rows) * words_per_row(s, v.padded_cols) * 2) {
    throw Corrupt("container payload length mismatch");
  }
  if (static_cast<uint64_t>(end - p) < len) throw Corrupt("truncated container");
  v.payload = p;
  v.payload_words = static_cast<size_t>(len / 2);
  return v;
}

}  // namespace amsqb
