// host_core.hpp -- host-side C++ core of the B200 AMS-Quant library.
//
// Scheme/format metadata, the reference packed-stream codec, the host quantizer
// (RTN + Adaptive Searching, which the north star keeps on the host) and the AMSQ
// container. Everything here is bit-identical to the reference
// (/root/reference/proj/include/amsq) -- tests/test_host.py checks it against
// the oracle and the compiled reference -- but is written fresh around flat
// constexpr tables instead of the reference's cached runtime tables.
#pragma once

#include <cstddef>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace amsqb {

// ---- errors: the reference throws std::invalid_argument / std::runtime_error;
// the C-ABI turns them into AMSQ_EINVAL / AMSQ_ECORRUPT.
struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct Corrupt : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ---- binary16 (half.hpp:16-71)
uint16_t f32_to_f16(float f);  // RNE, overflow -> inf, NaN stays NaN
float f16_to_f32(uint16_t h);  // exact

// ---- schemes (scheme.hpp:21-74) and their packing layouts (packing.hpp:6-25)
struct Segment {
  uint8_t word, bit, width, code_shift;
};

struct Scheme {
  int id;
  const char* name;
  int exp_bits, man_bits, bias, k;
  int block;            // weights per packing block
  int words_per_block;  // u16 words per block
  int segs_per_weight;
  int code_bits() const { return 1 + exp_bits + man_bits; }
  unsigned code_count() const { return 1u << code_bits(); }
  unsigned sign_mask() const { return 1u << (exp_bits + man_bits); }
};

constexpr int kNumSchemes = 8;
const Scheme& scheme(int id);  // throws InvalidArgument for unknown ids
int scheme_id_by_name(const std::string& name);

// Segment j of weight i in the block, and the shared slot of group g.
Segment segment(const Scheme& s, int weight, int j);
void shared_slot(const Scheme& s, int group, int* word, int* bit);
int shared_groups(const Scheme& s);  // groups carrying a shared bit per block (0 if k == 1)

size_t padded_cols(const Scheme& s, size_t cols);
size_t words_per_row(const Scheme& s, size_t padded_cols);
size_t packed_payload_bytes(const Scheme& s, size_t rows, size_t cols);

// ---- minifloat values (format.hpp:82-93, 190-198)
float decode(const Scheme& s, unsigned code);
uint16_t code_to_f16(const Scheme& s, unsigned code);  // normative to_fp16_bits
float max_magnitude(const Scheme& s);
uint8_t round_to_nearest(const Scheme& s, float w);  // format.hpp:165-182 semantics

// ---- codec (packing.hpp:159-266)
void pack_block(const Scheme& s, const uint8_t* codes, uint16_t* words);    // throws Corrupt
void unpack_block(const Scheme& s, const uint16_t* words, uint8_t* codes);
void pack_row(const Scheme& s, std::span<const uint8_t> codes, std::span<uint16_t> words);
void unpack_row(const Scheme& s, std::span<const uint16_t> words, std::span<uint8_t> codes);

// ---- quantizer (quantize.hpp:72-216). Returns scales; fills payload.
struct Quantized {
  size_t rows = 0, cols = 0, padded_cols = 0;
  std::vector<uint16_t> scales;
  std::vector<uint16_t> payload;
};
Quantized quantize_tensor(const Scheme& s, size_t rows, size_t cols, const float* w,
                          int threads);

// ---- container v1 (container.hpp:4-9, 63-127)
size_t container_bytes(const Scheme& s, size_t rows, size_t cols);
void container_write(const Scheme& s, size_t rows, size_t cols, size_t padded_cols,
                     const uint16_t* scales, const uint16_t* payload, size_t payload_words,
                     uint8_t* out, size_t out_bytes);
struct ContainerView {
  int scheme_id;
  size_t rows, cols, padded_cols;
  const uint8_t* scales;   // little-endian u16 x rows
  const uint8_t* payload;  // little-endian u16 x payload_words
  size_t payload_words;
};
ContainerView container_parse(const uint8_t* in, size_t in_bytes);

// ---- threading (parallel.hpp:15-53 semantics: static partition, first error rethrown)
int resolve_threads(int threads);
template <typename Body>
void parallel_rows(size_t n, int threads, Body&& body);

}  // namespace amsqb

#include "host_parallel.inl"
