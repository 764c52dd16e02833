/*
 * oracle/amsq_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's hot-path algorithms (AMS-Quant,
 * /root/reference/proj/include/amsq/ headers) used as the parity checker for the
 * B200 kernels. Only tests/, __graft_entry__.smoke() and bench.py's
 * `cpu_baseline` leg may load it; the product library never links or calls it.
 *
 * Parity of this restatement is PINNED: tests/test_oracle.py checks it against
 * (a) the golden vectors of the reference's own unit tests (packing_test.cc,
 * kernels_test.cc, half_test.cc, format_test.cc, quantize_test.cc) and
 * (b) byte-for-byte outputs of the unmodified reference compiled in place
 * (oracle/_ref/libamsq_ref.so, built by oracle/Makefile) and the fixtures that
 * tests/golden/make_golden.py generated from it.
 *
 * Build: gcc -std=c11 -O2 -ffp-contract=off (FMA contraction changes the
 * reference's gemv output bits).
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- binary16
 * half.hpp:16-47 float_bits_to_half: RNE narrowing, overflow -> inf, NaN kept. */
uint16_t orc_float_to_half(float f) {
  uint32_t fb;
  memcpy(&fb, &f, 4);
  const uint32_t sign = (fb >> 16) & 0x8000u;
  const uint32_t e8 = (fb >> 23) & 0xFFu;
  uint32_t man = fb & 0x7FFFFFu;
  if (e8 == 0xFFu) {
    uint32_t payload = man >> 13;
    if (man != 0 && payload == 0) payload = 1;
    return (uint16_t)(sign | 0x7C00u | payload);
  }
  const int32_t e = (int32_t)e8 - 127 + 15;
  if (e >= 31) return (uint16_t)(sign | 0x7C00u);
  if (e <= 0) {
    if (e < -10) return (uint16_t)sign;
    man |= 0x800000u;
    const uint32_t shift = (uint32_t)(14 - e);
    const uint32_t hm = man >> shift;
    const uint32_t rem = man & ((1u << shift) - 1u);
    const uint32_t halfway = 1u << (shift - 1);
    uint32_t out = sign | hm;
    if (rem > halfway || (rem == halfway && (hm & 1u))) ++out;
    return (uint16_t)out;
  }
  uint32_t out = sign | ((uint32_t)e << 10) | (man >> 13);
  const uint32_t rem = man & 0x1FFFu;
  if (rem > 0x1000u || (rem == 0x1000u && (out & 1u))) ++out;
  return (uint16_t)out;
}

/* half.hpp:49-63 half_bits_to_float_bits: exact widening. */
float orc_half_to_float(uint16_t h) {
  const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  const uint32_t e = (h >> 10) & 0x1Fu;
  const uint32_t m = h & 0x3FFu;
  uint32_t bits;
  if (e == 0) {
    if (m == 0) {
      bits = sign;
    } else {
      int lead = 31 - __builtin_clz(m);
      bits = sign | ((uint32_t)(103 + lead) << 23) | ((m ^ (1u << lead)) << (23 - lead));
    }
  } else if (e == 31) {
    bits = sign | 0x7F800000u | (m << 13);
  } else {
    bits = sign | ((e + 112u) << 23) | (m << 13);
  }
  float f;
  memcpy(&f, &bits, 4);
  return f;
}

/* ----------------------------------------------------------------- schemes
 * scheme.hpp:21-30 (ids), 59-74 (table); format.hpp:31-72 (bias 2^(e-1)-1). */
typedef struct {
  int e, m, bias, k;
} orc_scheme;

static const orc_scheme kSchemes[8] = {
    {2, 1, 1, 1}, /* 0 fp4-e2m1   */
    {2, 2, 1, 1}, /* 1 fp5-e2m2   */
    {2, 3, 1, 1}, /* 2 fp6-e2m3   */
    {3, 2, 3, 1}, /* 3 fp6-e3m2   */
    {2, 2, 1, 4}, /* 4 fp4.25-e2m2 */
    {2, 2, 1, 3}, /* 5 fp4.33-e2m2 */
    {2, 2, 1, 2}, /* 6 fp4.5-e2m2  */
    {2, 3, 1, 3}, /* 7 fp5.33-e2m3 */
};

int orc_scheme_valid(int id) { return id >= 0 && id < 8; }

/* format.hpp:82-93 decode: zero exponent field = subnormal (no implicit one). */
float orc_decode(unsigned code, int scheme_id) {
  const orc_scheme* s = &kSchemes[scheme_id];
  const unsigned ex = (code >> s->m) & ((1u << s->e) - 1u);
  const unsigned man = code & ((1u << s->m) - 1u);
  const float sgn = (code & (1u << (s->e + s->m))) ? -1.0f : 1.0f;
  if (ex == 0) return sgn * ldexpf((float)man, 1 - s->bias - s->m);
  return sgn * ldexpf((float)((1u << s->m) | man), (int)ex - s->bias - s->m);
}

/* format.hpp:109-132 build_tables -> to_fp16_bits (format.hpp:190): the
 * normative code -> binary16 pattern is float_to_half(decode(code)). */
uint16_t orc_to_fp16_bits(unsigned code, int scheme_id) {
  return orc_float_to_half(orc_decode(code, scheme_id));
}

/* ------------------------------------------------------------------ layout
 * packing.hpp:6-25 (normative table) and 67-138 (build_layout). A segment is
 * {word, bit, width, code_shift}; a shared slot is {word, bit}. */
typedef struct {
  int word, bit, width, code_shift;
} orc_seg;

typedef struct {
  int block, words, segs_per_weight, nshared;
  orc_seg seg[64 * 2];
  int sh_word[16], sh_bit[16];
} orc_layout;

void orc_layout_of(int id, orc_layout* L) {
  memset(L, 0, sizeof(*L));
  int i;
  switch (id) {
    case 0: /* fp4-e2m1: block 16, 4 words, weight i bits [4*(i%4),+4) of word i/4 */
      L->block = 16, L->words = 4, L->segs_per_weight = 1;
      for (i = 0; i < 16; ++i) L->seg[i] = (orc_seg){i / 4, 4 * (i % 4), 4, 0};
      break;
    case 1: /* fp5-e2m2: top 4 bits as fp4, LSB plane in word 4 */
      L->block = 16, L->words = 5, L->segs_per_weight = 2;
      for (i = 0; i < 16; ++i) {
        L->seg[2 * i] = (orc_seg){i / 4, 4 * (i % 4), 4, 1};
        L->seg[2 * i + 1] = (orc_seg){4, i, 1, 0};
      }
      break;
    case 2:
    case 3: /* fp6: top 4 bits as fp4, low 2 bits in words 4-5 */
      L->block = 16, L->words = 6, L->segs_per_weight = 2;
      for (i = 0; i < 16; ++i) {
        L->seg[2 * i] = (orc_seg){i / 4, 4 * (i % 4), 4, 2};
        L->seg[2 * i + 1] = (orc_seg){4 + i / 8, 2 * (i % 8), 2, 0};
      }
      break;
    case 7: /* fp5.33-e2m3: block 3, 1 word, 5-bit segments at 5j, shared bit 15 */
      L->block = 3, L->words = 1, L->segs_per_weight = 1;
      for (i = 0; i < 3; ++i) L->seg[i] = (orc_seg){0, 5 * i, 5, 1};
      L->nshared = 1, L->sh_word[0] = 0, L->sh_bit[0] = 15;
      break;
    case 4: /* fp4.25-e2m2: block 64, 17 words, shared bits in word 16 */
    case 5: /* fp4.33-e2m2: block 48, 13 words, shared bits in word 12 */
    case 6: /* fp4.5-e2m2: block 32, 9 words, shared bits in word 8 */
    {
      const int blk = id == 4 ? 64 : id == 5 ? 48 : 32;
      L->block = blk, L->words = blk / 4 + 1, L->segs_per_weight = 1;
      for (i = 0; i < blk; ++i) L->seg[i] = (orc_seg){i / 4, 4 * (i % 4), 4, 1};
      L->nshared = 16;
      for (i = 0; i < 16; ++i) L->sh_word[i] = blk / 4, L->sh_bit[i] = i;
      break;
    }
  }
}

/* packing.hpp:190-212 unpack_block: OR the segments, then OR each group's
 * shared bit into all k members. */
void orc_unpack_block(const uint16_t* words, const orc_layout* L, int k, uint8_t* codes) {
  int i, s, g, j;
  for (i = 0; i < L->block; ++i) {
    unsigned code = 0;
    for (s = 0; s < L->segs_per_weight; ++s) {
      const orc_seg* sg = &L->seg[i * L->segs_per_weight + s];
      code |= ((words[sg->word] >> sg->bit) & ((1u << sg->width) - 1u)) << sg->code_shift;
    }
    codes[i] = (uint8_t)code;
  }
  for (g = 0; g < L->nshared; ++g) {
    const unsigned bit = (words[L->sh_word[g]] >> L->sh_bit[g]) & 1u;
    for (j = 0; j < k; ++j) codes[g * k + j] |= (uint8_t)bit;
  }
}

/* packing.hpp:159-188 pack_block. Returns 2 (runtime_error) on a shared-bit
 * mismatch within a group (packing.hpp:176-179). */
int orc_pack_block(const uint8_t* codes, const orc_layout* L, int k, uint16_t* words) {
  int w, i, s, g, j;
  for (w = 0; w < L->words; ++w) words[w] = 0;
  for (i = 0; i < L->block; ++i) {
    for (s = 0; s < L->segs_per_weight; ++s) {
      const orc_seg* sg = &L->seg[i * L->segs_per_weight + s];
      const unsigned bits = ((unsigned)codes[i] >> sg->code_shift) & ((1u << sg->width) - 1u);
      words[sg->word] = (uint16_t)(words[sg->word] | (bits << sg->bit));
    }
  }
  for (g = 0; g < L->nshared; ++g) {
    const unsigned bit = codes[g * k] & 1u;
    for (j = 1; j < k; ++j)
      if ((codes[g * k + j] & 1u) != bit) return 2;
    if (bit) words[L->sh_word[g]] = (uint16_t)(words[L->sh_word[g]] | (1u << L->sh_bit[g]));
  }
  return 0;
}

/* packing.hpp:216-231 pack_row / 243-258 unpack_row (1 = invalid_argument). */
int orc_pack_row(int id, const uint8_t* codes, size_t n, uint16_t* words, size_t nw) {
  orc_layout L;
  size_t b;
  if (!orc_scheme_valid(id)) return 1;
  orc_layout_of(id, &L);
  if (n % (size_t)L.block) return 1;
  if (nw != n / (size_t)L.block * (size_t)L.words) return 1;
  for (b = 0; b < n / (size_t)L.block; ++b) {
    int rc = orc_pack_block(codes + b * L.block, &L, kSchemes[id].k, words + b * L.words);
    if (rc) return rc;
  }
  return 0;
}

int orc_unpack_row(int id, const uint16_t* words, size_t nw, uint8_t* codes, size_t n) {
  orc_layout L;
  size_t b;
  if (!orc_scheme_valid(id)) return 1;
  orc_layout_of(id, &L);
  if (nw % (size_t)L.words) return 1;
  if (n != nw / (size_t)L.words * (size_t)L.block) return 1;
  for (b = 0; b < nw / (size_t)L.words; ++b)
    orc_unpack_block(words + b * L.words, &L, kSchemes[id].k, codes + b * L.block);
  return 0;
}

/* packing.hpp:154-157 packed_words_per_row; quantize.hpp:64-69 packed_payload_bytes. */
size_t orc_padded_cols(int id, size_t cols) {
  orc_layout L;
  orc_layout_of(id, &L);
  return (cols + (size_t)L.block - 1) / (size_t)L.block * (size_t)L.block;
}

size_t orc_words_per_row(int id, size_t padded_cols) {
  orc_layout L;
  orc_layout_of(id, &L);
  return padded_cols / (size_t)L.block * (size_t)L.words;
}

size_t orc_packed_payload_bytes(int id, size_t rows, size_t cols) {
  return rows * orc_words_per_row(id, orc_padded_cols(id, cols)) * 2;
}

/* kernels.hpp:55-63 restore_block (table route): unpack, then look up the
 * binary16 pattern of every code. */
void orc_restore_block(int id, const uint16_t* words, uint16_t* out) {
  orc_layout L;
  uint8_t codes[64];
  int i;
  orc_layout_of(id, &L);
  orc_unpack_block(words, &L, kSchemes[id].k, codes);
  for (i = 0; i < L.block; ++i) out[i] = orc_to_fp16_bits(codes[i], id);
}

/* kernels.hpp:55-63 applied to a whole tensor: the binary16 grid bits of every
 * padded column ([rows][padded_cols]) -- "bit-exact dequantized weights". */
void orc_restore_grid(int id, size_t rows, size_t padded_cols, const uint16_t* payload,
                      uint16_t* out) {
  orc_layout L;
  size_t r, b;
  orc_layout_of(id, &L);
  const size_t wpr = padded_cols / (size_t)L.block * (size_t)L.words;
  for (r = 0; r < rows; ++r)
    for (b = 0; b < padded_cols / (size_t)L.block; ++b)
      orc_restore_block(id, payload + r * wpr + b * L.words, out + r * padded_cols + b * L.block);
}

/* kernels.hpp:100-124 restore_matrix: half_to_float(grid) * half_to_float(scale)
 * in single precision, logical columns only. */
void orc_restore_matrix(int id, size_t rows, size_t cols, size_t padded_cols,
                        const uint16_t* scales, const uint16_t* payload, float* out) {
  orc_layout L;
  uint16_t buf[64];
  size_t r, b, j;
  orc_layout_of(id, &L);
  const size_t wpr = padded_cols / (size_t)L.block * (size_t)L.words;
  for (r = 0; r < rows; ++r) {
    const float s = orc_half_to_float(scales[r]);
    for (b = 0; b * (size_t)L.block < padded_cols; ++b) {
      orc_restore_block(id, payload + r * wpr + b * L.words, buf);
      const size_t base = b * (size_t)L.block;
      size_t n = cols > base ? cols - base : 0;
      if (n > (size_t)L.block) n = (size_t)L.block;
      for (j = 0; j < n; ++j) out[r * cols + base + j] = orc_half_to_float(buf[j]) * s;
    }
  }
}

/* kernels.hpp:151-187 gemv: y[b][r] = fp16(sum_i (fp32(w_i) * s) * fp32(x_b,i)),
 * single-precision accumulation in ascending i, logical columns only.
 * Returns 1 (invalid_argument) on the check_gemv_shapes condition (137-143). */
int orc_gemv(int id, size_t rows, size_t cols, size_t padded_cols, const uint16_t* scales,
             const uint16_t* payload, const uint16_t* x, size_t x_len, size_t batch,
             uint16_t* y) {
  orc_layout L;
  uint16_t wbuf[64];
  size_t r, blk, bb, j;
  if (!orc_scheme_valid(id)) return 1;
  if (batch == 0 || x_len != batch * cols) return 1;
  orc_layout_of(id, &L);
  const size_t wpr = padded_cols / (size_t)L.block * (size_t)L.words;
  float* acc = (float*)calloc(batch, sizeof(float));
  if (!acc) return 3;
  for (r = 0; r < rows; ++r) {
    const float s = orc_half_to_float(scales[r]);
    for (bb = 0; bb < batch; ++bb) acc[bb] = 0.0f;
    for (blk = 0; blk * (size_t)L.block < padded_cols; ++blk) {
      orc_restore_block(id, payload + r * wpr + blk * L.words, wbuf);
      const size_t base = blk * (size_t)L.block;
      size_t n = cols > base ? cols - base : 0;
      if (n > (size_t)L.block) n = (size_t)L.block;
      for (bb = 0; bb < batch; ++bb) {
        const uint16_t* xb = x + bb * cols + base;
        float a = acc[bb];
        for (j = 0; j < n; ++j) {
          const float ws = orc_half_to_float(wbuf[j]) * s;
          a += ws * orc_half_to_float(xb[j]);
        }
        acc[bb] = a;
      }
    }
    for (bb = 0; bb < batch; ++bb) y[bb * rows + r] = orc_float_to_half(acc[bb]);
  }
  free(acc);
  return 0;
}

/* Float64 reference of the same linear (tolerance denominators for the kernel
 * tests): yabs[b][r] = sum_i |w_i s x_b,i| and yexact[b][r] = sum_i w_i s x_b,i. */
int orc_gemv_f64(int id, size_t rows, size_t cols, size_t padded_cols, const uint16_t* scales,
                 const uint16_t* payload, const uint16_t* x, size_t batch, double* yexact,
                 double* yabs) {
  size_t r, i, bb;
  float* w = (float*)malloc(sizeof(float) * rows * cols);
  if (!w) return 3;
  orc_restore_matrix(id, rows, cols, padded_cols, scales, payload, w);
  for (bb = 0; bb < batch; ++bb) {
    for (r = 0; r < rows; ++r) {
      double e = 0.0, a = 0.0;
      for (i = 0; i < cols; ++i) {
        const double p = (double)w[r * cols + i] * (double)orc_half_to_float(x[bb * cols + i]);
        e += p;
        a += fabs(p);
      }
      yexact[bb * rows + r] = e;
      yabs[bb * rows + r] = a;
    }
  }
  free(w);
  return 0;
}

/* --------------------------------------------------------------- quantizer
 * format.hpp:152-186 enumerate_values / round_to_nearest over the sorted grid
 * (negatives reversed, the canonical +0, positives), ties to the even code and,
 * when both neighbours are even, to the smaller magnitude. */
static int orc_grid(int id, float* val, uint8_t* code) {
  const orc_scheme* s = &kSchemes[id];
  const unsigned n = 1u << (1 + s->e + s->m), half_n = n / 2, sign = 1u << (s->e + s->m);
  int cnt = 0;
  unsigned mag;
  for (mag = half_n - 1; mag >= 1; --mag) {
    val[cnt] = orc_decode(sign | mag, id);
    code[cnt++] = (uint8_t)(sign | mag);
  }
  val[cnt] = 0.0f;
  code[cnt++] = 0;
  for (mag = 1; mag < half_n; ++mag) {
    val[cnt] = orc_decode(mag, id);
    code[cnt++] = (uint8_t)mag;
  }
  return cnt;
}

float orc_max_magnitude(int id) {
  float v[256];
  uint8_t c[256];
  const int n = orc_grid(id, v, c);
  return v[n - 1];
}

/* The sorted grid per scheme, built once (the reference caches it too,
 * format.hpp:134-146). Single-threaded test use only. */
static float g_grid_v[8][256];
static uint8_t g_grid_c[8][256];
static int g_grid_n[8];

uint8_t orc_round_to_nearest(float w, int id) {
  if (!g_grid_n[id]) g_grid_n[id] = orc_grid(id, g_grid_v[id], g_grid_c[id]);
  const float* v = g_grid_v[id];
  const uint8_t* c = g_grid_c[id];
  const int n = g_grid_n[id];
  int lo_i, hi_i, a, b;
  if (!(w > v[0])) return c[0];
  if (w >= v[n - 1]) return c[n - 1];
  /* lower_bound: first value >= w */
  a = 0, b = n;
  while (a < b) {
    const int mid = (a + b) / 2;
    if (v[mid] < w) a = mid + 1;
    else b = mid;
  }
  hi_i = a, lo_i = a - 1;
  const double dlo = (double)w - (double)v[lo_i];
  const double dhi = (double)v[hi_i] - (double)w;
  if (dlo < dhi) return c[lo_i];
  if (dhi < dlo) return c[hi_i];
  if ((c[lo_i] & 1u) == 0 && (c[hi_i] & 1u) == 0)
    return fabsf(v[lo_i]) <= fabsf(v[hi_i]) ? c[lo_i] : c[hi_i];
  return (c[lo_i] & 1u) == 0 ? c[lo_i] : c[hi_i];
}

/* quantize.hpp:72-82 channel_scale and 86-93 stored_scale_bits.
 * Returns 2 on a non-finite weight or half overflow (runtime_error). */
static int orc_stored_scale(const float* row, size_t n, int id, uint16_t* out) {
  float max_abs = 0.0f;
  size_t i;
  for (i = 0; i < n; ++i) {
    if (!isfinite(row[i])) return 2;
    const float a = fabsf(row[i]);
    if (a > max_abs) max_abs = a;
  }
  const float scale = max_abs == 0.0f ? 1.0f : max_abs / orc_max_magnitude(id);
  uint16_t h = (uint16_t)(orc_float_to_half(scale) & 0x7FFF);
  if (h >= 0x7C00) return 2;
  if (h == 0) h = 1;
  *out = h;
  return 0;
}

/* quantize.hpp:100-105 set_mantissa_lsb: -0 collapses to +0. */
static uint8_t orc_set_lsb(uint8_t code, unsigned bit, int id) {
  const orc_scheme* s = &kSchemes[id];
  uint8_t c = (uint8_t)((code & ~1u) | bit);
  if (c == (1u << (s->e + s->m))) c = 0;
  return c;
}

/* quantize.hpp:188-216 quantize_tensor = pad_cols_to(block) -> rtn_quantize
 * (112-131) -> ams_share (138-184, double-precision squared error, ties -> 0,
 * groups touching padding pinned to 0) -> pack_row. */
int orc_quantize_tensor(int id, size_t rows, size_t cols, const float* w, uint16_t* scales,
                        uint16_t* payload) {
  orc_layout L;
  size_t r, c, g;
  if (!orc_scheme_valid(id) || rows == 0 || cols == 0) return 1;
  orc_layout_of(id, &L);
  const int k = kSchemes[id].k;
  const size_t pc = orc_padded_cols(id, cols);
  const size_t wpr = orc_words_per_row(id, pc);
  float* prow = (float*)calloc(pc, sizeof(float));
  uint8_t* codes = (uint8_t*)calloc(pc, 1);
  if (!prow || !codes) return 3;
  int rc = 0;
  for (r = 0; r < rows && !rc; ++r) {
    memset(prow, 0, pc * sizeof(float));
    memcpy(prow, w + r * cols, cols * sizeof(float));
    rc = orc_stored_scale(prow, pc, id, &scales[r]);
    if (rc) break;
    const float s = orc_half_to_float(scales[r]);
    for (c = 0; c < pc; ++c) codes[c] = orc_round_to_nearest(prow[c] / s, id);
    if (k > 1) {
      const size_t gpr = (pc + (size_t)k - 1) / (size_t)k;
      for (g = 0; g < gpr; ++g) {
        const size_t begin = g * (size_t)k;
        const size_t end = begin + (size_t)k < pc ? begin + (size_t)k : pc;
        unsigned bit = 0, b;
        if (end <= cols) {
          double err[2] = {0.0, 0.0};
          for (b = 0; b < 2; ++b)
            for (c = begin; c < end; ++c) {
              const float restored = orc_decode(orc_set_lsb(codes[c], b, id), id) * s;
              const double d = (double)restored - (double)prow[c];
              err[b] += d * d;
            }
          bit = err[1] < err[0] ? 1u : 0u;
        }
        for (c = begin; c < end; ++c) codes[c] = orc_set_lsb(codes[c], bit, id);
      }
    }
    rc = orc_pack_row(id, codes, pc, payload + r * wpr, wpr);
  }
  free(prow);
  free(codes);
  return rc;
}
