// device_layout.cpp -- see device_layout.hpp for the bit map.
#include "device_layout.hpp"

#include <algorithm>
#include <cstring>
#include <vector>

#include "host_core.hpp"

#ifndef AMSQ_CLUSTER_COST_G  // plan cost of a cluster K split, in k-tiles (per row tile, fixed)
#define AMSQ_CLUSTER_COST_G 1.0
#endif
#ifndef AMSQ_CLUSTER_COST_0
#define AMSQ_CLUSTER_COST_0 25.0  // cluster barrier + DSMEM epilogue ~0.6 us (o_proj: C=1 wins)
#endif

namespace amsqb {

bool device_scheme_supported(int id) { return id >= 0 && id < kNumSchemes; }

namespace {
// (TK, tile bytes) per scheme: exactly the reference bits of a 16 x TK tile
constexpr int kTileTK[8] = {64, 64, 64, 64, 64, 48, 64, 48};
constexpr int kTileBytes[8] = {512, 640, 768, 768, 544, 416, 576, 512};
}  // namespace

DeviceLayout make_device_layout(int id, size_t rows, size_t cols, size_t pc) {
  const Scheme& s = scheme(id);
  if (!device_scheme_supported(id)) {
    throw InvalidArgument(std::string("device layout: scheme ") + s.name + " has no sm_100a kernel");
  }
  if (rows == 0 || cols == 0) throw InvalidArgument("device layout: empty tensor");
  if (pc != padded_cols(s, cols)) throw InvalidArgument("device layout: padded_cols mismatch");
  DeviceLayout L;
  L.scheme_id = id;
  L.rows = rows, L.cols = cols, L.padded_cols = pc;
  L.wpr = words_per_row(s, pc);
  L.tk = static_cast<size_t>(kTileTK[id]);
  L.tile_bytes = static_cast<size_t>(kTileBytes[id]);
  L.row_tiles = (rows + kRowsPerTile - 1) / kRowsPerTile;
  L.k_tiles = (pc + L.tk - 1) / L.tk;
  choose_plan(L.row_tiles, L.k_tiles, &L);
  return L;
}

// Per-CTA work = G row tiles x ceil(KT / C) k-tiles (G = ceil(RT / n_groups)); pick the
// plan with the least work per CTA, and among plans within 1 % of it the one that keeps the
// most SMs streaming (more CTAs = more bytes in flight), then the smaller K split.
void choose_plan(size_t RT, size_t KT, DeviceLayout* L) {
  struct Cand {
    double work;
    int ctas, C, ng, G;
  };
  std::vector<Cand> cands;
  for (int C = 1; C <= 8; C *= 2) {
    if (C > 1 && KT < 2 * static_cast<size_t>(C)) continue;
    const size_t max_groups = std::min<size_t>(RT, kMaxClusters[C]);
    for (size_t ng = 1; ng <= max_groups; ++ng) {
      const size_t G = (RT + ng - 1) / ng;
      if (G > static_cast<size_t>(kMaxGroupTiles) || (RT + G - 1) / G != ng) continue;
      // a cluster's DSMEM reduction (remote stores of G row tiles' partials + one cluster
      // barrier) costs about one k-tile per row tile plus ~3 k-tiles of barrier latency
      // a consumer warp reuses each k-tile's activation fragments over its <= 4 row tiles:
      // with fewer than 4 row tiles per CTA the per-byte cost rises (measured: 2 tiles ~1.15x)
      const double reuse = 1.0 + 0.3 * (4.0 - static_cast<double>(std::min<size_t>(G, 4))) / 4.0;
      const double work = static_cast<double>(G) * static_cast<double>((KT + C - 1) / C) * reuse +
                          (C > 1 ? AMSQ_CLUSTER_COST_G * G + AMSQ_CLUSTER_COST_0 : 0.0);
      cands.push_back({work, static_cast<int>(ng) * C, C, static_cast<int>(ng),
                       static_cast<int>(G)});
    }
  }
  if (cands.empty()) throw InvalidArgument("device layout: no work plan (too many rows per SM)");
  double best = cands[0].work;
  for (const Cand& c : cands) best = std::min(best, c.work);
  const Cand* pick = nullptr;
  for (const Cand& c : cands) {
    if (c.work > best * 1.01) continue;
    if (!pick || c.ctas > pick->ctas || (c.ctas == pick->ctas && c.C < pick->C)) pick = &c;
  }
  L->n_groups = pick->ng;
  L->g_big = pick->G;
  L->n_big = static_cast<int>(RT - static_cast<size_t>(pick->ng) * (pick->G - 1));
  L->csplit = pick->C;
}

namespace {

// ---------------------------------------------------------------- FP4.25
// Position of member i's mag3 (low half) and sign bit; +16 for the high half.
constexpr int kS4MagPos[4] = {9, 6, 3, 0};
constexpr int kS4SignPos[4] = {15, 12, 13, 14};

inline uint32_t s4_encode(const uint8_t nib_a[4], const uint8_t nib_b[4]) {
  uint32_t r = 0;
  for (int i = 0; i < 4; ++i) {
    const uint32_t a = nib_a[i], b = nib_b[i];
    r |= (a & 7u) << kS4MagPos[i] | (a >> 3) << kS4SignPos[i];
    r |= (b & 7u) << (kS4MagPos[i] + 16) | (b >> 3) << (kS4SignPos[i] + 16);
  }
  return r;
}

inline void s4_decode(uint32_t r, uint8_t nib_a[4], uint8_t nib_b[4]) {
  for (int i = 0; i < 4; ++i) {
    nib_a[i] = static_cast<uint8_t>(((r >> kS4MagPos[i]) & 7u) | ((r >> kS4SignPos[i]) & 1u) << 3);
    nib_b[i] = static_cast<uint8_t>(((r >> (kS4MagPos[i] + 16)) & 7u) |
                                    ((r >> (kS4SignPos[i] + 16)) & 1u) << 3);
  }
}

// One tile (rt, kt) of FP4.25 from the reference rows. Block kt of row n is the 17
// words at n*wpr + 17*kt: word G holds group G's four nibbles, word 16 the shared bits.
void s4_pack_tile(const DeviceLayout& L, const uint16_t* payload, size_t rt, size_t kt,
                  uint8_t* tile) {
  std::memset(tile, 0, L.tile_bytes);
  if (kt * 17 >= L.wpr) return;
  for (int lane = 0; lane < 32; ++lane) {
    const int g = lane >> 2, t = lane & 3;
    uint32_t R[4];
    uint8_t sh = 0;
    for (int q = 0; q < 4; ++q) {  // R_q: row g (q<2) / g+8 (q>=2), groups 4t+2(q&1) (+1)
      const size_t n = rt * 16 + static_cast<size_t>(g + (q >= 2 ? 8 : 0));
      const int ga = 4 * t + 2 * (q & 1), gb = ga + 1;
      uint8_t na[4] = {0, 0, 0, 0}, nb[4] = {0, 0, 0, 0};
      if (n < L.rows) {
        const uint16_t* blk = payload + n * L.wpr + kt * 17;
        for (int i = 0; i < 4; ++i) {
          na[i] = static_cast<uint8_t>((blk[ga] >> (4 * i)) & 0xFu);
          nb[i] = static_cast<uint8_t>((blk[gb] >> (4 * i)) & 0xFu);
        }
        sh = static_cast<uint8_t>(sh | ((blk[16] >> ga) & 1u) << q | ((blk[16] >> gb) & 1u) << (q + 4));
      }
      R[q] = s4_encode(na, nb);
    }
    std::memcpy(tile + lane * 16, R, 16);
    tile[512 + lane] = sh;
  }
}

void s4_unpack_tile(const DeviceLayout& L, const uint8_t* tile, size_t rt, size_t kt,
                    uint16_t* payload) {
  if (kt * 17 >= L.wpr) return;
  for (int lane = 0; lane < 32; ++lane) {
    const int g = lane >> 2, t = lane & 3;
    uint32_t R[4];
    std::memcpy(R, tile + lane * 16, 16);
    const uint8_t sh = tile[512 + lane];
    for (int q = 0; q < 4; ++q) {
      const size_t n = rt * 16 + static_cast<size_t>(g + (q >= 2 ? 8 : 0));
      if (n >= L.rows) continue;
      const int ga = 4 * t + 2 * (q & 1), gb = ga + 1;
      uint8_t na[4], nb[4];
      s4_decode(R[q], na, nb);
      uint16_t* blk = payload + n * L.wpr + kt * 17;
      uint16_t wa = 0, wb = 0;
      for (int i = 0; i < 4; ++i) {
        wa = static_cast<uint16_t>(wa | na[i] << (4 * i));
        wb = static_cast<uint16_t>(wb | nb[i] << (4 * i));
      }
      blk[ga] = wa, blk[gb] = wb;
      const uint16_t keep = static_cast<uint16_t>(~((1u << ga) | (1u << gb)));
      blk[16] = static_cast<uint16_t>((blk[16] & keep) | ((sh >> q) & 1u) << ga | ((sh >> (q + 4)) & 1u) << gb);
    }
  }
}

// ---------------------------------------------------------------- FP5.33
inline uint32_t s7_encode(uint16_t wa, uint16_t wb) {
  uint32_t r = 0;
  const uint16_t w[2] = {wa, wb};
  for (int h = 0; h < 2; ++h) {
    const uint32_t o = 16u * static_cast<uint32_t>(h);
    const uint32_t s0 = w[h] & 0x1Fu, s1 = (w[h] >> 5) & 0x1Fu, s2 = (w[h] >> 10) & 0x1Fu;
    const uint32_t sh = (w[h] >> 15) & 1u;
    r |= (s0 & 0xFu) << (8 + o) | (s0 >> 4) << (15 + o);
    r |= (s1 & 0xFu) << (0 + o) | (s1 >> 4) << (7 + o);
    r |= ((s2 & 0xFu) >> 1) << (4 + o) | (s2 & 1u) << (13 + o) | (s2 >> 4) << (14 + o);
    r |= sh << (12 + o);
  }
  return r;
}

inline void s7_decode(uint32_t r, uint16_t* wa, uint16_t* wb) {
  uint16_t w[2];
  for (int h = 0; h < 2; ++h) {
    const uint32_t x = r >> (16 * h);
    const uint32_t s0 = ((x >> 8) & 0xFu) | ((x >> 15) & 1u) << 4;
    const uint32_t s1 = (x & 0xFu) | ((x >> 7) & 1u) << 4;
    const uint32_t s2 = ((x >> 4) & 7u) << 1 | ((x >> 13) & 1u) | ((x >> 14) & 1u) << 4;
    const uint32_t sh = (x >> 12) & 1u;
    w[h] = static_cast<uint16_t>(s0 | s1 << 5 | s2 << 10 | sh << 15);
  }
  *wa = w[0], *wb = w[1];
}

// Tile (rt, kt) of FP5.33 covers reference words [16 kt, 16 kt + 16) of each row.
void s7_pack_tile(const DeviceLayout& L, const uint16_t* payload, size_t rt, size_t kt,
                  uint8_t* tile) {
  std::memset(tile, 0, L.tile_bytes);
  for (int lane = 0; lane < 32; ++lane) {
    const int g = lane >> 2, t = lane & 3;
    uint32_t R[4];
    for (int q = 0; q < 4; ++q) {
      const size_t n = rt * 16 + static_cast<size_t>(g + (q >= 2 ? 8 : 0));
      const size_t wa_i = kt * 16 + static_cast<size_t>(4 * t + 2 * (q & 1)), wb_i = wa_i + 1;
      uint16_t wa = 0, wb = 0;
      if (n < L.rows) {
        if (wa_i < L.wpr) wa = payload[n * L.wpr + wa_i];
        if (wb_i < L.wpr) wb = payload[n * L.wpr + wb_i];
      }
      R[q] = s7_encode(wa, wb);
    }
    std::memcpy(tile + lane * 16, R, 16);
  }
}

void s7_unpack_tile(const DeviceLayout& L, const uint8_t* tile, size_t rt, size_t kt,
                    uint16_t* payload) {
  for (int lane = 0; lane < 32; ++lane) {
    const int g = lane >> 2, t = lane & 3;
    uint32_t R[4];
    std::memcpy(R, tile + lane * 16, 16);
    for (int q = 0; q < 4; ++q) {
      const size_t n = rt * 16 + static_cast<size_t>(g + (q >= 2 ? 8 : 0));
      if (n >= L.rows) continue;
      const size_t wa_i = kt * 16 + static_cast<size_t>(4 * t + 2 * (q & 1)), wb_i = wa_i + 1;
      uint16_t wa, wb;
      s7_decode(R[q], &wa, &wb);
      if (wa_i < L.wpr) payload[n * L.wpr + wa_i] = wa;
      if (wb_i < L.wpr) payload[n * L.wpr + wb_i] = wb;
    }
  }
}

// ---------------------------------------------------------------- the nibble family
// Schemes 0, 1, 2, 3, 5, 6 (kernels_common.cuh "the other six schemes"): the code of each
// weight is split into its top nibble (sign + 3 magnitude bits) and its low bits (none, a
// per-weight LSB, two per-weight LSBs, or a group-shared LSB). The tile holds the nibbles in
// 32-bit registers (8 per register: members i = 0..3 of a pair a | b) and the low bits in a
// per-lane plane; see decode_frag for the exact bit positions the kernels expect.

// bit position of member i's mag bit b (0..2) and sign, low half; E3 = the fp6-e3m2 map
inline int nib_mag_pos(bool e3, int i, int b) {
  if (!e3) return (9 - 3 * i) + b;
  switch (i) {
    case 0: return 10 + b;
    case 1: return 4 + b;
    case 2: return b;
    default: return b == 0 ? 7 : b == 1 ? 8 : 3;
  }
}
inline int nib_sign_pos(bool e3, int i) {
  static constexpr int e2[4] = {15, 12, 13, 14}, e3p[4] = {15, 9, 13, 14};
  return e3 ? e3p[i] : e2[i];
}
inline uint32_t nib_put(bool e3, int i, int half, unsigned nib) {
  uint32_t r = 0;
  for (int b = 0; b < 3; ++b) r |= ((nib >> b) & 1u) << (nib_mag_pos(e3, i, b) + 16 * half);
  r |= ((nib >> 3) & 1u) << (nib_sign_pos(e3, i) + 16 * half);
  return r;
}
inline unsigned nib_get(bool e3, int i, int half, uint32_t r) {
  unsigned nib = 0;
  for (int b = 0; b < 3; ++b) nib |= ((r >> (nib_mag_pos(e3, i, b) + 16 * half)) & 1u) << b;
  nib |= ((r >> (nib_sign_pos(e3, i) + 16 * half)) & 1u) << 3;
  return nib;
}
inline int low_bits_of(int id) { return id == 0 ? 0 : (id == 2 || id == 3) ? 2 : 1; }

// The 16 x TK codes of tile (rt, kt) from the reference rows (0 past rows / padded_cols).
void tile_codes(const DeviceLayout& L, const Scheme& s, const uint16_t* payload, size_t rt,
                size_t kt, std::vector<uint8_t>& codes) {
  const size_t TK = L.tk, blocks_per_tile = TK / static_cast<size_t>(s.block);
  codes.assign(16 * TK, 0);
  const size_t blk0 = kt * blocks_per_tile, nblk_row = L.padded_cols / static_cast<size_t>(s.block);
  if (blk0 >= nblk_row) return;
  const size_t nblk = std::min(blocks_per_tile, nblk_row - blk0);
  for (size_t r = 0; r < 16; ++r) {
    const size_t n = rt * 16 + r;
    if (n >= L.rows) continue;
    const uint16_t* w = payload + n * L.wpr + blk0 * static_cast<size_t>(s.words_per_block);
    unpack_row(s, std::span<const uint16_t>(w, nblk * static_cast<size_t>(s.words_per_block)),
               std::span<uint8_t>(codes.data() + r * TK, nblk * static_cast<size_t>(s.block)));
  }
}

void tile_codes_store(const DeviceLayout& L, const Scheme& s, const std::vector<uint8_t>& codes,
                      size_t rt, size_t kt, uint16_t* payload) {
  const size_t TK = L.tk, blocks_per_tile = TK / static_cast<size_t>(s.block);
  const size_t blk0 = kt * blocks_per_tile, nblk_row = L.padded_cols / static_cast<size_t>(s.block);
  if (blk0 >= nblk_row) return;
  const size_t nblk = std::min(blocks_per_tile, nblk_row - blk0);
  for (size_t r = 0; r < 16; ++r) {
    const size_t n = rt * 16 + r;
    if (n >= L.rows) continue;
    uint16_t* w = payload + n * L.wpr + blk0 * static_cast<size_t>(s.words_per_block);
    pack_row(s, std::span<const uint8_t>(codes.data() + r * TK, nblk * static_cast<size_t>(s.block)),
             std::span<uint16_t>(w, nblk * static_cast<size_t>(s.words_per_block)));
  }
}

// (row, column) of output slot (q, i) of lane (g, t), half h (0 = a, 1 = b): family 4
inline void fam4_rc(int g, int t, int q, int i, int h, int* row, int* col) {
  *row = g + (q >= 2 ? 8 : 0);
  *col = 16 * t + 8 * (q & 1) + 4 * h + i;
}
// family 7 (fp4.33): flat output f = 4q + i; pair k = f / 3, member m = f % 3
inline void fam7_rc(int g, int t, int f, int h, int* row, int* col) {
  const int k = f / 3, m = f - 3 * k;
  *row = g + (k >= 2 ? 8 : 0);
  *col = 12 * t + 6 * (k & 1) + 3 * h + m;
}

void nib_pack_tile(const DeviceLayout& L, const uint16_t* payload, size_t rt, size_t kt,
                   uint8_t* tile) {
  const int id = L.scheme_id;
  const Scheme& s = scheme(id);
  const bool e3 = id == 3;
  const int lb = low_bits_of(id);
  const size_t TK = L.tk;
  std::vector<uint8_t> codes;
  tile_codes(L, s, payload, rt, kt, codes);
  std::memset(tile, 0, L.tile_bytes);
  auto code = [&](int row, int col) -> unsigned { return codes[static_cast<size_t>(row) * TK + col]; };
  for (int lane = 0; lane < 32; ++lane) {
    const int g = lane >> 2, t = lane & 3;
    if (id == 5) {
      uint32_t R[3] = {0, 0, 0};
      uint8_t sh = 0;
      for (int f = 0; f < 12; ++f) {
        for (int h = 0; h < 2; ++h) {
          int row, col;
          fam7_rc(g, t, f, h, &row, &col);
          R[f >> 2] |= nib_put(false, f & 3, h, code(row, col) >> 1);
          if (f % 3 == 0) sh = static_cast<uint8_t>(sh | (code(row, col) & 1u) << (f / 3 + 4 * h));
        }
      }
      std::memcpy(tile + lane * 8, R, 8);
      std::memcpy(tile + 256 + lane * 4, &R[2], 4);
      tile[384 + lane] = sh;
      continue;
    }
    uint32_t R[4] = {0, 0, 0, 0}, P = 0, Q[2] = {0, 0};
    uint16_t sh16 = 0;
    for (int q = 0; q < 4; ++q) {
      for (int i = 0; i < 4; ++i) {
        for (int h = 0; h < 2; ++h) {
          int row, col;
          fam4_rc(g, t, q, i, h, &row, &col);
          const unsigned c = code(row, col);
          R[q] |= nib_put(e3, i, h, c >> lb);
          const int p = 4 * q + i;
          if (id == 1) P |= (c & 1u) << (p + 16 * h);
          if (id == 2 || id == 3) Q[p >> 3] |= (c & 3u) << (2 * (p & 7) + 16 * h);
          if (id == 6 && (i == 0 || i == 2)) sh16 = static_cast<uint16_t>(sh16 | (c & 1u) << (8 * (i >> 1) + q + 4 * h));
        }
      }
    }
    std::memcpy(tile + lane * 16, R, 16);
    if (id == 1) std::memcpy(tile + 512 + lane * 4, &P, 4);
    if (id == 2 || id == 3) std::memcpy(tile + 512 + lane * 8, Q, 8);
    if (id == 6) std::memcpy(tile + 512 + lane * 2, &sh16, 2);
  }
}

void nib_unpack_tile(const DeviceLayout& L, const uint8_t* tile, size_t rt, size_t kt,
                     uint16_t* payload) {
  const int id = L.scheme_id;
  const Scheme& s = scheme(id);
  const bool e3 = id == 3;
  const int lb = low_bits_of(id);
  const size_t TK = L.tk;
  std::vector<uint8_t> codes(16 * TK, 0);
  auto set = [&](int row, int col, unsigned c) { codes[static_cast<size_t>(row) * TK + col] = static_cast<uint8_t>(c); };
  for (int lane = 0; lane < 32; ++lane) {
    const int g = lane >> 2, t = lane & 3;
    if (id == 5) {
      uint32_t R[3];
      std::memcpy(R, tile + lane * 8, 8);
      std::memcpy(&R[2], tile + 256 + lane * 4, 4);
      const uint8_t sh = tile[384 + lane];
      for (int f = 0; f < 12; ++f) {
        for (int h = 0; h < 2; ++h) {
          int row, col;
          fam7_rc(g, t, f, h, &row, &col);
          const unsigned shared = (sh >> (f / 3 + 4 * h)) & 1u;
          set(row, col, nib_get(false, f & 3, h, R[f >> 2]) << 1 | shared);
        }
      }
      continue;
    }
    uint32_t R[4], P = 0, Q[2] = {0, 0};
    uint16_t sh16 = 0;
    std::memcpy(R, tile + lane * 16, 16);
    if (id == 1) std::memcpy(&P, tile + 512 + lane * 4, 4);
    if (id == 2 || id == 3) std::memcpy(Q, tile + 512 + lane * 8, 8);
    if (id == 6) std::memcpy(&sh16, tile + 512 + lane * 2, 2);
    for (int q = 0; q < 4; ++q) {
      for (int i = 0; i < 4; ++i) {
        for (int h = 0; h < 2; ++h) {
          int row, col;
          fam4_rc(g, t, q, i, h, &row, &col);
          unsigned c = nib_get(e3, i, h, R[q]) << lb;
          const int p = 4 * q + i;
          if (id == 1) c |= (P >> (p + 16 * h)) & 1u;
          if (id == 2 || id == 3) c |= (Q[p >> 3] >> (2 * (p & 7) + 16 * h)) & 3u;
          if (id == 6) c |= (sh16 >> (8 * (i >> 1) + q + 4 * h)) & 1u;
          set(row, col, c);
        }
      }
    }
  }
  tile_codes_store(L, s, codes, rt, kt, payload);
}

}  // namespace

void repack_to_device(const DeviceLayout& L, const uint16_t* payload, uint8_t* out, int threads) {
  parallel_rows(L.row_tiles, threads, [&](size_t r0, size_t r1) {
    for (size_t rt = r0; rt < r1; ++rt) {
      for (size_t kt = 0; kt < L.k_tiles; ++kt) {
        uint8_t* tile = out + L.tile_offset(rt, kt);
        if (L.scheme_id == 4) {
          s4_pack_tile(L, payload, rt, kt, tile);
        } else if (L.scheme_id == 7) {
          s7_pack_tile(L, payload, rt, kt, tile);
        } else {
          nib_pack_tile(L, payload, rt, kt, tile);
        }
      }
    }
  });
}

void repack_from_device(const DeviceLayout& L, const uint8_t* in, uint16_t* payload, int threads) {
  parallel_rows(L.row_tiles, threads, [&](size_t r0, size_t r1) {
    for (size_t rt = r0; rt < r1; ++rt) {
      for (size_t kt = 0; kt < L.k_tiles; ++kt) {
        const uint8_t* tile = in + L.tile_offset(rt, kt);
        if (L.scheme_id == 4) {
          s4_unpack_tile(L, tile, rt, kt, payload);
        } else if (L.scheme_id == 7) {
          s7_unpack_tile(L, tile, rt, kt, payload);
        } else {
          nib_unpack_tile(L, tile, rt, kt, payload);
        }
      }
    }
  });
}

}  // namespace amsqb
