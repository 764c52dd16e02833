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

bool device_scheme_supported(int id) { return id == 4 || id == 7; }

DeviceLayout make_device_layout(int id, size_t rows, size_t cols, size_t pc) {
  const Scheme& s = scheme(id);
  if (!device_scheme_supported(id)) {
    throw InvalidArgument(std::string("device layout: scheme ") + s.name +
                          " has no sm_100a kernel (supported: fp4.25-e2m2, fp5.33-e2m3)");
  }
  if (rows == 0 || cols == 0) throw InvalidArgument("device layout: empty tensor");
  if (pc != padded_cols(s, cols)) throw InvalidArgument("device layout: padded_cols mismatch");
  DeviceLayout L;
  L.scheme_id = id;
  L.rows = rows, L.cols = cols, L.padded_cols = pc;
  L.wpr = words_per_row(s, pc);
  L.tk = id == 4 ? 64 : 48;
  L.tile_bytes = id == 4 ? 544 : 512;
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

}  // namespace

void repack_to_device(const DeviceLayout& L, const uint16_t* payload, uint8_t* out, int threads) {
  parallel_rows(L.row_tiles, threads, [&](size_t r0, size_t r1) {
    for (size_t rt = r0; rt < r1; ++rt) {
      for (size_t kt = 0; kt < L.k_tiles; ++kt) {
        uint8_t* tile = out + L.tile_offset(rt, kt);
        if (L.scheme_id == 4) {
          s4_pack_tile(L, payload, rt, kt, tile);
        } else {
          s7_pack_tile(L, payload, rt, kt, tile);
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
        } else {
          s7_unpack_tile(L, tile, rt, kt, payload);
        }
      }
    }
  });
}

}  // namespace amsqb
