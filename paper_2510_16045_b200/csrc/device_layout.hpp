// device_layout.hpp -- the sm_100a tile layout of the packed weights.
//
// The reference stream (packing.hpp:6-25; rows of `words_per_row` u16) is permuted,
// bit for bit, into 16-row x TK-column tiles whose bytes are exactly what one warp's
// mma.sync A-fragments need: lane (g = lane/4, t = lane%4) owns rows g and g+8 and
// four reference groups of each, as four 32-bit registers R0..R3 (16 B, one
// LDS.128). Each register holds two groups (a, b) of one row: output fp16x2 i of R is
// (a_i, b_i), so the shared LSB of a lands in bit 8/7 of the low half and b's in the
// high half. The bit positions inside R are chosen so that each fp16x2 is produced
// by at most {mask, IMAD, LOP3} (see decode_* in kernels_common.cuh).
//
//  FP4.25-e2m2 (scheme 4): TK = 64 (one reference block per row), 544 B per tile:
//    [lane*16, +16) R0..R3 (row g groups 4t,4t+1 | row g 4t+2,4t+3 | row g+8 ... )
//    [512 + lane]   shared byte: bit r = group a of R_r, bit r+4 = group b of R_r
//    R bits for member i (nibble = code bits 4..1 = s,E1,E0,M1; mag3 = E1,E0,M1):
//      i=0: mag3<<9,  sign@15 | high: mag3<<25, sign@31
//      i=1: mag3<<6,  sign@12 | high: mag3<<22, sign@28
//      i=2: mag3<<3,  sign@13 | high: mag3<<19, sign@29
//      i=3: mag3<<0,  sign@14 | high: mag3<<16, sign@30
//  FP5.33-e2m3 (scheme 7): TK = 48 (16 reference words per row), 512 B per tile:
//    [lane*16, +16) R0..R3, same row/group assignment, 2 reference words per R
//    R bits for member i (seg = code bits 5..1 = s,E1,E0,M2,M1; mag4 = E1,E0,M2,M1):
//      i=0: mag4<<8, sign@15            | high: mag4<<24, sign@31
//      i=1: mag4<<0, sign@7             | high: mag4<<16, sign@23
//      i=2: (mag4>>1)<<4, M1@13, sign@14 | high: (mag4>>1)<<20, M1@29, sign@30
//      shared: a@12, b@28
//
// Work plan and tile order (sm_100a, 148 SMs): the row tiles are split into `n_groups`
// contiguous row groups of g_big or g_big - 1 tiles (the first n_big groups are the big
// ones). Each group is processed by one CTA -- or by a cluster of `csplit` = 2/4/8 CTAs that
// split K and reduce through distributed shared memory -- over the FULL K range, so no
// partial sums ever leave the SM (cluster). The plan is chosen at upload from (row tiles,
// k tiles) alone to minimise the per-CTA tile count (SURVEY.md §7 hard part 4), so the
// fp32 summation order depends only on the shape.
// Tiles of a group are stored [k_tile][row_tile_in_group]: a CTA's whole weight range is
// one contiguous region and a pipeline stage (S k-tiles x G row tiles) is ONE
// cp.async.bulk. Padding rows (to a multiple of 16) and columns (to a multiple of TK)
// are zero and restore to +0.
#pragma once

#include <cstddef>
#include <cstdint>

namespace amsqb {

#ifndef AMSQ_CTAS_PER_SM  // K2 CTAs resident per SM the plan is built for (1 in the product)
#define AMSQ_CTAS_PER_SM 1
#endif
constexpr int kPlanSMs = 148 * AMSQ_CTAS_PER_SM;  // B200: 148 SMs
// Clusters of C CTAs that can be co-resident (C = 1, 2, 4, 8; index by C). Larger clusters
// must fit inside one GPC, which strands SMs: 4 -> 32 clusters, 8 -> 16 clusters assumed
// (conservative; tools/cluster_probe reports the device's own figure).
constexpr int kMaxClusters[9] = {0, 148 * AMSQ_CTAS_PER_SM, 74 * AMSQ_CTAS_PER_SM, 0,
                                 32 * AMSQ_CTAS_PER_SM, 0, 0, 0, 16 * AMSQ_CTAS_PER_SM};
constexpr int kMaxGroupTiles = 64;  // 16 consumer warps x 4 row tiles each

struct DeviceLayout {
  int scheme_id = -1;
  size_t rows = 0, cols = 0, padded_cols = 0;
  size_t wpr = 0;        // reference words per row
  size_t tk = 0;         // columns per k-tile
  size_t tile_bytes = 0;
  size_t row_tiles = 0;  // ceil(rows / 16)
  size_t k_tiles = 0;
  // plan
  int n_groups = 0, g_big = 0, n_big = 0, csplit = 1;
  int ctas() const { return n_groups * csplit; }
  size_t group_row0(size_t g) const {
    return g < static_cast<size_t>(n_big) ? g * g_big
                                          : n_big * static_cast<size_t>(g_big) +
                                                (g - n_big) * static_cast<size_t>(g_big - 1);
  }
  size_t group_size(size_t g) const { return g < static_cast<size_t>(n_big) ? g_big : g_big - 1; }
  size_t group_of(size_t rt) const {
    const size_t big_rows = static_cast<size_t>(n_big) * g_big;
    return rt < big_rows ? rt / g_big : n_big + (rt - big_rows) / (g_big - 1);
  }
  size_t bytes() const { return row_tiles * k_tiles * tile_bytes; }
  size_t tile_offset(size_t rt, size_t kt) const {
    const size_t g = group_of(rt), r0 = group_row0(g);
    return (r0 * k_tiles + kt * group_size(g) + (rt - r0)) * tile_bytes;
  }
};

constexpr size_t kRowsPerTile = 16;

bool device_scheme_supported(int scheme_id);
DeviceLayout make_device_layout(int scheme_id, size_t rows, size_t cols, size_t padded_cols);
// The plan for (row tiles, k tiles): fills n_groups, g_big, n_big, csplit.
void choose_plan(size_t row_tiles, size_t k_tiles, DeviceLayout* L);

// payload: reference rows [rows][wpr] (row-major). out: layout.bytes() bytes.
void repack_to_device(const DeviceLayout& L, const uint16_t* payload, uint8_t* out, int threads);
// Exact inverse: writes [rows][wpr].
void repack_from_device(const DeviceLayout& L, const uint8_t* in, uint16_t* payload, int threads);

}  // namespace amsqb
