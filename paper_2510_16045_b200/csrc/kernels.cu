// kernels.cu -- sm_100a kernels of the AMS-Quant weight-only linear.
//
//  K1 amsq_restore_kernel   restore_block / restore_matrix(_half) over the tile layout
//                           (kernels.hpp:55-133 of the reference), bit-exact.
//  K2 amsq_linear_kernel    fused restore + linear for batch M <= 16 (kernels.hpp:151-187):
//                           warp-specialised persistent CTA per SM (TMA-bulk producer warp,
//                           8 decode/MMA consumer warps), stream-K over (256-row block x
//                           k-tile) units, m16n8k16 tensor-core MMAs with fp32 accumulation,
//                           deterministic split-K fix-up (fixed order, no float atomics).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "kernels.h"
#include "kernels_common.cuh"

namespace amsqb {

static std::atomic<uint64_t> g_launches{0};
uint64_t kernel_launch_count() { return g_launches.load(); }
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

namespace dev {

// =====================================================================================
// K1: restore. One warp per tile; decode to placed fp16, rescale by 2^14 (exact in
// binary16), stage the 16 x TK tile in shared memory, write rows out coalesced.
// =====================================================================================
template <int SCHEME>
__global__ void __launch_bounds__(128) amsq_restore_kernel(RestoreParams p) {
  using T = Traits<SCHEME>;
  constexpr int TK = T::kTK;
  __shared__ __half tile_s[4][16][TK + 2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const long long tile = static_cast<long long>(blockIdx.x) * 4 + warp;
  const long long ntiles = static_cast<long long>(p.row_tiles) * p.k_tiles;
  if (tile >= ntiles) return;
  // tiles are enumerated in storage order [row_block][k_tile][row_tile_in_block]
  const long long rbk = tile / 16;
  const int rt = static_cast<int>(rbk / p.k_tiles) * 16 + static_cast<int>(tile % 16);
  const int kt = static_cast<int>(rbk % p.k_tiles);
  const uint8_t* src = p.w + tile * T::kTileBytes;
  const uint4 v = *reinterpret_cast<const uint4*>(src + lane * 16);
  const uint32_t R[4] = {v.x, v.y, v.z, v.w};
  const __half2 k2 = __floats2half2_rn(kPlaceScale, kPlaceScale);
  auto put = [&](uint32_t placed, int row, int klo, int khi) {
    __half2 h = *reinterpret_cast<const __half2*>(&placed);
    h = __hmul2(h, k2);  // exact: every grid value is a binary16 normal or zero
    tile_s[warp][row][klo] = __low2half(h);
    tile_s[warp][row][khi] = __high2half(h);
  };
  if constexpr (SCHEME == 4) {
    uint32_t A[4][4];
    decode_s4(R, src[512 + lane], A);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      put(A[j][0], g, 16 * t + j, 16 * t + 4 + j);
      put(A[j][1], g + 8, 16 * t + j, 16 * t + 4 + j);
      put(A[j][2], g, 16 * t + 8 + j, 16 * t + 12 + j);
      put(A[j][3], g + 8, 16 * t + 8 + j, 16 * t + 12 + j);
    }
  } else {
    uint32_t A[3][4];
    decode_s7(R, A);
#pragma unroll
    for (int j = 0; j < 3; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int o = 2 * j + h, pp = o / 3, i = o - 3 * pp;
        const int klo = 12 * t + 6 * pp + i, khi = klo + 3;
        put(A[j][2 * h], g, klo, khi);
        put(A[j][2 * h + 1], g + 8, klo, khi);
      }
    }
  }
  __syncwarp();
  const int k0 = kt * TK;
  for (int idx = lane; idx < 16 * TK; idx += 32) {
    const int r = idx / TK, c = idx - r * TK;
    const long long n = static_cast<long long>(rt) * 16 + r;
    const int k = k0 + c;
    if (n >= p.rows) continue;
    const __half h = tile_s[warp][r][c];
    if (p.grid_out && k < p.padded_cols) {
      p.grid_out[n * p.padded_cols + k] = __half_as_ushort(h);
    }
    if (k < p.cols && (p.f32_out || p.f16_out)) {
      const float ws = __half2float(h) * __half2float(__ushort_as_half(p.scales[n]));
      if (p.f32_out) p.f32_out[n * p.cols + k] = ws;
      if (p.f16_out) p.f16_out[n * p.cols + k] = __half_as_ushort(__float2half_rn(ws));
    }
  }
}

// =====================================================================================
// Activation prep for K2: x[M][cols] (fp16, row stride ldx) -> B-fragment units
// xp[kt][j][m][t] (8 bytes: the two fp16 pairs lane t of an m16n8k16 MMA j reads for batch
// row m), zero for m >= M and k >= cols. One thread per (k-tile, row, lane-column) item.
// =====================================================================================
template <int SCHEME>
__global__ void __launch_bounds__(256) amsq_xprep_kernel(const unsigned short* __restrict__ x,
                                                         long long ldx, long long cols, int M,
                                                         int MS, int KT, uint2* __restrict__ xp) {
  using T = Traits<SCHEME>;
  constexpr int J = T::kJ, LK = T::kLaneK, LW = LK / 2;
  pdl_launch_dependents();
  pdl_wait();  // x is produced by the previous kernel in the stream
  const int items = KT * MS * 4;
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < items; u += gridDim.x * blockDim.x) {
    const int kt = u / (MS * 4), r = u - kt * MS * 4, m = r >> 2, t = r & 3;
    const long long k = static_cast<long long>(kt) * T::kTK + t * LK;
    uint32_t w[LW];
#pragma unroll
    for (int i = 0; i < LW; ++i) {
      unsigned lo = 0, hi = 0;
      if (m < M) {
        if (k + 2 * i < cols) lo = __ldg(x + m * ldx + k + 2 * i);
        if (k + 2 * i + 1 < cols) hi = __ldg(x + m * ldx + k + 2 * i + 1);
      }
      w[i] = lo | hi << 16;
    }
    uint32_t B[J][2];
    if constexpr (SCHEME == 4) {
      bfrag_s4(w, B);
    } else {
      bfrag_s7(w, B);
    }
#pragma unroll
    for (int j = 0; j < J; ++j) {
      xp[((static_cast<long long>(kt) * J + j) * MS + m) * 4 + t] = make_uint2(B[j][0], B[j][1]);
    }
  }
}

// =====================================================================================
// K2: fused restore + linear, M <= 8*NB (NB = 1 or 2).
//
// Warp-specialised persistent CTA (one per SM): warp 8 is the producer -- its lane 0
// streams, per pipeline stage, kChunk k-tiles of the CTA's 16 row tiles (one
// cp.async.bulk per row tile) plus the matching activation rows (natural layout, one
// bulk copy per batch row, zero-filled past `cols`) into a 4-deep ring guarded by
// full/empty mbarriers. Warps 0..7 are consumers: warp w owns row tiles 2w, 2w+1,
// decodes its 16 B per tile in registers, gathers B fragments with PRMT and issues
// m16n8k16 MMAs (fp32 accumulation). Units are (256-row block, k-tile) pairs split
// evenly over the grid (stream-K); a row block cut between CTAs is finished by the
// last contributor, which sums the fp32 partials in CTA order (deterministic).
// =====================================================================================
constexpr int kGroupWarps = 8;                   // a consumer group covers a 256-row block
constexpr int kGroups = 2;                       // groups split every stage's k-tiles
constexpr int kConsumerWarps = kGroups * kGroupWarps;
constexpr int kK2Threads = (kConsumerWarps + 1) * 32;  // + the producer warp
constexpr int kChunk = 4;    // k-tiles per stage: 32-35 KB bulk copies (>= 16 KB, tools/tma_probe.cu)
constexpr int kGroupK = kChunk / kGroups;        // k-tiles of a stage each group consumes
constexpr int kMaxStages = 5;  // ring depth (fewer when the stage is large, see K2Layout);
                               // a <= 113 KB variant that lets PDL successors co-reside was
                               // measured slower (too few bytes in flight)

// One CTA per SM: co-resident CTAs were measured to starve each other at the warp arbiter
// (the lower-priority CTA finishes ~40% later), so each SM runs a single CTA whose two
// consumer groups each take half of every stage's k-tiles (balanced at segment ends).
template <int SCHEME, int NB>
struct K2Layout {
  using T = Traits<SCHEME>;
  static constexpr int kMS = 8 * NB;
  static constexpr int kWBytes = 16 * kChunk * T::kTileBytes;
  // Activations of a stage. M <= 8 (NB = 1): natural row-major rows loaded by LDGSTS, the
  // row stride padded so the lanes' LDS hit distinct banks (96 (mod 128) bytes for the
  // 24-byte FP5.33 lane runs, 16 (mod 128) for FP4.25) and B fragments gathered with PRMT.
  // M <= 16 (NB = 2): B-fragment-order units ((kk * J + j) * MS + m) * 4 + t written by
  // amsq_xprep_kernel and bulk-copied, one conflict-free LDS.64 per MMA.
  static constexpr bool kXPrep = NB == 2;
  static constexpr int kXRaw = kChunk * T::kTK * 2;
  static constexpr int kXTarget = SCHEME == 7 ? 96 : 16;
  static constexpr int kXRow = kXRaw + ((kXTarget - kXRaw % 128) + 128) % 128;
  static constexpr int kXBytes = kXPrep ? kChunk * T::kJ * kMS * 4 * 8 : kMS * kXRow;
  static constexpr int kStageBytes = kWBytes + kXBytes;
  static constexpr int kScratchBytes = kGroupWarps * 32 * 2 * NB * 4 * 4;
  static constexpr int kFit = (227 * 1024 - kScratchBytes - 1024) / kStageBytes;
  static constexpr int kStages = kFit < kMaxStages ? kFit : kMaxStages;
  static constexpr int kScratchOff = kStages * kStageBytes;  // group-1 accumulators
  static constexpr int kBarOff = kScratchOff + kScratchBytes;
  static constexpr int kBytes = kBarOff + 2 * kStages * 8 + 16;
  static_assert(kWBytes % 16 == 0 && kStageBytes % 16 == 0, "alignment");
  static_assert(kBytes <= 227 * 1024, "shared memory budget");
};

// Units are (256-row block, k-tile) pairs, u = rb * KT + kt; CTA c owns [start(c), start(c+1)).
__device__ __forceinline__ int unit_start(int c, int U, int G) {
  return static_cast<int>(static_cast<long long>(c) * U / G);
}
// CTA owning unit u: the largest c with unit_start(c) <= u (G <= U: every range non-empty).
__device__ __forceinline__ int unit_owner(int u, int U, int G) {
  return static_cast<int>((static_cast<long long>(u + 1) * G - 1) / U);
}

// One k-tile of the consumer loop for a warp's two row tiles: decode, gather the B
// fragments of every batch block from the natural-layout activations, 2*J*NB MMAs.
// Activation rows >= M are zero in shared memory, so the loads are unpredicated.
template <int SCHEME, int NB, int MODE = 0>  // MODE (profiling): 1 = no MMA, 2 = no decode
__device__ __forceinline__ void consume_ktile(const uint8_t* st, int kk, const uint4 (&wv)[2],
                                              const uint32_t (&sh)[2], float (&acc)[2][NB][4],
                                              int g, int t) {
  using T = Traits<SCHEME>;
  using LY = K2Layout<SCHEME, NB>;
  constexpr int J = T::kJ;
  uint32_t A[2][J][4];
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const uint32_t R[4] = {wv[rr].x, wv[rr].y, wv[rr].z, wv[rr].w};
    if constexpr (MODE == 2) {
#pragma unroll
      for (int j = 0; j < J; ++j)
#pragma unroll
        for (int q = 0; q < 4; ++q) A[rr][j][q] = R[(j + q) & 3] & 0x3F003F00u;
    } else if constexpr (SCHEME == 4) {
      decode_s4(R, sh[rr], A[rr]);
    } else {
      decode_s7(R, A[rr]);
    }
  }
#pragma unroll
  for (int nb = 0; nb < NB; ++nb) {
    uint32_t B[J][2];
    if constexpr (LY::kXPrep) {
      const uint2* xs = reinterpret_cast<const uint2*>(st + LY::kWBytes) +
                        ((kk * J) * LY::kMS + nb * 8 + g) * 4 + t;
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const uint2 b = xs[j * LY::kMS * 4];
        B[j][0] = b.x;
        B[j][1] = b.y;
      }
    } else {
      const uint8_t* xp =
          st + LY::kWBytes + (nb * 8 + g) * LY::kXRow + (kk * T::kTK + t * T::kLaneK) * 2;
      if constexpr (SCHEME == 4) {
        const uint4 a = *reinterpret_cast<const uint4*>(xp);
        const uint4 b = *reinterpret_cast<const uint4*>(xp + 16);
        const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        bfrag_s4(w, B);
      } else {
        const uint2 a = *reinterpret_cast<const uint2*>(xp);
        const uint2 b = *reinterpret_cast<const uint2*>(xp + 8);
        const uint2 d = *reinterpret_cast<const uint2*>(xp + 16);
        const uint32_t w[6] = {a.x, a.y, b.x, b.y, d.x, d.y};
        bfrag_s7(w, B);
      }
    }
#pragma unroll
    for (int j = 0; j < J; ++j) {
      if constexpr (MODE == 1) {  // keep the decode live without the tensor pipe
        acc[0][nb][j & 3] += __uint_as_float((A[0][j][0] ^ A[0][j][1] ^ A[0][j][2] ^ A[0][j][3] ^ B[j][0]) & 0x3F0F0F0Fu);
        acc[1][nb][j & 3] += __uint_as_float((A[1][j][0] ^ A[1][j][1] ^ A[1][j][2] ^ A[1][j][3] ^ B[j][1]) & 0x3F0F0F0Fu);
      } else {
        mma16816(acc[0][nb], A[0][j], B[j][0], B[j][1]);
        mma16816(acc[1][nb], A[1][j], B[j][0], B[j][1]);
      }
    }
  }
}

template <int SCHEME, int NB, int MODE>
__global__ void __launch_bounds__(kK2Threads, 1) amsq_linear_kernel(LinearParams p) {
  using T = Traits<SCHEME>;
  using LY = K2Layout<SCHEME, NB>;
  constexpr int TILE = T::kTileBytes;
  constexpr int MS = 8 * NB;
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int kStages = LY::kStages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + LY::kBarOff);
  uint64_t* empty = full + kStages;
  float* scratch = reinterpret_cast<float*>(smem + LY::kScratchOff);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KT = p.k_tiles;
  const int U = p.row_blocks * KT;
  const int G = gridDim.x;
  const int c = blockIdx.x;
  const int u0 = unit_start(c, U, G), u1 = unit_start(c + 1, U, G);
  const int rb_first = u0 / KT, rb_last = (u1 - 1) / KT;
  unsigned long long* trace = p.trace ? p.trace + blockIdx.x * 8 : nullptr;
  if (trace && threadIdx.x == 0) trace[0] = globaltimer();
  pdl_launch_dependents();

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      // the producer's arrive.expect_tx, plus one LDGSTS arrival per producer lane when the
      // activations are loaded in natural layout
      mbar_init(&full[s], LY::kXPrep ? 1 : 1 + 32);
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_barrier_init();
  }
  // natural-layout activation rows >= M are never written by the producer: zero them once
  if constexpr (!LY::kXPrep) {
    for (int s = 0; s < kStages; ++s) {
      uint4* xz = reinterpret_cast<uint4*>(smem + s * LY::kStageBytes + LY::kWBytes + p.M * LY::kXRow);
      const int n16 = (MS - p.M) * LY::kXRow / 16;
      for (int i = threadIdx.x; i < n16; i += blockDim.x) xz[i] = make_uint4(0, 0, 0, 0);
    }
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // ------------------------------------------------------------ producer warp
    // lane 0, per stage: one bulk copy of the 16*nk weight tiles (contiguous in the
    // [row_block][k_tile][row_tile] layout). Activations: NB = 2 -> one more bulk copy of the
    // prepped B-fragment units; NB = 1 -> all lanes LDGSTS the natural rows (zero-filled
    // past `cols`), each lane arriving once on the full barrier when its copies land.
    const uint64_t pol = policy_evict_first();
    constexpr uint32_t kXTileBytes = T::kJ * MS * 4 * 8;
    const bool x_vec = ((p.cols & 7) == 0) && ((p.ldx & 7) == 0) &&
                       ((reinterpret_cast<uintptr_t>(p.x) & 15) == 0);
    constexpr int kXUnits = kChunk * T::kTK * 2 / 16;  // 16-byte units per activation row
    const int units = p.M * kXUnits;
    int stage = 0;
    uint32_t phase = 0;
    bool waited = false;
    for (int rb = rb_first; rb <= rb_last; ++rb) {
      const int kt0 = rb == rb_first ? u0 - rb * KT : 0;
      const int kt1 = rb == rb_last ? u1 - rb * KT : KT;
      for (int kt = kt0; kt < kt1; kt += kChunk) {
        const int nk = min(kChunk, kt1 - kt);
        mbar_wait(&empty[stage], phase ^ 1u);
        uint8_t* st = smem + stage * LY::kStageBytes;
        uint64_t* fb = &full[stage];
        const uint32_t wbytes = static_cast<uint32_t>(16 * nk * TILE);
        const uint32_t xbytes =
            (LY::kXPrep && p.dry != 4) ? static_cast<uint32_t>(nk) * kXTileBytes : 0u;
        if (lane == 0) {
          fence_proxy_async_smem();
          mbar_arrive_expect_tx(fb, wbytes + xbytes);
          bulk_g2s(st, p.w + (static_cast<long long>(rb) * KT + kt) * 16LL * TILE, wbytes, fb,
                   pol);
        }
        if (!waited) {  // weights are independent of the previous kernel; activations not
          pdl_wait();
          waited = true;
        }
        if constexpr (LY::kXPrep) {
          if (lane == 0 && xbytes) {
            bulk_g2s(st + LY::kWBytes,
                     reinterpret_cast<const uint8_t*>(p.xperm) +
                         static_cast<long long>(kt) * kXTileBytes,
                     xbytes, fb, policy_evict_last());
          }
        } else {
          const long long k0 = static_cast<long long>(kt) * T::kTK;
          if (p.dry == 4) {  // profiling: stream weights only
            mbar_arrive(fb);
          } else if (x_vec) {
            for (int u = lane; u < units; u += 32) {
              const int m = u / kXUnits, q = u - m * kXUnits;
              const long long k = k0 + q * 8;
              const long long left = p.cols - k;
              const uint32_t nb =
                  left >= 8 ? 16u : (left > 0 ? static_cast<uint32_t>(left) * 2u : 0u);
              cp_async_16(st + LY::kWBytes + m * LY::kXRow + q * 16,
                          p.x + m * p.ldx + (nb ? k : 0), nb);
            }
            cp_async_mbar_arrive(fb);
          } else {  // unaligned activations: plain loads, then a regular arrival
            for (int u = lane; u < p.M * kChunk * T::kTK; u += 32) {
              const int m = u / (kChunk * T::kTK), e = u - m * (kChunk * T::kTK);
              unsigned short* xr =
                  reinterpret_cast<unsigned short*>(st + LY::kWBytes + m * LY::kXRow);
              xr[e] = (k0 + e < p.cols) ? __ldg(p.x + m * p.ldx + k0 + e)
                                        : static_cast<unsigned short>(0);
            }
            __threadfence_block();
            mbar_arrive(fb);
          }
        }
        if (++stage == kStages) stage = 0, phase ^= 1u;
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumer warps
  // group gr = warp / 8 consumes the stages of parity gr (chunks 2j + gr of the CTA's
  // sequence); warp wg = warp % 8 owns row tiles 2wg, 2wg+1 of the 256-row block.
  const int gr = warp / kGroupWarps, wg = warp % kGroupWarps;
  const int g = lane >> 2, t = lane & 3;
  constexpr int kCons = kConsumerWarps * 32;
  float acc[2][NB][4];
  bool waited = false;

  // End of a row-block segment: group 1 hands its accumulators to group 0 through shared
  // memory (sum order g0 + g1: deterministic). Group 0 then either stores y (the CTA
  // covered the whole K range) or publishes its 32-row slice as an fp32 partial and takes a
  // ticket on the slice's counter (release; result consumed after the main loop, when the
  // last contributor of a slice reduces it in CTA order).
  int pend_rb0 = -1, pend_t0 = 0, pend_rb1 = -1, pend_t1 = 0;
  const int rib0 = 32 * wg;
  float* my_scratch = scratch + (wg * 32 + lane) * (2 * NB * 4);
  auto finish_segment = [&](int rb, bool full_k) {
    if (!waited) {  // outputs / workspace may still be in use by the previous kernel
      pdl_wait();
      waited = true;
    }
    if (gr == 1) {
#pragma unroll
      for (int rr = 0; rr < 2; ++rr)
#pragma unroll
        for (int nb = 0; nb < NB; ++nb)
#pragma unroll
          for (int e = 0; e < 4; ++e) my_scratch[(rr * NB + nb) * 4 + e] = acc[rr][nb][e];
    }
    named_bar_sync(1, kCons);
    if (gr == 0) {
#pragma unroll
      for (int rr = 0; rr < 2; ++rr)
#pragma unroll
        for (int nb = 0; nb < NB; ++nb)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[rr][nb][e] += my_scratch[(rr * NB + nb) * 4 + e];
      if (full_k) {
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const long long n = static_cast<long long>(rb) * 256 + rib0 + rr * 16 + g + 8 * h;
            if (n >= p.rows) continue;
            const float sc = __half2float(__ushort_as_half(p.scales[n])) * kPlaceScale;
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) {
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int m = nb * 8 + 2 * t + e;
                if (m < p.M) {
                  p.y[static_cast<long long>(m) * p.ldy + n] =
                      __half_as_ushort(__float2half_rn(acc[rr][nb][2 * h + e] * sc));
                }
              }
            }
          }
        }
      } else {
        float* part = p.partials + (static_cast<long long>(c) + rb) * MS * 256;
#pragma unroll
        for (int rr = 0; rr < 2; ++rr)
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int nb = 0; nb < NB; ++nb)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int m = nb * 8 + 2 * t + e;
                part[m * 256 + rib0 + rr * 16 + g + 8 * h] = acc[rr][nb][2 * h + e];
              }
        __syncwarp();  // the warp's partial stores happen-before lane 0's release
        int ticket = 0;
        if (lane == 0) ticket = atomic_add_acq_rel_gpu(&p.counters[rb * kGroupWarps + wg], 1);
        if (pend_rb0 < 0) {
          pend_rb0 = rb, pend_t0 = ticket;
        } else {
          pend_rb1 = rb, pend_t1 = ticket;
        }
      }
    }
    named_bar_sync(1, kCons);  // scratch free for the next segment
  };

  // Deferred reduction of a 32-row slice whose partials are all published: the slice is
  // M x 8 float4 outputs, each the CTA-ordered sum of ncon partials. Every lane issues the
  // loads of all its (output, contributor) pairs before adding, four contributors at a time.
  auto reduce_slice = [&](int rb) {
    const int c_first = unit_owner(rb * KT, U, G);
    const int ncon = unit_owner((rb + 1) * KT - 1, U, G) - c_first + 1;
    const float4* base = reinterpret_cast<const float4*>(
        p.partials + (static_cast<long long>(c_first) + rb) * MS * 256 + rib0);
    const int nout = p.M * 8;  // outputs of the slice (<= 128): lane owns o = lane + 32 i
    float4 sum[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) sum[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int c0 = 0; c0 < ncon; c0 += 4) {  // 16 independent loads in flight per lane
      float4 v[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int o = lane + 32 * i;
          v[i][j] = (o < nout && c0 + j < ncon)
                        ? __ldcg(base + ((c0 + j) * MS + (o >> 3)) * 64 + (o & 7))
                        : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (c0 + j < ncon) {  // contributor order c0, c0+1, ... : deterministic
            sum[i].x += v[i][j].x, sum[i].y += v[i][j].y, sum[i].z += v[i][j].z,
                sum[i].w += v[i][j].w;
          }
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int o = lane + 32 * i;
      if (o >= nout) continue;
      const int m = o >> 3, q = o & 7;
      const float r4[4] = {sum[i].x, sum[i].y, sum[i].z, sum[i].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const long long n = static_cast<long long>(rb) * 256 + rib0 + 4 * q + e;
        if (n < p.rows) {
          const float sc = __half2float(__ushort_as_half(p.scales[n])) * kPlaceScale;
          p.y[static_cast<long long>(m) * p.ldy + n] = __half_as_ushort(__float2half_rn(r4[e] * sc));
        }
      }
    }
  };

  int stage = 0;
  uint32_t phase = 0;
  bool first = true;
  const uint8_t* wlane = smem + (2 * wg) * TILE + lane * 16;  // + stage base; [kk][16 row tiles]
  const int kkb = gr * kGroupK;  // this group's k-tiles of each stage: kkb .. kkb + kGroupK - 1
  for (int rb = rb_first; rb <= rb_last; ++rb) {
    const int kt0 = rb == rb_first ? u0 - rb * KT : 0;
    const int kt1 = rb == rb_last ? u1 - rb * KT : KT;
#pragma unroll
    for (int rr = 0; rr < 2; ++rr)
#pragma unroll
      for (int nb = 0; nb < NB; ++nb)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[rr][nb][e] = 0.0f;
    for (int kt = kt0; kt < kt1; kt += kChunk) {
      const int nk = min(kChunk, kt1 - kt);
      mbar_wait(&full[stage], phase);
      if (trace && first && threadIdx.x == 0) trace[1] = globaltimer();
      first = false;
      const uint8_t* st = smem + stage * LY::kStageBytes;
      const uint8_t* wt = wlane + stage * LY::kStageBytes;
      if (p.dry == 1 || p.dry == 4) {
        // profiling mode: stream only
      } else if (nk == kChunk) {
        // common case: guard-free and fully unrolled so the loads of the second k-tile
        // overlap the decode/MMA of the first
        uint4 wv[kGroupK][2];
        uint32_t sh[kGroupK][2];
#pragma unroll
        for (int i = 0; i < kGroupK; ++i)
#pragma unroll
          for (int rr = 0; rr < 2; ++rr) {
            const uint8_t* tp = wt + ((kkb + i) * 16 + rr) * TILE;
            wv[i][rr] = *reinterpret_cast<const uint4*>(tp);
            sh[i][rr] = SCHEME == 4 ? tp[512 - lane * 16 + lane] : 0u;
          }
#pragma unroll
        for (int i = 0; i < kGroupK; ++i)
          consume_ktile<SCHEME, NB, MODE>(st, kkb + i, wv[i], sh[i], acc, g, t);
      } else {
        for (int kk = kkb; kk < min(nk, kkb + kGroupK); ++kk) {
          uint4 wv[2];
          uint32_t sh[2];
#pragma unroll
          for (int rr = 0; rr < 2; ++rr) {
            const uint8_t* tp = wt + (kk * 16 + rr) * TILE;
            wv[rr] = *reinterpret_cast<const uint4*>(tp);
            sh[rr] = SCHEME == 4 ? tp[512 - lane * 16 + lane] : 0u;
          }
          consume_ktile<SCHEME, NB, MODE>(st, kk, wv, sh, acc, g, t);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == kStages) stage = 0, phase ^= 1u;
    }
    if (trace && rb == rb_last && threadIdx.x == 0) trace[2] = globaltimer();
    finish_segment(rb, kt0 == 0 && kt1 == KT);
  }
  // Slices this warp completed last: reduce them (the acquire in the ticket makes the other
  // contributors' partials visible to lane 0; __syncwarp extends that to the warp).
  if (gr == 0) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int rb = i == 0 ? pend_rb0 : pend_rb1;
      if (rb < 0) continue;
      const int ticket = i == 0 ? pend_t0 : pend_t1;
      const int ncon = unit_owner((rb + 1) * KT - 1, U, G) - unit_owner(rb * KT, U, G) + 1;
      const int last = __shfl_sync(0xffffffffu, ticket == ncon - 1 ? 1 : 0, 0);
      __syncwarp();
      if (last) {
        if (lane == 0) store_relaxed_gpu(&p.counters[rb * kGroupWarps + wg], 0);
        reduce_slice(rb);
      }
    }
  }
  if (trace && threadIdx.x == 0) trace[3] = globaltimer();
}

}  // namespace dev

// =====================================================================================
// launchers
// =====================================================================================
cudaError_t launch_restore(const RestoreParams& p, cudaStream_t s) {
  const long long ntiles = static_cast<long long>(p.row_tiles) * p.k_tiles;
  const unsigned blocks = static_cast<unsigned>((ntiles + 3) / 4);
  if (blocks == 0) return cudaSuccess;
  if (p.scheme_id == 4) {
    dev::amsq_restore_kernel<4><<<blocks, 128, 0, s>>>(p);
  } else {
    dev::amsq_restore_kernel<7><<<blocks, 128, 0, s>>>(p);
  }
  count_launch();
  return cudaGetLastError();
}

template <int SCHEME, int NB, int MODE>
static cudaError_t launch_linear_m(const LinearParams& p, int grid, cudaStream_t s) {
  using SM = dev::K2Layout<SCHEME, NB>;
  static bool configured = false;  // per template instance; attribute is per-function
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(dev::amsq_linear_kernel<SCHEME, NB, MODE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, SM::kBytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(dev::kK2Threads);
  cfg.dynamicSmemBytes = SM::kBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, dev::amsq_linear_kernel<SCHEME, NB, MODE>, p);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <int SCHEME, int NB>
static cudaError_t launch_linear_t(const LinearParams& p, int grid, cudaStream_t s) {
  if constexpr (NB == 2) {
  // activations first (PDL-chained: waits for whoever produced x, lets the linear start
  // streaming weights as soon as it is scheduled)
  const int MS = 8 * NB;
  const int items = p.k_tiles * MS * 4;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>((items + 255) / 256));
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, dev::amsq_xprep_kernel<SCHEME>, p.x, p.ldx, p.cols,
                                     p.M, MS, p.k_tiles, p.xperm);
  count_launch();
  if (e != cudaSuccess) return e;
  }
  if (p.dry == 2) return launch_linear_m<SCHEME, NB, 1>(p, grid, s);  // profiling: no MMA
  if (p.dry == 3) return launch_linear_m<SCHEME, NB, 2>(p, grid, s);  // profiling: no decode
  return launch_linear_m<SCHEME, NB, 0>(p, grid, s);
}

int linear_max_batch_per_launch() { return 16; }

long long linear_grid(long long units, int /*M*/) { return units < kSMs ? units : kSMs; }

cudaError_t launch_linear(const LinearParams& p, cudaStream_t s) {  // NOLINT
  const long long units = static_cast<long long>(p.row_blocks) * p.k_tiles;
  const int grid = static_cast<int>(linear_grid(units, p.M));
  if (grid <= 0) return cudaSuccess;
  if (p.scheme_id == 4) {
    return p.M <= 8 ? launch_linear_t<4, 1>(p, grid, s) : launch_linear_t<4, 2>(p, grid, s);
  }
  return p.M <= 8 ? launch_linear_t<7, 1>(p, grid, s) : launch_linear_t<7, 2>(p, grid, s);
}

// [P][batch][n] -> [batch][P*n]
__global__ void amsq_unshard_kernel(const unsigned short* __restrict__ in, int P, int batch, int n,
                                    unsigned short* __restrict__ out) {
  const long long total = static_cast<long long>(P) * batch * n;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = i / n, col = i - r * n;
    const long long pp = r / batch, b = r - pp * batch;
    out[b * (static_cast<long long>(P) * n) + pp * n + col] = in[i];
  }
}

cudaError_t launch_unshard(const unsigned short* in, int P, int batch, int n, unsigned short* out,
                           cudaStream_t s) {
  const long long total = static_cast<long long>(P) * batch * n;
  const int blocks = static_cast<int>(total < 148LL * 256 * 8 ? (total + 255) / 256 : 148 * 8);
  if (blocks == 0) return cudaSuccess;
  amsq_unshard_kernel<<<blocks, 256, 0, s>>>(in, P, batch, n, out);
  count_launch();
  return cudaGetLastError();
}

}  // namespace amsqb
