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
constexpr int kConsumerWarps = 8;
constexpr int kK2Threads = (kConsumerWarps + 1) * 32;
constexpr int kChunk = 2;    // k-tiles per stage
constexpr int kStages = 5;   // ring depth (two CTAs per SM share the 227 KB)
constexpr int kCtasPerSM = 2;

template <int SCHEME, int NB>
struct K2Layout {
  using T = Traits<SCHEME>;
  static constexpr int kMS = 8 * NB;
  static constexpr int kWBytes = 16 * kChunk * T::kTileBytes;
  // activation row stride padded so the lanes' LDS hit distinct banks:
  // stride = 96 (mod 128) bytes for the 24-byte FP5.33 lane runs, 16 (mod 128) for FP4.25
  static constexpr int kXRaw = kChunk * T::kTK * 2;
  static constexpr int kXTarget = SCHEME == 7 ? 96 : 16;
  static constexpr int kXRow = kXRaw + ((kXTarget - kXRaw % 128) + 128) % 128;
  static constexpr int kStageBytes = kWBytes + kMS * kXRow;
  static constexpr int kBarOff = kStages * kStageBytes;
  static constexpr int kBytes = kBarOff + 2 * kStages * 8 + 16;
  static_assert(kWBytes % 16 == 0 && kXRow % 16 == 0 && kStageBytes % 16 == 0, "alignment");
};

// Walks a CTA's unit range [u, u1) in chunks that never cross a row block.
struct ChunkIter {
  long long u, u1;
  int rb, kt, KT;
  __device__ ChunkIter(long long u0, long long u1_, int KT_) : u(u0), u1(u1_), KT(KT_) {
    rb = static_cast<int>(u0 / KT_);
    kt = static_cast<int>(u0 - static_cast<long long>(rb) * KT_);
  }
  __device__ bool valid() const { return u < u1; }
  __device__ int nk() const {
    const long long left = u1 - u;
    int n = KT - kt < kChunk ? KT - kt : kChunk;
    return left < n ? static_cast<int>(left) : n;
  }
  __device__ void next() {
    const int n = nk();
    u += n;
    kt += n;
    if (kt == KT) kt = 0, ++rb;
  }
};

__device__ __forceinline__ long long unit_start(long long c, long long U, long long G) {
  return c * U / G;
}
// CTA owning unit u: the largest c with unit_start(c) <= u (G <= U: every range non-empty).
__device__ __forceinline__ long long unit_owner(long long u, long long U, long long G) {
  return ((u + 1) * G - 1) / U;
}

// One k-tile of the consumer loop for a warp's two row tiles: decode, gather the B
// fragments of every batch block from the natural-layout activations, 2*J*NB MMAs.
template <int SCHEME, int NB>
__device__ __forceinline__ void consume_ktile(const uint8_t* st, int kk, const uint4 (&wv)[2],
                                              const uint32_t (&sh)[2], float (&acc)[2][NB][4],
                                              int g, int t, int M) {
  using T = Traits<SCHEME>;
  using LY = K2Layout<SCHEME, NB>;
  constexpr int J = T::kJ;
  uint32_t A[2][J][4];
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const uint32_t R[4] = {wv[rr].x, wv[rr].y, wv[rr].z, wv[rr].w};
    if constexpr (SCHEME == 4) {
      decode_s4(R, sh[rr], A[rr]);
    } else {
      decode_s7(R, A[rr]);
    }
  }
#pragma unroll
  for (int nb = 0; nb < NB; ++nb) {
    const int m = nb * 8 + g;
    const uint8_t* xp = st + LY::kWBytes + m * LY::kXRow + (kk * T::kTK + t * T::kLaneK) * 2;
    uint32_t B[J][2];
    if constexpr (SCHEME == 4) {
      uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      if (m < M) {
        const uint4 a = *reinterpret_cast<const uint4*>(xp);
        const uint4 b = *reinterpret_cast<const uint4*>(xp + 16);
        w[0] = a.x, w[1] = a.y, w[2] = a.z, w[3] = a.w;
        w[4] = b.x, w[5] = b.y, w[6] = b.z, w[7] = b.w;
      }
      bfrag_s4(w, B);
    } else {
      uint32_t w[6] = {0, 0, 0, 0, 0, 0};
      if (m < M) {
        const uint2 a = *reinterpret_cast<const uint2*>(xp);
        const uint2 b = *reinterpret_cast<const uint2*>(xp + 8);
        const uint2 d = *reinterpret_cast<const uint2*>(xp + 16);
        w[0] = a.x, w[1] = a.y, w[2] = b.x, w[3] = b.y, w[4] = d.x, w[5] = d.y;
      }
      bfrag_s7(w, B);
    }
#pragma unroll
    for (int j = 0; j < J; ++j) {
      mma16816(acc[0][nb], A[0][j], B[j][0], B[j][1]);
      mma16816(acc[1][nb], A[1][j], B[j][0], B[j][1]);
    }
  }
}

template <int SCHEME, int NB>
__global__ void __launch_bounds__(kK2Threads, kCtasPerSM) amsq_linear_kernel(LinearParams p) {
  using T = Traits<SCHEME>;
  using LY = K2Layout<SCHEME, NB>;
  constexpr int J = T::kJ;
  constexpr int TILE = T::kTileBytes;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + LY::kBarOff);
  uint64_t* empty = full + kStages;
  int* flag = reinterpret_cast<int*>(empty + kStages);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long U = static_cast<long long>(p.row_blocks) * p.k_tiles;
  const long long G = gridDim.x;
  const long long c = blockIdx.x;
  const long long u0 = unit_start(c, U, G), u1 = unit_start(c + 1, U, G);
  const int KT = p.k_tiles;
  unsigned long long* trace = p.trace ? p.trace + blockIdx.x * 8 : nullptr;
  if (trace && threadIdx.x == 0) trace[0] = globaltimer();

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1 + 32);  // expect_tx arrival + one per producer lane
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // ------------------------------------------------------------ producer warp
    // lane 0: one bulk copy of the stage's 16*nk weight tiles (contiguous in the
    // [row_block][k_tile][row_tile] layout); all lanes: the activation rows with 16-byte
    // LDGSTS (zero-filled past `cols`), each lane arriving once on the full barrier.
    const uint64_t pol = policy_evict_first();
    const bool x_vec = ((p.cols & 7) == 0) && ((p.ldx & 7) == 0) &&
                       ((reinterpret_cast<uintptr_t>(p.x) & 15) == 0);
    constexpr int kXUnits = kChunk * T::kTK * 2 / 16;  // 16-byte units per activation row
    ChunkIter it(u0, u1, KT);
    for (int i = 0; it.valid(); ++i, it.next()) {
      const int s = i % kStages;
      if (i >= kStages) mbar_wait(&empty[s], static_cast<uint32_t>((i / kStages) - 1) & 1u);
      const int nk = it.nk();
      uint8_t* st = smem + s * LY::kStageBytes;
      const long long k0 = static_cast<long long>(it.kt) * T::kTK;
      if (lane == 0) {
        fence_proxy_async_smem();
        const uint32_t wbytes = static_cast<uint32_t>(16 * nk * TILE);
        mbar_arrive_expect_tx(&full[s], wbytes);
        bulk_g2s(st, p.w + (static_cast<long long>(it.rb) * KT + it.kt) * 16LL * TILE, wbytes,
                 &full[s], pol);
      }
      const int units = p.M * kXUnits;
      if (x_vec) {
        for (int u = lane; u < units; u += 32) {
          const int m = u / kXUnits, q = u - m * kXUnits;
          const long long k = k0 + q * 8;
          const long long left = p.cols - k;
          const uint32_t nbytes = left >= 8 ? 16u : (left > 0 ? static_cast<uint32_t>(left) * 2u : 0u);
          const unsigned short* src = p.x + m * p.ldx + (nbytes ? k : 0);
          cp_async_16(st + LY::kWBytes + m * LY::kXRow + q * 16, src, nbytes);
        }
        cp_async_mbar_arrive(&full[s]);
      } else {  // unaligned activations: plain loads, then a regular arrival
        for (int u = lane; u < p.M * kChunk * T::kTK; u += 32) {
          const int m = u / (kChunk * T::kTK), e = u - m * (kChunk * T::kTK);
          unsigned short* xr = reinterpret_cast<unsigned short*>(st + LY::kWBytes + m * LY::kXRow);
          xr[e] = (k0 + e < p.cols) ? __ldg(p.x + m * p.ldx + k0 + e) : static_cast<unsigned short>(0);
        }
        __threadfence_block();
        mbar_arrive(&full[s]);
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumer warps
  const int g = lane >> 2, t = lane & 3;
  float acc[2][NB][4];
  auto zero_acc = [&] {
#pragma unroll
    for (int rr = 0; rr < 2; ++rr)
#pragma unroll
      for (int nb = 0; nb < NB; ++nb)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[rr][nb][e] = 0.0f;
  };
  zero_acc();
  int cur_rb = -1, seg_kt0 = 0, seg_kt1 = 0;
  constexpr int kCons = kConsumerWarps * 32;

  auto finish_segment = [&](int rb) {
    const int rib0 = 32 * warp;
    if (seg_kt0 == 0 && seg_kt1 == KT) {  // this CTA covered the whole K range
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
      return;
    }
    constexpr int MS = 8 * NB;
    const long long pid = c + rb;
    float* part = p.partials + pid * MS * 256;
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
    named_bar_sync(1, kCons);  // all partial stores of this CTA happen-before thread 0's ticket
    const long long c_first = unit_owner(static_cast<long long>(rb) * KT, U, G);
    const long long c_last = unit_owner(static_cast<long long>(rb + 1) * KT - 1, U, G);
    if (threadIdx.x == 0) {
      const int ncontrib = static_cast<int>(c_last - c_first + 1);
      const int old = atomic_add_acq_rel_gpu(&p.counters[rb], 1);
      const int last = (old == ncontrib - 1);
      if (last) store_relaxed_gpu(&p.counters[rb], 0);  // self-cleaning for the next launch
      *flag = last;
    }
    named_bar_sync(1, kCons);
    if (*flag) {
      // Sum the contributors' partials in CTA order (deterministic). All loads of a batch
      // are issued before any add so the L2 latency is paid once per batch, not per term.
      const int ncon = static_cast<int>(c_last - c_first + 1);
      const float4* base = reinterpret_cast<const float4*>(p.partials + (c_first + rb) * MS * 256);
      constexpr int kB = 8;
      for (int o = threadIdx.x; o < p.M * 64; o += kCons) {
        const int m = o >> 6, q = o & 63;
        float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int c0 = 0; c0 < ncon; c0 += kB) {
          float4 v[kB];
#pragma unroll
          for (int j = 0; j < kB; ++j) {
            v[j] = (c0 + j < ncon) ? __ldcg(base + ((c0 + j) * MS + m) * 64 + q)
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
          for (int j = 0; j < kB; ++j) {
            if (c0 + j < ncon) {
              sum.x += v[j].x, sum.y += v[j].y, sum.z += v[j].z, sum.w += v[j].w;
            }
          }
        }
        const float r4[4] = {sum.x, sum.y, sum.z, sum.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const long long n = static_cast<long long>(rb) * 256 + 4 * q + e;
          if (n < p.rows) {
            const float sc = __half2float(__ushort_as_half(p.scales[n])) * kPlaceScale;
            p.y[static_cast<long long>(m) * p.ldy + n] = __half_as_ushort(__float2half_rn(r4[e] * sc));
          }
        }
      }
    }
    named_bar_sync(1, kCons);
  };

  ChunkIter it(u0, u1, KT);
  for (int i = 0; it.valid(); ++i, it.next()) {
    const int s = i % kStages;
    const int nk = it.nk();
    if (it.rb != cur_rb) {
      if (cur_rb >= 0) finish_segment(cur_rb);
      zero_acc();
      cur_rb = it.rb;
      seg_kt0 = it.kt;
    }
    seg_kt1 = it.kt + nk;
    mbar_wait(&full[s], static_cast<uint32_t>(i / kStages) & 1u);
    if (trace && i == 0 && threadIdx.x == 0) trace[1] = globaltimer();
    const uint8_t* st = smem + s * LY::kStageBytes;
    const uint8_t* wt = st + (2 * warp) * TILE + lane * 16;  // stage: [kk][16 row tiles]
    if (p.dry) {
      // profiling mode: stream only
    } else if (nk == kChunk) {
      // common case: guard-free, fully unrolled so loads of later k-tiles overlap the
      // decode/MMA of earlier ones
      uint4 wv[kChunk][2];
      uint32_t sh[kChunk][2];
#pragma unroll
      for (int kk = 0; kk < kChunk; ++kk)
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          const uint8_t* tp = wt + (kk * 16 + rr) * TILE;
          wv[kk][rr] = *reinterpret_cast<const uint4*>(tp);
          sh[kk][rr] = SCHEME == 4 ? tp[512 - lane * 16 + lane] : 0u;
        }
#pragma unroll
      for (int kk = 0; kk < kChunk; ++kk) consume_ktile<SCHEME, NB>(st, kk, wv[kk], sh[kk], acc, g, t, p.M);
    } else {
      for (int kk = 0; kk < nk; ++kk) {
        uint4 wv[2];
        uint32_t sh[2];
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          const uint8_t* tp = wt + (kk * 16 + rr) * TILE;
          wv[rr] = *reinterpret_cast<const uint4*>(tp);
          sh[rr] = SCHEME == 4 ? tp[512 - lane * 16 + lane] : 0u;
        }
        consume_ktile<SCHEME, NB>(st, kk, wv, sh, acc, g, t, p.M);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if (trace && threadIdx.x == 0) trace[2] = globaltimer();
  if (cur_rb >= 0) finish_segment(cur_rb);
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

template <int SCHEME, int NB>
static cudaError_t launch_linear_t(const LinearParams& p, int grid, cudaStream_t s) {
  using SM = dev::K2Layout<SCHEME, NB>;
  static bool configured = false;  // per template instance; attribute is per-function
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(dev::amsq_linear_kernel<SCHEME, NB>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, SM::kBytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  dev::amsq_linear_kernel<SCHEME, NB><<<grid, dev::kK2Threads, SM::kBytes, s>>>(p);
  count_launch();
  return cudaGetLastError();
}

int linear_max_batch_per_launch() { return 16; }

long long linear_grid(long long units) { return units < kGridCTAs ? units : kGridCTAs; }

cudaError_t launch_linear(const LinearParams& p, cudaStream_t s) {
  const long long units = static_cast<long long>(p.row_blocks) * p.k_tiles;
  const int grid = static_cast<int>(linear_grid(units));
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
