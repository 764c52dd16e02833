// kernels.cu -- sm_100a kernels of the AMS-Quant weight-only linear.
//
//  K1 amsq_restore_kernel   restore_block / restore_matrix(_half) over the tile layout
//                           (kernels.hpp:55-133 of the reference), bit-exact.
//  K2 amsq_linear_kernel    fused restore + linear for batch M <= 16 (kernels.hpp:151-187):
//                           stream-K over (256-row block x k-tile) units, one persistent
//                           CTA per SM, 8 warps x 2 row tiles, packed tiles streamed by the
//                           TMA bulk engine into a per-warp mbarrier ring, decode in
//                           registers, m16n8k16 tensor-core MMAs with fp32 accumulation,
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
  const int rt = static_cast<int>(tile / p.k_tiles), kt = static_cast<int>(tile % p.k_tiles);
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
// K2: fused restore + linear, M <= 8*NB.
// =====================================================================================
constexpr int kWarps = 8;        // each warp: 2 row tiles = 32 rows; CTA: 256-row block
constexpr int kChunk = 4;        // k-tiles per pipeline stage
constexpr int kStages = 4;       // ring depth per warp
constexpr int kXWin = 16;        // k-tiles of activations staged per window

template <int SCHEME, int NB>
struct K2Smem {
  using T = Traits<SCHEME>;
  static constexpr int kMS = 8 * NB;
  static constexpr int kStageBytes = 2 * kChunk * T::kTileBytes;
  static constexpr int kRingBytes = kWarps * kStages * kStageBytes;
  static constexpr int kXsBytes = kXWin * T::kJ * kMS * 4 * 8;
  static constexpr int kBarOff = kRingBytes + kXsBytes;
  static constexpr int kBytes = kBarOff + kWarps * kStages * 8 + 16;
};

// Walks the CTA's unit range [u, u1) in chunks that never cross a row block.
struct ChunkIter {
  long long u, u1;
  int KT;
  __device__ bool valid() const { return u < u1; }
  __device__ void get(int& rb, int& kt, int& nk) const {
    rb = static_cast<int>(u / KT);
    kt = static_cast<int>(u - static_cast<long long>(rb) * KT);
    const long long seg_end = min(u1, static_cast<long long>(rb + 1) * KT);
    nk = static_cast<int>(min(static_cast<long long>(kChunk), seg_end - u));
  }
  __device__ void next() {
    int rb, kt, nk;
    get(rb, kt, nk);
    u += nk;
  }
};

__device__ __forceinline__ long long unit_start(long long c, long long U, long long G) {
  return c * U / G;
}
// CTA owning unit u: the largest c with unit_start(c) <= u (G <= U: every range non-empty).
__device__ __forceinline__ long long unit_owner(long long u, long long U, long long G) {
  return ((u + 1) * G - 1) / U;
}

template <int SCHEME, int NB>
__global__ void __launch_bounds__(kWarps * 32, 1) amsq_linear_kernel(LinearParams p) {
  using T = Traits<SCHEME>;
  using SM = K2Smem<SCHEME, NB>;
  constexpr int J = T::kJ;
  constexpr int MS = SM::kMS;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* ring = smem;
  uint2* xs = reinterpret_cast<uint2*>(smem + SM::kRingBytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::kBarOff);
  int* flag = reinterpret_cast<int*>(smem + SM::kBarOff + kWarps * kStages * 8);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const long long U = static_cast<long long>(p.row_blocks) * p.k_tiles;
  const long long G = gridDim.x;
  const long long c = blockIdx.x;
  const long long u0 = unit_start(c, U, G), u1 = unit_start(c + 1, U, G);
  const int KT = p.k_tiles;

  uint64_t* mybars = bars + warp * kStages;
  uint8_t* myring = ring + warp * kStages * SM::kStageBytes;
  if (lane == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&mybars[s], 1);
    fence_barrier_init();
  }
  __syncwarp();
  const uint64_t pol = policy_evict_first();

  // producer: lane 0 streams this warp's two row tiles of each chunk
  auto issue = [&](const ChunkIter& it, int stage) {
    int rb, kt, nk;
    it.get(rb, kt, nk);
    const int rt0 = rb * 16 + 2 * warp;
    const uint32_t bytes = static_cast<uint32_t>(nk * T::kTileBytes);
    uint8_t* dst = myring + stage * SM::kStageBytes;
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&mybars[stage], 2 * bytes);
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const uint8_t* src =
          p.w + (static_cast<long long>(rt0 + rr) * KT + kt) * static_cast<long long>(T::kTileBytes);
      bulk_g2s(dst + rr * kChunk * T::kTileBytes, src, bytes, &mybars[stage], pol);
    }
  };

  ChunkIter prod{u0, u1, KT}, cons{u0, u1, KT};
  if (lane == 0) {
    for (int s = 0; s < kStages && prod.valid(); ++s) {
      issue(prod, s);
      prod.next();
    }
  }

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

  int stage = 0;
  uint32_t phase = 0;
  int cur_rb = -1, seg_kt0 = 0, seg_kt1 = 0;
  int xw_lo = 0, xw_hi = 0;  // staged activation window [lo, hi) in k-tiles

  // Stage x[:, xw_lo*TK .. xw_hi*TK) permuted into the B-fragment order, zero padded.
  auto stage_x = [&](int lo) {
    __syncthreads();
    xw_lo = lo;
    xw_hi = min(lo + kXWin, KT);
    const int nkt = xw_hi - xw_lo;
    const int nunits = nkt * MS * 4;  // (ktl, m, t): one lane chunk of TK/4 columns
    for (int idx = threadIdx.x; idx < nunits; idx += blockDim.x) {
      const int tt = idx & 3;
      const int m = (idx >> 2) % MS;
      const int ktl = (idx >> 2) / MS;
      const long long kbase = static_cast<long long>(xw_lo + ktl) * T::kTK + tt * T::kLaneK;
      __half v[T::kLaneK];
      const bool live = m < p.M;
      const unsigned short* xr = p.x + static_cast<long long>(m) * p.ldx;
#pragma unroll
      for (int e = 0; e < T::kLaneK; ++e) {
        const long long k = kbase + e;
        v[e] = (live && k < p.cols) ? __ushort_as_half(__ldg(xr + k)) : __ushort_as_half(0);
      }
#pragma unroll
      for (int j = 0; j < J; ++j) {
        __half2 lo2 = __halves2half2(v[T::kofs(j, 0)], v[T::kofs(j, 1)]);
        __half2 hi2 = __halves2half2(v[T::kofs(j, 2)], v[T::kofs(j, 3)]);
        uint2 u;
        u.x = *reinterpret_cast<uint32_t*>(&lo2);
        u.y = *reinterpret_cast<uint32_t*>(&hi2);
        xs[((ktl * J + j) * MS + m) * 4 + tt] = u;
      }
    }
    __syncthreads();
  };

  // End of a row-block segment: direct store when this CTA covered the whole K range,
  // otherwise publish a partial and let the last contributor reduce in CTA order.
  auto finish_segment = [&](int rb) {
    const bool full = (seg_kt0 == 0 && seg_kt1 == KT);
    const int rib0 = 32 * warp;  // row-in-block of this warp's first row tile
    if (full) {
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
    __threadfence();
    __syncthreads();
    const long long c_first = unit_owner(static_cast<long long>(rb) * KT, U, G);
    const long long c_last = unit_owner(static_cast<long long>(rb + 1) * KT - 1, U, G);
    if (threadIdx.x == 0) {
      const int ncontrib = static_cast<int>(c_last - c_first + 1);
      const int old = atomicAdd(&p.counters[rb], 1);
      const int last = (old == ncontrib - 1);
      if (last) {
        __threadfence();
        p.counters[rb] = 0;  // self-cleaning for the next launch / graph replay
      }
      *flag = last;
    }
    __syncthreads();
    if (*flag) {
      for (int idx = threadIdx.x; idx < p.M * 256; idx += blockDim.x) {
        const int m = idx >> 8, rib = idx & 255;
        const long long n = static_cast<long long>(rb) * 256 + rib;
        if (n >= p.rows) continue;
        float s = 0.0f;
        for (long long cc = c_first; cc <= c_last; ++cc) {
          s += __ldcg(p.partials + ((cc + rb) * MS + m) * 256 + rib);
        }
        const float sc = __half2float(__ushort_as_half(p.scales[n])) * kPlaceScale;
        p.y[static_cast<long long>(m) * p.ldy + n] = __half_as_ushort(__float2half_rn(s * sc));
      }
    }
    __syncthreads();
  };

  while (cons.valid()) {
    int rb, kt, nk;
    cons.get(rb, kt, nk);
    if (rb != cur_rb) {
      if (cur_rb >= 0) finish_segment(cur_rb);
      zero_acc();
      cur_rb = rb;
      seg_kt0 = kt;
    }
    seg_kt1 = kt + nk;
    if (kt < xw_lo || kt + nk > xw_hi) stage_x(kt);

    mbar_wait(&mybars[stage], phase);
    const uint8_t* sbase = myring + stage * SM::kStageBytes;
    for (int kk = 0; kk < nk; ++kk) {
      uint32_t A[2][J][4];
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        const uint8_t* tp = sbase + (rr * kChunk + kk) * T::kTileBytes;
        const uint4 v = *reinterpret_cast<const uint4*>(tp + lane * 16);
        const uint32_t R[4] = {v.x, v.y, v.z, v.w};
        if constexpr (SCHEME == 4) {
          decode_s4(R, tp[512 + lane], A[rr]);
        } else {
          decode_s7(R, A[rr]);
        }
      }
      const int ktl = kt + kk - xw_lo;
#pragma unroll
      for (int j = 0; j < J; ++j) {
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) {
          const uint2 b = xs[((ktl * J + j) * MS + nb * 8 + g) * 4 + t];
          mma16816(acc[0][nb], A[0][j], b.x, b.y);
          mma16816(acc[1][nb], A[1][j], b.x, b.y);
        }
      }
    }
    __syncwarp();
    if (lane == 0 && prod.valid()) {
      issue(prod, stage);
      prod.next();
    }
    if (++stage == kStages) {
      stage = 0;
      phase ^= 1u;
    }
    cons.next();
  }
  if (cur_rb >= 0) finish_segment(cur_rb);
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
  using SM = dev::K2Smem<SCHEME, NB>;
  static bool configured = false;  // per template instance; attribute is per-function
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(dev::amsq_linear_kernel<SCHEME, NB>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, SM::kBytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  dev::amsq_linear_kernel<SCHEME, NB><<<grid, dev::kWarps * 32, SM::kBytes, s>>>(p);
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
