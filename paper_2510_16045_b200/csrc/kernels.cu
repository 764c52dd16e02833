// kernels.cu -- sm_100a kernels of the AMS-Quant weight-only linear.
//
//  K1 amsq_restore_kernel   restore_block / restore_matrix(_half) over the tile layout
//                           (kernels.hpp:55-133 of the reference), bit-exact.
//  K2 amsq_linear_kernel    fused restore + linear for batch M <= 32 per launch
//                           (kernels.hpp:151-187): k2.cuh, one translation unit per scheme
//                           (k2_s<id>.cu); launch_linear below dispatches on the scheme.
//  bf16 activation staging, and the TP unshard permutation.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <type_traits>
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
  // tiles are enumerated in storage order [group][k_tile][row_tile_in_group]
  const GroupPlan& P = p.plan;
  const long long KT = p.k_tiles;
  const long long big_tiles = static_cast<long long>(P.n_big) * P.g_big * KT;
  long long G, grp, rem;
  if (tile < big_tiles) {
    G = P.g_big;
    grp = tile / (G * KT);
    rem = tile - grp * G * KT;
  } else {
    G = P.g_big - 1;
    const long long t2 = tile - big_tiles;
    grp = P.n_big + t2 / (G * KT);
    rem = t2 - (grp - P.n_big) * G * KT;
  }
  const int kt = static_cast<int>(rem / G);
  const int rt = P.row0(static_cast<int>(grp)) + static_cast<int>(rem - kt * G);
  const uint8_t* src = p.w + tile * T::kTileBytes;
  const Frag<SCHEME> fr = load_frag<SCHEME>(src, lane);
  const __half2 k2 = __floats2half2_rn(T::kPlace, T::kPlace);
  auto put = [&](uint32_t placed, int row, int klo, int khi) {
    __half2 h = *reinterpret_cast<const __half2*>(&placed);
    h = __hmul2(h, k2);  // exact: every grid value is a binary16 normal or zero
    tile_s[warp][row][klo] = __low2half(h);
    tile_s[warp][row][khi] = __high2half(h);
  };
  uint32_t A[T::kJ][4];
  decode_frag<SCHEME>(fr, A);
  if constexpr (T::kFam == 4) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      put(A[j][0], g, 16 * t + j, 16 * t + 4 + j);
      put(A[j][1], g + 8, 16 * t + j, 16 * t + 4 + j);
      put(A[j][2], g, 16 * t + 8 + j, 16 * t + 12 + j);
      put(A[j][3], g + 8, 16 * t + 8 + j, 16 * t + 12 + j);
    }
  } else {
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

}  // namespace dev

// =====================================================================================
// launchers
// =====================================================================================
namespace {

int restore_ntiles(const RestoreParams& p) { return p.row_tiles * p.k_tiles; }

}  // namespace

cudaError_t launch_restore(const RestoreParams& p, cudaStream_t s) {
  const long long ntiles = restore_ntiles(p);
  const unsigned blocks = static_cast<unsigned>((ntiles + 3) / 4);
  if (blocks == 0) return cudaSuccess;
  switch (p.scheme_id) {
    case 0: dev::amsq_restore_kernel<0><<<blocks, 128, 0, s>>>(p); break;
    case 1: dev::amsq_restore_kernel<1><<<blocks, 128, 0, s>>>(p); break;
    case 2: dev::amsq_restore_kernel<2><<<blocks, 128, 0, s>>>(p); break;
    case 3: dev::amsq_restore_kernel<3><<<blocks, 128, 0, s>>>(p); break;
    case 4: dev::amsq_restore_kernel<4><<<blocks, 128, 0, s>>>(p); break;
    case 5: dev::amsq_restore_kernel<5><<<blocks, 128, 0, s>>>(p); break;
    case 6: dev::amsq_restore_kernel<6><<<blocks, 128, 0, s>>>(p); break;
    case 7: dev::amsq_restore_kernel<7><<<blocks, 128, 0, s>>>(p); break;
    default: return cudaErrorInvalidValue;
  }
  count_launch();
  return cudaGetLastError();
}

// Stage geometry for a plan: wr = smallest power of two with ceil(G / wr) <= 4 row tiles
// per consumer warp, S = 16 / wr k-tiles per stage (so a stage is <= 64 tiles, ~32 KB),
// as many ring stages as fit (<= 6).
int linear_max_batch_per_launch() { return AMSQ_K2_MAX_BATCH; }

cudaError_t launch_linear(const LinearParams& p, cudaStream_t s) {  // NOLINT
  switch (p.scheme_id) {
    case 0: return launch_linear_scheme<0>(p, s);
    case 1: return launch_linear_scheme<1>(p, s);
    case 2: return launch_linear_scheme<2>(p, s);
    case 3: return launch_linear_scheme<3>(p, s);
    case 4: return launch_linear_scheme<4>(p, s);
    case 5: return launch_linear_scheme<5>(p, s);
    case 6: return launch_linear_scheme<6>(p, s);
    case 7: return launch_linear_scheme<7>(p, s);
    default: return cudaErrorInvalidValue;
  }
}

// bf16 activations (the reference itself is fp16-only, half.hpp). One
// block per batch row: the row's largest |x| is brought into [2^14, 2^15) by 2^e, and every
// x * 2^e is rounded to fp16 -- exact for all |x| 2^e >= 2^-17 (bf16 has 8 significant bits,
// fp16 11 down to 2^-14 and fewer in its subnormals), so the fp16 kernels multiply the same
// numbers up to a power of two. yscale[m] = 2^-e undoes it in the epilogue, before the one
// rounding to bf16.
__global__ void __launch_bounds__(256) amsq_x_bf16_prep_kernel(const unsigned short* __restrict__ x,
                                                              long long ldx, long long cols,
                                                              unsigned short* __restrict__ xh,
                                                              float* __restrict__ yscale) {
  dev::pdl_launch_dependents();
  dev::pdl_wait();
  const int m = blockIdx.x;
  const unsigned short* xr = x + m * ldx;
  float mx = 0.0f;
  for (long long i = threadIdx.x; i < cols; i += blockDim.x) {
    mx = fmaxf(mx, fabsf(__bfloat162float(__ushort_as_bfloat16(xr[i]))));
  }
  __shared__ float red[8];
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = red[0];
  for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) mx = fmaxf(mx, red[w]);
  int e = 0;
  if (mx > 0.0f && mx <= 3.0e38f) {
    int ex;
    frexpf(mx, &ex);  // mx in [2^(ex-1), 2^ex)
    e = 15 - ex;
  }
  for (long long i = threadIdx.x; i < cols; i += blockDim.x) {
    const float v = __bfloat162float(__ushort_as_bfloat16(xr[i]));
    xh[m * cols + i] = __half_as_ushort(__float2half_rn(ldexpf(v, e)));
  }
  if (threadIdx.x == 0) yscale[m] = ldexpf(1.0f, -e);
}

cudaError_t launch_x_bf16_prep(const unsigned short* x, long long ldx, long long cols, int M,
                               unsigned short* xh, float* yscale, cudaStream_t s) {
  if (M <= 0) return cudaSuccess;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(M));
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, amsq_x_bf16_prep_kernel, x, ldx, cols, xh, yscale);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

// Fused-TP flag barrier: thread r < nranks publishes this rank's epoch into rank r's flags
// and then waits for rank r's epoch here. Release/acquire at system scope order the K2 peer
// stores (fenced at the end of every K2 CTA) before the flag, and the flag before any later
// read of the gathered output on this GPU.
__global__ void amsq_tp_barrier_kernel(unsigned int* const* __restrict__ peer_flags,
                                       unsigned int* __restrict__ my_flags,
                                       unsigned int* __restrict__ epoch,
                                       unsigned int* __restrict__ error, int rank, int nranks,
                                       unsigned long long timeout_ns) {
  dev::pdl_wait();  // the K2 launches before us have finished (and fenced) their stores
  const unsigned int e = *epoch + 1u;
  const int r = threadIdx.x;
  if (r < nranks) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(peer_flags[r] + rank), "r"(e) : "memory");
    const unsigned long long t0 = dev::globaltimer();
    unsigned int v;
    for (;;) {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(my_flags + r) : "memory");
      if (static_cast<int>(v - e) >= 0) break;
      if (dev::globaltimer() - t0 > timeout_ns) {
        atomicExch(error, 1u);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) *epoch = e;
}

cudaError_t launch_tp_barrier(unsigned int* const* peer_flags, unsigned int* my_flags,
                              unsigned int* epoch, unsigned int* error, int rank, int nranks,
                              unsigned long long timeout_ns, cudaStream_t s) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(static_cast<unsigned>((nranks + 31) / 32 * 32));
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, amsq_tp_barrier_kernel, peer_flags, my_flags, epoch,
                                           error, rank, nranks, timeout_ns);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
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
