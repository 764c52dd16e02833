// kernels_common.cuh -- sm_100a device helpers for the AMS-Quant kernels:
// mbarrier + cp.async.bulk (TMA bulk engine), mma.sync fragments, and the in-register
// decode of the tile layout (device_layout.hpp) into "placed" binary16 pairs.
//
// Placement (SURVEY.md §7 hard part 2): for a code with exponent field E and mantissa
// field M (m bits), the binary16 pattern sign<<15 | (E|M) << (10-m) equals
// decode(code) * 2^-(15-bias) exactly -- fp16 subnormals included -- so the kernels
// feed these patterns straight to the tensor cores and fold 2^(15-bias) = 2^14
// (both shipped formats have bias 1) into the per-row fp32 scale.
#pragma once

#include <cuda_fp16.h>
#include <cstdint>

namespace amsqb {
namespace dev {

constexpr float kPlaceScale = 16384.0f;  // 2^(15 - bias), bias = 1 for e2m2 and e2m3

template <int SCHEME>
struct Traits;

template <>
struct Traits<4> {                 // FP4.25-e2m2, k = 4
  static constexpr int kTK = 64;   // columns per k-tile (= one reference block)
  static constexpr int kJ = 4;     // m16n8k16 MMAs per k-tile
  static constexpr int kTileBytes = 544;
  static constexpr int kLaneK = 16;  // columns of one row a lane owns per tile
  // relative column (within the lane's 16) of B slot s of MMA j
  __device__ __forceinline__ static int kofs(int j, int s) { return 4 * s + j; }
};

template <>
struct Traits<7> {                 // FP5.33-e2m3, k = 3
  static constexpr int kTK = 48;   // 16 reference words per row
  static constexpr int kJ = 3;
  static constexpr int kTileBytes = 512;
  static constexpr int kLaneK = 12;
  __device__ __forceinline__ static int kofs(int j, int s) {
    const int o = 2 * j + (s >> 1), p = o / 3, i = o - 3 * p;
    return 6 * p + 3 * (s & 1) + i;
  }
};

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(a),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// TMA bulk engine: global -> shared, completion counted on `bar` in bytes.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// D[16x8,f32] += A[16x16,f16,row] * B[16x8,f16,col]
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// ------------------------------------------------------------------ decode
// FP4.25: R[0..3] (see device_layout.hpp), sh = the lane's shared byte.
// Output A[j] = the four A-fragment registers of MMA j:
//   {row g pair (k 16t+j, 16t+4+j), row g+8 same, row g (16t+8+j, 16t+12+j), row g+8 same}
__device__ __forceinline__ void decode_s4(const uint32_t (&R)[4], uint32_t sh,
                                          uint32_t (&A)[4][4]) {
  const uint32_t T = sh * 0x1001u;  // sh | sh << 12: bit q -> q, bit q+4 -> q+16
  uint32_t o[4][4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t S = (T << (8 - q)) & 0x01000100u;  // shared LSBs of groups a, b -> bits 8, 24
    const uint32_t r = R[q];
    o[q][0] = (r & 0x8E008E00u) | S;
    o[q][1] = ((r << 3) & 0x8E008E00u) | S;
    o[q][2] = (((r & 0x20382038u) * 68u) & 0x8E008E00u) | S;   // mag <<6, sign <<2
    o[q][3] = (((r & 0x40074007u) * 514u) & 0x8E008E00u) | S;  // mag <<9, sign <<1
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    A[j][0] = o[0][j];
    A[j][1] = o[2][j];
    A[j][2] = o[1][j];
    A[j][3] = o[3][j];
  }
}

// FP5.33: A[j] for MMA j in {0,1,2}; row-g outputs in order
// [R0.o0, R0.o1, R0.o2, R1.o0, R1.o1, R1.o2], MMA j takes entries 2j, 2j+1.
__device__ __forceinline__ void decode_s7(const uint32_t (&R)[4], uint32_t (&A)[3][4]) {
  uint32_t o[4][3];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t r = R[q];
    const uint32_t t5 = r >> 5;
    const uint32_t S = t5 & 0x00800080u;     // shared bits 12/28 -> 7/23
    const uint32_t SM1 = t5 & 0x01800180u;   // + member-2 M1 13/29 -> 8/24
    o[q][0] = (r & 0x8F008F00u) | S;
    o[q][1] = ((r << 8) & 0x8F008F00u) | S;
    o[q][2] = (((r & 0x40704070u) * 34u) & 0x8E008E00u) | SM1;  // mag-hi <<5, sign <<1
  }
  const uint32_t g0[6] = {o[0][0], o[0][1], o[0][2], o[1][0], o[1][1], o[1][2]};
  const uint32_t g8[6] = {o[2][0], o[2][1], o[2][2], o[3][0], o[3][1], o[3][2]};
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    A[j][0] = g0[2 * j];
    A[j][1] = g8[2 * j];
    A[j][2] = g0[2 * j + 1];
    A[j][3] = g8[2 * j + 1];
  }
}

}  // namespace dev
}  // namespace amsqb
