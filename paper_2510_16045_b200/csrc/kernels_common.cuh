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

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>

namespace amsqb {
namespace dev {

constexpr float kPlaceScale = 16384.0f;  // 2^(15 - bias), bias = 1 for e2m2 and e2m3

// Tile geometry families (device_layout.hpp):
//  * family 4: 16 x 64 tiles, 4 m16n8k16 MMAs per k-tile; a lane owns 16 columns of rows g and
//    g+8; A register pairs are columns (j, 4 + j) of an 8-column run (FP4.25's group pairs).
//  * family 7: 16 x 48 tiles, 3 MMAs; a lane owns 12 columns; pairs are (i, i + 3) of a
//    6-column run (FP5.33's word pairs).
struct Fam4 {
  static constexpr int kFam = 4;
  static constexpr int kTK = 64;     // columns per k-tile
  static constexpr int kJ = 4;       // m16n8k16 MMAs per k-tile
  static constexpr int kLaneK = 16;  // columns of one row a lane owns per tile
  // relative column (within the lane's 16) of B slot s of MMA j
  __device__ __forceinline__ static int kofs(int j, int s) { return 4 * s + j; }
};
struct Fam7 {
  static constexpr int kFam = 7;
  static constexpr int kTK = 48;
  static constexpr int kJ = 3;
  static constexpr int kLaneK = 12;
  __device__ __forceinline__ static int kofs(int j, int s) {
    const int o = 2 * j + (s >> 1), p = o / 3, i = o - 3 * p;
    return 6 * p + 3 * (s & 1) + i;
  }
};

template <int SCHEME>
struct Traits;
// kTileBytes = exactly the reference bits of a 16 x kTK tile (no padding); kPlace = 2^(15-bias).
template <> struct Traits<0> : Fam4 { static constexpr int kTileBytes = 512; static constexpr float kPlace = 16384.0f; };  // fp4-e2m1
template <> struct Traits<1> : Fam4 { static constexpr int kTileBytes = 640; static constexpr float kPlace = 16384.0f; };  // fp5-e2m2
template <> struct Traits<2> : Fam4 { static constexpr int kTileBytes = 768; static constexpr float kPlace = 16384.0f; };  // fp6-e2m3
template <> struct Traits<3> : Fam4 { static constexpr int kTileBytes = 768; static constexpr float kPlace = 4096.0f; };   // fp6-e3m2 (bias 3)
template <> struct Traits<4> : Fam4 { static constexpr int kTileBytes = 544; static constexpr float kPlace = 16384.0f; };  // fp4.25-e2m2
template <> struct Traits<5> : Fam7 { static constexpr int kTileBytes = 416; static constexpr float kPlace = 16384.0f; };  // fp4.33-e2m2
template <> struct Traits<6> : Fam4 { static constexpr int kTileBytes = 576; static constexpr float kPlace = 16384.0f; };  // fp4.5-e2m2
template <> struct Traits<7> : Fam7 { static constexpr int kTileBytes = 512; static constexpr float kPlace = 16384.0f; };  // fp5.33-e2m3

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

// Same, for a waiter with nothing else to do (the producer warp): each try_wait may suspend
// the thread for up to `ns` before re-polling, so a long wait does not spin on the issue slots
// the consumer warps of its SM sub-partition need.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t phase, uint32_t ns) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAITS_%=;\n}" ::"r"(a),
      "r"(phase), "r"(ns)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Named barrier among `nthreads` threads (the consumer warps of a warp-specialised CTA).
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

// Ticket for the split-K fix-up: acq_rel at gpu scope orders this CTA's partial stores
// (published to thread 0 by the preceding bar.sync) before the increment, and makes the
// other contributors' partials visible to the last arriver.
__device__ __forceinline__ int atomic_add_acq_rel_gpu(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v)
               : "memory");
  return old;
}

__device__ __forceinline__ void store_relaxed_gpu(int* p, int v) {
  asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Programmatic dependent launch: let the next kernel in the stream start its prologue
// (and its weight stream) as our CTAs retire; wait for the previous kernel's memory
// before touching anything it may have produced (activations, outputs, workspace).
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
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

// L2 prefetch of a contiguous range through the bulk engine (no shared-memory destination).
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// LDGSTS: 16-byte async global -> shared copy; bytes past `src_bytes` are zero-filled.
__device__ __forceinline__ void cp_async_16(void* dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(src_bytes)
               : "memory");
}

// One arrival on `bar` once all of this thread's prior cp.async have landed (the
// barrier's expected count must include it: .noinc).
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// D[16x8,f32] += A[16x16,f16,row] * B[16x8,f16,col]
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  // not volatile: no side effects beyond its outputs, so ptxas may interleave independent
  // MMAs (other accumulators) between dependent ones
  asm(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Output element: fp16 (the reference's y, half.hpp:65-67 RNE) or, for bf16 activations,
// bf16 after undoing the batch row's power-of-two activation scale (exact) -- one rounding.
__device__ __forceinline__ unsigned short out_bits(float v, const float* yscale, int m) {
  if (yscale == nullptr) return __half_as_ushort(__float2half_rn(v));
  return __bfloat16_as_ushort(__float2bfloat16_rn(v * yscale[m]));
}

// ------------------------------------------------------------------ decode
// Explicit LOP3s: (a & b) | c in one ALU op (0xEA), a & b (0x80). Shifts are written as
// multiplies / mul.hi so ptxas can issue them on the FMA pipe (IMAD / IMAD.HI), keeping
// the ALU pipe -- the decode's bottleneck -- for the masks.
__device__ __forceinline__ uint32_t and_or(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t and2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, 0, 0xC0;" : "=r"(d) : "r"(a), "r"(b));  // a & b
  return d;
}
__device__ __forceinline__ uint32_t imul(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("mul.lo.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

// FP4.25: R[0..3] (see device_layout.hpp), sh = the lane's shared byte.
// Output A[j] = the four A-fragment registers of MMA j:
//   {row g pair (k 16t+j, 16t+4+j), row g+8 same, row g (16t+8+j, 16t+12+j), row g+8 same}
// Per register: 7 ALU (LOP3) + 4 FMA-pipe (IMAD) ops for 8 weights.
__device__ __forceinline__ void decode_s4(const uint32_t (&R)[4], uint32_t sh,
                                          uint32_t (&A)[4][4]) {
  const uint32_t T = imul(sh, 0x1001u);  // sh | sh << 12: bit q -> q, bit q+4 -> q+16
  uint32_t o[4][4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    // shared LSBs of groups a, b -> bits 8, 24
    const uint32_t S = and2(imul(T, 1u << (8 - q)), 0x01000100u);
    const uint32_t r = R[q];
    o[q][0] = and_or(r, 0x8E008E00u, S);
    o[q][1] = and_or(imul(r, 8u), 0x8E008E00u, S);
    o[q][2] = and_or(imul(and2(r, 0x20382038u), 68u), 0x8E008E00u, S);   // mag <<6, sign <<2
    o[q][3] = and_or(imul(and2(r, 0x40074007u), 514u), 0x8E008E00u, S);  // mag <<9, sign <<1
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
// Per register: 6 ALU + 3 FMA-pipe ops for 6 weights.
__device__ __forceinline__ void decode_s7(const uint32_t (&R)[4], uint32_t (&A)[3][4]) {
  uint32_t o[4][3];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t r = R[q];
    const uint32_t t5 = __umulhi(r, 1u << 27);  // r >> 5 on the FMA pipe
    const uint32_t S = and2(t5, 0x00800080u);     // shared bits 12/28 -> 7/23
    const uint32_t SM1 = and2(t5, 0x01800180u);   // + member-2 M1 13/29 -> 8/24
    o[q][0] = and_or(r, 0x8F008F00u, S);
    o[q][1] = and_or(imul(r, 256u), 0x8F008F00u, S);
    o[q][2] = and_or(imul(and2(r, 0x40704070u), 34u), 0x8E008E00u, SM1);  // mag-hi <<5, sign <<1
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

// ------------------------------------------------------------------ the other six schemes
// Nibble family (device_layout.hpp): every scheme but FP5.33 stores a 4-bit "top" field per
// weight (s + 3 magnitude bits) plus low bits (a per-weight LSB plane, 2-bit planes, or a
// shared LSB per group of k). A 32-bit register R holds 8 top nibbles -- members i = 0..3 of
// a pair (a: low half, b: high half) -- at the bit positions below, and output i of R is the
// placed fp16x2 (a_i, b_i) = (shift_i(R) & M) | L_i, L_i carrying the low / shared bits.
//   E2 map (mag3 -> bits 9-11, e2m1 / e2m2 / e2m3): mag3<<9,6,3,0; sign @15,12,13,14
//   E3 map (mag3 -> bits 10-12, e3m2):  i=0 mag3<<10 sign@15 | i=1 mag3<<4 sign@9 |
//     i=2 mag3<<0 sign@13 | i=3 e2@3 e0@7 e1@8 sign@14   (each +16 for the high half)
// The multipliers never make two partial products overlap a masked bit (checked exhaustively
// by tests/test_host.py's repack round trips and the GPU restore tests).
template <bool E3>
__device__ __forceinline__ void nib_decode(uint32_t r, const uint32_t (&L)[4], uint32_t (&o)[4]) {
  if constexpr (!E3) {
    constexpr uint32_t M = 0x8E008E00u;
    o[0] = and_or(r, M, L[0]);
    o[1] = and_or(imul(r, 8u), M, L[1]);
    o[2] = and_or(imul(and2(r, 0x20382038u), 68u), M, L[2]);    // mag <<6, sign <<2
    o[3] = and_or(imul(and2(r, 0x40074007u), 514u), M, L[3]);   // mag <<9, sign <<1
  } else {
    constexpr uint32_t M = 0x9C009C00u;
    o[0] = and_or(r, M, L[0]);
    o[1] = and_or(imul(r, 64u), M, L[1]);                         // mag, sign <<6
    o[2] = and_or(imul(and2(r, 0x20072007u), 1028u), M, L[2]);  // mag <<10, sign <<2
    o[3] = and_or(imul(and2(r, 0x41884188u), 522u), M, L[3]);   // e2 <<9, e0/e1 <<3, sign <<1
  }
}

// shift left by s (s >= 0) or right by -s, on the FMA pipe
template <int S>
__device__ __forceinline__ uint32_t shl_signed(uint32_t x) {
  if constexpr (S >= 0) {
    return imul(x, 1u << S);
  } else {
    return __umulhi(x, 1u << (32 + S));
  }
}

// Per-lane data of one tile (the loads are issued before any decode, for ILP).
template <int SCHEME> struct Frag { uint32_t R[4]; uint32_t lo0, lo1; };
template <> struct Frag<5> { uint32_t R[3]; uint32_t lo0, lo1; };

template <int SCHEME>
__device__ __forceinline__ Frag<SCHEME> load_frag(const uint8_t* tile, int lane) {
  Frag<SCHEME> f{};
  if constexpr (SCHEME == 5) {
    const uint2 a = *reinterpret_cast<const uint2*>(tile + lane * 8);
    f.R[0] = a.x, f.R[1] = a.y;
    f.R[2] = *reinterpret_cast<const uint32_t*>(tile + 256 + lane * 4);
    f.lo0 = tile[384 + lane];
  } else {
    const uint4 v = *reinterpret_cast<const uint4*>(tile + lane * 16);
    f.R[0] = v.x, f.R[1] = v.y, f.R[2] = v.z, f.R[3] = v.w;
    if constexpr (SCHEME == 4) f.lo0 = tile[512 + lane];
    if constexpr (SCHEME == 6) f.lo0 = *reinterpret_cast<const unsigned short*>(tile + 512 + lane * 2);
    if constexpr (SCHEME == 1) f.lo0 = *reinterpret_cast<const uint32_t*>(tile + 512 + lane * 4);
    if constexpr (SCHEME == 2 || SCHEME == 3) {
      const uint2 q = *reinterpret_cast<const uint2*>(tile + 512 + lane * 8);
      f.lo0 = q.x, f.lo1 = q.y;
    }
  }
  return f;
}

// Family-4 output order (decode_s4's): A[j] = {o[0][j], o[2][j], o[1][j], o[3][j]}.
__device__ __forceinline__ void fam4_to_A(const uint32_t (&o)[4][4], uint32_t (&A)[4][4]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    A[j][0] = o[0][j];
    A[j][1] = o[2][j];
    A[j][2] = o[1][j];
    A[j][3] = o[3][j];
  }
}

// Low-plane OR-terms of output p (= 4q + i) for the per-weight planes:
//  fp5: P bit p (a) / p+16 (b) -> bits 8 / 24;  fp6: Q_{p/8} bits 2k,2k+1 (a) / +16 (b),
//  k = p % 8 -> bits 7-8 (e2m3) or 8-9 (e3m2).
template <int SCHEME, int P>
__device__ __forceinline__ uint32_t low_term(const Frag<SCHEME>& f) {
  if constexpr (SCHEME == 1) {
    return and2(shl_signed<8 - P>(f.lo0), 0x01000100u);
  } else {
    constexpr int k = P & 7, tgt = SCHEME == 2 ? 7 : 8;
    const uint32_t q = (P >> 3) ? f.lo1 : f.lo0;
    return and2(shl_signed<tgt - 2 * k>(q), SCHEME == 2 ? 0x01800180u : 0x03000300u);
  }
}

template <int SCHEME>
__device__ __forceinline__ void decode_frag(const Frag<SCHEME>& f,
                                            uint32_t (&A)[Traits<SCHEME>::kJ][4]) {
  if constexpr (SCHEME == 7) {
    decode_s7(f.R, A);
  } else if constexpr (SCHEME == 4) {
    decode_s4(f.R, f.lo0, A);
  } else if constexpr (SCHEME == 5) {
    // fp4.33: 12 outputs o_f (f = 4q + i) = pair k = f / 3 (row g: k = 0, 1; row g+8: 2, 3),
    // member f % 3; the shared byte holds group a of pair k at bit k, group b at k + 4
    const uint32_t T = imul(f.lo0, 0x1001u);
    uint32_t S[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) S[k] = and2(imul(T, 1u << (8 - k)), 0x01000100u);
    uint32_t o[3][4];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const uint32_t L[4] = {S[(4 * q) / 3], S[(4 * q + 1) / 3], S[(4 * q + 2) / 3], S[(4 * q + 3) / 3]};
      nib_decode<false>(f.R[q], L, o[q]);
    }
    // decode_s7's order: row g = flat 0..5, row g+8 = flat 6..11
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int a0 = 2 * j, a1 = 2 * j + 1, b0 = 6 + 2 * j, b1 = 7 + 2 * j;
      A[j][0] = o[a0 >> 2][a0 & 3];
      A[j][1] = o[b0 >> 2][b0 & 3];
      A[j][2] = o[a1 >> 2][a1 & 3];
      A[j][3] = o[b1 >> 2][b1 & 3];
    }
  } else {
    uint32_t o[4][4];
    if constexpr (SCHEME == 0) {  // fp4-e2m1: the nibble is the whole code
      const uint32_t L[4] = {0u, 0u, 0u, 0u};
#pragma unroll
      for (int q = 0; q < 4; ++q) nib_decode<false>(f.R[q], L, o[q]);
    } else if constexpr (SCHEME == 6) {  // fp4.5: byte 0 -> members 0,1; byte 1 -> members 2,3
      const uint32_t T0 = imul(and2(f.lo0, 0xFFu), 0x1001u);
      const uint32_t T1 = imul(__umulhi(f.lo0, 1u << 24), 0x1001u);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t S0 = and2(imul(T0, 1u << (8 - q)), 0x01000100u);
        const uint32_t S1 = and2(imul(T1, 1u << (8 - q)), 0x01000100u);
        const uint32_t L[4] = {S0, S0, S1, S1};
        nib_decode<false>(f.R[q], L, o[q]);
      }
    } else {  // fp5 (1), fp6-e2m3 (2), fp6-e3m2 (3): per-weight low planes
      uint32_t L[4][4];
      L[0][0] = low_term<SCHEME, 0>(f);  L[0][1] = low_term<SCHEME, 1>(f);
      L[0][2] = low_term<SCHEME, 2>(f);  L[0][3] = low_term<SCHEME, 3>(f);
      L[1][0] = low_term<SCHEME, 4>(f);  L[1][1] = low_term<SCHEME, 5>(f);
      L[1][2] = low_term<SCHEME, 6>(f);  L[1][3] = low_term<SCHEME, 7>(f);
      L[2][0] = low_term<SCHEME, 8>(f);  L[2][1] = low_term<SCHEME, 9>(f);
      L[2][2] = low_term<SCHEME, 10>(f); L[2][3] = low_term<SCHEME, 11>(f);
      L[3][0] = low_term<SCHEME, 12>(f); L[3][1] = low_term<SCHEME, 13>(f);
      L[3][2] = low_term<SCHEME, 14>(f); L[3][3] = low_term<SCHEME, 15>(f);
#pragma unroll
      for (int q = 0; q < 4; ++q) nib_decode<SCHEME == 3>(f.R[q], L[q], o[q]);
    }
    fam4_to_A(o, A);
  }
}

// ------------------------------------------------------------------ B fragments
// The lane (g, t) holds its LK contiguous activation columns of row g as 16-bit pairs
// w[i] = (x[2i], x[2i+1]); PRMT gathers the pairs each MMA's B slots name
// (Traits::kofs), so x can stay in its natural layout in shared memory.
__device__ __forceinline__ void bfrag_s7(const uint32_t (&w)[6], uint32_t (&B)[3][2]) {
  B[0][0] = prmt(w[0], w[1], 0x7610);  // (x0, x3)
  B[0][1] = prmt(w[0], w[2], 0x5432);  // (x1, x4)
  B[1][0] = prmt(w[1], w[2], 0x7610);  // (x2, x5)
  B[1][1] = prmt(w[3], w[4], 0x7610);  // (x6, x9)
  B[2][0] = prmt(w[3], w[5], 0x5432);  // (x7, x10)
  B[2][1] = prmt(w[4], w[5], 0x7610);  // (x8, x11)
}

__device__ __forceinline__ void bfrag_s4(const uint32_t (&w)[8], uint32_t (&B)[4][2]) {
  B[0][0] = prmt(w[0], w[2], 0x5410);  // (x0, x4)
  B[0][1] = prmt(w[4], w[6], 0x5410);  // (x8, x12)
  B[1][0] = prmt(w[0], w[2], 0x7632);  // (x1, x5)
  B[1][1] = prmt(w[4], w[6], 0x7632);  // (x9, x13)
  B[2][0] = prmt(w[1], w[3], 0x5410);  // (x2, x6)
  B[2][1] = prmt(w[5], w[7], 0x5410);  // (x10, x14)
  B[3][0] = prmt(w[1], w[3], 0x7632);  // (x3, x7)
  B[3][1] = prmt(w[5], w[7], 0x7632);  // (x11, x15)
}

}  // namespace dev
}  // namespace amsqb
