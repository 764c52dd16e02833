// kernels_tc.cu -- K3: fused restore + linear on the 5th-generation tensor cores
// (tcgen05.mma, TMEM accumulators) for large batches (16 < M <= 256 per launch), where the
// linear stops being HBM-bound (crossover M ~ 56 / 70).
//
// Swap-AB: D[128 weight rows][Np batch] += W[128 x K] . X^T[K x Np], D in TMEM (128 lanes x
// Np fp32 columns), one CTA per 128-row block (8 row tiles of the tile layout).
//  * warps 0..15 ("decode"): two per row tile (even / odd k-tiles of each stage); each reads
//    its tiles from the stage's weight buffer, decodes in registers (the same decode_s4 /
//    decode_s7 as K2) and stores the placed fp16 pairs into the stage's A buffer in the UMMA
//    canonical K-major no-swizzle layout [k/8][128 rows][8]; fence.proxy.async + one
//    mbarrier arrival per warp.
//  * warp 16 ("producer"): per stage, bulk copies of the block's weight tiles (one per row
//    group segment, see below) and of the activation image (prepped once per call by
//    amsq_xprep_tc_kernel into the same [k/8][Np][8] layout); owns the TMEM allocation.
//  * warp 17 ("MMA"): one elected thread issues tcgen05.mma.cta_group::1.kind::f16 (M=128,
//    N=Np, K=16) per 16 columns and tcgen05.commit's the stage back to the producers.
//  * epilogue (warps 0..7): tcgen05.ld 32x32b -> fp32 * scale * 2^14 -> fp16 y; a cluster of
//    2/4 CTAs that split K sums its TMEM partials through DSMEM first.
// The decode emits a lane's fp16 pairs in its own order, so the K axis is permuted inside
// every tile column chunk (tc_kperm); the activation prep applies the same permutation, so
// the contraction is unchanged. Accumulation order: k ascending per MMA -- deterministic.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <type_traits>

#include "kernels.h"
#include "kernels_common.cuh"

namespace amsqb {

void count_launch();

namespace dev {

#ifndef AMSQ_TC_KC4_MIN_STAGES  // fewest ring stages for which 4 k-tiles per stage are taken
#define AMSQ_TC_KC4_MIN_STAGES 3
#endif
#ifndef AMSQ_TC_BIG_STAGES  // 1: also try 8 and 6 k-tiles per stage (>= 2 stages)
#define AMSQ_TC_BIG_STAGES 1
#endif
#ifndef AMSQ_TC_ATMEM  // 1: the decoded A operand lives in TMEM (tcgen05.st); 0: shared memory
#define AMSQ_TC_ATMEM 1
#endif

// Natural column (within a k-tile) of logical K position p of the decoded A operand.
//  * A in TMEM: decode warp lane (g, t) stores MMA j's fragment {A0, A2, A1, A3} with
//    tcgen05.st.16x256b (measured map, tools/tmem_probe.cu: register r -> TMEM lane g + 8 (r >> 1),
//    column 2t + (r & 1)), and the MMA reads column c as K = 2c, 2c + 1. So K position
//    L = p mod 16 of MMA j = p / 16 is lane t = L / 4's mma.sync slot s = 2 ((L / 2) & 1) + (L & 1),
//    i.e. natural column t * kLaneK + kofs(j, s) -- the B-fragment columns of K2 (bfrag_s4/_s7).
//  * A in shared memory: a lane (g, t) covers columns [12t, 12t + 12) (FP5.33) / [16t, 16t + 16)
//    (FP4.25) of its rows and emits them as the pairs of decode_s7 / decode_s4.
template <int SCHEME>
__device__ __forceinline__ int tc_kperm(int p) {
#if AMSQ_TC_ATMEM
  using T = Traits<SCHEME>;
  const int j = p >> 4, L = p & 15;
  return (L >> 2) * T::kLaneK + T::kofs(j, ((L >> 1) & 1) * 2 + (L & 1));
#else
  if constexpr (SCHEME == 7) {
    const int t = p / 12, r = p - 12 * t;
    const int q = r / 6, i = (r - 6 * q) >> 1, h = r & 1;
    return 3 * (4 * t + 2 * q + h) + i;
  } else {
    const int t = p >> 4, r = p & 15;
    const int q = r >> 3, j = (r & 7) >> 1, h = r & 1;
    return 16 * t + 8 * q + 4 * h + j;
  }
#endif
}

// x[M][ldx] -> xk[KTOT/8][Np][8] (the UMMA no-swizzle K-major image), K permuted per tile.
// nh = 2 (CTA pairs): two images [2][KTOT/8][Np/2][8], one per CTA of a pair (its N half).
template <int SCHEME>
__global__ void __launch_bounds__(256) amsq_xprep_tc_kernel(const unsigned short* __restrict__ x,
                                                            long long ldx, long long cols, int M,
                                                            int Np, int KT, int nh,
                                                            unsigned short* __restrict__ xk) {
  constexpr int TK = Traits<SCHEME>::kTK;
  pdl_launch_dependents();
  pdl_wait();  // x is produced by the previous kernel in the stream
  const long long total = static_cast<long long>(KT) * TK * Np;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int Nh = Np / nh;
    const long long g8 = e / (8LL * Nh);                // (half, k8) flattened
    const int rem = static_cast<int>(e - g8 * 8LL * Nh);
    const long long hk = static_cast<long long>(KT) * TK / 8;
    const int h = static_cast<int>(g8 / hk);
    const long long grp = g8 - h * hk;
    const int m = h * Nh + (rem >> 3), kk = rem & 7;
    const long long kp = grp * 8 + kk;                // permuted column
    const long long kt = kp / TK;
    const long long k = kt * TK + tc_kperm<SCHEME>(static_cast<int>(kp - kt * TK));
    xk[e] = (m < M && k < cols) ? __ldg(x + m * ldx + k) : static_cast<unsigned short>(0);
  }
}

// ---------------------------------------------------------------- tcgen05 helpers
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  // SM100 shared-memory matrix descriptor: start >> 4 [0,14), LBO >> 4 [16,30),
  // SBO >> 4 [32,46), version 1 [46,48), base offset 0, layout SWIZZLE_NONE (0) [61,64)
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) |
         static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16 |
         static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32 | 1ull << 46;
}

__device__ __forceinline__ void tc_mma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}

// D[tmem] (+)= A[tmem] . B[smem desc]: the A operand read from tensor memory (128 lanes = rows,
// consecutive 32-bit columns = K pairs)
__device__ __forceinline__ void tc_mma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}

// one m16 x k16 A fragment into TMEM lanes [lane0, lane0 + 16) x 8 columns (mma.sync fragment order)
__device__ __forceinline__ void tc_st_frag(uint32_t taddr, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3) {
  asm volatile("tcgen05.st.sync.aligned.16x256b.x1.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(a0), "r"(a1),
               "r"(a2), "r"(a3)
               : "memory");
}

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tc_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

constexpr int kTcDecodeWarps = 16;  // two per row tile (even / odd k-tiles of each stage)
constexpr int kTcEpiWarps = 8;      // the epilogue's TMEM readers (4 lane quarters x 2 halves)
constexpr int kTcThreads = (kTcDecodeWarps + 2) * 32;  // + B producer + MMA issuer


struct TcGeom {
  int kchunk;   // k-tiles per stage
  int stages;
  int a_bytes;  // A buffer per stage: 128 rows x kchunk*TK fp16
  int b_bytes;  // B buffer per stage: Np rows x kchunk*TK fp16
  int stage;    // [A +] activation image + weight tiles (8 row tiles x kchunk), 1 KB aligned
  int tmem_cols;
  int a_col0;   // A in TMEM: first column of stage 0's A (after the Np accumulator columns)
  int cols_a;   // A in TMEM: columns per stage (kchunk * TK / 2 fp16 pairs)
};

__device__ __forceinline__ uint32_t tc_cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void tc_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

// CS CTAs of a cluster split K for one 128-row block; their TMEM partials are summed through
// distributed shared memory (each 16-column chunk has an owner rank, round robin).
//
// Weights reach shared memory through the producer's bulk copies: the block's 8 row tiles are
// cut into segments by the layout's row groups (device_layout.hpp); a segment that is a whole
// group is ONE copy per stage ([k_tile][row_tile] contiguous), a partial one is one copy per
// k-tile. Few large copies keep the bulk engine's per-copy cost off the critical path.
constexpr int kTcMaxSeg = 8;

// CS = 0: CTA-pair mode (cta_group::2). The two CTAs of a cluster own consecutive 128-row blocks
// (A and D in their own TMEM) and the two N halves of the activation image (B in their own shared
// memory); the leader (rank 0) issues M = 256 MMAs over both, the follower's MMA warp relays its
// stage readiness to the leader, and the leader's commits arrive on both CTAs' barriers. Each SM
// thus streams half the activation bytes per weight row (tools/pair_probe.cu checked the operand
// split on the B200).
template <int SCHEME, int CS>
__global__ void __launch_bounds__(kTcThreads, 1) amsq_linear_tc_kernel(TcParams p, TcGeom geo) {
  constexpr bool PAIR = CS == 0;
  constexpr int KS = PAIR ? 1 : CS;  // CTAs splitting K
  using T = Traits<SCHEME>;
  constexpr int TILE = T::kTileBytes, TK = T::kTK, J = T::kJ;
  constexpr int RUN = SCHEME == 7 ? 12 : 16;  // columns a lane emits per row and tile
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int blk = blockIdx.x / KS;
  const uint32_t crank = (PAIR || KS > 1) ? tc_cluster_rank() : 0u;  // pair rank or K-split rank
  const int KT = p.k_tiles;
  const int kper = (KT + KS - 1) / KS;
  const int kb = PAIR ? 0 : static_cast<int>(crank) * kper, ke = min(KT, kb + kper);
  const int nst = ke > kb ? (ke - kb + geo.kchunk - 1) / geo.kchunk : 0;
  uint64_t* fullA = reinterpret_cast<uint64_t*>(smem + geo.stages * geo.stage);
  uint64_t* fullB = fullA + geo.stages;  // activations + weights of the stage landed
  uint64_t* empty = fullB + geo.stages;
  uint64_t* done = empty + geo.stages;
  uint64_t* peer = done + 1;  // pair leader: the follower's stage s is ready (A decoded, B landed)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(peer + geo.stages);
  int* seg = reinterpret_cast<int*>(tmem_slot + 4);  // [kTcMaxSeg][4]: row0, rows, whole, src tile
  const int Nh = PAIR ? p.Np / 2 : p.Np;  // activation columns this CTA holds
  const uint32_t lboA = 128 * 16, lboB = static_cast<uint32_t>(Nh) * 16;
  const int rb0 = blk * 8, rb1 = min(rb0 + 8, p.row_tiles);
  const GroupPlan& P = p.plan;

  unsigned long long* trace = p.trace ? p.trace + blockIdx.x * 64 : nullptr;
  // profiling trace (clock64 unless noted): [0] start (globaltimer) [1] start [2]/[3] epilogue /
  // end (globaltimer); per stage st < 8: [8+] producer loop top [16+] producer issued [24+]
  // decode warp 0 weights landed [32+] warp 0 A ready [40+] MMA operands ready [48+] MMAs issued
  // [56+] decode warp 15 A ready
  const bool tr8 = trace != nullptr;
  if (trace && threadIdx.x == 0) trace[0] = globaltimer(), trace[1] = clock64();
  pdl_launch_dependents();
  if (threadIdx.x == 0) {
    for (int s = 0; s < geo.stages; ++s) {
      mbar_init(&fullA[s], kTcDecodeWarps);
      mbar_init(&fullB[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&peer[s], 1);
    }
    mbar_init(done, 1);
    fence_barrier_init();
    // segments of the block by row group
    int nseg = 0, r = rb0;
    const int big_rows = P.n_big * P.g_big;
    while (r < rb1 && nseg < kTcMaxSeg) {
      const int g = r < big_rows ? r / P.g_big : P.n_big + (r - big_rows) / (P.g_big - 1);
      const int g0 = P.row0(g), gs = P.size(g);
      const int end = min(rb1, g0 + gs);
      seg[nseg * 4 + 0] = r - rb0;
      seg[nseg * 4 + 1] = end - r;
      seg[nseg * 4 + 2] = (r == g0 && end == g0 + gs) ? gs : -gs;  // +G whole, -G partial
      seg[nseg * 4 + 3] = g0 * KT + (r - g0);                     // tile index of (r, kt = 0)
      ++nseg;
      r = end;
    }
    for (int i = nseg; i < kTcMaxSeg; ++i) seg[i * 4 + 1] = 0;
  }
  __syncwarp();  // reconverge warp 0 before the aligned barriers below
  if (warp == kTcDecodeWarps) {  // TMEM: Np fp32 columns x 128 lanes
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(geo.tmem_cols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(geo.tmem_cols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) tc_cluster_sync();  // the peer's barriers and TMEM exist before any remote use
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < kTcDecodeWarps) {
    // ------------------------------------------------------------------ decode warps
    // warp w: the k-tiles of parity w >> 3 of every stage, for row tile rtl. With A in TMEM a warp
    // may only touch TMEM lanes 32 (w % 4) .. + 31, i.e. row tiles 2 (w % 4) and 2 (w % 4) + 1.
#if AMSQ_TC_ATMEM
    const int rtl = 2 * (warp & 3) + ((warp >> 2) & 1), par = warp >> 3;
#else
    const int rtl = warp & 7, par = warp >> 3;
#endif
    const bool live = rb0 + rtl < rb1;
    const int g = lane >> 2, t = lane & 3;
    // where this row tile sits in a stage's weight buffer: segment base + [kk][row in segment]
    int wbase = 0, srows = 1, sr = 0;
    for (int i = 0; i < kTcMaxSeg; ++i) {
      const int r0 = seg[i * 4 + 0], n = seg[i * 4 + 1];
      if (n == 0) break;
      if (rtl >= r0 && rtl < r0 + n) {
        srows = n;
        sr = rtl - r0;
        break;
      }
      wbase += geo.kchunk * n * TILE;
    }
    int sidx = 0;
    uint32_t ph = 0;
    for (int st = 0; st < nst; ++st) {
      mbar_wait(&fullB[sidx], ph);  // this stage's weights (and activations) landed
      if (tr8 && warp == 0 && lane == 0 && st < 8) trace[24 + st] = clock64();
      if (st >= geo.stages) {
        // A[sidx] is free once the MMAs of its previous use completed; fullB implies that
        // the producer saw `empty` for this stage, so this wait returns at once
        mbar_wait(&empty[sidx], ph ^ 1u);
      }
      uint8_t* A = smem + sidx * geo.stage;
      const uint8_t* W = A + geo.a_bytes + geo.b_bytes + wbase;
      for (int kk = par; kk < geo.kchunk; kk += 2) {
        if (kb + st * geo.kchunk + kk < ke) {
#if AMSQ_TC_ATMEM
          if (!live) continue;  // rows past the tensor: D rows that are never stored
          const uint8_t* tp = W + (kk * srows + sr) * TILE;
          const uint4 wv = *reinterpret_cast<const uint4*>(tp + lane * 16);
          const uint32_t sh = SCHEME == 4 ? tp[512 + lane] : 0u;
          uint32_t Af[J][4];
          const uint32_t R[4] = {wv.x, wv.y, wv.z, wv.w};
          if constexpr (SCHEME == 4) {
            decode_s4(R, sh, Af);
          } else {
            decode_s7(R, Af);
          }
          const uint32_t ta = tmem + (static_cast<uint32_t>(rtl * 16) << 16) +
                              static_cast<uint32_t>(geo.a_col0 + sidx * geo.cols_a + kk * J * 8);
#pragma unroll
          for (int j = 0; j < J; ++j) tc_st_frag(ta + j * 8, Af[j][0], Af[j][2], Af[j][1], Af[j][3]);
#else
          uint4 wv = make_uint4(0, 0, 0, 0);
          uint32_t sh = 0;
          if (live) {
            const uint8_t* tp = W + (kk * srows + sr) * TILE;
            wv = *reinterpret_cast<const uint4*>(tp + lane * 16);
            if (SCHEME == 4) sh = tp[512 + lane];
          }
          uint32_t Af[J][4];
          const uint32_t R[4] = {wv.x, wv.y, wv.z, wv.w};
          uint32_t rowg[2 * J], rowg8[2 * J];  // a lane's RUN columns of rows g and g + 8
          if constexpr (SCHEME == 4) {
            decode_s4(R, sh, Af);
            // A[j] = {g:(16t+j,16t+4+j), g+8, g:(16t+8+j,16t+12+j), g+8}: emit q-major
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              rowg[jj] = Af[jj][0], rowg[4 + jj] = Af[jj][2];
              rowg8[jj] = Af[jj][1], rowg8[4 + jj] = Af[jj][3];
            }
          } else {
            decode_s7(R, Af);
            // A[j] = {g: pair 2j, g+8: pair 2j, g: pair 2j+1, g+8: pair 2j+1}
#pragma unroll
            for (int jj = 0; jj < 3; ++jj) {
              rowg[2 * jj] = Af[jj][0], rowg[2 * jj + 1] = Af[jj][2];
              rowg8[2 * jj] = Af[jj][1], rowg8[2 * jj + 1] = Af[jj][3];
            }
          }
          // [k/8][128][8] image: column c of row r at (c / 8) * lboA + r * 16 + (c % 8) * 2
          const int c0 = kk * TK + RUN * t;  // first (permuted) column of the run
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = rtl * 16 + g + 8 * h;
            const uint32_t* v = h ? rowg8 : rowg;
            if constexpr (RUN == 16) {  // two whole 8-column core rows
              *reinterpret_cast<uint4*>(A + (c0 >> 3) * lboA + r * 16) = make_uint4(v[0], v[1], v[2], v[3]);
              *reinterpret_cast<uint4*>(A + ((c0 >> 3) + 1) * lboA + r * 16) = make_uint4(v[4], v[5], v[6], v[7]);
            } else if ((t & 1) == 0) {  // 12 columns from a core-row boundary: 8 + 4
              *reinterpret_cast<uint4*>(A + (c0 >> 3) * lboA + r * 16) = make_uint4(v[0], v[1], v[2], v[3]);
              *reinterpret_cast<uint2*>(A + ((c0 >> 3) + 1) * lboA + r * 16) = make_uint2(v[4], v[5]);
            } else {  // 4 + 8
              *reinterpret_cast<uint2*>(A + (c0 >> 3) * lboA + r * 16 + 8) = make_uint2(v[0], v[1]);
              *reinterpret_cast<uint4*>(A + ((c0 >> 3) + 1) * lboA + r * 16) = make_uint4(v[2], v[3], v[4], v[5]);
            }
          }
#endif
        }
      }
#if AMSQ_TC_ATMEM
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();  // the TMEM stores, before the arrival the MMA thread acquires
      // the generic-proxy reads of this stage's weight tiles, before the producer's bulk copy
      // (async proxy) rewrites the stage once the MMAs release it (cross-proxy WAR)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#else
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic -> tensor core
#endif
      __syncwarp();
      if (lane == 0) mbar_arrive(&fullA[sidx]);
      if (tr8 && lane == 0 && st < 8 && (warp == 0 || warp == 15)) trace[(warp ? 56 : 32) + st] = clock64();
      if (++sidx == geo.stages) sidx = 0, ph ^= 1u;
    }
  } else if (warp == kTcDecodeWarps) {
    // ------------------------------------------------------------------ producer
    // per stage: the block's weight segments + the activation image, one full barrier. The
    // whole warp walks the loop (lane 0 issues): lanes parked at a later barrier while lane 0
    // runs alone would leave the warp diverged across barriers.
    const uint64_t pol = policy_evict_first();
    int sidx = 0;
    uint32_t ph = 0;
    for (int st = 0; st < nst; ++st) {
      if (tr8 && lane == 0 && st < 8) trace[8 + st] = clock64();
      if (st >= geo.stages) mbar_wait(&empty[sidx], ph ^ 1u);
      if (st == 0) pdl_wait();  // the prepped activations come from the previous kernel
      if (lane == 0) {
        const int kt0 = kb + st * geo.kchunk, nk = min(geo.kchunk, ke - kt0);
        const uint32_t xbytes = static_cast<uint32_t>(nk * TK / 8) * lboB;
        uint32_t wbytes = 0;
        for (int i = 0; i < kTcMaxSeg; ++i) wbytes += static_cast<uint32_t>(seg[i * 4 + 1] * nk * TILE);
        uint8_t* sp = smem + sidx * geo.stage;
        mbar_arrive_expect_tx(&fullB[sidx], xbytes + wbytes);
        uint8_t* wdst = sp + geo.a_bytes + geo.b_bytes;
        for (int i = 0; i < kTcMaxSeg; ++i) {
          const int n = seg[i * 4 + 1];
          if (n == 0) break;
          const int gsz = seg[i * 4 + 2];
          const long long t0 = seg[i * 4 + 3];
          if (gsz > 0) {  // whole group: [k_tile][row_tile] contiguous
            bulk_g2s(wdst, p.w + (t0 + static_cast<long long>(kt0) * gsz) * TILE,
                     static_cast<uint32_t>(nk * n * TILE), &fullB[sidx], pol);
          } else {  // partial group: one copy of n row tiles per k-tile (row stride -gsz)
            for (int kk = 0; kk < nk; ++kk) {
              bulk_g2s(wdst + kk * n * TILE,
                       p.w + (t0 + static_cast<long long>(kt0 + kk) * (-gsz)) * TILE,
                       static_cast<uint32_t>(n * TILE), &fullB[sidx], pol);
            }
          }
          wdst += geo.kchunk * n * TILE;
        }
        const long long himg = PAIR ? static_cast<long long>(crank) * KT * TK * Nh : 0;  // this CTA's half
        bulk_g2s(sp + geo.a_bytes, p.xk + himg + static_cast<long long>(kt0) * TK * Nh, xbytes,
                 &fullB[sidx], policy_evict_last());
        if (tr8 && st < 8) trace[16 + st] = clock64();
      }
      __syncwarp();
      if (++sidx == geo.stages) sidx = 0, ph ^= 1u;
    }
  } else {
    // ------------------------------------------------------------------ MMA issuer
    // whole warp waits, one thread issues
    const uint32_t idesc = (1u << 4)                                      // D: f32
                           | (static_cast<uint32_t>(p.Np >> 3) << 17)     // N
                           | (static_cast<uint32_t>((PAIR ? 256 : 128) >> 4) << 24);  // M
    int sidx = 0;
    uint32_t ph = 0;
    if (PAIR && crank != 0) {
      // follower: relay each stage's readiness (A decoded into this CTA's TMEM, B half landed)
      // to the leader, which issues the pair's MMAs
      uint32_t lead_peer;
      asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(lead_peer) : "r"(smem_u32(peer)));
      for (int st = 0; st < nst; ++st) {
        mbar_wait(&fullA[sidx], ph);
        mbar_wait(&fullB[sidx], ph);
        if (lane == 0) {
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(lead_peer + sidx * 8)
                       : "memory");
        }
        __syncwarp();
        if (++sidx == geo.stages) sidx = 0, ph ^= 1u;
      }
    } else
    for (int st = 0; st < nst; ++st) {
      mbar_wait(&fullA[sidx], ph);
      mbar_wait(&fullB[sidx], ph);
      if constexpr (PAIR) {
        asm volatile(
            "{\n\t.reg .pred p;\n"
            "WPEER_%=:\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
            "@!p bra WPEER_%=;\n}" ::"r"(smem_u32(&peer[sidx])),
            "r"(ph)
            : "memory");
      }
      tc_fence_after();
      if (tr8 && lane == 0 && st < 8) trace[40 + st] = clock64();
      if (lane == 0) {
        const int nk = min(geo.kchunk, ke - (kb + st * geo.kchunk));
        const uint32_t a0 = smem_u32(smem + sidx * geo.stage);
        const uint32_t b0 = a0 + geo.a_bytes;
        for (int k16 = 0; k16 < nk * TK / 16; ++k16) {
          const uint64_t bd = umma_desc(b0 + k16 * 2 * lboB, lboB, 128);
#if AMSQ_TC_ATMEM
          const uint32_t at = tmem + static_cast<uint32_t>(geo.a_col0 + sidx * geo.cols_a + k16 * 8);
          if constexpr (PAIR) {
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
                "r"(at), "l"(bd), "r"(idesc), "r"((st > 0 || k16 > 0) ? 1u : 0u)
                : "memory");
          } else {
            tc_mma_f16_ts(tmem, at, bd, idesc, (st > 0 || k16 > 0) ? 1u : 0u);
          }
#else
          const uint64_t ad = umma_desc(a0 + k16 * 2 * lboA, lboA, 128);
          tc_mma_f16(tmem, ad, bd, idesc, (st > 0 || k16 > 0) ? 1u : 0u);
#endif
        }
        if constexpr (PAIR) {  // both CTAs' stage s: their A (TMEM) and B halves were read
          asm volatile(
              "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                  smem_u32(&empty[sidx])),
              "h"(static_cast<uint16_t>(3))
              : "memory");
        } else {
          tc_commit(&empty[sidx]);  // frees the stage once these MMAs have read it
        }
        if (tr8 && st < 8) trace[48 + st] = clock64();
      }
      __syncwarp();
      if (++sidx == geo.stages) sidx = 0, ph ^= 1u;
    }
    if (lane == 0 && !(PAIR && crank != 0)) {
      if constexpr (PAIR) {
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(done)),
            "h"(static_cast<uint16_t>(3))
            : "memory");
      } else {
        tc_commit(done);
      }
    }
    __syncwarp();
  }

  // ------------------------------------------------------------------ epilogue
  // warp w reads TMEM lanes 32*(w%4).. (its rows) for columns of half w/4, 16 at a time
  const int quarter = warp & 3, half = warp >> 2;
  const int row = quarter * 32 + lane;
  const long long n = static_cast<long long>(blk) * 128 + row;
  const int nchunks = p.Np / 16, ncap = (nchunks + KS - 1) / KS * 16;  // owned columns / rank
  const int nch_half = (nchunks + 1) / 2;  // 16-column chunks per epilogue warp half
  float* recv = reinterpret_cast<float*>(smem);  // [CS][ncap][128] (the idle stage ring)
  auto store_y = [&](int m, float v) {
    if (m < p.M && n < p.rows) {
      const float sc = __half2float(__ushort_as_half(p.scales[n])) * kPlaceScale;
      p.y[static_cast<long long>(m) * p.ldy + n] = out_bits(v * sc, p.yscale, m);
    }
  };
  if (warp < kTcEpiWarps && nst > 0) {
    mbar_wait(done, 0);
    tc_fence_after();
  }
  if (trace && threadIdx.x == 0) trace[2] = globaltimer();
  if constexpr (KS > 1) {
    // every rank's MMAs have finished reading its stage ring before any rank writes partials
    // into a peer's (reused) ring
    __syncwarp();
    tc_fence_before();
    tc_cluster_sync();
    tc_fence_after();
  } else {
    pdl_wait();  // y may still be read by the previous kernel
  }
  if (warp < kTcEpiWarps) {
    for (int ci = half * nch_half; ci < min(nchunks, (half + 1) * nch_half); ++ci) {
      const int c0 = ci * 16;
      uint32_t v[16];
      if (nst > 0) {
        tc_ld16(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + static_cast<uint32_t>(c0), v);
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = 0u;  // empty K range: a zero partial
      }
      if constexpr (KS == 1) {
#pragma unroll
        for (int j = 0; j < 16; ++j) store_y(c0 + j, __uint_as_float(v[j]));
      } else {
        const int owner = ci % KS, slot = (ci / KS) * 16;
        // [rank][column][row]: consecutive lanes (rows) hit consecutive banks
        float* dst = recv + (static_cast<long long>(crank) * ncap + slot) * 128 + row;
        uint32_t remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(dst)), "r"(owner));
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          asm volatile("st.shared::cluster.b32 [%0], %1;" ::"r"(remote + j * 128 * 4), "r"(v[j])
                       : "memory");
        }
      }
    }
  }
  if constexpr (KS > 1) {
    __syncwarp();
    tc_fence_before();
    tc_cluster_sync();  // all remote partials have landed
    if (warp < kTcEpiWarps) {
      pdl_wait();
      for (int ci = half * nch_half; ci < min(nchunks, (half + 1) * nch_half); ++ci) {
        const int c0 = ci * 16;
        if (ci % KS != static_cast<int>(crank)) continue;
        const int slot = (ci / KS) * 16;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          float v = 0.0f;
#pragma unroll
          for (int r = 0; r < KS; ++r) v += recv[(static_cast<long long>(r) * ncap + slot + j) * 128 + row];
          store_y(c0 + j, v);  // rank order: deterministic
        }
      }
    }
  }
  if (trace && threadIdx.x == 0) trace[3] = globaltimer();
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) {
    tc_cluster_sync();  // the leader's MMAs wrote this CTA's TMEM; both are done with it
    if (warp == kTcDecodeWarps) {
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "r"(geo.tmem_cols));
    }
  } else if (warp == kTcDecodeWarps) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(geo.tmem_cols));
  }
}

}  // namespace dev

// ---------------------------------------------------------------- launchers
template <int SCHEME, int CS>
static cudaError_t launch_tc_m(const TcParams& p, const dev::TcGeom& geo, int smem, int rb,
                               cudaStream_t s) {
  static std::atomic<uint64_t> configured{0};  // per template instance, one bit per device
  if (const cudaError_t e = opt_in_max_smem(dev::amsq_linear_tc_kernel<SCHEME, CS>, configured);
      e != cudaSuccess) {
    return e;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(CS == 0 ? (rb + 1) / 2 * 2 : rb * CS));  // CS = 0: CTA pairs
  cfg.blockDim = dim3(dev::kTcThreads);
  cfg.dynamicSmemBytes = static_cast<size_t>(smem);
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  int na = 1;
  if constexpr (CS != 1) {
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = CS == 0 ? 2 : CS;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    na = 2;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, dev::amsq_linear_tc_kernel<SCHEME, CS>, p, geo);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

int tc_pair_knob();

template <int SCHEME>
static cudaError_t launch_tc_t(const TcParams& p, const unsigned short* x, long long ldx,
                               long long cols, cudaStream_t s) {
  using T = dev::Traits<SCHEME>;
  // stage geometry for an activation image of nb columns per CTA
  auto geometry = [&](int nb) {
    dev::TcGeom geo{}, best{};
    best.stages = 0;
    const int budget = 227 * 1024 - 2048;
    // k-tiles per stage (even: two decode warps per row tile): the largest that leaves enough
    // stages -- per-stage synchronisation, not ring depth, is what K3 pays for
#if AMSQ_TC_BIG_STAGES
    for (int kc : {8, 6, 4, 2}) {
#else
    for (int kc : {4, 2}) {
#endif
      geo.kchunk = kc;
      geo.a_bytes = AMSQ_TC_ATMEM ? 0 : 128 * kc * T::kTK * 2;
      geo.b_bytes = nb * kc * T::kTK * 2;
      geo.stage = (geo.a_bytes + geo.b_bytes + 8 * kc * T::kTileBytes + 1023) / 1024 * 1024;
      geo.stages = budget / geo.stage;
      if (AMSQ_TC_ATMEM) {  // the A ring shares TMEM with the Np accumulator columns
        geo.a_col0 = p.Np <= 128 ? 128 : 256;
        geo.cols_a = kc * T::kTK / 2;
        geo.stages = std::min(geo.stages, (512 - geo.a_col0) / geo.cols_a);
      }
      const int need = kc > 4 ? 2 : AMSQ_TC_KC4_MIN_STAGES;
      if (geo.stages >= need || geo.stages > best.stages) best = geo;
      if (geo.stages >= need) break;
    }
    geo = best;
    if (geo.stages > (AMSQ_TC_ATMEM ? 8 : 6)) geo.stages = AMSQ_TC_ATMEM ? 8 : 6;
    geo.tmem_cols = 32;
    while (geo.tmem_cols < p.Np) geo.tmem_cols *= 2;
    if (AMSQ_TC_ATMEM) geo.tmem_cols = 512;
    return geo;
  };
  dev::TcGeom geo = geometry(p.Np);
  if (geo.stages < 2) return cudaErrorInvalidConfiguration;
  // split K over a cluster when the 128-row blocks alone leave SMs idle
  const int rb = (p.row_tiles + 7) / 8;
  int cs = 1;
  while (cs < 4 && rb * cs * 2 <= 148 && p.k_tiles >= 8 * cs * 2 &&
         (cs * 2 != 4 || rb <= 32)) {
    cs *= 2;
  }
  const int nchunks = p.Np / 16;
  const long long recv = static_cast<long long>(cs) * 128 * ((nchunks + cs - 1) / cs * 16) * 4;
  if (cs > 1 && geo.stages * geo.stage < recv) cs = 1;
  // otherwise CTA pairs (cta_group::2, M = 256): each CTA streams half the activation image. The
  // pair's per-stage handshake pays off only for large stages full of activations: measured 1.25x
  // at 128 batch rows where the halved image admits 4 k-tiles per stage (the single CTA then runs 2),
  // 4-7 % slower elsewhere (profiles/r02/k3_pair_ab.txt)
  const int knob = tc_pair_knob();
  const dev::TcGeom pgeo = geometry(p.Np / 2);  // halving the image lets a pair take bigger stages
  const bool pair_ok = AMSQ_TC_ATMEM && cs == 1 && rb >= 2 && pgeo.stages >= 2;
  const bool pair = pair_ok && (knob == 1 || (knob < 0 && pgeo.kchunk >= 4 && p.Np >= 128));
  if (pair) geo = pgeo;
  const int smem = geo.stages * geo.stage + (4 * geo.stages + 1) * 8 + 16 + dev::kTcMaxSeg * 16;
  // activation prep (PDL-chained): one image, or the two N halves of a pair
  {
    const long long total = static_cast<long long>(p.k_tiles) * T::kTK * p.Np;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(total / 256 + 1 < 148 * 16 ? total / 256 + 1 : 148 * 16));
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, dev::amsq_xprep_tc_kernel<SCHEME>, x, ldx, cols, p.M,
                                       p.Np, p.k_tiles, pair ? 2 : 1, const_cast<unsigned short*>(p.xk));
    count_launch();
    if (e != cudaSuccess) return e;
  }
  if (pair) return launch_tc_m<SCHEME, 0>(p, geo, smem, rb, s);
  switch (cs) {
    case 2: return launch_tc_m<SCHEME, 2>(p, geo, smem, rb, s);
    case 4: return launch_tc_m<SCHEME, 4>(p, geo, smem, rb, s);
    default: return launch_tc_m<SCHEME, 1>(p, geo, smem, rb, s);
  }
}

static std::atomic<int> g_tc_pair{-1};
int tc_pair_knob() { return g_tc_pair.load(std::memory_order_relaxed); }
int tc_set_pair_knob(int v) { return g_tc_pair.exchange(v < 0 ? -1 : (v ? 1 : 0)); }

cudaError_t launch_linear_tc(const TcParams& p, const unsigned short* x, long long ldx,
                             long long cols, cudaStream_t s) {
  if (p.row_tiles <= 0) return cudaSuccess;
  return p.scheme_id == 4 ? launch_tc_t<4>(p, x, ldx, cols, s) : launch_tc_t<7>(p, x, ldx, cols, s);
}

}  // namespace amsqb
