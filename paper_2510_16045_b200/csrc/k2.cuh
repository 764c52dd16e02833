// k2.cuh -- K2, the fused restore + linear for batch M <= 32 per launch (mma.sync), and its
// activation prep: templates over the scheme, instantiated one scheme per translation unit
// (k2_s<id>.cu) so the 8 x 12 kernel instances compile in parallel. See kernels.cu for K1.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <type_traits>

#include "kernels.h"
#include "kernels_common.cuh"

namespace amsqb {

void count_launch();

namespace dev {
// =====================================================================================
// Activation prep for K2: x[M][cols] (fp16, row stride ldx) -> B-fragment units
// xp[kt][j][m][t] (8 bytes: the two fp16 pairs lane t of an m16n8k16 MMA j reads for batch
// row m), zero for m >= M and k >= cols. One thread per (k-tile, row, lane-column) item.
// =====================================================================================
template <int SCHEME>
__global__ void __launch_bounds__(128) amsq_xprep_kernel(const unsigned short* __restrict__ x,
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
    const unsigned short* xr = x + m * ldx + k;
    // the lane's LK columns are one aligned 24-byte (FP5.33 family) or 32-byte run: vector loads
    // when the row and base alignment allow and the run lies inside `cols`
    constexpr int VB = LW % 4 == 0 ? 16 : 8;
    const bool vec = m < M && k + LK <= cols && (reinterpret_cast<uintptr_t>(xr) & (VB - 1)) == 0;
    if (vec) {
      if constexpr (VB == 16) {
#pragma unroll
        for (int i = 0; i < LW; i += 4) {
          const uint4 v = __ldg(reinterpret_cast<const uint4*>(xr) + i / 4);
          w[i] = v.x, w[i + 1] = v.y, w[i + 2] = v.z, w[i + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < LW; i += 2) {
          const uint2 v = __ldg(reinterpret_cast<const uint2*>(xr) + i / 2);
          w[i] = v.x, w[i + 1] = v.y;
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < LW; ++i) {
        unsigned lo = 0, hi = 0;
        if (m < M) {
          if (k + 2 * i < cols) lo = __ldg(xr + 2 * i);
          if (k + 2 * i + 1 < cols) hi = __ldg(xr + 2 * i + 1);
        }
        w[i] = lo | hi << 16;
      }
    }
    uint32_t B[J][2];
    if constexpr (T::kFam == 4) {
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
// K2: fused restore + linear, M <= 8*NB per launch (NB = 1 or 2).
//
// One CTA (or a cluster of CS = 2/4/8 CTAs splitting K) per row group of the weight's plan
// (device_layout.hpp): the CTA owns G row tiles over its whole K range, so partial sums
// never leave the SM / cluster and there is no global split-K fix-up.
//  * warp 16 = producer: per pipeline stage ONE cp.async.bulk of S k-tiles x G row tiles
//    (contiguous in the [group][k_tile][row_tile] layout) plus the stage's activations
//    (LDGSTS natural rows for M <= 8, bulk copy of B-fragment units for M <= 16), into a
//    ring guarded by full/empty mbarriers; weights are requested before griddepcontrol.wait
//    (they never depend on the previous kernel).
//  * warps 0..15 = consumers: warp w takes k-slot w / wr of every stage and the row tiles
//    r = w % wr + i*wr (i < 4); per k-tile it gathers the B fragments once and reuses them
//    for its row tiles: LDS.128 + in-register decode + m16n8k16 MMAs, fp32 accumulation.
//  * epilogue: the S k-slot partials are summed in k-slot order through shared memory, the
//    CTAs of a cluster are summed in rank order through DSMEM, scale * 2^14, fp16 round.
//    Deterministic: the summation order depends only on the shape.
// =====================================================================================
#ifndef AMSQ_K2_WARPS
#define AMSQ_K2_WARPS 16
#endif
#ifndef AMSQ_CTAS_PER_SM  // K2 CTAs per SM the plan assumes (device_layout.hpp); 1 in the product
#define AMSQ_CTAS_PER_SM 1
#endif
#ifndef AMSQ_K2_XPREP  // 1: M <= 16 reads activations pre-permuted by amsq_xprep_kernel (an extra
#define AMSQ_K2_XPREP 1  // launch); 0: natural rows + PRMT like M <= 8 (measured slower)
#endif
#ifndef AMSQ_RECV_STEAL  // 1: a ring of >= 4 stages gives one up for an out-of-ring receive buffer
#define AMSQ_RECV_STEAL 1
#endif
#ifndef AMSQ_KPW2_MIN_STAGES  // fewest ring stages for which a warp takes 2 k-tiles per stage
#define AMSQ_KPW2_MIN_STAGES 2  // (M <= 16)
#endif
#ifndef AMSQ_KPW2_MIN_STAGES1  // (M <= 8)
#define AMSQ_KPW2_MIN_STAGES1 1
#endif
#ifndef AMSQ_OWN_TARGET  // row tiles per consumer warp the stage geometry aims for (<= 4)
#define AMSQ_OWN_TARGET 4
#endif
#ifndef AMSQ_L2_PREFETCH  // pull the next ring's worth of weights into L2 ahead of the copies
#define AMSQ_L2_PREFETCH 0
#endif
#ifndef AMSQ_PRODUCER_SLEEP_NS  // try_wait suspend hint of the producer's empty-slot waits
#define AMSQ_PRODUCER_SLEEP_NS 200
#endif
#ifndef AMSQ_CONSUMER_PROXY_FENCE  // consumers fence.proxy.async before releasing a stage
#define AMSQ_CONSUMER_PROXY_FENCE 0
#endif
#ifndef AMSQ_K2_PRE_W  // ring stages whose weights are requested before griddepcontrol.wait
#define AMSQ_K2_PRE_W 1
#endif
#ifndef AMSQ_K2_PIPE  // issue both k-tiles' fragment loads before decoding the first (kpw = 2)
#define AMSQ_K2_PIPE 0
#endif
#ifndef AMSQ_K2_LEAN
#define AMSQ_K2_LEAN 0
#endif
#ifndef AMSQ_EPI_OLD
#define AMSQ_EPI_OLD 0
#endif
#ifndef AMSQ_TRACE_STAGES
#define AMSQ_TRACE_STAGES 0
#endif
#ifndef AMSQ_K2_MODE  // profiling variants only (tools/build_variants.sh): 1 = stream only,
#define AMSQ_K2_MODE 0  // 2 = decode without MMA, 3 = MMA without decode, 4 = consume without copies
#endif
constexpr int kConsumerWarps = AMSQ_K2_WARPS;
constexpr bool kK2XStage = AMSQ_K2_XSTAGE != 0;
// the separate prep kernel only when the producer does not permute the activations itself
constexpr bool kK2XPrep = AMSQ_K2_XPREP != 0 && !kK2XStage;
constexpr int kK2Threads = (kConsumerWarps + 1) * 32;  // + the producer warp
#ifndef AMSQ_MAX_OWN1  // row tiles a consumer warp may own at M <= 8 (4 or 8)
#define AMSQ_MAX_OWN1 4
#endif
constexpr int kMaxOwn = 4;  // row tiles per consumer warp at M <= 16
#ifndef AMSQ_MAX_OWN4  // row tiles a consumer warp may own at M <= 32 (accumulators: 16 fp32 each)
#define AMSQ_MAX_OWN4 2
#endif
template <int NB>
struct OwnCap {
  static constexpr int value = NB == 1 ? AMSQ_MAX_OWN1 : NB == 2 ? kMaxOwn : AMSQ_MAX_OWN4;
};

struct K2Geom {
  int S, wr;         // k-tiles per stage; warps sharing a k-slot (row-tile interleave)
  int kpw;           // k-tiles per warp per stage (S = kpw * 16 / wr)
  int w_stage;       // weight bytes reserved per stage (max group)
  int x_row;         // natural-layout activation row stride (bytes), M <= 8
  int xrows;         // natural-layout activation rows held per stage (= M)
  int stage;         // bytes per stage (weights + activations), 128-aligned
  int stages;        // ring depth
  int recv_off;      // byte offset of the cluster reduction's receive buffer
  int recv_in_ring;  // 1: it overlaps the ring, so peers may only store after a cluster barrier
  int bar_off;       // byte offset of the mbarriers (then the staged scales)
  int xnat_off;      // AMSQ_K2_XSTAGE: natural activation rows, from the stage's activation area
};

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}

template <int SCHEME, int NB>
__device__ __forceinline__ void load_bfrag(const uint8_t* xs, const K2Geom& geo, int ks,
                                           int g, int t, uint32_t (&B)[NB][Traits<SCHEME>::kJ][2]) {
  using T = Traits<SCHEME>;
  constexpr int J = T::kJ, MS = 8 * NB;
#pragma unroll
  for (int nb = 0; nb < NB; ++nb) {
    if constexpr ((kK2XPrep && NB >= 2) || kK2XStage) {
      const uint2* xu = reinterpret_cast<const uint2*>(xs) + ((ks * J) * MS + nb * 8 + g) * 4 + t;
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const uint2 b = xu[j * MS * 4];
        B[nb][j][0] = b.x;
        B[nb][j][1] = b.y;
      }
    } else {
      // batch rows >= M only feed accumulator columns that are never stored: read row M-1
      const uint8_t* xp =
          xs + min(nb * 8 + g, geo.xrows - 1) * geo.x_row + (ks * T::kTK + t * T::kLaneK) * 2;
      if constexpr (T::kFam == 4) {
        const uint4 a = *reinterpret_cast<const uint4*>(xp);
        const uint4 b = *reinterpret_cast<const uint4*>(xp + 16);
        const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        bfrag_s4(w, B[nb]);
      } else {
        const uint2 a = *reinterpret_cast<const uint2*>(xp);
        const uint2 b = *reinterpret_cast<const uint2*>(xp + 8);
        const uint2 d = *reinterpret_cast<const uint2*>(xp + 16);
        const uint32_t w[6] = {a.x, a.y, b.x, b.y, d.x, d.y};
        bfrag_s7(w, B[nb]);
      }
    }
  }
}

template <int SCHEME, int NB, int CS>
__global__ void __launch_bounds__(kK2Threads, AMSQ_CTAS_PER_SM) amsq_linear_kernel(LinearParams p, K2Geom geo) {
  using T = Traits<SCHEME>;
  constexpr int TILE = T::kTileBytes, J = T::kJ, TK = T::kTK, MS = 8 * NB;
  constexpr bool kXPrep = kK2XPrep && NB >= 2;
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int grp = blockIdx.x / CS;
  const uint32_t crank = CS > 1 ? cluster_ctarank() : 0u;
  const int G = p.plan.size(grp), rt0 = p.plan.row0(grp);
  const int KT = p.k_tiles;
  const int kper = (KT + CS - 1) / CS;
  const int kb = static_cast<int>(crank) * kper, ke = min(KT, kb + kper);
  const int S = geo.S;
  const int nst = ke > kb ? (ke - kb + S - 1) / S : 0;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + geo.bar_off);
  uint64_t* empty = full + geo.stages;
  // the group's row scales (fp32, x 2^14), staged once so the epilogue does not wait on HBM
  uint64_t* xland = empty + geo.stages;  // kK2XStage: a stage's natural activation rows landed
  float* sscale = reinterpret_cast<float*>(empty + geo.stages * (kK2XStage ? 2 : 1));
  unsigned long long* trace = p.trace ? p.trace + blockIdx.x * 64 : nullptr;
  if (trace && threadIdx.x == 0) {
    trace[0] = globaltimer();
    trace[63] = clock64();
  }
  pdl_launch_dependents();

  if (threadIdx.x == 0) {
    for (int s = 0; s < geo.stages; ++s) {
      // arrival 1: the producer's arrive.expect_tx (weights + bulk activations); arrival 2:
      // after the activations were issued / plain-stored (release of the zero tails)
      mbar_init(&full[s], 2);
      mbar_init(&empty[s], kConsumerWarps);
      if constexpr (kK2XStage) mbar_init(&xland[s], 1);
    }
    fence_barrier_init();
  }
  __syncwarp();  // reconverge warp 0 before the aligned CTA barrier
  __syncthreads();
  // DSMEM rule: a peer's shared memory may only be written once that peer is known to be
  // running. Arrive now (nothing to publish yet: relaxed) and wait right before the first
  // remote store in the epilogue, by which time every peer has long arrived.
  if constexpr (CS > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");

  constexpr int MAXOWN = OwnCap<NB>::value;
  float acc[MAXOWN][NB][4];
#pragma unroll
  for (int i = 0; i < MAXOWN; ++i)
#pragma unroll
    for (int nb = 0; nb < NB; ++nb)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[i][nb][e] = 0.0f;
  // k-slot (kpw k-tiles per stage) and row lane of the warp. Warp w runs on SM sub-partition
  // w % 4; numbering row lanes slowest spreads the lanes that own one extra row tile (when wr
  // does not divide G) over the sub-partitions instead of stacking them on one.
  const int nks = kConsumerWarps / geo.wr;
  const int ks = warp % nks, rl = warp / nks;
  const int nown = warp < kConsumerWarps && rl < G ? min(MAXOWN, (G - rl + geo.wr - 1) / geo.wr) : 0;

  // The CTA's K range [kb, ke) is walked from a per-group rotation rho: every CTA reads
  // the SAME activations, and all of them starting at k = 0 would hammer the same L2
  // lines (measured: ~1 us per stage at M = 1, ~3 us at M = 8). Logical position q maps to
  // k-tile kb + (rho + q) mod L; a stage may wrap once (two contiguous runs). The fp32
  // order stays a function of the shape only.
  const int L = ke - kb;
  const int rho = L > 0 ? static_cast<int>(static_cast<long long>(grp) * L / p.plan.n_groups) : 0;

  if (warp == kConsumerWarps) {
    // ------------------------------------------------------------------ producer
    const uint64_t pol = policy_evict_first();
    const uint8_t* wgrp = p.w + static_cast<long long>(rt0) * KT * TILE;
    // bulk copies need 16-byte aligned rows (cols, ldx multiples of 8, 16-byte aligned x)
    const bool x_bulk = ((p.cols & 7) == 0) && ((p.ldx & 7) == 0) &&
                        ((reinterpret_cast<uintptr_t>(p.x) & 15) == 0);
    constexpr uint32_t kXTileBytes = J * MS * 4 * 8;
    // runs of stage st: [k0, k0 + n0) then [k1, k1 + n1) (n1 = 0 when it does not wrap)
    auto runs = [&](int st, int& k0, int& n0, int& k1, int& n1) {
      const int q0 = st * S, nk = min(S, L - q0);
      const int start = rho + q0 >= L ? rho + q0 - L : rho + q0;  // rho, q0 < L: no division
      k0 = kb + start;
      n0 = min(nk, L - start);
      k1 = kb;
      n1 = nk - n0;
    };
    // activation bytes of row m that a run [kt, kt + nr) covers (the rest is past `cols`)
    auto xvalid = [&](int kt, int nr) -> uint32_t {
      const long long left = p.cols - static_cast<long long>(kt) * TK;
      return static_cast<uint32_t>(left <= 0 ? 0 : (left >= nr * TK ? nr * TK : left) * 2);
    };
    auto issue_w = [&](int st, int sidx) {  // lane 0
#if AMSQ_K2_MODE == 4  // profiling variant: no copies (consumers run on whatever the ring holds)
      mbar_arrive(&full[sidx]);
      return;
#endif
      int k0, n0, k1, n1;
      runs(st, k0, n0, k1, n1);
      uint8_t* sp = smem + sidx * geo.stage;
      const uint32_t wbytes = static_cast<uint32_t>((n0 + n1) * G * TILE);
      uint32_t xbytes = 0;
      if constexpr (kXPrep) {
        xbytes = static_cast<uint32_t>(n0 + n1) * kXTileBytes;
      } else if constexpr (!kK2XStage) {
        if (x_bulk) xbytes = static_cast<uint32_t>(p.M) * (xvalid(k0, n0) + (n1 ? xvalid(k1, n1) : 0u));
      }
      // no fence.proxy.async: the empty-barrier acquire already orders the consumers' reads
      // before this async-proxy write (a proxy fence here serialises the copies: measured)
      mbar_arrive_expect_tx(&full[sidx], wbytes + xbytes);  // arrival 1 of 2
      bulk_g2s(sp, wgrp + static_cast<long long>(k0) * G * TILE, static_cast<uint32_t>(n0 * G * TILE),
               &full[sidx], pol);
      if (n1) {
        bulk_g2s(sp + n0 * G * TILE, wgrp + static_cast<long long>(k1) * G * TILE,
                 static_cast<uint32_t>(n1 * G * TILE), &full[sidx], pol);
      }
    };
    // DRAM latency under full load (~3 us) is longer than a ~200 KB ring can cover at the
    // consumers' pace, so stage st + stages is pulled into L2 when stage st is issued: the
    // ring's own copies then hit L2.
    auto prefetch_w = [&](int st) {  // lane 0
#if AMSQ_L2_PREFETCH
      if (st >= nst) return;
      int k0, n0, k1, n1;
      runs(st, k0, n0, k1, n1);
      bulk_prefetch_l2(wgrp + static_cast<long long>(k0) * G * TILE, static_cast<uint32_t>(n0 * G * TILE));
      if (n1) bulk_prefetch_l2(wgrp + static_cast<long long>(k1) * G * TILE, static_cast<uint32_t>(n1 * G * TILE));
#else
      (void)st;
#endif
    };
    auto issue_x = [&](int st, int sidx) {  // whole warp; ends with arrival 2 of 2
#if AMSQ_K2_MODE == 4
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[sidx]);
      return;
#endif
      int k0, n0, k1, n1;
      runs(st, k0, n0, k1, n1);
      uint8_t* xs = smem + sidx * geo.stage + geo.w_stage + (kK2XStage ? geo.xnat_off : 0);
      uint64_t* xbar = kK2XStage ? &xland[sidx] : &full[sidx];
      if constexpr (kK2XStage) {
        // natural rows land on xland; the permute into B-fragment units arrives on full
        if (lane == 0) {
          const uint32_t xb = x_bulk ? static_cast<uint32_t>(p.M) * (xvalid(k0, n0) + (n1 ? xvalid(k1, n1) : 0u)) : 0u;
          mbar_arrive_expect_tx(xbar, xb);
        }
        __syncwarp();
      }
      if constexpr (kXPrep) {
        if (lane == 0) {
          const uint8_t* xp = reinterpret_cast<const uint8_t*>(p.xperm);
          bulk_g2s(xs, xp + static_cast<long long>(k0) * kXTileBytes, n0 * kXTileBytes, &full[sidx],
                   policy_evict_last());
          if (n1) {
            bulk_g2s(xs + n0 * kXTileBytes, xp + static_cast<long long>(k1) * kXTileBytes,
                     n1 * kXTileBytes, &full[sidx], policy_evict_last());
          }
        }
      } else {
        for (int run = 0; run < 2; ++run) {
          const int kt = run ? k1 : k0, nr = run ? n1 : n0, off = run ? n0 : 0;
          if (nr == 0) continue;
          const long long kx = static_cast<long long>(kt) * TK;
          if (x_bulk) {
            // rows m < M: one bulk copy each (lane m); the part past `cols` is zeroed with
            // plain stores (only the final k-tile of K has one)
            const uint32_t vb = xvalid(kt, nr);
            const int tail16 = (nr * TK * 2 - static_cast<int>(vb)) / 16;
            for (int u = lane; u < p.M * tail16; u += 32) {
              const int m = u / tail16, q = u - m * tail16;
              *reinterpret_cast<uint4*>(xs + m * geo.x_row + off * TK * 2 + vb + q * 16) =
                  make_uint4(0, 0, 0, 0);
            }
            if (lane < p.M && vb) {
              bulk_g2s(xs + lane * geo.x_row + off * TK * 2, p.x + lane * p.ldx + kx, vb, xbar,
                       policy_evict_last());
            }
          } else {  // unaligned activations: plain loads
            const int per_row = nr * TK;
            for (int u = lane; u < p.M * per_row; u += 32) {
              const int m = u / per_row, e = u - m * per_row;
              unsigned short* xr = reinterpret_cast<unsigned short*>(xs + m * geo.x_row) + off * TK;
              xr[e] = (kx + e < p.cols) ? __ldg(p.x + m * p.ldx + kx + e) : static_cast<unsigned short>(0);
            }
          }
        }
      }
      __syncwarp();  // the lanes' plain stores happen-before lane 0's release
      if (!kK2XStage && lane == 0) mbar_arrive(&full[sidx]);
    };
    // kK2XStage: once stage st's natural rows landed, the producer warp permutes them into the
    // B-fragment units the consumers read (what amsq_xprep_kernel writes to global memory):
    // item (k-tile, batch row m, lane column tt) -> J 8-byte units; rows m >= M are zero
    auto permute_x = [&](int st, int sidx, uint32_t phase) {
      mbar_wait(&xland[sidx], phase);
      const uint8_t* xn = smem + sidx * geo.stage + geo.w_stage + geo.xnat_off;
      uint2* xf = reinterpret_cast<uint2*>(smem + sidx * geo.stage + geo.w_stage);
      const int nk = min(S, L - st * S), items = nk * MS * 4;
      constexpr int LK = T::kLaneK;
      for (int u = lane; u < items; u += 32) {
        const int ktl = u / (MS * 4), r = u - ktl * (MS * 4), m = r >> 2, tt = r & 3;
        uint32_t B[J][2];
        if (m < p.M) {
          const uint8_t* src = xn + m * geo.x_row + (ktl * TK + tt * LK) * 2;
          if constexpr (T::kFam == 4) {
            const uint4 a = *reinterpret_cast<const uint4*>(src);
            const uint4 b = *reinterpret_cast<const uint4*>(src + 16);
            const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
            bfrag_s4(w, B);
          } else {
            const uint2 a = *reinterpret_cast<const uint2*>(src);
            const uint2 b = *reinterpret_cast<const uint2*>(src + 8);
            const uint2 d = *reinterpret_cast<const uint2*>(src + 16);
            const uint32_t w[6] = {a.x, a.y, b.x, b.y, d.x, d.y};
            bfrag_s7(w, B);
          }
        } else {
#pragma unroll
          for (int j = 0; j < J; ++j) B[j][0] = B[j][1] = 0u;
        }
#pragma unroll
        for (int j = 0; j < J; ++j) xf[((ktl * J + j) * MS + m) * 4 + tt] = make_uint2(B[j][0], B[j][1]);
      }
      __syncwarp();  // every lane's units happen-before lane 0's release
      if (lane == 0) mbar_arrive(&full[sidx]);
    };
    // the group's row scales (fp32, x 2^14) for the epilogue, staged after the last copy is
    // issued: the consumers still have a ring's worth of stages to go, which hides the loads
    auto stage_scales = [&]() {
      for (int i = lane; i < G * 16; i += 32) {
        const long long n = static_cast<long long>(rt0) * 16 + i;
        sscale[i] = n < p.rows ? __half2float(__ushort_as_half(__ldg(p.scales + n))) * T::kPlace : 0.0f;
      }
    };
    // weights of the first ring-full of stages are independent of the previous kernel:
    // request them before griddepcontrol.wait
    // stage 0's weights do not depend on the previous kernel: request them before
    // griddepcontrol.wait. Later stages go weights-then-activations, so the TMA queue never
    // holds a ring's worth of weights in front of the activations the first stage needs.
    const int pre = min(nst, min(geo.stages, AMSQ_K2_PRE_W));
    if (lane == 0 && nst > 0) {
      for (int st = 0; st < pre; ++st) issue_w(st, st);
      for (int st = 1; st < 2 * geo.stages; ++st) prefetch_w(st);  // stages 1 .. 2*ring - 1
    }
    pdl_wait();  // activations may be produced by the previous kernel
    if (trace && lane == 0) trace[4] = clock64();
    int sidx = 0;
    uint32_t ph = 0;
    // kK2XStage: stage st - 1 is permuted after stage st's copies are issued (its rows are
    // then in flight behind them) when the ring is deep enough to hide the lag
    const bool xlag = geo.stages >= 3;
    int psidx = -1;
    uint32_t pph = 0;
    for (int st = 0; st < nst; ++st) {
      if (st >= pre) {
        if (st >= geo.stages) {
#if AMSQ_PRODUCER_SLEEP_NS > 0
          mbar_wait_sleep(&empty[sidx], ph ^ 1u, AMSQ_PRODUCER_SLEEP_NS);
#else
          mbar_wait(&empty[sidx], ph ^ 1u);
#endif
        }
        if (lane == 0) {
          issue_w(st, sidx);
          if (st >= geo.stages) prefetch_w(st + geo.stages);
        }
      }
      issue_x(st, sidx);
      if constexpr (kK2XStage) {
        if (!xlag) {
          permute_x(st, sidx, ph);
        } else {
          if (psidx >= 0) permute_x(st - 1, psidx, pph);
          psidx = sidx;
          pph = ph;
        }
      }
#if AMSQ_TRACE_STAGES
      if (trace && lane == 0 && st < 24) trace[32 + st] = clock64();
#endif
      if (++sidx == geo.stages) sidx = 0, ph ^= 1u;
    }
    if constexpr (kK2XStage) {
      if (psidx >= 0) permute_x(nst - 1, psidx, pph);
    }
    stage_scales();
    // the next call's first stages into L2 (its CTA j starts on an SM this grid frees): the
    // same group / rank / rotation arithmetic as above, on the successor's plan
    if (!AMSQ_K2_LEAN && p.next_w != nullptr && lane == 0) {
      const GroupPlan& Q = p.next_plan;
      const int nct = Q.n_groups * Q.csplit, KTn = p.next_k_tiles;
      for (int b = blockIdx.x; b < nct; b += gridDim.x) {
        const int gq = b / Q.csplit, rq = b - gq * Q.csplit;
        const int Gq = Q.size(gq), kpq = (KTn + Q.csplit - 1) / Q.csplit;
        const int kb2 = rq * kpq, ke2 = min(KTn, kb2 + kpq), L2n = ke2 - kb2;
        if (L2n <= 0) continue;
        const int rho2 = static_cast<int>(static_cast<long long>(gq) * L2n / Q.n_groups);
        const long long tile_b = static_cast<long long>(Gq) * p.next_tile_bytes;  // one k-tile
        const long long base = static_cast<long long>(Q.row0(gq)) * KTn * p.next_tile_bytes;
        long long want = p.next_pf_bytes;
        // from k-tile kb2 + rho2 to the end of the range, then wrapping to kb2
        const long long run0 = min(want, (L2n - rho2) * tile_b) & ~15LL;
        if (run0 > 0) bulk_prefetch_l2(p.next_w + base + (kb2 + rho2) * tile_b, static_cast<uint32_t>(run0));
        want -= run0;
        const long long run1 = min(want, rho2 * tile_b) & ~15LL;
        if (run1 > 0) bulk_prefetch_l2(p.next_w + base + kb2 * tile_b, static_cast<uint32_t>(run1));
      }
    }
  } else {
    // ------------------------------------------------------------------ consumers
    // the warp's kpw k-tiles x NOWN row tiles of a stage, branch-free for a fixed NOWN
    auto consume = [&](const uint8_t* sp, int nk, auto nown_c) {
      constexpr int NOWN = decltype(nown_c)::value;
#if AMSQ_K2_PIPE
      // both k-tiles of the warp's k-slot present: issue every shared-memory load of the two
      // k-tiles first, so the second k-tile's loads land under the first one's decode + MMAs
      if (geo.kpw == 2 && 2 * ks + 1 < nk) {
        uint32_t B0[NB][J][2], B1[NB][J][2];
        Frag<SCHEME> w0[NOWN], w1[NOWN];
        const uint8_t* tb0 = sp + (2 * ks * G + rl) * TILE;
        const uint8_t* tb1 = tb0 + G * TILE;
        load_bfrag<SCHEME, NB>(sp + geo.w_stage, geo, 2 * ks, g, t, B0);
#pragma unroll
        for (int i = 0; i < NOWN; ++i) w0[i] = load_frag<SCHEME>(tb0 + i * geo.wr * TILE, lane);
        load_bfrag<SCHEME, NB>(sp + geo.w_stage, geo, 2 * ks + 1, g, t, B1);
#pragma unroll
        for (int i = 0; i < NOWN; ++i) w1[i] = load_frag<SCHEME>(tb1 + i * geo.wr * TILE, lane);
#pragma unroll
        for (int i = 0; i < NOWN; ++i) {
          uint32_t A[J][4];
          decode_frag<SCHEME>(w0[i], A);
#pragma unroll
          for (int j = 0; j < J; ++j)
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) mma16816(acc[i][nb], A[j], B0[nb][j][0], B0[nb][j][1]);
        }
#pragma unroll
        for (int i = 0; i < NOWN; ++i) {
          uint32_t A[J][4];
          decode_frag<SCHEME>(w1[i], A);
#pragma unroll
          for (int j = 0; j < J; ++j)
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) mma16816(acc[i][nb], A[j], B1[nb][j][0], B1[nb][j][1]);
        }
        return;
      }
#endif
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const int kq = geo.kpw * ks + kk;
        if (kk < geo.kpw && kq < nk) {
          uint32_t B[NB][J][2];
          load_bfrag<SCHEME, NB>(sp + geo.w_stage, geo, kq, g, t, B);
          const uint8_t* tb = sp + (kq * G + rl) * TILE;
          Frag<SCHEME> wv[NOWN];
#pragma unroll
          for (int i = 0; i < NOWN; ++i) wv[i] = load_frag<SCHEME>(tb + i * geo.wr * TILE, lane);
#pragma unroll
          for (int i = 0; i < NOWN; ++i) {
            uint32_t A[J][4];
#if AMSQ_K2_MODE == 3  // profiling variant: MMA on masked raw words (no decode)
#pragma unroll
            for (int j = 0; j < J; ++j)
#pragma unroll
              for (int q = 0; q < 4; ++q) A[j][q] = wv[i].R[(j + q) & 3] & 0x3F003F00u;
#else
            decode_frag<SCHEME>(wv[i], A);
#endif
#if AMSQ_K2_MODE == 2  // profiling variant: decode without the tensor cores
#pragma unroll
            for (int j = 0; j < J; ++j)
              acc[i][0][j & 3] += __uint_as_float((A[j][0] ^ A[j][1] ^ A[j][2] ^ A[j][3] ^ B[0][j][0]) & 0x3F0F0F0Fu);
#else
#pragma unroll
            for (int j = 0; j < J; ++j)  // k-step outer: consecutive MMAs hit different accumulators
#pragma unroll
              for (int nb = 0; nb < NB; ++nb) mma16816(acc[i][nb], A[j], B[nb][j][0], B[nb][j][1]);
#endif
          }
        }
      }
    };
    int sidx = 0;
    uint32_t ph = 0;
    for (int st = 0; st < nst; ++st) {
      mbar_wait(&full[sidx], ph);
      if (trace && st == 0 && threadIdx.x == 0) trace[1] = globaltimer();
#if AMSQ_TRACE_STAGES  // profiling variant: stage landed (warp 0) / stage issued (producer)
      if (trace && threadIdx.x == 0 && st < 24) trace[8 + st] = clock64();
#endif
      const int nk = min(S, L - st * S);
      const uint8_t* sp = smem + sidx * geo.stage;
#if AMSQ_K2_MODE == 1
      if (false)
#endif
      switch (nown) {  // warp-uniform and fixed per warp
        case 1: consume(sp, nk, std::integral_constant<int, 1>{}); break;
        case 2: consume(sp, nk, std::integral_constant<int, 2>{}); break;
        case 3: if constexpr (MAXOWN >= 3) consume(sp, nk, std::integral_constant<int, 3>{}); break;
        case 4: if constexpr (MAXOWN >= 4) consume(sp, nk, std::integral_constant<int, 4>{}); break;
#if AMSQ_MAX_OWN1 > 4
        case 5: if constexpr (MAXOWN >= 5) consume(sp, nk, std::integral_constant<int, 5>{}); break;
        case 6: if constexpr (MAXOWN >= 6) consume(sp, nk, std::integral_constant<int, 6>{}); break;
        case 7: if constexpr (MAXOWN >= 7) consume(sp, nk, std::integral_constant<int, 7>{}); break;
        case 8: if constexpr (MAXOWN >= 8) consume(sp, nk, std::integral_constant<int, 8>{}); break;
#endif
        default: break;
      }
#if AMSQ_CONSUMER_PROXY_FENCE
      // generic-proxy reads of the stage before the producer's async-proxy (bulk copy)
      // rewrite of it (PTX memory model: cross-proxy WAR)
      fence_proxy_async_smem();
#endif
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[sidx]);
#if AMSQ_TRACE_STAGES
      if (trace && warp == kConsumerWarps - 1 && lane == 0 && st < 7) trace[56 + st] = clock64();
#endif
      if (++sidx == geo.stages) sidx = 0, ph ^= 1u;
    }
    if (trace && threadIdx.x == 0) trace[2] = globaltimer();
  }

  // ------------------------------------------------------------------ epilogue
  __syncwarp();
  __syncthreads();  // every stage consumed: the ring is free for the reduction
  if constexpr (CS > 1) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");  // peers started
  if (CS > 1 && geo.recv_in_ring) {
    // peers store their partials into this CTA's ring (recv below): announce that the ring is
    // idle here, and wait for the peers' announcements before storing into theirs
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  }
#if AMSQ_EPI_OLD  // A/B only: the round-1 epilogue (all 8*NB columns, integer indexing)
  const int nslots = S / geo.kpw;               // k-slots (a warp covers kpw k-tiles of a stage)
  float* red = reinterpret_cast<float*>(smem);  // [nslots][G][32][NB4]
  constexpr int NB4 = NB * 4;
  const int items = G * 32 * NB4;
  if (warp < kConsumerWarps) {
#pragma unroll
    for (int i = 0; i < MAXOWN; ++i) {
      if (i < nown) {
        float* dst = red + (static_cast<long long>(ks) * G + rl + i * geo.wr) * 32 * NB4 + lane * NB4;
#pragma unroll
        for (int nb = 0; nb < NB; ++nb)
#pragma unroll
          for (int e = 0; e < 4; ++e) dst[nb * 4 + e] = acc[i][nb][e];
      }
    }
  }
  __syncthreads();
  pdl_wait();  // outputs may still be read by the previous kernel
  // clusters: recv[C][items] -- rank q's partial of the items rank r finalises lands in
  // rank r's recv[q] (remote stores), one cluster barrier, then rank r sums in rank order
  const int Gs = (G + CS - 1) / CS;  // row tiles each rank finalises
  const int owned = Gs * 32 * NB4;   // items per rank
  float* recv = reinterpret_cast<float*>(smem + geo.recv_off);  // [CS][owned]
  auto store_y = [&](int it, float v) {
    const int r = it / (32 * NB4), rem = it - r * 32 * NB4;
    const int ln = rem / NB4, q = rem - ln * NB4, nb = q >> 2, e = q & 3;
    const int m = nb * 8 + 2 * (ln & 3) + (e & 1);
    const long long n = static_cast<long long>(rt0 + r) * 16 + (ln >> 2) + 8 * (e >> 1);
    if (m < p.M && n < p.rows) {
      const float sc = sscale[n - static_cast<long long>(rt0) * 16];
      p.y[static_cast<long long>(m) * p.ldy + n] = out_bits(v * sc, p.yscale, m);
    }
  };
  if (CS > 1 && geo.recv_in_ring) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    float v = 0.0f;
    for (int k = 0; k < nslots; ++k) v += red[static_cast<long long>(k) * items + it];  // slot order
    if constexpr (CS == 1) {
      store_y(it, v);
    } else {
      const uint32_t owner = static_cast<uint32_t>((it / (32 * NB4)) / Gs);
      float* dst = recv + static_cast<long long>(crank) * owned + (it - static_cast<int>(owner) * owned);
      if (owner == crank) {
        *dst = v;
      } else {
        uint32_t remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(dst)), "r"(owner));
        asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(remote), "f"(v) : "memory");
      }
    }
  }
  if constexpr (CS > 1) {
    __syncwarp();
    cluster_sync_all();  // every rank's partials have landed in their owners' recv
    const int i0 = min(G, static_cast<int>(crank) * Gs) * 32 * NB4;
    const int i1 = min(G, static_cast<int>(crank + 1) * Gs) * 32 * NB4;
    for (int it = i0 + threadIdx.x; it < i1; it += blockDim.x) {
      float v = 0.0f;
#pragma unroll
      for (int r = 0; r < CS; ++r) v += recv[static_cast<long long>(r) * owned + (it - i0)];  // rank order
      store_y(it, v);
    }
  }
#else
  // Only the M valid batch columns are reduced (at M = 1 that is 1/8 of the accumulator
  // elements), in a [slot][row tile][m][16 rows] layout, with no runtime integer division.
  const int nslots = S / geo.kpw;               // k-slots (a warp covers kpw k-tiles of a stage)
  float* red = reinterpret_cast<float*>(smem);  // [nslots][G][MS][16]
  const int M = p.M;
  if (warp < kConsumerWarps) {
#pragma unroll
    for (int i = 0; i < MAXOWN; ++i) {
      if (i < nown) {
        float* dst = red + ((static_cast<long long>(ks) * G + rl + i * geo.wr) * MS) * 16;
#pragma unroll
        for (int nb = 0; nb < NB; ++nb)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int m = nb * 8 + 2 * t + (e & 1), row = g + 8 * (e >> 1);
            if (m < M) dst[m * 16 + row] = acc[i][nb][e];
          }
      }
    }
  }
  __syncthreads();
  pdl_wait();  // outputs may still be read by the previous kernel
  const int M16 = M * 16;                      // items per row tile: (m, row), m < M
  const int items = G * M16;
  const int slot = G * MS * 16;                // floats per k-slot in red
  const float inv_m16 = 1.0f / static_cast<float>(M16);
  // item -> (row tile r, q = m*16 + row); exact: (it + 0.5) / M16 is never within 2^-9 of an
  // integer for it < 2^16, far above fp32 rounding
  auto split = [&](int it, int& r, int& q) {
    r = __float2int_rz((static_cast<float>(it) + 0.5f) * inv_m16);
    q = it - r * M16;
  };
  auto store_y = [&](int r, int q, float v) {
    const int m = q >> 4, row = q & 15;
    const long long n = static_cast<long long>(rt0 + r) * 16 + row;
    if (n < p.rows) {
#if AMSQ_K2_LEAN  // A/B only: no bf16 / fused-TP epilogue branches
      const unsigned short b = __half_as_ushort(__float2half_rn(v * sscale[r * 16 + row]));
      constexpr bool tp_off = true;
#else
      const unsigned short b = out_bits(v * sscale[r * 16 + row], p.yscale, m);
      const bool tp_off = p.tp_ranks == 0;
#endif
      if (tp_off) {
        p.y[static_cast<long long>(m) * p.ldy + n] = b;
      } else {  // fused TP: the element lands in every rank's gathered output (NVLink stores)
        const long long off = static_cast<long long>(m) * p.ldy + p.tp_col0 + n;
        for (int rr = 0; rr < p.tp_ranks; ++rr) p.tp_y[rr][off] = b;
      }
    }
  };
  if constexpr (CS == 1) {
    for (int it = threadIdx.x; it < items; it += blockDim.x) {
      int r, q;
      split(it, r, q);
      const float* src = red + r * MS * 16 + q;
      float v = 0.0f;
      for (int k = 0; k < nslots; ++k) v += src[k * slot];  // slot order
      store_y(r, q, v);
    }
  } else {
    // clusters: rank r finalises row tiles [r*Gs, (r+1)*Gs); rank q's partial of them lands in
    // rank r's recv[q] (remote stores), one cluster barrier, then rank r sums in rank order
    const int Gs = (G + CS - 1) / CS;
    const int owned = Gs * M16;  // items per rank
    const float inv_gs = 1.0f / static_cast<float>(Gs);
    float* recv = reinterpret_cast<float*>(smem + geo.recv_off);  // [CS][owned]
    if (geo.recv_in_ring) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    for (int it = threadIdx.x; it < items; it += blockDim.x) {
      int r, q;
      split(it, r, q);
      const float* src = red + r * MS * 16 + q;
      float v = 0.0f;
      for (int k = 0; k < nslots; ++k) v += src[k * slot];
      const int owner = __float2int_rz((static_cast<float>(r) + 0.5f) * inv_gs);
      float* dst = recv + static_cast<long long>(crank) * owned + (it - owner * owned);
      if (owner == static_cast<int>(crank)) {
        *dst = v;
      } else {
        uint32_t remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(dst)), "r"(owner));
        asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(remote), "f"(v) : "memory");
      }
    }
    __syncwarp();
    cluster_sync_all();  // every rank's partials have landed in their owners' recv
    const int i0 = min(G, static_cast<int>(crank) * Gs) * M16;
    const int i1 = min(G, static_cast<int>(crank + 1) * Gs) * M16;
    for (int it = i0 + threadIdx.x; it < i1; it += blockDim.x) {
      float v = 0.0f;
#pragma unroll
      for (int rr = 0; rr < CS; ++rr) v += recv[static_cast<long long>(rr) * owned + (it - i0)];  // rank order
      int r, q;
      split(it, r, q);
      store_y(r, q, v);
    }
  }
#endif
  if (p.tp_ranks) asm volatile("fence.acq_rel.sys;" ::: "memory");  // peer stores before the barrier
  if (trace && threadIdx.x == 0) trace[3] = globaltimer();
}

}  // namespace dev

template <int SCHEME, int NB>
static dev::K2Geom k2_geometry(const LinearParams& p, int* smem_bytes) {
  // wr = warps sharing a k-slot (row-tile interleave): the smallest power of two giving each
  // consumer warp <= 2 row tiles (<= 4 beyond 32 tiles); every warp takes 2 k-tiles of each
  // stage, so a stage is S = 2 * 16 / wr k-tiles x G row tiles (<= 64 tiles, ~32 KB)
  using T = dev::Traits<SCHEME>;
  dev::K2Geom geo{};
  const int G = p.plan.g_big;
  // wr: the smallest divisor of the consumer-warp count giving each warp <= 2 row tiles
  // (<= 4 when even all warps on one k-slot cannot)
  const int own_target = NB == 1   ? (AMSQ_MAX_OWN1 > AMSQ_OWN_TARGET ? AMSQ_MAX_OWN1 : AMSQ_OWN_TARGET)
                         : NB == 2 ? AMSQ_OWN_TARGET
                                   : AMSQ_MAX_OWN4;
  int wr = dev::kConsumerWarps;
  for (int d = 1; d <= dev::kConsumerWarps; ++d) {
    if (dev::kConsumerWarps % d == 0 && (G + d - 1) / d <= own_target) {
      wr = d;
      break;
    }
  }
  geo.wr = wr;
  // kpw k-tiles per warp and stage: 2 (B fragments and loop overhead amortised over twice the
  // tiles) unless that leaves fewer than AMSQ_KPW2_MIN_STAGES ring stages (large G x S tiles,
  // or M <= 16's double activation bytes), or a warp already owns > 4 row tiles
  const int budget = (AMSQ_CTAS_PER_SM > 1 ? 113 : 227) * 1024 - 1024 - G * 16 * 4;
  const int target = T::kFam == 7 ? 96 : 16;  // lanes' LDS hit distinct banks
  auto shape = [&](int kpw) {
    geo.kpw = kpw;
    geo.S = kpw * (dev::kConsumerWarps / wr);
    geo.w_stage = (geo.S * G * T::kTileBytes + 127) / 128 * 128;
    const int x_raw = geo.S * T::kTK * 2;
    geo.x_row = x_raw + ((target - x_raw % 128) + 128) % 128;
    geo.xrows = (dev::kK2XPrep && NB >= 2) ? 8 * NB : p.M;
    const int x_frag = geo.S * T::kJ * 8 * NB * 4 * 8;  // B-fragment units of a stage
    geo.xnat_off = dev::kK2XStage ? x_frag : 0;        // natural rows behind them
    const int x_stage = dev::kK2XStage                   ? x_frag + geo.xrows * geo.x_row
                        : (dev::kK2XPrep && NB >= 2) ? x_frag
                                                       : geo.xrows * geo.x_row;
    geo.stage = (geo.w_stage + x_stage + 127) / 128 * 128;
    geo.stages = budget / geo.stage;
    if (geo.stages > 6) geo.stages = 6;
  };
  shape(2);
  if ((G + wr - 1) / wr > dev::OwnCap<NB>::value || geo.stages < (NB >= 2 ? AMSQ_KPW2_MIN_STAGES : AMSQ_KPW2_MIN_STAGES1)) {
    shape(1);
  }
  // the epilogue reuses the ring for the k-slot partials: (S/kpw) x G x 32 x NB*4 floats. A
  // cluster's receive buffer ([C][ceil(G/C) x 32 x NB*4] floats) goes after the ring when the
  // leftover space holds it -- peers may then store as soon as they are done -- else into the
  // ring behind the partials, fenced by an extra cluster barrier.
  const long long red = static_cast<long long>(geo.S / geo.kpw) * G * 32 * NB * 4 * 4;
  const int C = p.plan.csplit;
  const long long recv = C > 1 ? static_cast<long long>(C) * ((G + C - 1) / C) * 32 * NB * 4 * 4 : 0;
  if (AMSQ_RECV_STEAL && recv > 0 && geo.stages >= 4 && geo.stages * geo.stage + recv > budget) {
    --geo.stages;  // give a ring stage to the receive buffer rather than fence it with a barrier
  }
  if (recv > 0 && geo.stages * geo.stage + recv <= budget && geo.stages * geo.stage >= red) {
    geo.recv_off = geo.stages * geo.stage;
    geo.recv_in_ring = 0;
  } else {
    while (geo.stages * geo.stage < red + recv) ++geo.stages;
    geo.recv_off = static_cast<int>(red);
    geo.recv_in_ring = recv > 0 ? 1 : 0;
  }
  geo.bar_off = geo.recv_in_ring || recv == 0 ? geo.stages * geo.stage
                                              : static_cast<int>((geo.recv_off + recv + 127) / 128 * 128);
  *smem_bytes = geo.bar_off + (dev::kK2XStage ? 3 : 2) * geo.stages * 8 + G * 16 * 4 + 16;
  return geo;
}

template <int SCHEME, int NB, int CS>
static cudaError_t launch_linear_m(const LinearParams& p, cudaStream_t s) {
  int smem = 0;
  const dev::K2Geom geo = k2_geometry<SCHEME, NB>(p, &smem);
  if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
  static std::atomic<uint64_t> configured{0};  // per template instance, one bit per device
  if (const cudaError_t e = opt_in_max_smem(dev::amsq_linear_kernel<SCHEME, NB, CS>, configured);
      e != cudaSuccess) {
    return e;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(p.plan.n_groups * CS));
  cfg.blockDim = dim3(dev::kK2Threads);
  cfg.dynamicSmemBytes = static_cast<size_t>(smem);
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  int na = 1;
  if constexpr (CS > 1) {
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = CS;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    na = 2;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, dev::amsq_linear_kernel<SCHEME, NB, CS>, p, geo);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <int SCHEME, int NB>
static cudaError_t launch_linear_t(const LinearParams& p, cudaStream_t s) {
  if constexpr (NB >= 2 && dev::kK2XPrep) {
    // activations first (PDL-chained: waits for whoever produced x, lets the linear start
    // streaming weights as soon as it is scheduled)
    const int MS = 8 * NB;
    const int items = p.k_tiles * MS * 4;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>((items + 127) / 128));  // more SMs: latency-bound
    cfg.blockDim = dim3(128);
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
  switch (p.plan.csplit) {
    case 1: return launch_linear_m<SCHEME, NB, 1>(p, s);
    case 2: return launch_linear_m<SCHEME, NB, 2>(p, s);
    case 4: return launch_linear_m<SCHEME, NB, 4>(p, s);
    case 8: return launch_linear_m<SCHEME, NB, 8>(p, s);
    default: return cudaErrorInvalidConfiguration;
  }
}

// batches of <= 32 rows of one scheme (the caller splits larger batches)
template <int SCHEME>
cudaError_t launch_linear_scheme(const LinearParams& p, cudaStream_t s) {
  if (p.plan.n_groups <= 0) return cudaSuccess;
  if (p.M > 16 && p.plan.g_big > dev::kConsumerWarps * dev::OwnCap<4>::value) {
    // groups too tall for the M <= 32 kernel's accumulators: two M <= 16 launches
    LinearParams a = p, b = p;
    a.M = 16;
    b.M = p.M - 16;
    b.x = p.x + 16 * p.ldx;
    b.y = p.y + 16 * p.ldy;
    if (p.yscale) b.yscale = p.yscale + 16;
    if (p.tp_ranks) b.tp_col0 = p.tp_col0 + 16 * p.ldy;
    const cudaError_t e = launch_linear_scheme<SCHEME>(a, s);
    return e != cudaSuccess ? e : launch_linear_scheme<SCHEME>(b, s);
  }
  if (p.M <= 8) return launch_linear_t<SCHEME, 1>(p, s);
  if (p.M <= 16 || AMSQ_K2_MAX_BATCH <= 16) return launch_linear_t<SCHEME, 2>(p, s);
  return launch_linear_t<SCHEME, 4>(p, s);
}

}  // namespace amsqb
