// kernels.h -- host-visible launch interface of the sm_100a kernels (kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <vector_types.h>

namespace amsqb {

// The row-group plan of a weight (device_layout.hpp): group g covers row tiles
// [row0(g), row0(g) + size(g)), g_big tiles for g < n_big, g_big - 1 after.
struct GroupPlan {
  int n_groups, g_big, n_big, csplit;
  __host__ __device__ int row0(int g) const {
    return g < n_big ? g * g_big : n_big * g_big + (g - n_big) * (g_big - 1);
  }
  __host__ __device__ int size(int g) const { return g < n_big ? g_big : g_big - 1; }
};

struct RestoreParams {
  int scheme_id;
  const uint8_t* w;
  const unsigned short* scales;  // fp16 bits [rows]
  long long rows, cols, padded_cols;
  int row_tiles, k_tiles;
  GroupPlan plan;
  unsigned short* grid_out;  // [rows][padded_cols] grid bits, or null
  float* f32_out;            // [rows][cols] w*s, or null
  unsigned short* f16_out;   // [rows][cols] fp16(w*s), or null
};

struct LinearParams {
  int scheme_id;
  const uint8_t* w;
  const unsigned short* scales;
  const unsigned short* x;  // [M][ldx] fp16 (logical cols)
  uint2* xperm;             // workspace: x in B-fragment order, [k_tiles][J][8*NB][4] units
  unsigned short* y;        // [M][ldy] fp16 (bf16 when yscale != null)
  const float* yscale;      // bf16 activations: per batch row 2^-e (undoes amsq_x_bf16 scaling)
  // fused tensor-parallel epilogue (amsq_linear_tp_fused; tp_ranks = 0: off): every output
  // element also goes to column tp_col0 + n of each rank's [M][ldy] buffer tp_y[r] (peer
  // memory over NVLink), and each CTA ends with a system-scope fence
  int tp_ranks;
  unsigned short* const* tp_y;  // device array [tp_ranks]
  long long tp_col0;             // element offset of this launch's (m = 0, n = 0) in tp_y[r]
  // cross-call L2 prefetch (amsq_linear_chain): once its last stage is issued, CTA j pulls the
  // first next_pf_bytes of what CTA j (j + grid, ...) of the NEXT call will stream into L2
  const uint8_t* next_w;        // null: off
  GroupPlan next_plan;
  int next_k_tiles, next_tile_bytes, next_pf_bytes;
  long long rows, cols, ldx, ldy;
  int M;                    // <= 16 per launch
  int row_tiles, k_tiles;
  GroupPlan plan;
  unsigned long long* trace;  // profiling only: per-CTA globaltimer stamps (null = off)
};

// K3 (kernels_tc.cu): tcgen05 fused linear for 16 < M <= 256 per launch.
struct TcParams {
  int scheme_id;
  const uint8_t* w;
  const unsigned short* scales;
  const unsigned short* xk;  // workspace: activations prepped into [K/8][Np][8] (>= Np*KT*TK)
  unsigned short* y;         // [M][ldy] fp16 (bf16 when yscale != null)
  const float* yscale;       // bf16 activations: per batch row 2^-e, or null
  long long rows, ldy;
  int M, Np;                 // batch rows; Np = round_up(M, 16) <= 256
  int row_tiles, k_tiles;
  GroupPlan plan;
  unsigned long long* trace;  // profiling only: per-CTA globaltimer stamps (null = off)
};

// Opt a kernel into 227 KB of dynamic shared memory on the CURRENT device. The attribute is
// per function and per device, so `done` keeps one bit per device ordinal; two first callers
// racing both set it (idempotent), never neither.
template <typename Kernel>
cudaError_t opt_in_max_smem(Kernel* fn, std::atomic<uint64_t>& done) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = dev < 64 ? (1ull << dev) : 0ull;
  if (bit && (done.load(std::memory_order_acquire) & bit)) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (e == cudaSuccess && bit) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

cudaError_t launch_restore(const RestoreParams& p, cudaStream_t s);

// Device quantize (quantize.cu): per-scheme value grid and packing map, passed by value.
struct QuantTables {
  int scheme_id, block, wpb, segs, k, sign_mask, ngrid, nshared;
  float maxmag;
  float val[64];      // value of each raw code (format.hpp:82-93)
  float grid_v[64];   // sorted grid (format.hpp:119-131) and its codes
  uint8_t grid_c[64];
  uint8_t seg_word[128], seg_bit[128], seg_width[128], seg_shift[128];  // [weight * segs + j]
  uint8_t sh_word[16], sh_bit[16];                                      // shared slot of group g
};
struct Scheme;
QuantTables make_quant_tables(const Scheme& s);
// err: device int, OR-ed with 1 (non-finite weight) / 2 (scale overflows binary16).
cudaError_t launch_quantize(const QuantTables& tb, const float* w, long long rows, long long ldw,
                            long long cols, long long pc, long long wpr, unsigned short* scales,
                            unsigned short* payload, int* err, cudaStream_t s);
cudaError_t launch_linear_tc(const TcParams& p, const unsigned short* x, long long ldx,
                             long long cols, cudaStream_t s);
constexpr int kTcMaxBatch = 256;
// K3 CTA-pair mode (cta_group::2): -1 = the measured rule, 0 = never, 1 = whenever no K split is
// chosen and there are >= 2 row blocks. Returns the previous setting.
int tc_set_pair_knob(int v);
cudaError_t launch_linear(const LinearParams& p, cudaStream_t s);
// Fused-TP flag barrier (one tiny launch per call): publish epoch e = *epoch + 1 into every
// rank's flag array at index `rank`, wait until all ranks published e here, then *epoch = e.
// Gives up after timeout_ns and sets *error (no hang on a missing peer).
cudaError_t launch_tp_barrier(unsigned int* const* peer_flags, unsigned int* my_flags,
                              unsigned int* epoch, unsigned int* error, int rank, int nranks,
                              unsigned long long timeout_ns, cudaStream_t s);
cudaError_t launch_unshard(const unsigned short* in, int P, int batch, int n, unsigned short* out,
                           cudaStream_t s);
#ifndef AMSQ_K2_XSTAGE  // 1: K2's producer warp permutes natural activation rows into B-fragment
#define AMSQ_K2_XSTAGE 0  // units in shared memory (no prep kernel, no consumer PRMTs)
#endif
#ifndef AMSQ_K2_MAX_BATCH  // batch rows per K2 launch: 16 (NB <= 2) or 32 (NB = 4 for 17..32)
#define AMSQ_K2_MAX_BATCH 32
#endif
int linear_max_batch_per_launch();
// K2 for one scheme (k2.cuh; explicit instances in k2_s<id>.cu), batch <= AMSQ_K2_MAX_BATCH.
template <int SCHEME>
cudaError_t launch_linear_scheme(const LinearParams& p, cudaStream_t s);
// bf16 activations -> fp16 scaled by 2^e per row (max |x| 2^e in [2^14, 2^15)); yscale[m] = 2^-e.
cudaError_t launch_x_bf16_prep(const unsigned short* x, long long ldx, long long cols, int M,
                               unsigned short* xh, float* yscale, cudaStream_t s);
uint64_t kernel_launch_count();

}  // namespace amsqb
