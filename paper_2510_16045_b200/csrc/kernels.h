// kernels.h -- host-visible launch interface of the sm_100a kernels (kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector_types.h>

namespace amsqb {

// Fixed persistent grid of the stream-K linear (one CTA per SM of the 148-SM B200): the
// split-K partition, and therefore the fp32 reduction order, depends only on the shape,
// never on the device it runs on.
constexpr long long kSMs = 148;
constexpr long long kMaxGridCTAs = kSMs;

struct RestoreParams {
  int scheme_id;
  const uint8_t* w;
  const unsigned short* scales;  // fp16 bits [rows]
  long long rows, cols, padded_cols;
  int row_tiles, k_tiles;
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
  unsigned short* y;        // [M][ldy] fp16
  float* partials;          // [(grid + row_blocks)][16][256] fp32
  int* counters;            // [row_blocks][8 32-row slices], zero between launches
  long long rows, cols, ldx, ldy;
  int M;                    // <= 16 per launch
  int row_blocks, k_tiles;
  int dry;                  // profiling only: consumers skip decode/MMA (measures the stream)
  unsigned long long* trace;  // profiling only: per-CTA globaltimer stamps (null = off)
};

cudaError_t launch_restore(const RestoreParams& p, cudaStream_t s);
cudaError_t launch_linear(const LinearParams& p, cudaStream_t s);
cudaError_t launch_unshard(const unsigned short* in, int P, int batch, int n, unsigned short* out,
                           cudaStream_t s);
long long linear_grid(long long units, int M);
int linear_max_batch_per_launch();
uint64_t kernel_launch_count();

}  // namespace amsqb
