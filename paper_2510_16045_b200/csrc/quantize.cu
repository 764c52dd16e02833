// quantize.cu -- device-side quantize: the reference's quantize_tensor
// (quantize.hpp:188-216 = pad_cols_to + rtn_quantize 112-131 + ams_share 138-184 + pack_row,
// packing.hpp:216-239) on the GPU, producing the reference stream (scales u16[rows], payload
// u16[rows][wpr]) bit for bit. The offline Adaptive Searching stays the reference's algorithm;
// this only moves it off the host for 70B-scale tensors (the CPU quantizer does ~10-20 M
// weights/s).
//
// One CTA per row: (1) max |w| and the non-finite check (block reduction), the binary16 stored
// scale (quantize.hpp:72-93); (2) every thread quantizes whole packing blocks: round-to-nearest
// over the sorted value grid (format.hpp:165-182), the per-group shared-LSB search scored in
// double (ties keep bit 0; groups reaching into padding pinned to 0), then the block's segments
// and shared slots are packed into its words. All float / double arithmetic is written with
// explicit _rn intrinsics, so no FMA contraction can change a bit relative to the host.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "host_core.hpp"
#include "kernels.h"

namespace amsqb {

void count_launch();

namespace dev {

__global__ void __launch_bounds__(128) amsq_quantize_kernel(QuantTables tb, const float* __restrict__ w,
                                                            long long ldw, long long cols, long long pc,
                                                            long long wpr, unsigned short* __restrict__ scales,
                                                            unsigned short* __restrict__ payload,
                                                            int* __restrict__ err) {
  __shared__ float red[4];
  __shared__ float s_scale;
  const long long r = blockIdx.x;
  const float* row = w + r * ldw;
  // (1) max |w| over the logical columns (padding is 0), non-finite check
  float mx = 0.0f;
  bool bad = false;
  for (long long c = threadIdx.x; c < cols; c += blockDim.x) {
    const float v = row[c];
    bad |= !isfinite(v);
    mx = fmaxf(mx, fabsf(v));
  }
  if (__syncthreads_or(bad)) {
    if (threadIdx.x == 0) atomicOr(err, 1);  // quantize.hpp:77 "non-finite weight"
    return;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    mx = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
    const float scale = mx == 0.0f ? 1.0f : __fdiv_rn(mx, tb.maxmag);
    unsigned short h = static_cast<unsigned short>(__half_as_ushort(__float2half_rn(scale)) & 0x7FFFu);
    if (h >= 0x7C00u) atomicOr(err, 2);  // quantize.hpp:89 "channel scale overflows"
    if (h == 0) h = 1;
    scales[r] = h;
    s_scale = __half2float(__ushort_as_half(h));
  }
  __syncthreads();
  const float sc = s_scale;
  // (2) blocks of the padded row
  const int B = tb.block;
  const long long nblk = pc / B;
  for (long long blk = threadIdx.x; blk < nblk; blk += blockDim.x) {
    uint8_t code[64];
    const long long c0 = blk * B;
    for (int i = 0; i < B; ++i) {
      const float v = c0 + i < cols ? row[c0 + i] : 0.0f;
      const float q = __fdiv_rn(v, sc);
      // round_to_nearest (format.hpp:165-182)
      uint8_t cd;
      if (!(q > tb.grid_v[0])) {
        cd = tb.grid_c[0];
      } else if (q >= tb.grid_v[tb.ngrid - 1]) {
        cd = tb.grid_c[tb.ngrid - 1];
      } else {
        int lo = 0, hi = tb.ngrid - 1;  // grid_v[lo] < q <= grid_v[hi]: lower_bound = hi
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (tb.grid_v[mid] < q) lo = mid; else hi = mid;
        }
        const double dlo = __dsub_rn(static_cast<double>(q), static_cast<double>(tb.grid_v[lo]));
        const double dhi = __dsub_rn(static_cast<double>(tb.grid_v[hi]), static_cast<double>(q));
        const uint8_t cl = tb.grid_c[lo], ch = tb.grid_c[hi];
        if (dlo != dhi) {
          cd = dlo < dhi ? cl : ch;
        } else if ((cl & 1u) == 0 && (ch & 1u) == 0) {
          cd = fabsf(tb.grid_v[lo]) <= fabsf(tb.grid_v[hi]) ? cl : ch;
        } else {
          cd = (cl & 1u) == 0 ? cl : ch;
        }
      }
      code[i] = cd;
    }
    // ams_share over groups of k (quantize.hpp:138-184); with_lsb collapses -0 to +0
    if (tb.k > 1) {
      for (int g0 = 0; g0 < B; g0 += tb.k) {
        unsigned bit = 0;
        if (c0 + g0 + tb.k <= cols) {
          double e0 = 0.0, e1 = 0.0;
          for (int i = g0; i < g0 + tb.k; ++i) {
            const float v = row[c0 + i];
            const unsigned a0 = code[i] & ~1u, a1 = a0 | 1u;
            const unsigned z0 = a0 == static_cast<unsigned>(tb.sign_mask) ? 0u : a0;
            const unsigned z1 = a1 == static_cast<unsigned>(tb.sign_mask) ? 0u : a1;
            const double d0 = __dsub_rn(static_cast<double>(__fmul_rn(tb.val[z0], sc)), static_cast<double>(v));
            const double d1 = __dsub_rn(static_cast<double>(__fmul_rn(tb.val[z1], sc)), static_cast<double>(v));
            e0 = __dadd_rn(e0, __dmul_rn(d0, d0));
            e1 = __dadd_rn(e1, __dmul_rn(d1, d1));
          }
          bit = e1 < e0 ? 1u : 0u;
        }
        for (int i = g0; i < g0 + tb.k; ++i) {
          unsigned c = (code[i] & ~1u) | bit;
          if (c == static_cast<unsigned>(tb.sign_mask)) c = 0;
          code[i] = static_cast<uint8_t>(c);
        }
      }
    }
    // pack_block (packing.hpp:159-181): segments, then the groups' shared bits
    uint16_t words[17];
    for (int q = 0; q < tb.wpb; ++q) words[q] = 0;
    for (int i = 0; i < B; ++i) {
      for (int j = 0; j < tb.segs; ++j) {
        const int e = i * tb.segs + j;
        const unsigned bits = (static_cast<unsigned>(code[i]) >> tb.seg_shift[e]) & ((1u << tb.seg_width[e]) - 1u);
        words[tb.seg_word[e]] = static_cast<uint16_t>(words[tb.seg_word[e]] | (bits << tb.seg_bit[e]));
      }
    }
    for (int gq = 0; gq < tb.nshared; ++gq) {
      const unsigned bit = code[gq * tb.k] & 1u;
      words[tb.sh_word[gq]] = static_cast<uint16_t>(words[tb.sh_word[gq]] | (bit << tb.sh_bit[gq]));
    }
    unsigned short* out = payload + r * wpr + blk * tb.wpb;
    for (int q = 0; q < tb.wpb; ++q) out[q] = words[q];
  }
}

}  // namespace dev

QuantTables make_quant_tables(const Scheme& s) {
  QuantTables t{};
  t.scheme_id = s.id;
  t.block = s.block;
  t.wpb = s.words_per_block;
  t.segs = s.segs_per_weight;
  t.k = s.k;
  t.sign_mask = static_cast<int>(s.sign_mask());
  const unsigned n = s.code_count();
  for (unsigned c = 0; c < n; ++c) t.val[c] = decode(s, c);
  // format.hpp:119-131: negatives reversed, the canonical +0, positives
  int g = 0;
  for (unsigned mag = n / 2 - 1; mag >= 1; --mag) {
    t.grid_v[g] = t.val[s.sign_mask() | mag];
    t.grid_c[g++] = static_cast<uint8_t>(s.sign_mask() | mag);
  }
  t.grid_v[g] = 0.0f;
  t.grid_c[g++] = 0;
  for (unsigned mag = 1; mag < n / 2; ++mag) {
    t.grid_v[g] = t.val[mag];
    t.grid_c[g++] = static_cast<uint8_t>(mag);
  }
  t.ngrid = g;
  t.maxmag = t.grid_v[g - 1];
  for (int i = 0; i < s.block; ++i) {
    for (int j = 0; j < s.segs_per_weight; ++j) {
      const Segment sg = segment(s, i, j);
      const int e = i * s.segs_per_weight + j;
      t.seg_word[e] = sg.word, t.seg_bit[e] = sg.bit, t.seg_width[e] = sg.width, t.seg_shift[e] = sg.code_shift;
    }
  }
  t.nshared = shared_groups(s);
  for (int q = 0; q < t.nshared; ++q) {
    int wd, bt;
    shared_slot(s, q, &wd, &bt);
    t.sh_word[q] = static_cast<uint8_t>(wd), t.sh_bit[q] = static_cast<uint8_t>(bt);
  }
  return t;
}

cudaError_t launch_quantize(const QuantTables& tb, const float* w, long long rows, long long ldw,
                            long long cols, long long pc, long long wpr, unsigned short* scales,
                            unsigned short* payload, int* err, cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  dev::amsq_quantize_kernel<<<static_cast<unsigned>(rows), 128, 0, s>>>(tb, w, ldw, cols, pc, wpr, scales,
                                                                      payload, err);
  count_launch();
  return cudaGetLastError();
}

}  // namespace amsqb
