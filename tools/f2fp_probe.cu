// tools/f2fp_probe.cu -- is the sm_100a hardware FP6 unpack (cvt.rn.f16x2.e2m3x2 ->
// F2FP.F16.E2M3.UNPACK_B) usable as the AMS decode?
//  (1) semantics: every byte value 0..255 (top two bits = garbage?) vs the e2m3 table;
//  (2) throughput per SM of F2FP alone, LOP3 alone, IMAD alone, and F2FP mixed with LOP3 /
//      IMAD (does it issue on a third pipe?).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/f2fp_probe tools/f2fp_probe.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t f2fp(uint32_t a) {
  uint32_t r;
  asm volatile("{.reg .b16 lo, hi; mov.b32 {lo, hi}, %1; cvt.rn.f16x2.e2m3x2 %0, lo;}"
               : "=r"(r) : "r"(a));
  return r;
}
__device__ __forceinline__ uint32_t f2fp_hi(uint32_t a) {
  uint32_t r;
  asm volatile("{.reg .b16 lo, hi; mov.b32 {lo, hi}, %1; cvt.rn.f16x2.e2m3x2 %0, hi;}"
               : "=r"(r) : "r"(a));
  return r;
}
__device__ __forceinline__ uint32_t lop(uint32_t a, uint32_t b) {
  uint32_t d;
  asm volatile("lop3.b32 %0, %1, %2, 0x3E3E3E3E, 0xEA;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b) {
  uint32_t d;
  asm volatile("mad.lo.u32 %0, %1, 5, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

__global__ void semantics(uint32_t* out) {
  const uint32_t b = threadIdx.x;  // byte value 0..255, paired with itself
  out[b] = f2fp(b | (b << 8));
}

template <int MODE>
__global__ void tput(uint32_t seed, uint32_t* sink, long long* cycles, int iters) {
  uint32_t v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = seed * (threadIdx.x + 1) + i * 0x01010101u;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) v[i] = f2fp(v[i]);                              // F2FP only
      if (MODE == 1) v[i] = lop(v[i], v[(i + 1) & 7]);                // LOP3 only
      if (MODE == 2) v[i] = imad(v[i], v[(i + 1) & 7]);               // IMAD only
      if (MODE == 3) { v[i] = f2fp(v[i]); v[i] = lop(v[i], v[(i + 3) & 7]); }   // F2FP + LOP3
      if (MODE == 4) { v[i] = f2fp(v[i]); v[i] = imad(v[i], v[(i + 3) & 7]); }  // F2FP + IMAD
      if (MODE == 5) { v[i] = lop(v[i], v[(i + 3) & 7]); v[i] = imad(v[i], v[(i + 5) & 7]); }
      if (MODE == 6) { v[i] = f2fp(v[i]) ^ f2fp_hi(v[i]); }          // 2 F2FP + LOP3
    }
  }
  const long long t1 = clock64();
  uint32_t x = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) x ^= v[i];
  if (x == 0x1234567u) *sink = x;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

static float e2m3(uint32_t c) {
  const int s = (c >> 5) & 1, e = (c >> 3) & 3, m = c & 7;
  const float v = e == 0 ? m * 0.125f : std::ldexp(1.0f + m / 8.0f, e - 1);
  return s ? -v : v;
}

int main() {
  uint32_t *d, h[256];
  cudaMalloc(&d, 256 * 4);
  semantics<<<1, 256>>>(d);
  cudaMemcpy(h, d, 256 * 4, cudaMemcpyDeviceToHost);
  int bad = 0, bad_low6 = 0;
  for (uint32_t b = 0; b < 256; ++b) {
    __half_raw lo;
    lo.x = static_cast<unsigned short>(h[b] & 0xFFFF);
    const float got = __half2float(__half(lo));
    const float want = e2m3(b & 63);
    if (got != want || std::signbit(got) != std::signbit(want)) {
      ++bad;
      if (b < 64) ++bad_low6;
      if (bad <= 4) printf("byte 0x%02x -> %04x (%g) want %g\n", b, h[b] & 0xFFFF, got, want);
    }
  }
  printf("semantics: %d/256 bytes differ from e2m3(byte & 63) (%d of the 64 canonical codes)\n",
         bad, bad_low6);
  long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, 148 * 8 * sizeof(long long));
  cudaMalloc(&sink, 8);
  const int iters = 4096, threads = 1024;
  const char* names[] = {"F2FP", "LOP3", "IMAD", "F2FP+LOP3", "F2FP+IMAD", "LOP3+IMAD",
                         "2xF2FP+LOP3"};
  const int ops[] = {1, 1, 1, 2, 2, 2, 3};
  for (int mode = 0; mode < 7; ++mode) {
    auto run = [&](int blocks) {
      switch (mode) {
        case 0: tput<0><<<blocks, threads>>>(3, sink, cyc, iters); break;
        case 1: tput<1><<<blocks, threads>>>(3, sink, cyc, iters); break;
        case 2: tput<2><<<blocks, threads>>>(3, sink, cyc, iters); break;
        case 3: tput<3><<<blocks, threads>>>(3, sink, cyc, iters); break;
        case 4: tput<4><<<blocks, threads>>>(3, sink, cyc, iters); break;
        case 5: tput<5><<<blocks, threads>>>(3, sink, cyc, iters); break;
        case 6: tput<6><<<blocks, threads>>>(3, sink, cyc, iters); break;
      }
    };
    run(148);
    cudaDeviceSynchronize();
    run(148);
    long long hc[148];
    cudaMemcpy(hc, cyc, sizeof(hc), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += hc[i];
    avg /= 148;
    const double warp_instr = double(iters) * 8 * ops[mode] * (threads / 32);
    printf("%-12s %6.2f warp-instr/clk/SM  (%6.1f thread-ops/clk/SM)\n", names[mode],
           warp_instr / avg, warp_instr * 32 / avg);
  }
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
