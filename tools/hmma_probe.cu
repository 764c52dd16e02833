// tools/hmma_probe.cu -- legacy mma.sync.m16n8k16 (HMMA.16816.F32) throughput per SM on
// sm_100a: independent accumulator chains, 4..16 warps per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/hmma_probe tools/hmma_probe.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__global__ void hmma(float* out, int iters, long long* cyc) {
  float acc[8][4] = {};
  uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, threadIdx.x * 5u, threadIdx.x * 7u};
  uint32_t b0 = threadIdx.x * 11u, b1 = threadIdx.x * 13u;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(acc[c][0]), "+f"(acc[c][1]), "+f"(acc[c][2]), "+f"(acc[c][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
    }
  }
  const long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
  if (s == 1.2345f) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 4);
  cudaMalloc(&cyc, 148 * 8);
  const int iters = 2048;
  for (int warps : {4, 8, 16, 32}) {
    hmma<<<148, warps * 32>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    hmma<<<148, warps * 32>>>(out, iters, cyc);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    const double hmmas = double(iters) * 8 * warps;  // per SM
    printf("%2d warps/SM: %.2f cycles per HMMA.16816 per SM  (%.1f per SMSP), %.0f dense fp16 TFLOP/s at 1.9 GHz\n",
           warps, avg / hmmas, avg / hmmas * 4, hmmas / avg * 4096 * 1.9e9 * 148 / 1e12);
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
