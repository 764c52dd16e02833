// tools/bulk_issue_probe.cu -- does cp.async.bulk block the issuing thread? One CTA per SM,
// lane 0 issues N bulk copies of B bytes back to back (clock64 after each issue), then waits.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/bulk_issue_probe tools/bulk_issue_probe.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void probe(const uint8_t* src, size_t span, int n, int bytes, long long* out) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 200 * 1024);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint8_t* base = src + (size_t)blockIdx.x * span;
  long long t[17];
  t[0] = clock64();
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(n * bytes));
  for (int i = 0; i < n; ++i) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(smem + (i * bytes) % (192 * 1024))),
        "l"(base + (size_t)i * bytes), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
    t[1 + i] = clock64();
  }
  asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(
      smem_u32(bar)));
  const long long done = clock64();
  if (blockIdx.x == 0 || blockIdx.x == 77) {
    for (int i = 0; i <= n; ++i) out[blockIdx.x * 20 + i] = t[i] - t[0];
    out[blockIdx.x * 20 + 19] = done - t[0];
  }
}

int main() {
  uint8_t* buf;
  const size_t span = 4 << 20;
  cudaMalloc(&buf, span * 148);
  cudaMemset(buf, 1, span * 148);
  long long* out;
  cudaMalloc(&out, 148 * 20 * 8);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 201 * 1024);
  for (int bytes : {8192, 32768}) {
    for (int grid : {1, 148}) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(out, 0, 148 * 20 * 8);
        probe<<<grid, 32, 201 * 1024>>>(buf, span, 16, bytes, out);
        cudaDeviceSynchronize();
      }
      long long h[20];
      cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
      printf("bytes %6d grid %3d: issue stamps (cycles):", bytes, grid);
      for (int i = 1; i <= 16; ++i) printf(" %lld", h[i]);
      printf(" | all landed %lld\n", h[19]);
    }
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
