// pair_probe.cu -- B200 probe of the CTA-pair (cta_group::2) MMA with the A operand in TMEM:
// D[256 x N] = A[256 x 16] . B[16 x N], CTA r of a 2-CTA cluster holding A/D rows [128 r, 128 r + 128)
// in its own TMEM and the B columns [N/2 r, N/2 r + N/2) in its own shared memory (hypothesis 1),
// or all N columns in both (hypothesis 2, mode 1). Prints the max error of each CTA's D rows vs a
// CPU product. Build: nvcc -gencode arch=compute_100a,code=sm_100a -o build/pair_probe tools/pair_probe.cu
#include <cuda_fp16.h>
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16 |
         static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32 | 1ull << 46;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

constexpr int N = 32;

__global__ void __cluster_dims__(2, 1, 1) probe(const __half* A, const __half* B, float* D, int mode) {
  __shared__ uint32_t slot;
  __shared__ __align__(128) __half bs[2 * N * 8];
  __shared__ __align__(8) uint64_t bar;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int warp = threadIdx.x >> 5, row = threadIdx.x;  // 128 threads: row of this CTA's half
  // B image [k/8][n][8]: hypothesis 1 -> this CTA's N/2 columns; 2 -> all N
  const int nb = mode == 0 ? N / 2 : N, n0 = mode == 0 ? static_cast<int>(rank) * (N / 2) : 0;
  for (int i = threadIdx.x; i < 16 * nb; i += blockDim.x) {
    const int k = i / nb, n = i % nb;
    bs[(k / 8) * nb * 8 + n * 8 + (k % 8)] = B[k * N + n0 + n];
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  // A rows of this CTA -> TMEM lanes 0..127, columns 64..71
  uint32_t a[8];
  const int grow = static_cast<int>(rank) * 128 + row;
  for (int c = 0; c < 8; ++c) {
    const __half2 h = __halves2half2(A[grow * 16 + 2 * c], A[grow * 16 + 2 * c + 1]);
    a[c] = *reinterpret_cast<const uint32_t*>(&h);
  }
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                   tm + ((static_cast<uint32_t>(32 * warp)) << 16) + 64),
               "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]));
  asm volatile("tcgen05.wait::st.sync.aligned;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (rank == 0 && threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(256 >> 4) << 24);
    const uint64_t bd = umma_desc(smem_u32(bs), nb * 16, 128);
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm),
        "r"(tm + 64), "l"(bd), "r"(idesc)
        : "memory");
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&bar)),
        "h"(static_cast<uint16_t>(3))
        : "memory");
  }
  asm volatile(
      "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(
          smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t r[N];
  for (int c0 = 0; c0 < N; c0 += 16) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[c0 + 0]), "=r"(r[c0 + 1]), "=r"(r[c0 + 2]), "=r"(r[c0 + 3]), "=r"(r[c0 + 4]), "=r"(r[c0 + 5]),
          "=r"(r[c0 + 6]), "=r"(r[c0 + 7]), "=r"(r[c0 + 8]), "=r"(r[c0 + 9]), "=r"(r[c0 + 10]), "=r"(r[c0 + 11]),
          "=r"(r[c0 + 12]), "=r"(r[c0 + 13]), "=r"(r[c0 + 14]), "=r"(r[c0 + 15])
        : "r"(tm + ((static_cast<uint32_t>(32 * warp)) << 16) + c0));
  }
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int n = 0; n < N; ++n) D[grow * N + n] = __uint_as_float(r[n]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  cluster_sync();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 128;" ::"r"(tm));
}

int main() {
  __half hA[256 * 16], hB[16 * N];
  float ref[256 * N], got[256 * N];
  srand(3);
  for (int i = 0; i < 256 * 16; ++i) hA[i] = __float2half((rand() % 17 - 8) / 8.0f);
  for (int i = 0; i < 16 * N; ++i) hB[i] = __float2half((rand() % 17 - 8) / 8.0f);
  for (int m = 0; m < 256; ++m)
    for (int n = 0; n < N; ++n) {
      float s = 0;
      for (int k = 0; k < 16; ++k) s += __half2float(hA[m * 16 + k]) * __half2float(hB[k * N + n]);
      ref[m * N + n] = s;
    }
  __half *dA, *dB;
  float* dD;
  cudaMalloc(&dA, sizeof(hA));
  cudaMalloc(&dB, sizeof(hB));
  cudaMalloc(&dD, sizeof(got));
  cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(dD, 0, sizeof(got));
    probe<<<2, 128>>>(dA, dB, dD, mode);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(got, dD, sizeof(got), cudaMemcpyDeviceToHost);
    double e0 = 0, e1 = 0;
    for (int m = 0; m < 256; ++m)
      for (int n = 0; n < N; ++n) {
        const double d = fabs(got[m * N + n] - ref[m * N + n]);
        if (m < 128) e0 = fmax(e0, d); else e1 = fmax(e1, d);
      }
    printf("mode %d (%s): %s; max |err| rows 0-127 %.3g, rows 128-255 %.3g; D[0][0..3] %g %g %g %g ref %g %g %g %g; D[128][0] %g ref %g\n",
           mode, mode == 0 ? "B split by N" : "full B in both", cudaGetErrorString(e), e0, e1, got[0], got[1],
           got[2], got[3], ref[0], ref[1], ref[2], ref[3], got[128 * N], ref[128 * N]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
