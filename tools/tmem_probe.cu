// tmem_probe.cu -- B200 probe: the register -> (TMEM lane, column) map of
// tcgen05.st.16x256b.x1 (read back with tcgen05.ld.32x32b, whose map is thread i -> lane i), and
// a tcgen05.mma kind::f16 with A from TMEM vs a CPU reference (the K3 "A in TMEM" design).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o build/tmem_probe tools/tmem_probe.cu
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void probe_st(uint32_t* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  // warp q stores at lanes 32q (half 0) and 32q + 16 (half 1); value = (half, lane, reg)
  for (int half = 0; half < 2; ++half) {
    const uint32_t addr = tm + ((static_cast<uint32_t>(32 * warp + 16 * half)) << 16) + 8 * half;
    const uint32_t v0 = (half << 12) | (lane << 4) | 0, v1 = (half << 12) | (lane << 4) | 1;
    const uint32_t v2 = (half << 12) | (lane << 4) | 2, v3 = (half << 12) | (lane << 4) | 3;
    asm volatile("tcgen05.st.sync.aligned.16x256b.x1.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v0),
                 "r"(v1), "r"(v2), "r"(v3));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(tm + ((static_cast<uint32_t>(32 * warp)) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int c = 0; c < 16; ++c) out[(32 * warp + lane) * 16 + c] = r[c];
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

// D[128][N=16] = A[128][16] (TMEM, written with 32x32b: thread r holds row r, 8 columns = 16 K values)
// * B[16][16] (smem, K-major no-swizzle [k/8][N][8])
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16 |
         static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32 | 1ull << 46;
}

__global__ void probe_mma(const __half* A, const __half* B, float* D) {
  __shared__ uint32_t slot;
  __shared__ __align__(128) __half bs[2 * 16 * 8];
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, row = threadIdx.x;
  // B image: [k/8][n][8]
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    const int k = i / 16, n = i % 16;
    bs[(k / 8) * 128 + n * 8 + (k % 8)] = B[k * 16 + n];
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  // A row `row` -> TMEM lane row, columns 32..39 (pairs of K)
  uint32_t a[8];
  for (int c = 0; c < 8; ++c) {
    const __half2 h = __halves2half2(A[row * 16 + 2 * c], A[row * 16 + 2 * c + 1]);
    a[c] = *reinterpret_cast<const uint32_t*>(&h);
  }
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                   tm + ((static_cast<uint32_t>(32 * warp)) << 16) + 32),
               "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]));
  asm volatile("tcgen05.wait::st.sync.aligned;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (static_cast<uint32_t>(16 >> 3) << 17) | (static_cast<uint32_t>(128 >> 4) << 24);
    const uint64_t bd = umma_desc(smem_u32(bs), 16 * 16, 128);
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm),
        "r"(tm + 32), "l"(bd), "r"(idesc)
        : "memory");
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
  }
  asm volatile(
      "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(
          smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(tm + ((static_cast<uint32_t>(32 * warp)) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int n = 0; n < 16; ++n) D[row * 16 + n] = __uint_as_float(r[n]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tm));
}

int main() {
  uint32_t* d_out;
  cudaMalloc(&d_out, 128 * 16 * 4);
  cudaMemset(d_out, 0xFF, 128 * 16 * 4);
  probe_st<<<1, 128>>>(d_out);
  uint32_t h[128 * 16];
  cudaError_t e = cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
  printf("probe_st: %s\n", cudaGetErrorString(e));
  // print the map for TMEM lanes 0..31, columns 0..15: (half, writer lane, reg)
  for (int l = 0; l < 32; ++l) {
    printf("lane %2d:", l);
    for (int c = 0; c < 16; ++c) {
      const uint32_t v = h[l * 16 + c];
      if (v == 0xFFFFFFFFu) printf("   --   ");
      else printf(" h%ul%02ur%u", v >> 12, (v >> 4) & 0xFF, v & 0xF);
    }
    printf("\n");
  }
  // mma with A from TMEM
  __half hA[128 * 16], hB[16 * 16];
  float ref[128 * 16], got[128 * 16];
  srand(1);
  for (int i = 0; i < 128 * 16; ++i) hA[i] = __float2half((rand() % 17 - 8) / 8.0f);
  for (int i = 0; i < 16 * 16; ++i) hB[i] = __float2half((rand() % 17 - 8) / 8.0f);
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 16; ++n) {
      float s = 0;
      for (int k = 0; k < 16; ++k) s += __half2float(hA[m * 16 + k]) * __half2float(hB[k * 16 + n]);
      ref[m * 16 + n] = s;
    }
  __half *dA, *dB;
  float* dD;
  cudaMalloc(&dA, sizeof(hA));
  cudaMalloc(&dB, sizeof(hB));
  cudaMalloc(&dD, sizeof(got));
  cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
  probe_mma<<<1, 128>>>(dA, dB, dD);
  e = cudaMemcpy(got, dD, sizeof(got), cudaMemcpyDeviceToHost);
  double maxerr = 0;
  for (int i = 0; i < 128 * 16; ++i) maxerr = fmax(maxerr, fabs(got[i] - ref[i]));
  printf("probe_mma (A from TMEM): %s, max |err| %.3g (D[0][0..3] = %g %g %g %g, ref %g %g %g %g)\n",
         cudaGetErrorString(e), maxerr, got[0], got[1], got[2], got[3], ref[0], ref[1], ref[2], ref[3]);
  return 0;
}
