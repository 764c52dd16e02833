// tools/tma_probe.cu -- measures HBM read bandwidth of cp.async.bulk streaming (the
// producer pattern of the fused linear) against plain LDG.128, for a range of copy
// sizes / ring depths / CTAs per SM. Build + run on the B200 box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/tma_probe tools/tma_probe.cu
//   build/tma_probe
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Each CTA streams [begin, end) of `src` in `chunk`-byte bulk copies through a ring of
// `stages` buffers; one producer thread, consumer warps only read one word per stage.
__global__ void bulk_stream(const uint8_t* __restrict__ src, size_t total, int chunk, int stages,
                            unsigned long long* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * chunk);
  uint64_t* empty = full + stages;
  const int nconsumer = (blockDim.x / 32) - 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&empty[s])),
                   "r"(nconsumer));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const size_t nchunks = total / chunk;
  const size_t per = (nchunks + gridDim.x - 1) / gridDim.x;
  const size_t c0 = blockIdx.x * per, c1 = c0 + per < nchunks ? c0 + per : nchunks;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (warp == nconsumer) {
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      for (size_t i = 0; c0 + i < c1; ++i) {
        const int s = i % stages;
        if (i >= (size_t)stages) {
          const uint32_t ph = ((i / stages) - 1) & 1;
          asm volatile(
              "{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
              "@!p bra W%=;\n}" ::"r"(smem_u32(&empty[s])),
              "r"(ph));
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                         smem_u32(&full[s])),
                     "r"(chunk));
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
            "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(smem + s * chunk)),
            "l"(src + (c0 + i) * chunk), "r"(chunk), "r"(smem_u32(&full[s])), "l"(pol)
            : "memory");
      }
    }
    return;
  }
  unsigned long long acc = 0;
  for (size_t i = 0; c0 + i < c1; ++i) {
    const int s = i % stages;
    const uint32_t ph = (i / stages) & 1;
    asm volatile(
        "{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra W%=;\n}" ::"r"(smem_u32(&full[s])),
        "r"(ph));
    acc += reinterpret_cast<const uint32_t*>(smem + s * chunk)[threadIdx.x];
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])));
  }
  if (acc == 0x12345) *sink = acc;
}

__global__ void ldg_stream(const uint4* __restrict__ src, size_t n, unsigned long long* sink) {
  unsigned long long acc = 0;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    uint4 a = __ldcs(src + i), b = __ldcs(src + i + stride), c = __ldcs(src + i + 2 * stride),
          d = __ldcs(src + i + 3 * stride);
    acc += a.x ^ b.y ^ c.z ^ d.w;
  }
  for (; i < n; i += stride) acc += __ldcs(src + i).x;
  if (acc == 0x12345) *sink = acc;
}

int main() {
  const size_t total = 1ull << 30;  // 1 GiB >> 126 MB L2
  uint8_t* buf;
  cudaMalloc(&buf, total);
  cudaMemset(buf, 1, total);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto time = [&](auto launch) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return total * 5 / (ms * 1e-3) / 1e9;
  };
  printf("SMs %d\n", sms);
  for (int blocks_per_sm : {1, 2, 4}) {
    for (int threads : {256, 512, 1024}) {
      const double gbs = time([&] {
        ldg_stream<<<sms * blocks_per_sm, threads>>>(reinterpret_cast<const uint4*>(buf),
                                                     total / 16, sink);
      });
      printf("LDG.128 x4 unroll: %d CTA/SM x %d thr: %.0f GB/s\n", blocks_per_sm, threads, gbs);
    }
  }
  for (int ctas : {1, 2, 3, 4}) {
    for (int chunk : {4096, 8192, 16384, 32768}) {
      for (int stages : {2, 4, 6, 8}) {
        const int smem = stages * chunk + 2 * stages * 8;
        if (smem * ctas > 220 * 1024 || smem > 227 * 1024) continue;
        cudaFuncSetAttribute(bulk_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const double gbs = time([&] {
          bulk_stream<<<sms * ctas, 288, smem>>>(buf, total, chunk, stages, sink);
        });
        printf("bulk: %d CTA/SM chunk %6d stages %d (%3d KB/SM in flight): %.0f GB/s\n", ctas,
               chunk, stages, ctas * stages * chunk / 1024, gbs);
      }
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
