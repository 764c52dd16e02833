// tools/stream_probe.cu -- the read-only HBM ceiling per call size: how fast can ONE kernel
// launch stream S bytes (S = the packed weight of one Llama-3.1-8B layer), back to back in a
// CUDA graph with rotating source offsets (> L2), using (a) LDG.128 with several loads in
// flight per thread, (b) cp.async.bulk rings, one CTA per SM. This bounds what the fused
// linear can reach at each shape, fixed launch/ramp/tail costs included.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/stream_probe tools/stream_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int U>
__global__ void __launch_bounds__(512) ldg_stream(const uint4* __restrict__ src, size_t n,
                                                  unsigned* sink) {
  unsigned acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(src + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  for (; i < n; i += stride) acc ^= __ldcs(src + i).x;
  if (acc == 0x9E3779B9u) *sink = acc;
}

// contiguous per-CTA ranges (the fused linear's split), LDG.128, U loads in flight per thread
template <int U>
__global__ void __launch_bounds__(512) ldg_range(const uint4* __restrict__ src, size_t n,
                                                 unsigned* sink) {
  const size_t per = (n + gridDim.x - 1) / gridDim.x;
  const size_t b = blockIdx.x * per, e = b + per < n ? b + per : n;
  unsigned acc = 0;
  size_t i = b + threadIdx.x;
  for (; i + (U - 1) * blockDim.x < e; i += U * blockDim.x) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(src + i + u * blockDim.x);
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  for (; i < e; i += blockDim.x) acc ^= __ldcs(src + i).x;
  if (acc == 0x9E3779B9u) *sink = acc;
}

__global__ void bulk_stream(const uint8_t* __restrict__ src, size_t total, int chunk, int stages,
                            unsigned* sink) {
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
  const size_t nchunks = (total + chunk - 1) / chunk;
  const size_t c0 = blockIdx.x * nchunks / gridDim.x, c1 = (blockIdx.x + 1) * nchunks / gridDim.x;
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
        const size_t off = (c0 + i) * chunk;
        const uint32_t bytes = static_cast<uint32_t>(off + chunk <= total ? chunk : total - off);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                         smem_u32(&full[s])),
                     "r"(bytes));
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
            "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(smem + s * chunk)),
            "l"(src + off), "r"(bytes), "r"(smem_u32(&full[s])), "l"(pol)
            : "memory");
      }
    }
    return;
  }
  unsigned acc = 0;
  for (size_t i = 0; c0 + i < c1; ++i) {
    const int s = i % stages;
    const uint32_t ph = (i / stages) & 1;
    asm volatile(
        "{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra W%=;\n}" ::"r"(smem_u32(&full[s])),
        "r"(ph));
    acc ^= reinterpret_cast<const uint32_t*>(smem + s * chunk)[threadIdx.x];
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])));
  }
  if (acc == 0x9E3779B9u) *sink = acc;
}

__global__ void empty_kernel(unsigned* sink) {
  if (threadIdx.x == 1023) *sink = 1;
}

int main() {
  const size_t total = 2ull << 30;
  uint8_t* buf;
  cudaMalloc(&buf, total);
  cudaMemset(buf, 1, total);
  unsigned* sink;
  cudaMalloc(&sink, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  // graph of R back-to-back launches over rotating sources (sum > 2x L2), replayed
  auto time_graph = [&](size_t bytes, auto launch) {
    const int R = 16;
    const size_t step = (total / R) & ~size_t(4095);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int r = 0; r < R; ++r) launch(buf + (r * step) % (total - bytes), bytes);
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, st);
    cudaStreamSynchronize(st);
    const int reps = 20;
    cudaEventRecord(a, st);
    for (int i = 0; i < reps; ++i) cudaGraphLaunch(ge, st);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    return ms * 1e3 / (reps * R);  // us per launch
  };
  printf("SMs %d\n", sms);
  const double empty_us = time_graph(0, [&](const uint8_t*, size_t) {
    empty_kernel<<<sms, 1024, 0, st>>>(sink);
  });
  printf("empty kernel 148x1024 in graph: %.2f us\n", empty_us);
  const size_t sizes[] = {11190272, 16785408, 39149568, 78331904, 249561088};
  for (size_t S : sizes) {
    printf("--- S = %.1f MB\n", S / 1e6);
    for (int bps : {1, 2, 4}) {
      for (int thr : {256, 512}) {
        double us = time_graph(S, [&](const uint8_t* src, size_t n) {
          ldg_stream<4><<<sms * bps, thr, 0, st>>>(reinterpret_cast<const uint4*>(src), n / 16, sink);
        });
        printf("  ldg_stream U4 %d CTA/SM x %d: %7.2f us  %6.0f GB/s\n", bps, thr, us, S / us / 1e3);
        us = time_graph(S, [&](const uint8_t* src, size_t n) {
          ldg_stream<8><<<sms * bps, thr, 0, st>>>(reinterpret_cast<const uint4*>(src), n / 16, sink);
        });
        printf("  ldg_stream U8 %d CTA/SM x %d: %7.2f us  %6.0f GB/s\n", bps, thr, us, S / us / 1e3);
        us = time_graph(S, [&](const uint8_t* src, size_t n) {
          ldg_range<8><<<sms * bps, thr, 0, st>>>(reinterpret_cast<const uint4*>(src), n / 16, sink);
        });
        printf("  ldg_range  U8 %d CTA/SM x %d: %7.2f us  %6.0f GB/s\n", bps, thr, us, S / us / 1e3);
      }
    }
    for (int chunk : {8192, 16384, 32768}) {
      for (int stages : {4, 6}) {
        const int smem = stages * chunk + 2 * stages * 8;
        if (smem > 227 * 1024) continue;
        cudaFuncSetAttribute(bulk_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const double us = time_graph(S, [&](const uint8_t* src, size_t n) {
          bulk_stream<<<sms, 288, smem, st>>>(src, n, chunk, stages, sink);
        });
        printf("  bulk chunk %5d x %d stages: %7.2f us  %6.0f GB/s\n", chunk, stages, us,
               S / us / 1e3);
      }
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
