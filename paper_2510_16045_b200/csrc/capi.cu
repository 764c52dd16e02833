// capi.cu -- implementation of the C-ABI declared in include/amsq_b200.h.
//
// Exceptions never cross the boundary: InvalidArgument -> AMSQ_EINVAL, Corrupt ->
// AMSQ_ECORRUPT, CUDA/NCCL failures -> AMSQ_ECUDA/AMSQ_ENCCL, with a thread-local
// message. Device entry points never fall back to the CPU: without a device they
// fail with AMSQ_ENODEV.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <nccl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "amsq_b200.h"
#include "device_layout.hpp"
#include "host_core.hpp"
#include "kernels.h"

struct amsq_weight_s {
  amsqb::DeviceLayout L;
  int device = 0;
  uint8_t* d_w = nullptr;
  unsigned short* d_scales = nullptr;
  // K2's activation workspace for batches of 9..64 rows (x in B-fragment order, <= 32 rows
  // per launch): one buffer per stream that used this handle, so calls on different
  // streams never share one; calls on one stream are ordered by the stream itself.
  std::mutex ws_mu;
  std::vector<std::pair<void*, uint2*>> ws;
};

// One rank's view of a fused-TP group (amsq_linear_tp_fused). Each rank owns a segment of
// device memory [flags: nranks u32 | epoch u32 | error u32 | arena]; every rank can store into
// every segment (peer access in one process, CUDA IPC across processes).
struct amsq_tp_s {
  int nranks = 0, rank = 0, device = 0;
  uint8_t* seg = nullptr;          // this rank's segment (owned)
  size_t arena_bytes = 0;
  std::vector<uint8_t*> peer_seg;  // every rank's segment as seen from this device
  std::vector<uint8_t*> opened;    // IPC-opened peer segments (to close)
  unsigned short** d_y = nullptr;  // device array [nranks]: peers' arena bases
  unsigned int** d_flags = nullptr;
};

namespace {

constexpr size_t kTpHeader = 512;  // flags at 0, epoch at 256, error at 260, arena at 512

thread_local std::string g_error;
unsigned long long* g_trace = nullptr;  // amsq_debug_set_trace(): per-CTA timestamps
// batches of at least this many rows run K3 (tcgen05); smaller ones run K2 in chunks of
// linear_max_batch_per_launch() rows (measured crossover)
std::atomic<int> g_k3_min_batch{-1};
std::atomic<int> g_host_direct{1};  // amsq_gemv_host: epilogue stores into page-locked host y  // > 0: a process-wide override of k3_min_batch()

// Batches of at least this many rows run K3 (tcgen05), smaller ones K2 in 32-row chunks: the
// measured crossover per scheme (profiles/r02/k3_crossover_final.txt, K3 with A in TMEM, 2-8
// k-tiles per stage and CTA pairs): K3 wins FP5.33 from M = 33 (past one K2 launch), FP4.25 from 40.
int k3_min_batch(int scheme_id) {
  const int v = g_k3_min_batch.load(std::memory_order_relaxed);
  if (v > 0) return v;
  return scheme_id == 7 ? 33 : 40;
}
bool uses_k3(int scheme_id, size_t batch) {
  return (scheme_id == 4 || scheme_id == 7) && batch >= static_cast<size_t>(k3_min_batch(scheme_id));
}
// bytes of the successor's stream each CTA of amsq_linear_chain pulls into L2
std::atomic<int> g_chain_pf_bytes{65536};

struct CudaError : std::runtime_error {
  cudaError_t code;
  CudaError(cudaError_t c, const char* what)
      : std::runtime_error(std::string(what) + ": " + cudaGetErrorString(c)), code(c) {}
};
struct NoDevice : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NcclError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(e, what);
}

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return AMSQ_OK;
  } catch (const amsqb::InvalidArgument& e) {
    g_error = e.what();
    return AMSQ_EINVAL;
  } catch (const amsqb::Corrupt& e) {
    g_error = e.what();
    return AMSQ_ECORRUPT;
  } catch (const NoDevice& e) {
    g_error = e.what();
    return AMSQ_ENODEV;
  } catch (const NcclError& e) {
    g_error = e.what();
    return AMSQ_ENCCL;
  } catch (const CudaError& e) {
    g_error = e.what();
    return e.code == cudaErrorMemoryAllocation ? AMSQ_ENOMEM : AMSQ_ECUDA;
  } catch (const std::bad_alloc&) {
    g_error = "host allocation failed";
    return AMSQ_ENOMEM;
  } catch (const std::exception& e) {
    g_error = e.what();
    return AMSQ_ECORRUPT;
  }
}

void require_device(int device) {
  int n = 0;
  const cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    throw NoDevice(std::string("no CUDA device available (") + cudaGetErrorString(e) +
                   "): the AMS-Quant kernels run on sm_100a only, there is no CPU fallback");
  }
  if (device < 0 || device >= n) throw amsqb::InvalidArgument("device index out of range");
  cudaDeviceProp prop{};
  ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
  // keep the stream-ordered pool's memory cached (the per-call scratch of amsq_gemv_host and
  // K3 would otherwise be unmapped and re-mapped on every synchronising call)
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  if (prop.major != 10) {
    throw NoDevice("device is sm_" + std::to_string(prop.major) + std::to_string(prop.minor) +
                   "; this library is built for sm_100a (B200) only");
  }
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) ck(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// Device scratch of the synchronous host-buffer entry points (amsq_gemv_host): one grow-only
// buffer per calling thread and device. Never freed -- a thread-exit cudaFree could run after
// the driver has shut down -- so at most one (largest x + y) buffer per thread and device.
uint8_t* host_call_scratch(int device, size_t bytes) {
  struct Buf {
    void* p = nullptr;
    size_t n = 0;
  };
  thread_local Buf bufs[16];
  if (device < 0 || device >= 16) throw amsqb::InvalidArgument("device ordinal out of range");
  Buf& b = bufs[device];
  if (b.n < bytes) {
    if (b.p) ck(cudaFree(b.p), "cudaFree(scratch)");
    b.p = nullptr;
    b.n = 0;
    ck(cudaMalloc(&b.p, bytes), "cudaMalloc(scratch)");
    b.n = bytes;
  }
  return static_cast<uint8_t*>(b.p);
}

// The device address of page-locked host memory, or nullptr for pageable memory.
void* host_mapped(void* p) {
  if (g_host_direct.load(std::memory_order_relaxed) == 0) return nullptr;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();  // pageable pointers on old drivers: clear the sticky-free error
    return nullptr;
  }
  return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

amsqb::GroupPlan plan_of(const amsqb::DeviceLayout& L) {
  return amsqb::GroupPlan{L.n_groups, L.g_big, L.n_big, L.csplit};
}

void check_handle(amsq_weight_t h) {
  if (!h || !h->d_w) throw amsqb::InvalidArgument("null weight handle");
}

amsq_weight_t upload_impl(int scheme_id, size_t rows, size_t cols, size_t pc,
                          const uint16_t* scales, const uint16_t* payload, size_t words,
                          size_t row0, size_t nrows, int device, void* stream) {
  const amsqb::Scheme& s = amsqb::scheme(scheme_id);
  if (!scales || !payload) throw amsqb::InvalidArgument("upload: null host buffer");
  if (rows == 0 || cols == 0) throw amsqb::InvalidArgument("upload: empty tensor");
  if (pc != amsqb::padded_cols(s, cols)) throw amsqb::InvalidArgument("upload: padded_cols mismatch");
  const size_t wpr = amsqb::words_per_row(s, pc);
  if (words != rows * wpr) throw amsqb::InvalidArgument("upload: payload size mismatch");
  if (nrows == 0 || row0 >= rows || nrows > rows - row0) {
    throw amsqb::InvalidArgument("upload: row range out of bounds");
  }
  require_device(device);
  DeviceGuard dg(device);
  auto h = std::make_unique<amsq_weight_s>();
  h->device = device;
  h->L = amsqb::make_device_layout(scheme_id, nrows, cols, pc);
  std::vector<uint8_t> tiles(h->L.bytes());
  amsqb::repack_to_device(h->L, payload + row0 * wpr, tiles.data(), 0);
  std::vector<unsigned short> sc(h->L.row_tiles * 16, 0);
  std::memcpy(sc.data(), scales + row0, nrows * sizeof(uint16_t));
  cudaStream_t st = as_stream(stream);
  ck(cudaMalloc(&h->d_w, tiles.size()), "cudaMalloc(weights)");
  ck(cudaMalloc(&h->d_scales, sc.size() * sizeof(unsigned short)), "cudaMalloc(scales)");
  ck(cudaMemcpyAsync(h->d_w, tiles.data(), tiles.size(), cudaMemcpyHostToDevice, st), "H2D weights");
  ck(cudaMemcpyAsync(h->d_scales, sc.data(), sc.size() * 2, cudaMemcpyHostToDevice, st), "H2D scales");
  ck(cudaStreamSynchronize(st), "upload sync");  // host staging buffers die here
  return h.release();
}

void free_impl(amsq_weight_t h) {
  if (!h) return;
  DeviceGuard dg(h->device);
  cudaFree(h->d_w);
  cudaFree(h->d_scales);
  for (auto& e : h->ws) cudaFree(e.second);
  delete h;
}

// The stream's K2 activation workspace on h (created on first use). A stream that is being
// captured into a CUDA graph and has none yet gets a stream-ordered allocation for this call
// instead (cudaMalloc is not capturable); the caller frees *async_ws after the launches.
uint2* k2_workspace(amsq_weight_t h, cudaStream_t st, void** async_ws) {
  const size_t bytes = h->L.k_tiles * 4 * 32 * 4 * sizeof(uint2);
  std::lock_guard<std::mutex> lk(h->ws_mu);
  for (auto& e : h->ws) {
    if (e.first == static_cast<void*>(st)) return e.second;
  }
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  ck(cudaStreamIsCapturing(st, &cs), "cudaStreamIsCapturing");
  if (cs != cudaStreamCaptureStatusNone) {
    ck(cudaMallocAsync(async_ws, bytes, st), "cudaMallocAsync(xperm)");
    return static_cast<uint2*>(*async_ws);
  }
  uint2* d = nullptr;
  ck(cudaMalloc(&d, bytes), "cudaMalloc(xperm)");
  h->ws.emplace_back(static_cast<void*>(st), d);
  return d;
}

struct TpArgs {
  int nranks;
  unsigned short* const* d_y;  // peers' output bases (already offset)
  long long col0;
};

void linear_impl(amsq_weight_t h, const uint16_t* d_x, size_t batch, uint16_t* d_y, size_t ldy,
                 cudaStream_t st, const float* yscale = nullptr, const TpArgs* tp = nullptr,
                 amsq_weight_t next = nullptr) {
  check_handle(h);
  if (batch == 0) throw amsqb::InvalidArgument("gemv: activation shape mismatch");
  if (!d_x || (!d_y && !tp)) throw amsqb::InvalidArgument("linear: null device buffer");
  if (ldy < h->L.rows) throw amsqb::InvalidArgument("linear: ldy < rows");
  DeviceGuard dg(h->device);
  amsqb::LinearParams p{};
  p.scheme_id = h->L.scheme_id;
  p.w = h->d_w;
  p.scales = h->d_scales;
  p.rows = static_cast<long long>(h->L.rows);
  p.cols = static_cast<long long>(h->L.cols);
  p.ldx = p.cols;
  p.ldy = static_cast<long long>(ldy);
  p.row_tiles = static_cast<int>(h->L.row_tiles);
  p.k_tiles = static_cast<int>(h->L.k_tiles);
  p.plan = plan_of(h->L);
  p.trace = g_trace;
  if (next && next->device == h->device && next->d_w) {
    p.next_w = next->d_w;
    p.next_plan = plan_of(next->L);
    p.next_k_tiles = static_cast<int>(next->L.k_tiles);
    p.next_tile_bytes = static_cast<int>(next->L.tile_bytes);
    p.next_pf_bytes = g_chain_pf_bytes.load(std::memory_order_relaxed);
  }
  if (tp) {
    p.tp_ranks = tp->nranks;
    p.tp_y = tp->d_y;
    p.tp_col0 = tp->col0;
  }
  if (!tp && uses_k3(h->L.scheme_id, batch)) {  // K3: the two AMS schemes
    // K3: tcgen05 tiles, up to 256 batch rows per launch (weights streamed once per launch)
    // the activation image is stream-ordered scratch (cudaMallocAsync: capturable in CUDA
    // graphs, pooled, and private to this call -- no race between streams)
    void* xk = nullptr;
    const size_t mb_max = batch < static_cast<size_t>(amsqb::kTcMaxBatch) ? batch : amsqb::kTcMaxBatch;
    ck(cudaMallocAsync(&xk, (mb_max + 15) / 16 * 16 * h->L.k_tiles * h->L.tk * 2, st),
       "cudaMallocAsync(xk)");
    amsqb::TcParams q{};
    q.scheme_id = h->L.scheme_id;
    q.w = h->d_w;
    q.scales = h->d_scales;
    q.xk = static_cast<const unsigned short*>(xk);
    q.rows = p.rows;
    q.ldy = p.ldy;
    q.row_tiles = p.row_tiles;
    q.k_tiles = p.k_tiles;
    q.plan = p.plan;
    q.trace = g_trace;
    for (size_t b0 = 0; b0 < batch; b0 += amsqb::kTcMaxBatch) {
      q.yscale = yscale ? yscale + b0 : nullptr;
      const size_t mb = batch - b0 < static_cast<size_t>(amsqb::kTcMaxBatch) ? batch - b0 : amsqb::kTcMaxBatch;
      q.M = static_cast<int>(mb);
      q.Np = static_cast<int>((mb + 15) / 16 * 16);
      q.y = reinterpret_cast<unsigned short*>(d_y) + b0 * ldy;
      ck(amsqb::launch_linear_tc(q, reinterpret_cast<const unsigned short*>(d_x) + b0 * h->L.cols,
                                 p.cols, p.cols, st),
         "amsq_linear_tc_kernel launch");
    }
    ck(cudaFreeAsync(xk, st), "cudaFreeAsync(xk)");
    return;
  }
  const size_t step = static_cast<size_t>(amsqb::linear_max_batch_per_launch());
  void* async_ws = nullptr;
  if (batch > 8 && !AMSQ_K2_XSTAGE) p.xperm = k2_workspace(h, st, &async_ws);
  for (size_t b0 = 0; b0 < batch; b0 += step) {
    const size_t mb = batch - b0 < step ? batch - b0 : step;
    p.x = reinterpret_cast<const unsigned short*>(d_x) + b0 * h->L.cols;
    p.y = reinterpret_cast<unsigned short*>(d_y) + b0 * ldy;
    p.yscale = yscale ? yscale + b0 : nullptr;
    if (tp) p.tp_col0 = tp->col0 + static_cast<long long>(b0 * ldy);
    p.M = static_cast<int>(mb);
    ck(amsqb::launch_linear(p, st), "amsq_linear_kernel launch");
  }
  if (async_ws) ck(cudaFreeAsync(async_ws, st), "cudaFreeAsync(xperm)");
}

void restore_impl(amsq_weight_t h, uint16_t* grid, float* f32, uint16_t* f16, cudaStream_t st) {
  check_handle(h);
  DeviceGuard dg(h->device);
  amsqb::RestoreParams p{};
  p.scheme_id = h->L.scheme_id;
  p.w = h->d_w;
  p.scales = h->d_scales;
  p.rows = static_cast<long long>(h->L.rows);
  p.cols = static_cast<long long>(h->L.cols);
  p.padded_cols = static_cast<long long>(h->L.padded_cols);
  p.row_tiles = static_cast<int>(h->L.row_tiles);
  p.k_tiles = static_cast<int>(h->L.k_tiles);
  p.plan = plan_of(h->L);
  p.grid_out = reinterpret_cast<unsigned short*>(grid);
  p.f32_out = f32;
  p.f16_out = reinterpret_cast<unsigned short*>(f16);
  ck(amsqb::launch_restore(p, st), "amsq_restore_kernel launch");
}

// A parsed container (container.hpp:79-115) -> device. The container stores little-endian
// u16 runs; on this (little-endian) host they are used in place when 2-byte aligned -- the
// repack then reads only the requested rows straight from the caller's (or the mmap's)
// bytes -- and decoded into a copy otherwise.
amsq_weight_t upload_container_view(const amsqb::ContainerView& v, size_t row0, size_t nrows,
                                    int device, void* stream) {
  if (row0 >= v.rows) throw amsqb::InvalidArgument("upload_container: row0 out of bounds");
  if (nrows == 0) nrows = v.rows - row0;
  static_assert(__BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__, "container runs are little-endian");
  const bool aligned = (reinterpret_cast<uintptr_t>(v.scales) % 2 == 0) &&
                       (reinterpret_cast<uintptr_t>(v.payload) % 2 == 0);
  if (aligned) {
    return upload_impl(v.scheme_id, v.rows, v.cols, v.padded_cols,
                       reinterpret_cast<const uint16_t*>(v.scales),
                       reinterpret_cast<const uint16_t*>(v.payload), v.payload_words, row0, nrows,
                       device, stream);
  }
  std::vector<uint16_t> scales(v.rows), payload(v.payload_words);
  std::memcpy(scales.data(), v.scales, v.rows * 2);
  std::memcpy(payload.data(), v.payload, v.payload_words * 2);
  return upload_impl(v.scheme_id, v.rows, v.cols, v.padded_cols, scales.data(), payload.data(),
                     payload.size(), row0, nrows, device, stream);
}

}  // namespace

extern "C" {

const char* amsq_last_error(void) { return g_error.c_str(); }
const char* amsq_version(void) { return "amsq-b200 0.1 (sm_100a)"; }

int amsq_scheme_info(int id, amsq_scheme_info_t* out) {
  return guarded([&] {
    if (!out) throw amsqb::InvalidArgument("null output");
    const amsqb::Scheme& s = amsqb::scheme(id);
    out->id = s.id;
    out->exp_bits = s.exp_bits;
    out->man_bits = s.man_bits;
    out->bias = s.bias;
    out->k = s.k;
    out->block = static_cast<size_t>(s.block);
    out->words_per_block = static_cast<size_t>(s.words_per_block);
    out->name = s.name;
    out->device_supported = amsqb::device_scheme_supported(id) ? 1 : 0;
  });
}

int amsq_scheme_by_name(const char* name, int* id) {
  return guarded([&] {
    if (!name || !id) throw amsqb::InvalidArgument("null argument");
    *id = amsqb::scheme_id_by_name(name);
  });
}

size_t amsq_packed_payload_bytes(int id, size_t rows, size_t cols) {
  if (id < 0 || id >= amsqb::kNumSchemes) return 0;
  return amsqb::packed_payload_bytes(amsqb::scheme(id), rows, cols);
}

uint16_t amsq_float_to_half(float f) { return amsqb::f32_to_f16(f); }
float amsq_half_to_float(uint16_t h) { return amsqb::f16_to_f32(h); }

int amsq_restore_table(int id, uint16_t* table, size_t n) {
  return guarded([&] {
    const amsqb::Scheme& s = amsqb::scheme(id);
    if (!table || n < s.code_count()) throw amsqb::InvalidArgument("restore_table: buffer too small");
    for (unsigned c = 0; c < s.code_count(); ++c) table[c] = amsqb::code_to_f16(s, c);
  });
}

int amsq_pack_row(int id, const uint8_t* codes, size_t n, uint16_t* words, size_t nw) {
  return guarded([&] {
    amsqb::pack_row(amsqb::scheme(id), std::span<const uint8_t>(codes, n),
                    std::span<uint16_t>(words, nw));
  });
}

int amsq_unpack_row(int id, const uint16_t* words, size_t nw, uint8_t* codes, size_t n) {
  return guarded([&] {
    amsqb::unpack_row(amsqb::scheme(id), std::span<const uint16_t>(words, nw),
                      std::span<uint8_t>(codes, n));
  });
}

int amsq_quantize_tensor(int id, size_t rows, size_t cols, const float* w, int threads,
                         size_t* padded, size_t* words, uint16_t* scales, uint16_t* payload) {
  return guarded([&] {
    const amsqb::Scheme& s = amsqb::scheme(id);
    if (rows == 0 || cols == 0) throw amsqb::InvalidArgument("quantize_tensor: empty matrix");
    const size_t pc = amsqb::padded_cols(s, cols);
    const size_t nw = rows * amsqb::words_per_row(s, pc);
    if (padded) *padded = pc;
    if (words) *words = nw;
    if (!scales && !payload) return;
    if (!scales || !payload || !w) throw amsqb::InvalidArgument("quantize_tensor: null buffer");
    auto q = amsqb::quantize_tensor(s, rows, cols, w, threads);
    std::memcpy(scales, q.scales.data(), rows * sizeof(uint16_t));
    std::memcpy(payload, q.payload.data(), nw * sizeof(uint16_t));
  });
}

int amsq_quantize_device(int id, const float* d_w, size_t rows, size_t cols, size_t ldw,
                         uint16_t* d_scales, uint16_t* d_payload, size_t words, int device,
                         void* stream) {
  return guarded([&] {
    const amsqb::Scheme& s = amsqb::scheme(id);
    if (rows == 0 || cols == 0) throw amsqb::InvalidArgument("quantize_tensor: empty matrix");
    if (ldw == 0) ldw = cols;
    if (ldw < cols) throw amsqb::InvalidArgument("quantize_device: ldw < cols");
    const size_t pc = amsqb::padded_cols(s, cols), wpr = amsqb::words_per_row(s, pc);
    if (words != rows * wpr) throw amsqb::InvalidArgument("quantize_device: payload size mismatch");
    if (!d_w || !d_scales || !d_payload) throw amsqb::InvalidArgument("quantize_device: null device buffer");
    require_device(device);
    DeviceGuard dg(device);
    cudaStream_t st = as_stream(stream);
    int* d_err = nullptr;
    ck(cudaMallocAsync(reinterpret_cast<void**>(&d_err), sizeof(int), st), "cudaMallocAsync(err)");
    ck(cudaMemsetAsync(d_err, 0, sizeof(int), st), "memset(err)");
    static const amsqb::QuantTables kTables[amsqb::kNumSchemes] = {
        amsqb::make_quant_tables(amsqb::scheme(0)), amsqb::make_quant_tables(amsqb::scheme(1)),
        amsqb::make_quant_tables(amsqb::scheme(2)), amsqb::make_quant_tables(amsqb::scheme(3)),
        amsqb::make_quant_tables(amsqb::scheme(4)), amsqb::make_quant_tables(amsqb::scheme(5)),
        amsqb::make_quant_tables(amsqb::scheme(6)), amsqb::make_quant_tables(amsqb::scheme(7))};
    ck(amsqb::launch_quantize(kTables[id], d_w, static_cast<long long>(rows), static_cast<long long>(ldw),
                              static_cast<long long>(cols), static_cast<long long>(pc),
                              static_cast<long long>(wpr), d_scales, d_payload, d_err, st),
       "amsq_quantize_kernel launch");
    int h_err = 0;
    ck(cudaMemcpyAsync(&h_err, d_err, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H err");
    ck(cudaFreeAsync(d_err, st), "cudaFreeAsync(err)");
    ck(cudaStreamSynchronize(st), "quantize sync");
    if (h_err & 1) throw amsqb::Corrupt("non-finite weight");                       // quantize.hpp:77
    if (h_err & 2) throw amsqb::Corrupt("channel scale overflows half precision");  // quantize.hpp:89
  });
}

int amsq_quantize_device_host(int id, size_t rows, size_t cols, const float* w, int device,
                              size_t* padded, size_t* words, uint16_t* scales, uint16_t* payload) {
  return guarded([&] {
    const amsqb::Scheme& s = amsqb::scheme(id);
    if (rows == 0 || cols == 0) throw amsqb::InvalidArgument("quantize_tensor: empty matrix");
    const size_t pc = amsqb::padded_cols(s, cols), nw = rows * amsqb::words_per_row(s, pc);
    if (padded) *padded = pc;
    if (words) *words = nw;
    if (!scales && !payload) return;
    if (!scales || !payload || !w) throw amsqb::InvalidArgument("quantize_tensor: null buffer");
    require_device(device);
    DeviceGuard dg(device);
    // stream-ordered scratch on a private stream: w in, scales + payload out (synchronous call)
    cudaStream_t st = nullptr;
    ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
    struct StreamGone {
      cudaStream_t s;
      ~StreamGone() { cudaStreamDestroy(s); }
    } gone{st};
    const size_t wb = (rows * cols * sizeof(float) + 255) / 256 * 256, sb = (rows * 2 + 255) / 256 * 256;
    void* d = nullptr;
    ck(cudaMallocAsync(&d, wb + sb + nw * 2, st), "cudaMallocAsync(quantize)");
    auto* dw = static_cast<float*>(d);
    auto* ds = reinterpret_cast<uint16_t*>(static_cast<uint8_t*>(d) + wb);
    auto* dp = reinterpret_cast<uint16_t*>(static_cast<uint8_t*>(d) + wb + sb);
    ck(cudaMemcpyAsync(dw, w, rows * cols * sizeof(float), cudaMemcpyHostToDevice, st), "H2D w");
    const int rc = amsq_quantize_device(id, dw, rows, cols, cols, ds, dp, nw, device, st);
    if (rc != AMSQ_OK) {
      const std::string msg = g_error;
      cudaFreeAsync(d, st);
      cudaStreamSynchronize(st);
      if (rc == AMSQ_ECORRUPT) throw amsqb::Corrupt(msg);
      throw amsqb::InvalidArgument(msg);
    }
    ck(cudaMemcpyAsync(scales, ds, rows * 2, cudaMemcpyDeviceToHost, st), "D2H scales");
    ck(cudaMemcpyAsync(payload, dp, nw * 2, cudaMemcpyDeviceToHost, st), "D2H payload");
    ck(cudaFreeAsync(d, st), "cudaFreeAsync(quantize)");
    ck(cudaStreamSynchronize(st), "quantize sync");
  });
}

int amsq_container_size(int id, size_t rows, size_t cols, size_t* bytes) {
  return guarded([&] { *bytes = amsqb::container_bytes(amsqb::scheme(id), rows, cols); });
}

int amsq_container_write(int id, size_t rows, size_t cols, size_t pc, const uint16_t* scales,
                         const uint16_t* payload, size_t words, uint8_t* out, size_t out_bytes) {
  return guarded([&] {
    amsqb::container_write(amsqb::scheme(id), rows, cols, pc, scales, payload, words, out, out_bytes);
  });
}

int amsq_container_read(const uint8_t* in, size_t n, int* id, size_t* rows, size_t* cols,
                        size_t* pc, uint16_t* scales, size_t n_scales, uint16_t* payload,
                        size_t words) {
  return guarded([&] {
    if (!in) throw amsqb::InvalidArgument("null container");
    const auto v = amsqb::container_parse(in, n);
    if (id) *id = v.scheme_id;
    if (rows) *rows = v.rows;
    if (cols) *cols = v.cols;
    if (pc) *pc = v.padded_cols;
    if (scales) {
      if (n_scales != v.rows) throw amsqb::InvalidArgument("container_read: scales size mismatch");
      for (size_t i = 0; i < v.rows; ++i) scales[i] = static_cast<uint16_t>(v.scales[2 * i] | v.scales[2 * i + 1] << 8);
    }
    if (payload) {
      if (words != v.payload_words) throw amsqb::InvalidArgument("container_read: payload size mismatch");
      for (size_t i = 0; i < words; ++i) payload[i] = static_cast<uint16_t>(v.payload[2 * i] | v.payload[2 * i + 1] << 8);
    }
  });
}

size_t amsq_device_layout_bytes(int id, size_t rows, size_t cols) {
  try {
    const amsqb::Scheme& s = amsqb::scheme(id);
    return amsqb::make_device_layout(id, rows, cols, amsqb::padded_cols(s, cols)).bytes();
  } catch (const std::exception& e) {
    g_error = e.what();
    return 0;
  }
}

int amsq_device_layout_plan(int id, size_t rows, size_t cols, int* plan) {
  return guarded([&] {
    if (!plan) throw amsqb::InvalidArgument("null output");
    const amsqb::Scheme& s = amsqb::scheme(id);
    const auto L = amsqb::make_device_layout(id, rows, cols, amsqb::padded_cols(s, cols));
    plan[0] = L.n_groups, plan[1] = L.g_big, plan[2] = L.n_big, plan[3] = L.csplit;
  });
}

int amsq_repack(int id, size_t rows, size_t cols, size_t pc, const uint16_t* payload,
                size_t words, uint8_t* tiles, size_t tile_bytes) {
  return guarded([&] {
    const auto L = amsqb::make_device_layout(id, rows, cols, pc);
    if (words != rows * L.wpr) throw amsqb::InvalidArgument("repack: payload size mismatch");
    if (tile_bytes != L.bytes()) throw amsqb::InvalidArgument("repack: tile buffer size mismatch");
    amsqb::repack_to_device(L, payload, tiles, 0);
  });
}

int amsq_unrepack(int id, size_t rows, size_t cols, size_t pc, const uint8_t* tiles,
                  size_t tile_bytes, uint16_t* payload, size_t words) {
  return guarded([&] {
    const auto L = amsqb::make_device_layout(id, rows, cols, pc);
    if (words != rows * L.wpr) throw amsqb::InvalidArgument("unrepack: payload size mismatch");
    if (tile_bytes != L.bytes()) throw amsqb::InvalidArgument("unrepack: tile buffer size mismatch");
    amsqb::repack_from_device(L, tiles, payload, 0);
  });
}

int amsq_weight_upload(int id, size_t rows, size_t cols, size_t pc, const uint16_t* scales,
                       const uint16_t* payload, size_t words, int device, void* stream,
                       amsq_weight_t* out) {
  return guarded([&] {
    if (!out) throw amsqb::InvalidArgument("null output handle");
    *out = upload_impl(id, rows, cols, pc, scales, payload, words, 0, rows, device, stream);
  });
}

int amsq_weight_upload_rows(int id, size_t rows, size_t cols, size_t pc, const uint16_t* scales,
                            const uint16_t* payload, size_t words, size_t row0, size_t nrows,
                            int device, void* stream, amsq_weight_t* out) {
  return guarded([&] {
    if (!out) throw amsqb::InvalidArgument("null output handle");
    *out = upload_impl(id, rows, cols, pc, scales, payload, words, row0, nrows, device, stream);
  });
}



int amsq_weight_upload_container(const uint8_t* in, size_t n, size_t row0, size_t nrows,
                                 int device, void* stream, amsq_weight_t* out) {
  return guarded([&] {
    if (!out || !in) throw amsqb::InvalidArgument("null argument");
    *out = upload_container_view(amsqb::container_parse(in, n), row0, nrows, device, stream);
  });
}

int amsq_weight_upload_file(const char* path, size_t row0, size_t nrows, int device,
                            void* stream, amsq_weight_t* out) {
  return guarded([&] {
    if (!out || !path) throw amsqb::InvalidArgument("null argument");
    const int fd = ::open(path, O_RDONLY | O_CLOEXEC);
    if (fd < 0) throw amsqb::Corrupt(std::string("cannot open container ") + path);
    struct stat st {};
    if (::fstat(fd, &st) != 0 || st.st_size <= 0) {
      ::close(fd);
      throw amsqb::Corrupt(std::string("cannot stat container ") + path);
    }
    const size_t n = static_cast<size_t>(st.st_size);
    void* m = ::mmap(nullptr, n, PROT_READ, MAP_PRIVATE, fd, 0);
    ::close(fd);
    if (m == MAP_FAILED) throw amsqb::Corrupt(std::string("cannot map container ") + path);
    ::madvise(m, n, MADV_SEQUENTIAL);
    struct Unmap {
      void* p;
      size_t n;
      ~Unmap() { ::munmap(p, n); }
    } unmap{m, n};
    *out = upload_container_view(amsqb::container_parse(static_cast<const uint8_t*>(m), n), row0,
                                 nrows, device, stream);
  });
}

int amsq_weight_download(amsq_weight_t h, uint16_t* scales, size_t n_scales, uint16_t* payload,
                         size_t words) {
  return guarded([&] {
    check_handle(h);
    DeviceGuard dg(h->device);
    const auto& L = h->L;
    if (scales) {
      if (n_scales != L.rows) throw amsqb::InvalidArgument("download: scales size mismatch");
      ck(cudaMemcpy(scales, h->d_scales, L.rows * 2, cudaMemcpyDeviceToHost), "D2H scales");
    }
    if (payload) {
      if (words != L.rows * L.wpr) throw amsqb::InvalidArgument("download: payload size mismatch");
      std::vector<uint8_t> tiles(L.bytes());
      ck(cudaMemcpy(tiles.data(), h->d_w, tiles.size(), cudaMemcpyDeviceToHost), "D2H weights");
      amsqb::repack_from_device(L, tiles.data(), payload, 0);
    }
  });
}

int amsq_weight_clone(amsq_weight_t h, void* stream, amsq_weight_t* out) {
  return guarded([&] {
    check_handle(h);
    if (!out) throw amsqb::InvalidArgument("null output handle");
    DeviceGuard dg(h->device);
    auto c = std::make_unique<amsq_weight_s>();
    c->device = h->device;
    c->L = h->L;
    cudaStream_t st = as_stream(stream);
    ck(cudaMalloc(&c->d_w, h->L.bytes()), "cudaMalloc(weights)");
    ck(cudaMalloc(&c->d_scales, h->L.row_tiles * 16 * sizeof(unsigned short)), "cudaMalloc(scales)");
    ck(cudaMemcpyAsync(c->d_w, h->d_w, h->L.bytes(), cudaMemcpyDeviceToDevice, st), "D2D weights");
    ck(cudaMemcpyAsync(c->d_scales, h->d_scales, h->L.row_tiles * 16 * 2, cudaMemcpyDeviceToDevice, st),
       "D2D scales");
    ck(cudaStreamSynchronize(st), "clone sync");
    *out = c.release();
  });
}

int amsq_weight_free(amsq_weight_t h) {
  return guarded([&] { free_impl(h); });
}

int amsq_weight_info(amsq_weight_t h, amsq_weight_info_t* out) {
  return guarded([&] {
    check_handle(h);
    if (!out) throw amsqb::InvalidArgument("null output");
    const auto& L = h->L;
    out->scheme_id = L.scheme_id;
    out->rows = L.rows;
    out->cols = L.cols;
    out->padded_cols = L.padded_cols;
    out->payload_bytes = L.rows * L.wpr * 2;
    out->device_bytes = L.bytes();
    out->row_tiles = L.row_tiles;
    out->n_groups = L.n_groups;
    out->g_big = L.g_big;
    out->n_big = L.n_big;
    out->csplit = L.csplit;
    out->k_tiles = L.k_tiles;
    out->device = h->device;
  });
}

int amsq_restore_grid_f16(amsq_weight_t h, uint16_t* d_out, void* stream) {
  return guarded([&] {
    if (!d_out) throw amsqb::InvalidArgument("null output");
    restore_impl(h, d_out, nullptr, nullptr, as_stream(stream));
  });
}

int amsq_restore_f32(amsq_weight_t h, float* d_out, void* stream) {
  return guarded([&] {
    if (!d_out) throw amsqb::InvalidArgument("null output");
    restore_impl(h, nullptr, d_out, nullptr, as_stream(stream));
  });
}

int amsq_restore_f16(amsq_weight_t h, uint16_t* d_out, void* stream) {
  return guarded([&] {
    if (!d_out) throw amsqb::InvalidArgument("null output");
    restore_impl(h, nullptr, nullptr, d_out, as_stream(stream));
  });
}

int amsq_restore_to_host(amsq_weight_t h, int what, void* host_out, size_t bytes, void* stream) {
  return guarded([&] {
    check_handle(h);
    if (!host_out) throw amsqb::InvalidArgument("restore_to_host: null output");
    const auto& L = h->L;
    size_t need = 0;
    if (what == AMSQ_RESTORE_GRID) need = L.rows * L.padded_cols * 2;
    else if (what == AMSQ_RESTORE_F32) need = L.rows * L.cols * 4;
    else if (what == AMSQ_RESTORE_F16) need = L.rows * L.cols * 2;
    else throw amsqb::InvalidArgument("restore_to_host: unknown output kind");
    if (bytes != need) throw amsqb::InvalidArgument("restore_to_host: output size mismatch");
    DeviceGuard dg(h->device);
    cudaStream_t st = as_stream(stream);
    void* d = nullptr;
    ck(cudaMallocAsync(&d, need, st), "cudaMallocAsync(restore)");
    restore_impl(h, what == AMSQ_RESTORE_GRID ? static_cast<uint16_t*>(d) : nullptr,
                 what == AMSQ_RESTORE_F32 ? static_cast<float*>(d) : nullptr,
                 what == AMSQ_RESTORE_F16 ? static_cast<uint16_t*>(d) : nullptr, st);
    ck(cudaMemcpyAsync(host_out, d, need, cudaMemcpyDeviceToHost, st), "D2H restore");
    ck(cudaFreeAsync(d, st), "cudaFreeAsync");
    ck(cudaStreamSynchronize(st), "restore sync");
  });
}

int amsq_linear(amsq_weight_t h, const uint16_t* d_x, size_t batch, uint16_t* d_y, void* stream) {
  return guarded([&] {
    check_handle(h);
    linear_impl(h, d_x, batch, d_y, h->L.rows, as_stream(stream));
  });
}

int amsq_linear_chain(amsq_weight_t h, const uint16_t* d_x, size_t batch, uint16_t* d_y,
                      amsq_weight_t next, void* stream) {
  return guarded([&] {
    check_handle(h);
    linear_impl(h, d_x, batch, d_y, h->L.rows, as_stream(stream), nullptr, nullptr, next);
  });
}

int amsq_debug_set_chain_prefetch(int bytes) {
  const int prev = g_chain_pf_bytes.load();
  if (bytes >= 0) g_chain_pf_bytes.store(bytes);
  return prev;
}

int amsq_linear_ld(amsq_weight_t h, const uint16_t* d_x, size_t batch, uint16_t* d_y, size_t ldy,
                   void* stream) {
  return guarded([&] { linear_impl(h, d_x, batch, d_y, ldy, as_stream(stream)); });
}

int amsq_linear_ex(amsq_weight_t h, const void* d_x, int x_dtype, size_t batch, void* d_y,
                   int y_dtype, size_t ldy, void* stream) {
  return guarded([&] {
    check_handle(h);
    if (x_dtype != y_dtype || (x_dtype != AMSQ_DTYPE_F16 && x_dtype != AMSQ_DTYPE_BF16)) {
      throw amsqb::InvalidArgument("linear_ex: supported dtypes are f16->f16 and bf16->bf16");
    }
    if (ldy == 0) ldy = h->L.rows;
    cudaStream_t st = as_stream(stream);
    if (x_dtype == AMSQ_DTYPE_F16) {
      linear_impl(h, static_cast<const uint16_t*>(d_x), batch, static_cast<uint16_t*>(d_y), ldy, st);
      return;
    }
    if (batch == 0) throw amsqb::InvalidArgument("gemv: activation shape mismatch");
    if (!d_x || !d_y) throw amsqb::InvalidArgument("linear: null device buffer");
    DeviceGuard dg(h->device);
    // stream-ordered scratch (pooled; capturable): x as scaled fp16 + the per-row scales
    const size_t xb = (batch * h->L.cols * 2 + 255) / 256 * 256;
    void* ws = nullptr;
    ck(cudaMallocAsync(&ws, xb + batch * sizeof(float), st), "cudaMallocAsync(bf16 prep)");
    auto* xh = static_cast<unsigned short*>(ws);
    auto* ys = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + xb);
    ck(amsqb::launch_x_bf16_prep(static_cast<const unsigned short*>(d_x),
                                 static_cast<long long>(h->L.cols), static_cast<long long>(h->L.cols),
                                 static_cast<int>(batch), xh, ys, st),
       "amsq_x_bf16_prep launch");
    linear_impl(h, reinterpret_cast<const uint16_t*>(xh), batch, static_cast<uint16_t*>(d_y), ldy, st, ys);
    ck(cudaFreeAsync(ws, st), "cudaFreeAsync(bf16 prep)");
  });
}

int amsq_gemv_host(amsq_weight_t h, const uint16_t* x, size_t x_len, size_t batch, uint16_t* y,
                   void* stream) {
  return guarded([&] {
    check_handle(h);
    if (batch == 0 || x_len != batch * h->L.cols) {
      throw amsqb::InvalidArgument("gemv: activation shape mismatch");  // kernels.hpp:137-143
    }
    if (!x || !y) throw amsqb::InvalidArgument("gemv: null host buffer");
    DeviceGuard dg(h->device);
    cudaStream_t st = as_stream(stream);
    // per-thread, per-device scratch for x and y, grown on demand and reused: the call is
    // synchronous, so a thread's previous call has finished with it before the next starts
    const size_t xb = (x_len * 2 + 255) / 256 * 256, yb = batch * h->L.rows * 2;
    uint8_t* scratch = host_call_scratch(h->device, xb + yb);
    void* dx = scratch;
    void* dy = scratch + xb;
    ck(cudaMemcpyAsync(dx, x, x_len * 2, cudaMemcpyHostToDevice, st), "H2D x");
    // y in page-locked host memory (cudaHostAlloc / cudaHostRegister, e.g. torch pin_memory):
    // the epilogue stores each output element straight into it over the host link, which
    // saves the D2H copy's launch and completion latency. Pageable y: device scratch + D2H.
    void* hy = host_mapped(y);
    linear_impl(h, static_cast<const uint16_t*>(dx), batch, static_cast<uint16_t*>(hy ? hy : dy),
                h->L.rows, st);
    if (!hy) ck(cudaMemcpyAsync(y, dy, yb, cudaMemcpyDeviceToHost, st), "D2H y");
    ck(cudaStreamSynchronize(st), "gemv sync");
  });
}

int amsq_tp_unshard(const uint16_t* d_in, size_t P, size_t batch, size_t n, uint16_t* d_y,
                    void* stream) {
  return guarded([&] {
    if (!d_in || !d_y) throw amsqb::InvalidArgument("null buffer");
    ck(amsqb::launch_unshard(reinterpret_cast<const unsigned short*>(d_in), static_cast<int>(P),
                             static_cast<int>(batch), static_cast<int>(n),
                             reinterpret_cast<unsigned short*>(d_y), as_stream(stream)),
       "unshard launch");
  });
}

int amsq_linear_tp(amsq_weight_t shard, const uint16_t* d_x, size_t batch, uint16_t* d_y,
                   void* d_scratch, size_t scratch_bytes, void* nccl_comm, int nranks,
                   void* stream) {
  return guarded([&] {
    check_handle(shard);
    if (nranks < 1) throw amsqb::InvalidArgument("linear_tp: nranks < 1");
    if (!nccl_comm && nranks > 1) throw amsqb::InvalidArgument("linear_tp: null communicator");
    const size_t n = shard->L.rows;
    const size_t need = 2 * batch * n * (static_cast<size_t>(nranks) + 1);
    if (!d_scratch || scratch_bytes < need) throw amsqb::InvalidArgument("linear_tp: scratch too small");
    cudaStream_t st = as_stream(stream);
    if (nranks == 1 && !nccl_comm) {
      linear_impl(shard, d_x, batch, d_y, n, st);
      return;
    }
    uint16_t* local = static_cast<uint16_t*>(d_scratch);
    uint16_t* gathered = local + batch * n;
    linear_impl(shard, d_x, batch, local, n, st);
    DeviceGuard dg(shard->device);
    const ncclResult_t r = ncclAllGather(local, gathered, batch * n, ncclFloat16,
                                         static_cast<ncclComm_t>(nccl_comm), st);
    if (r != ncclSuccess) throw NcclError(std::string("ncclAllGather: ") + ncclGetErrorString(r));
    ck(amsqb::launch_unshard(gathered, nranks, static_cast<int>(batch), static_cast<int>(n),
                             reinterpret_cast<unsigned short*>(d_y), st),
       "unshard launch");
  });
}

int amsq_linear_tp_group(int nranks, const amsq_weight_t* shards, const uint16_t* const* d_x,
                         size_t batch, uint16_t* const* d_y, void* const* d_scratch,
                         size_t scratch_bytes, void* const* nccl_comms, void* const* streams) {
  return guarded([&] {
    if (nranks < 1 || !shards || !d_x || !d_y || !d_scratch || !nccl_comms || !streams) {
      throw amsqb::InvalidArgument("linear_tp_group: null argument");
    }
    const size_t n = shards[0] ? shards[0]->L.rows : 0;
    for (int r = 0; r < nranks; ++r) {
      check_handle(shards[r]);
      if (shards[r]->L.rows != n) throw amsqb::InvalidArgument("linear_tp_group: unequal shards");
      if (!nccl_comms[r]) throw amsqb::InvalidArgument("linear_tp_group: null communicator");
      if (!d_scratch[r] || scratch_bytes < 2 * batch * n * (static_cast<size_t>(nranks) + 1)) {
        throw amsqb::InvalidArgument("linear_tp_group: scratch too small");
      }
    }
    // 1) every rank's fused linear on its own device/stream
    for (int r = 0; r < nranks; ++r) {
      linear_impl(shards[r], d_x[r], batch, static_cast<uint16_t*>(d_scratch[r]), n,
                  as_stream(streams[r]));
    }
    // 2) one thread drives all communicators: the gathers must be one NCCL group
    ncclResult_t res = ncclGroupStart();
    for (int r = 0; r < nranks && res == ncclSuccess; ++r) {
      DeviceGuard dg(shards[r]->device);
      uint16_t* local = static_cast<uint16_t*>(d_scratch[r]);
      res = ncclAllGather(local, local + batch * n, batch * n, ncclFloat16,
                          static_cast<ncclComm_t>(nccl_comms[r]), as_stream(streams[r]));
    }
    const ncclResult_t end = ncclGroupEnd();
    if (res == ncclSuccess) res = end;
    if (res != ncclSuccess) throw NcclError(std::string("ncclAllGather (group): ") + ncclGetErrorString(res));
    // 3) [P][batch][n] -> [batch][P*n] on every rank
    for (int r = 0; r < nranks; ++r) {
      DeviceGuard dg(shards[r]->device);
      const uint16_t* gathered = static_cast<const uint16_t*>(d_scratch[r]) + batch * n;
      ck(amsqb::launch_unshard(reinterpret_cast<const unsigned short*>(gathered), nranks,
                               static_cast<int>(batch), static_cast<int>(n),
                               reinterpret_cast<unsigned short*>(d_y[r]), as_stream(streams[r])),
         "unshard launch");
    }
  });
}

namespace {
uint8_t* tp_segment_alloc(int device, int nranks, size_t arena_bytes) {
  if (nranks < 1 || nranks > 64) throw amsqb::InvalidArgument("tp: 1 <= nranks <= 64");
  require_device(device);
  DeviceGuard dg(device);
  uint8_t* seg = nullptr;
  ck(cudaMalloc(&seg, kTpHeader + arena_bytes), "cudaMalloc(tp segment)");
  ck(cudaMemset(seg, 0, kTpHeader + arena_bytes), "memset(tp segment)");
  return seg;
}

// device arrays of the peers' arena bases and flag arrays, on the rank's device
void tp_publish(amsq_tp_s* t) {
  DeviceGuard dg(t->device);
  std::vector<unsigned short*> y(static_cast<size_t>(t->nranks));
  std::vector<unsigned int*> f(static_cast<size_t>(t->nranks));
  for (int r = 0; r < t->nranks; ++r) {
    y[static_cast<size_t>(r)] = reinterpret_cast<unsigned short*>(t->peer_seg[static_cast<size_t>(r)] + kTpHeader);
    f[static_cast<size_t>(r)] = reinterpret_cast<unsigned int*>(t->peer_seg[static_cast<size_t>(r)]);
  }
  ck(cudaMalloc(&t->d_y, y.size() * sizeof(void*)), "cudaMalloc(tp ptrs)");
  ck(cudaMalloc(&t->d_flags, f.size() * sizeof(void*)), "cudaMalloc(tp ptrs)");
  ck(cudaMemcpy(t->d_y, y.data(), y.size() * sizeof(void*), cudaMemcpyHostToDevice), "H2D tp ptrs");
  ck(cudaMemcpy(t->d_flags, f.data(), f.size() * sizeof(void*), cudaMemcpyHostToDevice), "H2D tp ptrs");
}

void tp_free(amsq_tp_s* t) {
  if (!t) return;
  DeviceGuard dg(t->device);
  for (uint8_t* p : t->opened) cudaIpcCloseMemHandle(p);
  cudaFree(t->d_y);
  cudaFree(t->d_flags);
  cudaFree(t->seg);
  delete t;
}
}  // namespace

int amsq_tp_create_local(int nranks, const int* devices, size_t arena_bytes, amsq_tp_t* out) {
  return guarded([&] {
    if (!devices || !out) throw amsqb::InvalidArgument("tp_create_local: null argument");
    std::vector<std::unique_ptr<amsq_tp_s, void (*)(amsq_tp_s*)>> ts;
    for (int r = 0; r < nranks; ++r) {
      ts.emplace_back(new amsq_tp_s, tp_free);
      amsq_tp_s* t = ts.back().get();
      t->nranks = nranks, t->rank = r, t->device = devices[r], t->arena_bytes = arena_bytes;
      t->seg = tp_segment_alloc(devices[r], nranks, arena_bytes);
    }
    for (int r = 0; r < nranks; ++r) {  // NVLink peer access between distinct devices
      for (int q = 0; q < nranks; ++q) {
        if (devices[r] == devices[q]) continue;
        int ok = 0;
        ck(cudaDeviceCanAccessPeer(&ok, devices[r], devices[q]), "cudaDeviceCanAccessPeer");
        if (!ok) throw NoDevice("tp_create_local: no peer access between the GPUs");
        DeviceGuard dg(devices[r]);
        const cudaError_t e = cudaDeviceEnablePeerAccess(devices[q], 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) {
          cudaGetLastError();
        } else {
          ck(e, "cudaDeviceEnablePeerAccess");
        }
      }
    }
    for (auto& t : ts) {
      for (auto& q : ts) t->peer_seg.push_back(q->seg);
      tp_publish(t.get());
    }
    for (int r = 0; r < nranks; ++r) out[r] = ts[static_cast<size_t>(r)].release();
  });
}

int amsq_tp_segment_create(int nranks, int rank, int device, size_t arena_bytes,
                           void* ipc_handle_out, amsq_tp_t* out) {
  return guarded([&] {
    if (!ipc_handle_out || !out) throw amsqb::InvalidArgument("tp_segment_create: null argument");
    if (rank < 0 || rank >= nranks) throw amsqb::InvalidArgument("tp_segment_create: bad rank");
    std::unique_ptr<amsq_tp_s, void (*)(amsq_tp_s*)> t(new amsq_tp_s, tp_free);
    t->nranks = nranks, t->rank = rank, t->device = device, t->arena_bytes = arena_bytes;
    t->seg = tp_segment_alloc(device, nranks, arena_bytes);
    DeviceGuard dg(device);
    cudaIpcMemHandle_t hnd;
    ck(cudaIpcGetMemHandle(&hnd, t->seg), "cudaIpcGetMemHandle");
    std::memcpy(ipc_handle_out, &hnd, sizeof(hnd));
    *out = t.release();
  });
}

int amsq_tp_attach(amsq_tp_t t, const void* ipc_handles) {
  return guarded([&] {
    if (!t || !ipc_handles) throw amsqb::InvalidArgument("tp_attach: null argument");
    if (!t->peer_seg.empty()) throw amsqb::InvalidArgument("tp_attach: already attached");
    DeviceGuard dg(t->device);
    const auto* hs = static_cast<const cudaIpcMemHandle_t*>(ipc_handles);
    for (int r = 0; r < t->nranks; ++r) {
      if (r == t->rank) {
        t->peer_seg.push_back(t->seg);
        continue;
      }
      void* p = nullptr;
      ck(cudaIpcOpenMemHandle(&p, hs[r], cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
      t->opened.push_back(static_cast<uint8_t*>(p));
      t->peer_seg.push_back(static_cast<uint8_t*>(p));
    }
    tp_publish(t);
  });
}

int amsq_tp_arena(amsq_tp_t t, void** arena, size_t* bytes) {
  return guarded([&] {
    if (!t || !arena) throw amsqb::InvalidArgument("tp_arena: null argument");
    *arena = t->seg + kTpHeader;
    if (bytes) *bytes = t->arena_bytes;
  });
}

int amsq_tp_destroy(amsq_tp_t t) {
  return guarded([&] { tp_free(t); });
}

int amsq_linear_tp_fused(amsq_weight_t shard, amsq_tp_t t, const uint16_t* d_x, size_t batch,
                         size_t y_offset, void* stream) {
  return guarded([&] {
    check_handle(shard);
    if (!t || t->peer_seg.empty()) throw amsqb::InvalidArgument("linear_tp_fused: group not attached");
    if (shard->device != t->device) throw amsqb::InvalidArgument("linear_tp_fused: shard on another device");
    const size_t n = shard->L.rows, N = n * static_cast<size_t>(t->nranks);
    if (y_offset % 2 || y_offset + 2 * batch * N > t->arena_bytes) {
      throw amsqb::InvalidArgument("linear_tp_fused: output does not fit the arena");
    }
    DeviceGuard dg(t->device);
    cudaStream_t st = as_stream(stream);
    // peers' output bases at y_offset (a small device array per call shape, cached per handle
    // would be an optimisation; the offset is folded into tp_col0 instead)
    TpArgs tp{t->nranks, t->d_y, static_cast<long long>(y_offset / 2) +
                                     static_cast<long long>(t->rank) * static_cast<long long>(n)};
    linear_impl(shard, d_x, batch, nullptr, N, st, nullptr, &tp);
    unsigned int* flags = reinterpret_cast<unsigned int*>(t->seg);
    ck(amsqb::launch_tp_barrier(t->d_flags, flags, flags + 64, flags + 65, t->rank, t->nranks,
                                2000000000ull, st),
       "amsq_tp_barrier_kernel launch");
  });
}

int amsq_tp_error(amsq_tp_t t, int* error) {
  return guarded([&] {
    if (!t || !error) throw amsqb::InvalidArgument("tp_error: null argument");
    DeviceGuard dg(t->device);
    unsigned int e = 0;
    ck(cudaMemcpy(&e, t->seg + 260, 4, cudaMemcpyDeviceToHost), "D2H tp error");
    *error = static_cast<int>(e);
  });
}

int amsq_nccl_unique_id(void* id_out, size_t bytes) {
  return guarded([&] {
    if (!id_out || bytes < sizeof(ncclUniqueId)) throw amsqb::InvalidArgument("nccl_unique_id: buffer < 128 bytes");
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) throw NcclError(std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    std::memcpy(id_out, &id, sizeof(id));
  });
}

int amsq_nccl_comm_init_rank(const void* id, size_t bytes, int nranks, int rank, int device,
                             void** comm) {
  return guarded([&] {
    if (!id || bytes < sizeof(ncclUniqueId) || !comm) throw amsqb::InvalidArgument("nccl_comm_init_rank: bad argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) throw amsqb::InvalidArgument("nccl_comm_init_rank: bad rank");
    require_device(device);
    DeviceGuard dg(device);
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    ncclComm_t c = nullptr;
    const ncclResult_t r = ncclCommInitRank(&c, nranks, uid, rank);
    if (r != ncclSuccess) throw NcclError(std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    *comm = c;
  });
}

int amsq_nccl_comm_init_all(int ndev, const int* devices, void** comms) {
  return guarded([&] {
    if (ndev < 1 || !devices || !comms) throw amsqb::InvalidArgument("nccl_comm_init_all: bad argument");
    for (int i = 0; i < ndev; ++i) require_device(devices[i]);
    std::vector<ncclComm_t> cs(static_cast<size_t>(ndev));
    const ncclResult_t r = ncclCommInitAll(cs.data(), ndev, devices);
    if (r != ncclSuccess) throw NcclError(std::string("ncclCommInitAll: ") + ncclGetErrorString(r));
    for (int i = 0; i < ndev; ++i) comms[i] = cs[static_cast<size_t>(i)];
  });
}

int amsq_nccl_comm_destroy(void* comm) {
  return guarded([&] {
    if (!comm) return;
    const ncclResult_t r = ncclCommDestroy(static_cast<ncclComm_t>(comm));
    if (r != ncclSuccess) throw NcclError(std::string("ncclCommDestroy: ") + ncclGetErrorString(r));
  });
}

uint64_t amsq_kernel_launch_count(void) { return amsqb::kernel_launch_count(); }

void amsq_debug_set_trace(void* d_buf) { g_trace = static_cast<unsigned long long*>(d_buf); }

int amsq_debug_set_k3_min_batch(int rows) {
  const int prev = g_k3_min_batch.load();
  if (rows != 0) g_k3_min_batch.store(rows > 0 ? rows : -1);
  return prev;
}

int amsq_linear_uses_tc(int scheme_id, size_t batch) { return uses_k3(scheme_id, batch) ? 1 : 0; }

int amsq_debug_set_k3_pair(int mode) { return amsqb::tc_set_pair_knob(mode); }

int amsq_debug_set_host_direct(int on) { return g_host_direct.exchange(on ? 1 : 0); }

}  // extern "C"
