/*
 * amsq_b200.h -- C-ABI of the B200-native AMS-Quant weight-only linear.
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/proj/include/amsq): every entry point below names the
 * reference interface it replaces. Plain pointers and sizes only; no C++ or
 * torch types cross it. Device pointers are caller-owned and `stream` is a
 * cudaStream_t (NULL = legacy default stream); all device entry points are
 * stream-ordered and asynchronous unless stated otherwise.
 *
 * Errors: every function returns an amsq_status; amsq_last_error() gives the
 * thread-local message of the last failure. The C++ wrapper (amsq_b200.hpp)
 * maps AMSQ_EINVAL -> std::invalid_argument and everything else ->
 * std::runtime_error, preserving the reference tests' exception types
 * (SURVEY.md §8(b)).
 */
#ifndef AMSQ_B200_H_
#define AMSQ_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  AMSQ_OK = 0,
  AMSQ_EINVAL = 1,   /* std::invalid_argument in the reference */
  AMSQ_ECORRUPT = 2, /* std::runtime_error: data (shared-bit mismatch, non-finite, overflow, container) */
  AMSQ_ECUDA = 3,    /* CUDA runtime / launch failure */
  AMSQ_ENCCL = 4,    /* NCCL failure (tensor-parallel path) */
  AMSQ_ENOMEM = 5,
  AMSQ_ENODEV = 6    /* no CUDA device: the product never falls back to the CPU */
} amsq_status;

/* Scheme ids are the container/ABI enum of scheme.hpp:21-30. */
enum {
  AMSQ_FP4_E2M1 = 0,
  AMSQ_FP5_E2M2 = 1,
  AMSQ_FP6_E2M3 = 2,
  AMSQ_FP6_E3M2 = 3,
  AMSQ_FP4_25_E2M2 = 4,
  AMSQ_FP4_33_E2M2 = 5,
  AMSQ_FP4_5_E2M2 = 6,
  AMSQ_FP5_33_E2M3 = 7
};

typedef struct {
  int id;
  int exp_bits, man_bits, bias; /* FloatFormat, format.hpp:31-72 */
  int k;                        /* weights sharing one mantissa LSB */
  size_t block;                 /* PackLayout::block, packing.hpp:51-63 */
  size_t words_per_block;       /* PackLayout::words_per_block */
  const char* name;             /* QuantScheme::name, scheme.hpp:59-74 */
  int device_supported;         /* 1 if the sm_100a kernels implement this scheme */
} amsq_scheme_info_t;

const char* amsq_last_error(void);
const char* amsq_version(void);

/* ---- scheme / layout metadata (scheme.hpp:76-89, packing.hpp:143-157, quantize.hpp:64-69) */
int amsq_scheme_info(int scheme_id, amsq_scheme_info_t* out);
int amsq_scheme_by_name(const char* name, int* scheme_id);
size_t amsq_packed_payload_bytes(int scheme_id, size_t rows, size_t cols);

/* ---- binary16 (half.hpp:16-71) */
uint16_t amsq_float_to_half(float f);
float amsq_half_to_float(uint16_t h);
/* to_fp16_bits / restore_table (format.hpp:190-198): table[code], n >= 2^(1+e+m) */
int amsq_restore_table(int scheme_id, uint16_t* table, size_t n);

/* ---- host codec of the reference stream (packing.hpp:216-266) */
int amsq_pack_row(int scheme_id, const uint8_t* codes, size_t n_codes, uint16_t* words,
                  size_t n_words);
int amsq_unpack_row(int scheme_id, const uint16_t* words, size_t n_words, uint8_t* codes,
                    size_t n_codes);

/* ---- host quantizer, kept on the host by design (quantize.hpp:188-216 quantize_tensor:
 * RTN + Adaptive Searching + pack). `w` is row-major [rows][cols] fp32. Pass
 * scales == payload == NULL to query *padded_cols and *payload_words. threads <= 0
 * means all hardware threads (parallel.hpp:15-19). */
int amsq_quantize_tensor(int scheme_id, size_t rows, size_t cols, const float* w, int threads,
                         size_t* padded_cols, size_t* payload_words, uint16_t* scales,
                         uint16_t* payload);

/* ---- device quantizer: quantize_tensor (quantize.hpp:188-216) on the GPU,
 * bit-identical to amsq_quantize_tensor. d_w is device fp32 [rows][ldw] (ldw = 0: cols); the
 * outputs are the reference stream in device memory: d_scales u16[rows], d_payload u16[words]
 * (words = rows * words_per_row, see amsq_quantize_tensor's query). Synchronous: it waits for
 * the stream to report a non-finite weight or a scale overflow as AMSQ_ECORRUPT (quantize.hpp:77,
 * 89). */
int amsq_quantize_device(int scheme_id, const float* d_w, size_t rows, size_t cols, size_t ldw,
                         uint16_t* d_scales, uint16_t* d_payload, size_t words, int device,
                         void* stream);

/* The same with host buffers (the reference's quantize_tensor call shape): w is host fp32
 * [rows][cols]; pass scales == payload == NULL to query *padded_cols and *payload_words.
 * Synchronous (its own stream). */
int amsq_quantize_device_host(int scheme_id, size_t rows, size_t cols, const float* w, int device,
                              size_t* padded_cols, size_t* payload_words, uint16_t* scales,
                              uint16_t* payload);

/* ---- AMSQ container v1 (container.hpp:63-127), host buffers. */
int amsq_container_size(int scheme_id, size_t rows, size_t cols, size_t* bytes);
int amsq_container_write(int scheme_id, size_t rows, size_t cols, size_t padded_cols,
                         const uint16_t* scales, const uint16_t* payload, size_t payload_words,
                         uint8_t* out, size_t out_bytes);
/* Validating reader: parses the header into the outputs; copies scales/payload when the
 * pointers are non-NULL (sizes checked). */
int amsq_container_read(const uint8_t* in, size_t in_bytes, int* scheme_id, size_t* rows,
                        size_t* cols, size_t* padded_cols, uint16_t* scales, size_t n_scales,
                        uint16_t* payload, size_t payload_words);

/* ---- the device tile layout on the host: exposed so the layout and its
 * exact inverse can be checked without a GPU. tiles must hold amsq_device_layout_bytes(). */
size_t amsq_device_layout_bytes(int scheme_id, size_t rows, size_t cols);
/* The work plan the layout is built for: plan[4] = {n_groups, g_big, n_big, csplit}
 * (row tiles split into n_groups contiguous groups, the first n_big of g_big tiles, the
 * rest of g_big - 1; csplit CTAs per group split K). */
int amsq_device_layout_plan(int scheme_id, size_t rows, size_t cols, int* plan);
int amsq_repack(int scheme_id, size_t rows, size_t cols, size_t padded_cols,
                const uint16_t* payload, size_t payload_words, uint8_t* tiles, size_t tile_bytes);
int amsq_unrepack(int scheme_id, size_t rows, size_t cols, size_t padded_cols,
                  const uint8_t* tiles, size_t tile_bytes, uint16_t* payload,
                  size_t payload_words);

/* ---- device weights: the QuantizedTensor (quantize.hpp:45-61) uploaded into the
 * sm_100a tile layout. The repack is a pure bit permutation of the
 * reference stream: amsq_weight_download() returns the identical words. */
typedef struct amsq_weight_s* amsq_weight_t;

int amsq_weight_upload(int scheme_id, size_t rows, size_t cols, size_t padded_cols,
                       const uint16_t* scales, const uint16_t* payload, size_t payload_words,
                       int device, void* stream, amsq_weight_t* out);
/* N-shard [row0, row0+nrows) of a full tensor (column-parallel TP). */
int amsq_weight_upload_rows(int scheme_id, size_t rows, size_t cols, size_t padded_cols,
                            const uint16_t* scales, const uint16_t* payload,
                            size_t payload_words, size_t row0, size_t nrows, int device,
                            void* stream, amsq_weight_t* out);
/* Container bytes -> device in one step (container.hpp:79-115 read_amsq + upload). */
int amsq_weight_upload_container(const uint8_t* in, size_t in_bytes, size_t row0, size_t nrows,
                                 int device, void* stream, amsq_weight_t* out);
/* The same from a container FILE: mmap'd read-only, validated (container.hpp:79-115), and
 * only the pages of rows [row0, row0+nrows) are read by the repack (nrows = 0: to the end). */
int amsq_weight_upload_file(const char* path, size_t row0, size_t nrows, int device,
                            void* stream, amsq_weight_t* out);
int amsq_weight_download(amsq_weight_t h, uint16_t* scales, size_t n_scales, uint16_t* payload,
                         size_t payload_words);
/* A second, independent device copy of h (same device; a device-to-device copy of the tile
 * layout -- e.g. to lay out many layers of identical shape without re-uploading). */
int amsq_weight_clone(amsq_weight_t h, void* stream, amsq_weight_t* out);
int amsq_weight_free(amsq_weight_t h);

typedef struct {
  int scheme_id;
  size_t rows, cols, padded_cols;
  size_t payload_bytes;        /* reference stream bytes, packed_payload_bytes() */
  size_t device_bytes;         /* bytes of the device tile layout (>= payload_bytes) */
  size_t row_tiles, k_tiles;   /* 16-row x (64|48)-col tiles */
  int device;
  int n_groups, g_big, n_big, csplit; /* work plan: row groups (one CTA or CTA pair each) */
} amsq_weight_info_t;
int amsq_weight_info(amsq_weight_t h, amsq_weight_info_t* out);

/* ---- the hot path (kernels.hpp), device buffers, stream-ordered ----------------- */

/* restore_block over the whole tensor (kernels.hpp:55-63): binary16 grid bits,
 * [rows][padded_cols]. Bit-exact bar #1. */
int amsq_restore_grid_f16(amsq_weight_t h, uint16_t* d_out, void* stream);
/* restore_matrix (kernels.hpp:100-124): fp32 w*s, [rows][cols]. Bit-exact. */
int amsq_restore_f32(amsq_weight_t h, float* d_out, void* stream);
/* restore_matrix_half (kernels.hpp:127-133): fp16(w*s), [rows][cols]. Bit-exact. */
int amsq_restore_f16(amsq_weight_t h, uint16_t* d_out, void* stream);

/* The three restores above into a HOST buffer (device scratch + D2H inside; synchronous):
 * what = AMSQ_RESTORE_GRID (u16 [rows][padded_cols]), AMSQ_RESTORE_F32 (f32 [rows][cols]) or
 * AMSQ_RESTORE_F16 (u16 [rows][cols]); bytes must equal that size. */
enum { AMSQ_RESTORE_GRID = 0, AMSQ_RESTORE_F32 = 1, AMSQ_RESTORE_F16 = 2 };
int amsq_restore_to_host(amsq_weight_t h, int what, void* host_out, size_t bytes, void* stream);

/* gemv (kernels.hpp:151-187): y[b][r] = fp16(sum_i w_i s_r x_b,i), fp32 accumulation.
 * d_x is [batch][cols] fp16 (logical cols), d_y is [batch][rows] fp16.
 * batch >= 1 (check_gemv_shapes, kernels.hpp:137-143 -> AMSQ_EINVAL).
 * Reentrant: batches of 9..64 rows stage their activations in a per-(handle, stream)
 * workspace, so calls on one handle from different streams may overlap. */
int amsq_linear(amsq_weight_t h, const uint16_t* d_x, size_t batch, uint16_t* d_y, void* stream);

/* amsq_linear, and while it runs, the first stages of the NEXT call's weights (`next`, the
 * weight of the call that follows on this stream; NULL = none) are pulled into L2, so that
 * call's ramp starts from L2 instead of HBM (decode steps: layer after layer, graph-replayed).
 * Results are identical to amsq_linear. */
int amsq_linear_chain(amsq_weight_t h, const uint16_t* d_x, size_t batch, uint16_t* d_y,
                      amsq_weight_t next, void* stream);
/* Tuning knob: bytes per CTA amsq_linear_chain prefetches (default 64 KiB; 0 = off, < 0 only
 * queries). Returns the previous value. Process-wide. */
int amsq_debug_set_chain_prefetch(int bytes);

/* Same with an explicit output row stride (elements) for writing into a wider buffer. */
int amsq_linear_ld(amsq_weight_t h, const uint16_t* d_x, size_t batch, uint16_t* d_y,
                   size_t ldy, void* stream);

/* Activation dtypes (the reference is fp16-only, half.hpp; bf16 is the north star's
 * addition). bf16 rows are brought to fp16 exactly up to a per-row power of two, which the
 * epilogue undoes before the single rounding of y to bf16. y has the activations' dtype.
 * ldy = 0 means rows. */
enum { AMSQ_DTYPE_F16 = 0, AMSQ_DTYPE_BF16 = 1 };
int amsq_linear_ex(amsq_weight_t h, const void* d_x, int x_dtype, size_t batch, void* d_y,
                   int y_dtype, size_t ldy, void* stream);

/* The reference call shape end to end: host x in, host y out (H2D, kernel, D2H on
 * `stream`, synchronous on return). x_len must equal batch*cols. The device copies of x and
 * y live in a grow-only scratch buffer per calling thread and device (reused across calls,
 * never freed); pinned host buffers avoid a staging copy in the driver. A page-locked y is
 * written by the kernel's epilogue directly (no D2H copy); a pageable y goes through the
 * device scratch and a D2H copy. */
int amsq_gemv_host(amsq_weight_t h, const uint16_t* x, size_t x_len, size_t batch, uint16_t* y,
                   void* stream);

/* ---- column-parallel tensor parallelism ----------------------
 * `shard` holds rows [rank*N/P, (rank+1)*N/P). Computes the local [batch][N/P] output,
 * all-gathers it with ncclAllGather over `nccl_comm` (an ncclComm_t), and writes the
 * reference-layout [batch][N] result into d_y. d_scratch must hold
 * 2*batch*(N/P)*(P+1) bytes. With nranks == 1 and no communicator it is amsq_linear_ld. */
int amsq_linear_tp(amsq_weight_t shard, const uint16_t* d_x, size_t batch, uint16_t* d_y,
                   void* d_scratch, size_t scratch_bytes, void* nccl_comm, int nranks,
                   void* stream);
/* Single-process multi-GPU form (one process drives every GPU through
 * ncclCommInitAll communicators): rank r's shard, activations, output, scratch, communicator
 * and stream are element r of each array; the all-gathers are issued as one NCCL group. */
int amsq_linear_tp_group(int nranks, const amsq_weight_t* shards, const uint16_t* const* d_x,
                         size_t batch, uint16_t* const* d_y, void* const* d_scratch,
                         size_t scratch_bytes, void* const* nccl_comms, void* const* streams);
/* ---- fused column-parallel TP: no NCCL collective. Every rank owns a
 * device segment (flag words + an output arena) that all ranks can store into -- peer access
 * in one process, CUDA IPC across processes. amsq_linear_tp_fused computes the rank's shard
 * and its epilogue stores every output element straight into EVERY rank's arena at
 * [m][rank*n + j] (NVLink stores, overlapped with the other CTAs' math); a one-block flag
 * barrier (system-scope release/acquire, epoch counters kept on the device so the call is
 * CUDA-graph replayable) then guarantees, in stream order, that this rank's arena holds the
 * whole [batch][N] output at byte offset y_offset. Callers must not overwrite an arena
 * region a peer may still be reading (use distinct offsets per layer, like NCCL user
 * buffers). A peer that never arrives fails the barrier after 2 s (amsq_tp_error). The fused
 * epilogue is K2's: every batch runs K2 (in 32-row chunks), also past the K2/K3 crossover
 * where amsq_linear_tp would run K3 on the shard -- outputs are within the same bar, not
 * bit-identical to the K3 path there. */
typedef struct amsq_tp_s* amsq_tp_t;
/* One process, every rank's view at once (out[r]); devices may repeat (virtual ranks). */
int amsq_tp_create_local(int nranks, const int* devices, size_t arena_bytes, amsq_tp_t* out);
/* Multi-process: create this rank's segment and its 64-byte cudaIpcMemHandle; exchange the
 * handles out of band (nranks x 64 bytes, rank order) and attach. */
int amsq_tp_segment_create(int nranks, int rank, int device, size_t arena_bytes,
                           void* ipc_handle_out, amsq_tp_t* out);
int amsq_tp_attach(amsq_tp_t tp, const void* ipc_handles);
int amsq_tp_arena(amsq_tp_t tp, void** arena, size_t* bytes);
int amsq_tp_error(amsq_tp_t tp, int* error);
int amsq_tp_destroy(amsq_tp_t tp);
int amsq_linear_tp_fused(amsq_weight_t shard, amsq_tp_t tp, const uint16_t* d_x, size_t batch,
                         size_t y_offset, void* stream);
/* [P][batch][n] -> [batch][P*n] permutation used after the gather (exposed for tests). */
int amsq_tp_unshard(const uint16_t* d_gathered, size_t nranks, size_t batch, size_t n_local,
                    uint16_t* d_y, void* stream);

/* NCCL plumbing for hosts that do not own a communicator (the bench, the Python TP driver):
 * a 128-byte ncclUniqueId made on one rank and shared out of band, then one ncclComm_t per
 * rank (ncclCommInitRank), or all ranks' communicators of a single process
 * (ncclCommInitAll over `devices`). The returned void* is an ncclComm_t. */
int amsq_nccl_unique_id(void* id_out, size_t bytes);
int amsq_nccl_comm_init_rank(const void* id, size_t bytes, int nranks, int rank, int device,
                             void** comm);
int amsq_nccl_comm_init_all(int ndev, const int* devices, void** comms);
int amsq_nccl_comm_destroy(void* comm);

/* Number of this library's kernels launched so far in this process (bench accounting). */
uint64_t amsq_kernel_launch_count(void);
/* Profiling knob: device buffer of >= 64 u64 per CTA receiving %globaltimer stamps of
 * each fused-linear CTA (0 start, 1 first stage landed, 2 stream done, 3 end, 4..7 the
 * producer's first issues, 8+2s / 9+2s stage s landed / consumed); NULL = off. */
void amsq_debug_set_trace(void* d_buf);
/* Dispatch knob: batches of >= rows run the tcgen05 kernel (K3, schemes 4 and 7), smaller ones
 * the mma.sync kernel (K2) in 32-row chunks. rows > 0 overrides the per-scheme measured crossover
 * (FP5.33: 33, FP4.25: 40), rows < 0 restores it, 0 only queries. Returns the previous setting
 * (-1 = the per-scheme defaults). Process-wide. */
int amsq_debug_set_k3_min_batch(int rows);
/* K3 CTA-pair knob (cta_group::2 M = 256 MMAs, the activation image split across the pair):
 * -1 the measured rule (128 batch rows when the halved image admits >= 4 k-tiles per stage), 0 never, 1 whenever K is not split across
 * a cluster. Returns the previous setting. Test / tuning use. */
int amsq_debug_set_k3_pair(int mode);
/* amsq_gemv_host into page-locked host y: 1 (default) the epilogue stores into y directly, 0 device
 * scratch + a D2H copy as for pageable y. Returns the previous setting. Test / tuning use. */
int amsq_debug_set_host_direct(int on);
/* 1 when amsq_linear on a batch of `batch` rows of this scheme runs K3 (tcgen05), 0 for K2. */
int amsq_linear_uses_tc(int scheme_id, size_t batch);

#ifdef __cplusplus
}
#endif

#endif /* AMSQ_B200_H_ */
