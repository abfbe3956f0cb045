/* bbm_capi.h — C ABI of libbbm, the B200-native Binary Block Masking engine.
 *
 * This is the drop-in boundary below the reference's C++ API (namespace blockmask in
 * /root/reference/proj/include/blockmask). Plain pointers and sizes only; no torch or C++ types.
 * The C++ drop-in headers in include/blockmask/ and the Python package
 * paper_2409_15097_b200/ both bind exactly these symbols.
 *
 * Each entry point names the reference interface it replaces (file:line under proj/include).
 * Error convention: every call returns a bbm_status; on failure bbm_last_error() holds a
 * thread-local message. BBM_ERR_INVALID corresponds to the reference's
 * require() -> std::invalid_argument (matrix.hpp:47-49) and is raised on the same triggers
 * (engine.hpp:244-258, 493-496); the C++ wrappers rethrow it as std::invalid_argument.
 * There is no CPU fallback: compute entry points fail with BBM_ERR_CUDA when no device exists.
 *
 * Mask layout (input): the reference's bit-packed rows, u64 words, words_per_row = ceil(n/64),
 * bit j of row i at word j>>6 bit j&63, tail bits zero (mask.hpp:17-52); or a dense n x n bool
 * (uint8) mask on the device. Attention tensors: bf16 [slots][n][d], d in {64,128}, row-major.
 */
#ifndef BBM_CAPI_H
#define BBM_CAPI_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BBM_ABI_VERSION 2

typedef enum {
  BBM_OK = 0,
  BBM_ERR_INVALID = 1,     /* bad argument: reference would throw std::invalid_argument */
  BBM_ERR_CUDA = 2,        /* CUDA runtime / device failure (including "no device") */
  BBM_ERR_UNSUPPORTED = 3, /* valid for the reference, not for the sm_100a kernel (e.g. d=5) */
  BBM_ERR_INTERNAL = 4,
  /* MaskIoError kinds (mask_io.hpp:24-42) from the mask-file entry points */
  BBM_ERR_IO_FAILURE = 10,
  BBM_ERR_IO_BAD_MAGIC = 11,
  BBM_ERR_IO_BAD_VERSION = 12,
  BBM_ERR_IO_DIMENSION_OVERFLOW = 13,
  BBM_ERR_IO_TRUNCATED = 14,
  BBM_ERR_IO_TRAILING_DATA = 15
} bbm_status;

/* Variant (engine.hpp:21-26); same numbering as the reference enum. */
typedef enum {
  BBM_VARIANT_DENSE = 0,
  BBM_VARIANT_NAIVE = 1,
  BBM_VARIANT_BINBLK = 2,
  BBM_VARIANT_DENSE_BINBLK = 3
} bbm_variant;

/* BlockStats (mask.hpp:156-162) */
typedef struct {
  uint64_t blocks_total, blocks_nonzero, blocks_full;
  double block_density, element_density;
} bbm_block_stats;

/* EngineCounters (engine.hpp:49-66) */
typedef struct {
  uint64_t blocks_visited, blocks_processed, mask_block_reads, skipped_by_binblk,
      skipped_mask_reads_by_run;
} bbm_counters;

typedef struct {
  uint64_t n, block_i, block_j, rows, cols; /* caller's BlockSpec view (BlockSums geometry) */
  uint32_t ktile, krows, kcols;             /* attention kernel's 128x128 view */
  uint64_t knnz, kfull;                     /* occupied / full tiles in the kernel view */
  int device;
} bbm_prep_info;

/* Opaque MaskPrep (engine.hpp:71-78): host copies of sums/occupancy/runs/stats plus the
 * device-resident kernel metadata (compacted tile lists, tile-major partial bitmaps).
 * Like the reference's MaskPrep ("built once and shared across heads, runs and both passes",
 * engine.hpp:68-70) a prep may be used from any number of threads and streams concurrently:
 * everything a launch mutates (work counters, split-KV workspace, launch plans) is private to the
 * launching stream. */
typedef struct bbm_prep_s* bbm_prep;

int bbm_abi_version(void);
const char* bbm_last_error(void);
bbm_status bbm_device_count(int* count);

/* ---- preprocess_mask (engine.hpp:80-91): block_sums + build_block_occupancy +
 *      build_dense_runs + block_stats (mask.hpp:184-247), computed on the GPU. Any BlockSpec
 *      with block_i, block_j >= 1 (BlockSpec::validate, mask.hpp:61-63); n >= 1. ---- */
bbm_status bbm_preprocess_packed_host(const uint64_t* words, uint64_t n, uint64_t block_i,
                                      uint64_t block_j, int device, bbm_prep* out);
bbm_status bbm_preprocess_packed_device(const uint64_t* d_words, uint64_t n, uint64_t block_i,
                                        uint64_t block_j, void* stream, bbm_prep* out);
/* Dense bool mask on the device (K1: pack + sums fused), row stride in bytes. */
bbm_status bbm_preprocess_bool_device(const uint8_t* d_mask, uint64_t n, uint64_t row_stride,
                                      uint64_t block_i, uint64_t block_j, void* stream,
                                      bbm_prep* out);
/* Rebuild an existing prep for a new mask of the same n (the per-batch path when every batch
 * packs different sequences), fully asynchronously on `stream`: no host copies, no allocation.
 * The update is ordered after every launch already queued on the prep (any stream), and every
 * later launch (any stream) is ordered after the update; launch plans are rebuilt on the device.
 * The caller-spec metadata (sums/occupancy/runs/stats getters, counters, info) is recomputed on
 * the next getter call (one synchronization there), and replicas made for the multi-GPU driver
 * are dropped and re-made from the new mask on their next use. */
bbm_status bbm_prep_update_bool_device(bbm_prep prep, const uint8_t* d_mask, uint64_t row_stride,
                                       void* stream);
bbm_status bbm_prep_update_packed_device(bbm_prep prep, const uint64_t* d_words, void* stream);
bbm_status bbm_prep_destroy(bbm_prep prep);
bbm_status bbm_prep_get_info(bbm_prep prep, bbm_prep_info* info);
/* BlockSums::sum(p,q) row-major [rows][cols] (mask.hpp:71-109) */
bbm_status bbm_prep_get_sums(bbm_prep prep, uint32_t* sums);
/* BlockOccupancy (mask.hpp:113-132), u8 [rows][cols] */
bbm_status bbm_prep_get_occupancy(bbm_prep prep, uint8_t* occ);
/* DenseRuns offset / total_ones, u32 [rows] each (mask.hpp:139-154) */
bbm_status bbm_prep_get_runs(bbm_prep prep, uint32_t* offset, uint32_t* total_ones);
/* BlockStats (mask.hpp:230-247) */
bbm_status bbm_prep_get_stats(bbm_prep prep, bbm_block_stats* stats);
/* Kernel view: row_cnt[krows], list[krows*kcols] (bit31 = full tile), LPT order[krows].
 * Any pointer may be NULL. */
bbm_status bbm_prep_get_kernel_lists(bbm_prep prep, uint32_t* row_cnt, uint32_t* list,
                                     uint32_t* order);
/* Per list position of the kernel view, u8 [krows*kcols]: bit 0 / bit 1 = key columns 0-63 /
 * 64-127 of that occupied 128x128 tile are empty for all of its rows (the forward neither loads
 * nor multiplies that half). No reference counterpart (a finer-grained classify_tile,
 * engine.hpp:118-153); exposed for tests. */
bbm_status bbm_prep_get_tile_halves(bbm_prep prep, uint8_t* halves);
/* EngineCounters a blocked_forward over `slots` slots reports for `variant`
 * (classify_tile, engine.hpp:118-153; summed as run_attention does, engine.hpp:500-503). */
bbm_status bbm_prep_counters(bbm_prep prep, int variant, uint64_t slots, bbm_counters* out);
/* build_block_occupancy + build_dense_runs + block_stats (mask.hpp:203-247) for a caller-held
 * BlockSums (u32 [ceil(n/bi)][ceil(n/bj)], row-major), on `device`: the same per-row-tile
 * kernel the preprocessor runs after its sums pass. Any output pointer may be NULL. */
bbm_status bbm_sums_metadata(const uint32_t* sums, uint64_t n, uint64_t block_i, uint64_t block_j,
                             int device, uint8_t* occ, uint32_t* offset, uint32_t* total_ones,
                             bbm_block_stats* stats);
/* Peer-to-peer copy of the device metadata to another GPU (NVLink), for the multi-GPU driver.
 * The result is an independent prep bound to `device`. The kernel view is one device arena, so
 * this is one cudaMemcpyPeerAsync. */
bbm_status bbm_prep_replicate(bbm_prep prep, int device, void* stream, bbm_prep* out);
/* The same replication across processes (one process per GPU): export writes a flat blob (the
 * arena's cudaIpcMemHandle + the host metadata; blob == NULL queries *size), import opens the
 * handle on `device`, copies the arena peer to peer and returns an independent prep. The exporting
 * prep must stay alive and un-updated until every importer has returned. */
bbm_status bbm_prep_export_ipc(bbm_prep prep, void* blob, size_t* size);
bbm_status bbm_prep_import_ipc(const void* blob, size_t size, int device, void* stream,
                               bbm_prep* out);

/* ---- blocked_forward (engine.hpp:282-341) over `slots` independent (batch, head) slots that
 *      share one mask (run_attention, engine.hpp:489-505). Device pointers, bf16 [slots][n][d];
 *      row_max / row_sum fp32 [slots][n] in natural-log units (NULL to skip). Asynchronous on
 *      `stream` (a cudaStream_t, NULL = legacy default stream). ---- */
bbm_status bbm_attn_fwd(bbm_prep prep, int variant, const void* q, const void* k, const void* v,
                        void* out, float* row_max, float* row_sum, uint64_t slots,
                        uint32_t head_dim, double scale, void* stream);

/* The same forward with the RCM permutation applied on the device (reorder.hpp:156-189):
 * `prep` was built from permute_mask(mask, perm), d_forward = perm.forward (new -> old, device
 * u32 [n]), and q/k/v/out/row stats stay in the ORIGINAL token order. Four implementations, equal
 * results bit for bit: mode 4 (the default) gathers every Q / K / V row inside the kernel with LSU
 * cp.async and writes O rows / row stats to their tokens (no scratch); mode 3 permutes K and V into
 * per-stream scratch (2 x slots*n*d bf16) and gathers Q / scatters O with TMA tile::gather4 /
 * scatter4; mode 1 permutes Q/K/V into scratch (4 x slots*n*d bf16 + 2 x slots*n fp32), runs the
 * plain kernel and scatters O / row stats back; mode 2 gathers every row with tile::gather4 (bound
 * by the TMA instruction rate). Modes 2-4 require slots * n < 2^31. bbm_attn_fwd_gather = mode 0 =
 * the default (env BBM_GATHER=passes|tma|hybrid|lsu overrides). */
bbm_status bbm_attn_fwd_gather(bbm_prep prep, int variant, const uint32_t* d_forward, const void* q,
                               const void* k, const void* v, void* out, float* row_max, float* row_sum,
                               uint64_t slots, uint32_t head_dim, double scale, void* stream);
bbm_status bbm_attn_fwd_gather_ex(bbm_prep prep, int variant, const uint32_t* d_forward, const void* q,
                                  const void* k, const void* v, void* out, float* row_max, float* row_sum,
                                  uint64_t slots, uint32_t head_dim, double scale, void* stream, int mode);

/* Same, host buffers (bf16 bits as uint16): copies in, runs, copies out, synchronizes.
 * Pinned buffers get full PCIe bandwidth. Validates finiteness (engine.hpp:237-258). */
bbm_status bbm_attn_fwd_host_bf16(bbm_prep prep, int variant, const uint16_t* q,
                                  const uint16_t* k, const uint16_t* v, uint16_t* out,
                                  float* row_max, float* row_sum, uint64_t slots,
                                  uint32_t head_dim, double scale);

/* The reordered pipeline end to end (bench.hpp:448-467 with reorder.hpp:156-189 on the device):
 * q/k/v/out/row stats in the ORIGINAL token order, `prep` built from permute_mask(mask, perm),
 * `forward` = perm.forward (new -> old, host u32 [n]). Rows are gathered into the reordered
 * layout, attended with the reordered mask, and O / row stats scattered back, on the device,
 * pipelined with the PCIe copies. Equals the attention with the original mask (equivariance). */
bbm_status bbm_attn_fwd_rcm_host_bf16(bbm_prep prep, int variant, const uint32_t* forward,
                                      const uint16_t* q, const uint16_t* k, const uint16_t* v,
                                      uint16_t* out, float* row_max, float* row_sum, uint64_t slots,
                                      uint32_t head_dim, double scale);

/* Same, float host buffers (the reference's Matrix<float> storage, matrix.hpp:14-45); inputs
 * rounded to bf16 (RNE) on the device, output widened back to float; row stats as double.
 * Validates finiteness like validate_forward_args (engine.hpp:244-258). Copy/compute pipeline
 * over slot chunks, like the bf16 form. The float host-buffer entries take any head dim in
 * [1, 128] (the device-pointer entries: 64 or 128): the device copy is zero-padded to 64 or 128
 * columns, which leaves every score and output unchanged. */
bbm_status bbm_attn_fwd_host_f32(bbm_prep prep, int variant, const float* q, const float* k,
                                 const float* v, float* out, double* row_max, double* row_sum,
                                 uint64_t slots, uint32_t head_dim, double scale);
/* run_attention<float> (engine.hpp:489-505) with the reference's per-slot storage: slot i's
 * Matrix<float> q/k/v (n x d, row-major) at q[i]/k[i]/v[i], ForwardResult<float>::out at out[i]
 * and its double row_max / row_sum at row_max[i] / row_sum[i] (the arrays may be NULL). */
bbm_status bbm_run_attention_host_f32(bbm_prep prep, int variant, const float* const* q,
                                      const float* const* k, const float* const* v,
                                      float* const* out, double* const* row_max,
                                      double* const* row_sum, uint64_t slots, uint32_t head_dim,
                                      double scale);
/* The same with the value head dim independent of the key head dim
 * (EngineForward.ValueHeadDimMayDifferFromKeyDim, test_engine.cpp:198-209): q/k are n x d_k,
 * v/out n x d_v; 1 <= d_k <= 128, d_v >= 1 (d_v above 128 runs as column passes over V, each
 * recomputing the same softmax). */
bbm_status bbm_run_attention_host_f32_dims(bbm_prep prep, int variant, const float* const* q,
                                           const float* const* k, const float* const* v,
                                           float* const* out, double* const* row_max,
                                           double* const* row_sum, uint64_t slots, uint32_t d_k,
                                           uint32_t d_v, double scale);

/* ---- blocked_backward (engine.hpp:346-471): dq, dk, dv of L = sum(out * d_out) from the forward's
 *      saved row statistics (row_max / row_sum as bbm_attn_fwd returns them), over the same tiles
 *      the forward processed. Deterministic (no atomics on gradients). Device pointers, bf16
 *      [slots][n][d]; asynchronous on `stream`. The first call after each mask version builds
 *      the column view (column tile lists + transposed partial-tile bitmaps) on the device. ---- */
bbm_status bbm_attn_bwd(bbm_prep prep, int variant, const void* q, const void* k, const void* v,
                        const void* out, const float* row_max, const float* row_sum,
                        const void* d_out, void* dq, void* dk, void* dv, uint64_t slots,
                        uint32_t head_dim, double scale, void* stream);
/* Same, float host buffers (Matrix<float>) with the reference's double row statistics; q, k, v,
 * d_out are rounded to bf16 on the device, out stays fp32 for delta = rowsum(d_out * out).
 * Validates finiteness of q, k, v, d_out (engine.hpp:244-258, 358). Synchronous. */
bbm_status bbm_attn_bwd_host_f32(bbm_prep prep, int variant, const float* q, const float* k,
                                 const float* v, const float* out, const double* row_max,
                                 const double* row_sum, const float* d_out, float* dq, float* dk,
                                 float* dv, uint64_t slots, uint32_t head_dim, double scale);
/* The same with d_v != d_k allowed: q, k, dq, dk are n x d_k; v, out, d_out, dv are n x d_v
 * (d_v above 128: column passes over V, dq / dk summed over the passes in order). */
bbm_status bbm_attn_bwd_host_f32_dims(bbm_prep prep, int variant, const float* q, const float* k,
                                      const float* v, const float* out, const double* row_max,
                                      const double* row_sum, const float* d_out, float* dq, float* dk,
                                      float* dv, uint64_t slots, uint32_t d_k, uint32_t d_v, double scale);

/* Multi-GPU run_attention: slots sharded contiguously over `n_devices` GPUs
 * ([g*S/G, (g+1)*S/G)), metadata replicated peer-to-peer from prep's device, one stream per
 * GPU, no collective. Host bf16 buffers. elapsed_ms (may be NULL) = device time, max over GPUs
 * of the kernel span measured from a common start. */
bbm_status bbm_run_attention_multi(bbm_prep prep, int variant, int n_devices,
                                   const int* devices, const uint16_t* q, const uint16_t* k,
                                   const uint16_t* v, uint16_t* out, float* row_max,
                                   float* row_sum, uint64_t slots, uint32_t head_dim,
                                   double scale, double* elapsed_ms);

/* ---- tracing (no reference counterpart; the reference only has steady_clock timings,
 *      bench.hpp:155-159): every attention launch made after this call records per-role events
 *      (TMA issue, MMA issue, softmax waits/arrivals; clock64 cycles) for CTAs [0, ctas) into
 *      d_buffer (device, ctas * 8192 u64). NULL disables. Format in attn_fwd.cu (trace_ev). ---- */
bbm_status bbm_set_trace(void* d_buffer, uint32_t ctas);

/* ---- forward engine builds (diagnostics, no reference counterpart): how many forward launches
 *      of this process ran the plain softmax engine build and how many the build that skips
 *      empty score halves (chosen per launch plan from its occupied/full tile counts). ---- */
bbm_status bbm_fwd_build_counts(uint64_t* plain, uint64_t* skipping);

/* ---- forward kernel selection (diagnostics and tests, no reference counterpart): 0 = default
 *      (attn_fwd.cu, one query tile per item with the softmax split over two warpgroups),
 *      1 = the same, 2 = the two-stream kernel attn_fwd_pair.cu wherever it can run (two query
 *      tiles per CTA sharing K/V loads, one softmax thread per row; bit-identical results where
 *      attn_fwd.cu splits no row, measured slower on B200). Process-wide; the environment
 *      variable BBM_FWD_KERNEL=single|pair sets the initial value. ---- */
bbm_status bbm_set_fwd_kernel(int mode);

/* ---- reorder.hpp ---- */
/* rcm_order(build_graph(mask)) (reorder.hpp:28-133): forward[new] = old. Host. */
bbm_status bbm_rcm_order(const uint64_t* words, uint64_t n, uint32_t* forward);
/* bandwidth (reorder.hpp:137-153). Host. */
bbm_status bbm_bandwidth(const uint64_t* words, uint64_t n, uint64_t* bandwidth);
/* permute_rows / unpermute_rows (reorder.hpp:167-189) on the device over `slots` matrices
 * [slots][n][row_bytes]; inverse != 0 scatters (unpermute). d_forward: u32 [n] on device. */
bbm_status bbm_permute_rows_device(const void* src, void* dst, const uint32_t* d_forward,
                                   uint64_t slots, uint64_t n, uint64_t row_bytes, int inverse,
                                   void* stream);
/* permute_mask (reorder.hpp:156-163) on the device: mask'(a,b) = mask(fwd[a], fwd[b]);
 * both masks in the reference packed layout (ceil(n/64) words per row). */
bbm_status bbm_permute_mask_device(const uint64_t* d_src, uint64_t* d_dst,
                                   const uint32_t* d_forward, uint64_t n, void* stream);

/* Host-buffer forms of the two kernels above (upload, permute on `device`, download), for the
 * Matrix<T>/Mask overloads of the C++ drop-in headers. Any row_bytes >= 1. `forward` must be a
 * bijection (Permutation::from_forward, reorder.hpp:57-68) or BBM_ERR_INVALID is returned. */
bbm_status bbm_permute_rows_host(const void* src, void* dst, const uint32_t* forward,
                                 uint64_t slots, uint64_t n, uint64_t row_bytes, int inverse,
                                 int device);
bbm_status bbm_permute_mask_host(const uint64_t* src, uint64_t* dst, const uint32_t* forward,
                                 uint64_t n, int device);
/* build_graph (reorder.hpp:28-49) as CSR: offsets u64 [n+1]; neighbors u32 [offsets[n]] sorted
 * ascending per node (NULL to query offsets only). Host. */
bbm_status bbm_graph_csr(const uint64_t* words, uint64_t n, uint64_t* offsets, uint32_t* neighbors);

/* ---- mask_io.hpp: BBMK mask files and BBLK occupancy sidecars (mask_io.hpp:14-207), same
 *      byte layout, 4M-token cap and error kinds (BBM_ERR_IO_*). Host, except
 *      bbm_preprocess_mask_file, which uploads the file's byte rows as-is and unpacks them on
 *      the device straight into the preprocessor (read_mask + preprocess_mask). ---- */
bbm_status bbm_write_mask_file(const char* path, const uint64_t* words, uint64_t n);
/* words == NULL: query n only. Else words receives n * ceil(n/64) u64 (the Mask layout). */
bbm_status bbm_read_mask_file(const char* path, uint64_t* n, uint64_t* words);
/* occ: u8 [ceil(n/bi)][ceil(n/bj)] (BlockOccupancy) */
bbm_status bbm_write_occupancy_file(const char* path, const uint8_t* occ, uint64_t n_tokens,
                                    uint64_t block_i, uint64_t block_j);
/* occ == NULL: query n_tokens / block sizes only. */
bbm_status bbm_read_occupancy_file(const char* path, uint64_t* n_tokens, uint64_t* block_i,
                                   uint64_t* block_j, uint8_t* occ);
bbm_status bbm_preprocess_mask_file(const char* path, uint64_t block_i, uint64_t block_j,
                                    int device, bbm_prep* out);

/* ---- generators.hpp (host fixtures): MaskSpec grammar (generators.hpp:364-438); families with
 *      a free n take n_free. Call with words == NULL to query n. ---- */
bbm_status bbm_generate(const char* spec, uint64_t n_free, uint64_t* n_out, uint64_t* words);
/* The same, generated straight into DEVICE memory (d_words: n * ceil(n/64) u64 on the current
 * device, NULL to query n), asynchronously on `stream`: causal, all-ones, windowed, dilated,
 * global and random (one mt19937_64 stream over the n^2 entries, as generators.hpp:171-183) run
 * as kernels, bit-identical to the reference; the other families are built on the host and
 * uploaded. */
bbm_status bbm_generate_device(const char* spec, uint64_t n_free, uint64_t* n_out, uint64_t* d_words,
                               void* stream);
/* make_problem's input stream (bench.hpp:320-337, rng.hpp:15-42): per slot q, k, v, d_out
 * (n x d each, uniform [-1,1) from one mt19937_64(seed), drawn in that order), as float. Host. */
bbm_status bbm_make_problem(uint64_t seed, uint64_t slots, uint64_t n, uint64_t d, float* q,
                            float* k, float* v, float* d_out);
/* Relabel a mask's tokens by a std::shuffle(mt19937_64(seed)) permutation:
 * out(label[i], label[j]) = in(i, j) (the test_reorder.cpp relabel fixture). */
bbm_status bbm_relabel(const uint64_t* words, uint64_t n, uint64_t seed, uint64_t* out_words);

#ifdef __cplusplus
}
#endif
#endif /* BBM_CAPI_H */
