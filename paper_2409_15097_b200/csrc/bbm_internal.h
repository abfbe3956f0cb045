// bbm_internal.h — shared host/device declarations for libbbm (not part of the public ABI).
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <type_traits>
#include <vector>

namespace bbm {

// Tile shape of the attention kernel (BLOCK_M query rows x BLOCK_N key rows). The preprocessor
// supports any BlockSpec; the kernel metadata is always also built at this shape.
constexpr uint32_t kTile = 128;

extern thread_local std::string g_last_error;  // capi.cu

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ArgError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

inline void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}
#define BBM_CUDA(x) ::bbm::check_cuda((x), #x)

inline void require(bool cond, const std::string& msg) {
  if (!cond) throw ArgError(msg);
}

// Kernel attributes (e.g. the opt-in shared memory size) belong to a device context: set them
// once per (kernel, device). `done` is a per-kernel bitmask of devices (threads of the
// multi-GPU driver launch on different devices concurrently).
template <class Set>
void once_per_device(std::atomic<uint64_t>& done, Set&& set) {
  int dev = 0;
  check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
  const uint64_t bit = uint64_t{1} << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return;
  set();
  done.fetch_or(bit, std::memory_order_release);
}

// Device metadata at the kernel tile shape (128 x 128), carved out of ONE device allocation (the
// arena) so that replication to another GPU is a single peer copy and an IPC export is a single
// handle. Layouts (all device memory):
//   mask      : padded bit-packed mask, ktiles*128 rows x kcols*2 u64 words (zero padded)
//   bitmaps   : uint4 [krows*kcols][128] tile-major copy of every occupied tile's mask bits at
//                                        its LIST position: row r of list entry (p,k) at
//                                        (p*kcols + k)*128 + r (16 bytes), written sparsely
//   sums      : u32 [krows][kcols]
//   list      : u32 [krows][kcols]       ascending occupied column tiles, bit 31 = full tile
//                                        (never set on a ragged right-edge tile)
//   row_cnt   : u32 [krows]              occupied tiles per query row tile
//   order     : u32 [krows]              scratch for the row tiles' LPT order
//   occ, run_off, run_len, row_stats, totals: the per-row pass's outputs at 128 x 128
struct KernelMeta {
  uint32_t krows = 0, kcols = 0;
  uint8_t* arena = nullptr;
  size_t arena_bytes = 0;
  uint64_t* mask = nullptr;
  uint4* bitmaps = nullptr;
  uint32_t* sums = nullptr;
  uint32_t* list = nullptr;
  uint32_t* row_cnt = nullptr;
  uint32_t* order = nullptr;
  uint8_t* occ = nullptr;
  // [krows][kcols] at list positions: bit 0 / bit 1 = key columns 0-63 / 64-127 of the tile are
  // empty for all 128 rows (the forward then loads and multiplies only the other 64 keys)
  uint8_t* halves = nullptr;
  uint32_t* run_off = nullptr;
  uint32_t* run_len = nullptr;
  uint64_t* row_stats = nullptr;
  uint64_t* totals = nullptr;
  uint32_t* scratch = nullptr;  // [krows + kcols + 2] ordering scratch (device LPT sort)
  uint32_t* partial = nullptr;  // [8][krows][kcols] fused preprocessor's per-slab tile sums
  uint32_t* ctr = nullptr;      // [krows + 1] fused preprocessor's finish counters (zero at rest)
};
void carve_kernel_meta(KernelMeta& km, uint64_t n, uint8_t* arena);  // sets pointers + bytes
size_t kernel_meta_bytes(uint64_t n);

// Per-spec metadata that mirrors the reference's MaskPrep (engine.hpp:71-78), host side.
struct SpecMeta {
  uint64_t bi = 0, bj = 0, rows = 0, cols = 0;
  std::vector<uint32_t> sums;
  std::vector<uint8_t> occ;
  std::vector<uint32_t> offset, total_ones;
  uint64_t blocks_total = 0, blocks_nonzero = 0, blocks_full = 0, ones = 0;
  uint64_t knnz = 0, kfull = 0;  // occupied / full tiles of the 128 x 128 kernel view
};

// Work decomposition of one attention launch (plan class x slots x SMs), BUILT ON THE DEVICE from
// row_cnt / list (plan.cu), so a mask update never needs the host: row units (whole row tiles, or
// balanced chunks of long ones = split-KV) in longest-first order. Header + arrays in one buffer.
struct PlanHdr {
  uint32_t units, split_rows, split_chunks, unit_len;
  uint32_t occupied, full;  // list plans: occupied tiles of the view and how many are full (bit 31)
  uint32_t halves;          // row view: occupied tiles with an empty 64-key half
};
struct DevPlan {
  uint64_t version = 0;  // mask version the plan was built from
  uint8_t* mem = nullptr;
  uint32_t cap_units = 0, cap_split = 0;
  PlanHdr* hdr = nullptr;
  uint4* unit_desc = nullptr;   // [cap_units] {row tile, j0, tiles, split | kNoSplit}
  uint2* split_info = nullptr;  // [cap_split] {chunks, first workspace chunk}
  uint4* tmp = nullptr;         // [cap_units] units in row order (before the LPT sort)
  uint32_t* hist = nullptr;     // [kcols + 2] sort scratch
  // {occupied, full} of the header, read back without blocking (pinned copy + event): the
  // forward picks its engine build from it once it has arrived (results do not depend on it)
  uint32_t* host_hdr = nullptr;
  cudaEvent_t hdr_ev = nullptr;
  uint64_t known_version = 0;
  bool partial_heavy = false;
  bool half_heavy = false;  // enough tiles with an empty key half for the forward to skip them
};

// Backward metadata (attn_bwd.cu): the column view of the kernel tiles — for key tile q, the
// ascending occupied query row tiles (bit 31 = full tile), and every
// occupied tile's mask bits TRANSPOSED (key-major) at its column-list position: key row c of
// column entry (q, k) at (q*krows + k)*128 + c (16 bytes over queries). Built on the device, on
// first backward use after each mask version (stream-ordered; no host sync).
struct BwdMeta {
  uint64_t version = 0;          // mask version of the column view (0 = never built)
  cudaEvent_t ready = nullptr;   // recorded after the latest column-view build
  uint32_t* col_cnt = nullptr;   // [kcols]
  uint32_t* col_list = nullptr;  // [kcols][krows]
  uint4* tbitmaps = nullptr;     // [kcols*krows][128]
  uint8_t* col_halves = nullptr; // [kcols*krows] per column-list position: bit h = query rows
                                 // 64h..64h+63 of the tile see no key (dkdv skips that half)
  uint32_t* scratch = nullptr;   // [kcols + krows + 2] ordering scratch
};

// Everything ONE launch mutates lives in a per-(prep, stream) context: launches on one stream
// are ordered by the stream, launches on different streams never share mutable device state.
struct StreamCtx {
  uint64_t seen_version = 0;     // mask version this stream has been ordered after
  cudaEvent_t done = nullptr;    // recorded after this stream's latest launch on the prep
  uint32_t* ctr = nullptr;       // device [8]: fwd next item / finished CTAs, bwd dq, bwd dkdv
  float* ws = nullptr;           // split-KV workspace
  size_t ws_floats = 0;
  uint32_t* split_ctr = nullptr; // split-KV finished-chunk counters
  size_t split_ctr_n = 0;
  float* rowws = nullptr;        // backward lse2 | delta
  size_t rowws_floats = 0;
  uint8_t* perm = nullptr;       // RCM pass-mode scratch: permuted Q/K/V/O + row statistics
  size_t perm_bytes = 0;
  std::map<std::tuple<int, uint64_t, uint32_t>, DevPlan> plans;
};

// Host-buffer pipeline of one prep's device (host_io.cu): persistent device buffers (grow-only)
// and three streams, so a host-buffer call overlaps H2D of slot chunk c+1, the kernel on chunk c
// and D2H of chunk c-1 instead of running copy -> kernel -> copy serially.
class HostPool;  // host_io.cu: persistent host threads for float -> bf16 conversion
struct HostPipe {
  cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
  std::vector<cudaEvent_t> ev_in, ev_out;
  uint8_t* buf = nullptr;
  size_t cap = 0;
  int* bad = nullptr;  // device finiteness flags (q, k, v, d_out)
  // float host path: slots converted to bf16 on the host go through two pinned staging buffers
  uint8_t* stage = nullptr;
  size_t stage_cap = 0;  // bytes per staging buffer
  cudaEvent_t ev_stage[2] = {nullptr, nullptr};
  HostPool* pool = nullptr;
  ~HostPipe();
};

// MaskPrep (engine.hpp:71-91): immutable between updates and shareable across threads and
// streams. The device metadata carries a version; bbm_prep_update_* rebuilds it on the caller's
// stream, bumps the version and records `ready`; every later launch orders its stream after
// `ready` (cudaStreamWaitEvent) and rebuilds its device plans, and the host-side caller-spec
// metadata (sums / occupancy / runs / stats / counters) is recomputed on the next getter call.
struct Prep {
  int device = 0;
  uint64_t n = 0;
  uint64_t bi = 0, bj = 0;       // the caller's BlockSpec
  KernelMeta kmeta;              // the kernel's 128x128 view (device)
  mutable std::recursive_mutex mu;  // guards everything below
  mutable uint64_t version = 1;     // bumped by each update
  cudaEvent_t ready = nullptr;      // recorded after the latest build / update of kmeta
  mutable SpecMeta spec;            // host metadata at the caller's spec ...
  mutable uint64_t spec_version = 0;  // ... valid for this version
  mutable BwdMeta bwd;
  mutable std::map<cudaStream_t, StreamCtx> streams;
  mutable std::mutex pipe_mu;       // host-buffer calls on one prep run one at a time
  mutable HostPipe* pipe = nullptr;

  // Context of stream `s` (created on first use), ordered after the latest metadata version.
  StreamCtx& ctx_for(cudaStream_t s) const;
  // Host-side caller-spec metadata for the current version (synchronous refresh if stale).
  const SpecMeta& spec_now() const;
  ~Prep();
};

// ---- kernel launchers (prep.cu) ----
void launch_pack_bool(const uint8_t* d_bool, uint64_t n, uint64_t row_stride, const KernelMeta& km,
                      cudaStream_t s);
void launch_pad_packed(const uint64_t* d_words, uint64_t n, const KernelMeta& km, cudaStream_t s);
// the whole kernel view (padded mask, sums, lists, bitmaps, totals, LPT order) in ONE launch;
// false when the input does not fit the fused path (the caller falls back to the chain)
bool launch_prep_fused_bool(const uint8_t* d_bool, uint64_t n, uint64_t stride, const KernelMeta& km,
                            cudaStream_t s);
bool launch_prep_fused_words(const uint64_t* d_words, uint64_t in_wpr, uint64_t n, const KernelMeta& km,
                             cudaStream_t s);
void launch_sums128(const KernelMeta& km, cudaStream_t s);
void launch_sums_generic(const KernelMeta& km, uint64_t n, uint64_t bi, uint64_t bj,
                         uint64_t rows, uint64_t cols, uint32_t* d_sums, cudaStream_t s);
void launch_rowmeta(const uint32_t* d_sums, uint64_t n, uint64_t bi, uint64_t bj, uint64_t rows,
                    uint64_t cols, uint8_t* d_occ, uint32_t* d_offset, uint32_t* d_total,
                    uint64_t* d_row_stats /* rows x 3 */, uint32_t* d_list, uint32_t* d_cnt,
                    cudaStream_t s);
void launch_compact_bitmaps(const KernelMeta& km, cudaStream_t s);
void launch_finalize(const uint64_t* d_row_stats, uint64_t rows, const uint32_t* d_cnt,
                     uint32_t* d_order, uint64_t* d_totals /* 3 */, cudaStream_t s);

// ---- device mask generators (gen.cu; spec parsing in host_generators.cpp) ----
enum GenFamily : int { kGenCausal = 0, kGenAllOnes, kGenWindowed, kGenDilated, kGenGlobal, kGenRandom };
struct GenSpec {
  int family = 0;
  uint64_t n = 0, w = 0, d = 1, g = 0, seed = 0;
  double p = 0.0;
  bool causal = false, diag = true;
};
// true (and `out` filled, validated like the reference) for the families generated on the device
bool parse_device_family(const std::string& spec, uint64_t n_free, GenSpec& out);
void launch_generate(const GenSpec& g, uint64_t* d_words, cudaStream_t s);

// ---- mask files (mask_io.cu) ----
void launch_bbmk_unpack(const uint8_t* d_payload, uint64_t n, uint64_t* d_words, uint64_t wpr,
                        uint64_t rows_out, cudaStream_t s);

// ---- permutation kernels (permute.cu) ----
void launch_permute_rows(const void* src, void* dst, const uint32_t* d_fwd, uint64_t slots,
                         uint64_t n, uint64_t row_bytes, bool inverse, cudaStream_t s);
void launch_permute_mask(const uint64_t* d_src, uint64_t* d_dst, const uint32_t* d_fwd,
                         uint64_t n, uint64_t src_wpr, uint64_t dst_wpr, cudaStream_t s);

// ---- attention (attn_fwd.cu) ----
struct AttnArgs {
  const void* q;
  const void* k;
  const void* v;
  void* o;
  float* row_max;
  float* row_sum;
  uint64_t slots;
  uint64_t n;
  uint32_t d;
  float scale;
  int variant;
  // optional in-kernel RCM application (reorder.hpp:156-189): device u32 [n], forward map new ->
  // old. q/k/v/o and the row statistics are then in the ORIGINAL token order while the prep holds
  // the permuted mask: rows are gathered / scattered by TMA inside the kernel (kGatherTma), or
  // permuted into per-stream scratch by HBM-bound passes around the plain kernel (kGatherPasses),
  // or K / V permuted by passes while Q / O rows are gathered / scattered in the kernel
  // (kGatherHybrid), or every row gathered inside the kernel by LSU cp.async (kGatherLsu, the
  // default: gather_mode_of in attn_fwd.cu).
  const uint32_t* rows = nullptr;
  int gather_mode = 0;
};
enum GatherMode : int { kGatherAuto = 0, kGatherPasses = 1, kGatherTma = 2, kGatherHybrid = 3, kGatherLsu = 4 };
// Process-wide kernel event trace (bbm_set_trace): device buffer of ctas * 8192 u64 events.
struct TraceConfig {
  void* buffer = nullptr;
  uint32_t ctas = 0;
};
extern TraceConfig g_trace;
// the fused preprocessor splits a tile row's 128 rows over this many CTAs (KernelMeta.partial)
#ifndef BBM_PREP_SPLITS
#define BBM_PREP_SPLITS 8
#endif
constexpr uint32_t kPrepRowSplits = BBM_PREP_SPLITS;
// forward launches so far per softmax engine build (plain, empty-half skipping)
void fwd_build_counts(uint64_t& plain, uint64_t& skipping);

void launch_attn_fwd(const Prep& prep, const AttnArgs& a, cudaStream_t s, int num_sms);
// the two-stream forward (attn_fwd_pair.cu) when selected with set_fwd_kernel(2); false = not
// selected or not applicable (the caller runs attn_fwd.cu)
bool launch_attn_fwd_pair(const Prep& prep, const AttnArgs& a, cudaStream_t s, int num_sms);
void set_fwd_kernel(int mode);  // 0 default (single-stream), 1 single-stream, 2 pair wherever it can run

// ---- device launch plans (plan.cu) ----
enum PlanClass : int { kPlanDense = 0, kPlanNaive = 1, kPlanList = 2 };
constexpr uint32_t kNoSplit = 0xFFFFFFFFu;
// upper bound on row units per slot of a plan and on workspace chunk blocks of one launch
uint32_t plan_cap_units(uint32_t krows, uint32_t kcols, uint64_t slots, uint32_t workers);
uint64_t plan_cap_chunks(uint64_t slots, uint32_t workers);
// The tile lists a plan cuts into units: the forward / dq walk the row view (row_cnt, list),
// dkdv the column view (col_cnt, col_list).
struct TileView {
  const uint32_t* cnt;
  const uint32_t* list;  // [tiles][partners]
  uint32_t tiles, partners;
  int id;  // plan-cache key: 0 rows, 1 columns
  const uint8_t* halves = nullptr;  // row view: per list position, the tile's empty key halves
};
inline TileView row_view(const KernelMeta& km) { return {km.row_cnt, km.list, km.krows, km.kcols, 0, km.halves}; }
// (re)build `plan` on stream s for the current metadata (kernel, no host sync)
void build_plan(const TileView& v, int cls, uint64_t slots, uint32_t workers, DevPlan& plan,
                cudaStream_t s);
const DevPlan& plan_for(const Prep& prep, StreamCtx& ctx, const TileView& v, int cls, uint64_t slots,
                        uint32_t workers, cudaStream_t s);
// LPT order of `count` keys (descending key, ties by index) into out[count], one CTA on s
void launch_lpt_order(const uint32_t* keys, uint32_t count, uint32_t max_key, uint32_t* scratch,
                      uint32_t* out, cudaStream_t s);
// record ctx.done after a launch on s (bbm_prep_update_* orders itself after it)
void mark_launch_done(StreamCtx& ctx, cudaStream_t s);
// grow-only per-stream scratch
float* ctx_workspace(StreamCtx& ctx, size_t floats, cudaStream_t s);
uint32_t* ctx_split_ctr(StreamCtx& ctx, size_t count, cudaStream_t s);
uint8_t* ctx_perm_scratch(StreamCtx& ctx, size_t bytes, cudaStream_t s);

// ---- attention backward (attn_bwd.cu) ----
struct BwdArgs {
  const void* q;  // bf16 [slots][n][d]
  const void* k;
  const void* v;
  const void* o;        // forward output: bf16 (o_f32 == false) or fp32 [slots][n][d]
  bool o_f32;
  const float* row_max;  // [slots][n] natural-log units (ForwardResult::row_max)
  const float* row_sum;  // [slots][n]
  const void* d_out;     // bf16 [slots][n][d]
  void* dq;              // bf16 [slots][n][d]
  void* dk;
  void* dv;
  uint64_t slots;
  uint64_t n;
  uint32_t d;
  float scale;
  int variant;
};
// column view for the current version, built on stream s if stale (stream-ordered, no host sync)
void ensure_bwd_meta(const Prep& prep, cudaStream_t s);
void launch_attn_bwd(const Prep& prep, const BwdArgs& a, cudaStream_t s, int num_sms);
void free_bwd_meta(BwdMeta& b);
int attn_fwd_kernel_launches_per_call();

// host-buffer forward through the prep's pipeline (host_io.cu): bf16 host q/k/v/out (pinned for
// full PCIe bandwidth), optional fp32 row stats; synchronous. Returns the device-side span in ms
// (first H2D issued -> last D2H done) when `span_ms` is non-null.
void run_fwd_host_pipelined(const Prep& prep, int variant, const uint16_t* q, const uint16_t* k,
                            const uint16_t* v, uint16_t* out, float* row_max, float* row_sum,
                            uint64_t slots, uint32_t d, float scale, int num_sms, double* span_ms);
// the reference's Matrix<float> signature: per-slot float host buffers in, float out, double row
// statistics (row_max / row_sum arrays, or their entries, may be null); synchronous. Any head dims
// d_k, d_v <= 128: the kernel runs at kernel_dim(d_k, d_v) with the inputs zero-padded on the
// device (zero Q/K columns add exact zeros to every score, zero V columns give output columns
// that are dropped).
void run_fwd_host_f32(const Prep& prep, int variant, const float* const* q, const float* const* k,
                      const float* const* v, float* const* out, double* const* row_max,
                      double* const* row_sum, uint64_t slots, uint32_t d_k, uint32_t d_v, float scale,
                      int num_sms, double* span_ms);
// blocked_backward over float host buffers (q, k, dq, dk: d_k wide; v, out, d_out, dv: d_v wide),
// double row statistics; synchronous, on the prep's pipeline stream and buffers
void run_bwd_host_f32(const Prep& prep, int variant, const float* q, const float* k, const float* v,
                      const float* out, const double* row_max, const double* row_sum, const float* d_out,
                      float* dq, float* dk, float* dv, uint64_t slots, uint32_t d_k, uint32_t d_v,
                      float scale, int num_sms);
// the kernels' head dim for caller dims d_k, d_v in [1, 128]
inline uint32_t kernel_dim(uint32_t d_k, uint32_t d_v) { return (d_k > 64 || d_v > 64) ? 128u : 64u; }
// row-pitch changes between the caller's dims and the kernel's (host_io.cu), on stream s:
// float [rows][w] -> bf16 [rows][D] (zero columns w..D-1; RNE; any inf / NaN sets *bad if non-null),
// float [rows][w] -> float [rows][D] (zero-padded), bf16 [rows][D] -> float [rows][w] (cropped)
void launch_pad_to_bf16(const float* in, void* out, uint64_t rows, uint32_t w, uint32_t D, int* bad,
                        cudaStream_t s);
void launch_pad_f32(const float* in, float* out, uint64_t rows, uint32_t w, uint32_t D, cudaStream_t s);
void launch_crop_to_f32(const void* in, float* out, uint64_t rows, uint32_t D, uint32_t w, cudaStream_t s);
// the RCM path end to end: original-order host buffers, prep built from the permuted mask
void run_fwd_host_rcm(const Prep& prep, int variant, const uint32_t* forward, const uint16_t* q,
                      const uint16_t* k, const uint16_t* v, uint16_t* out, float* row_max,
                      float* row_sum, uint64_t slots, uint32_t d, float scale, int num_sms,
                      double* span_ms);

}  // namespace bbm
