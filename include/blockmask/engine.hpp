// blockmask/engine.hpp — drop-in for the reference's attention engine (proj/include/blockmask/
// engine.hpp:21-505). Same types and entry points; the work runs on the B200:
//
//   preprocess_mask (engine.hpp:80-91)      -> bbm_preprocess_packed_host (GPU preprocessor; the
//                                              MaskPrep keeps the device metadata alive)
//   blocked_forward (engine.hpp:282-341)    -> bbm_run_attention_host_f32_dims (sm_100a kernel)
//   blocked_backward (engine.hpp:346-471)   -> bbm_attn_bwd_host_f32_dims
//   run_attention (engine.hpp:489-505)      -> bbm_run_attention_host_f32_dims over all slots (each
//                                              slot's Matrix<float> storage used in place)
//
// Numerics: Q/K/V are rounded to bf16 (RNE) on the device and the kernel accumulates in fp32, so
// outputs agree with the reference to a bf16 tolerance (max-abs <= 2e-2; tests/), not bit for
// bit. Counters (engine.hpp:47-66) are exact: they depend on the mask and spec only.
// New rejection (std::invalid_argument): key head dim d_k above 128 (the kernels hold one
// 128-column head-dim tile of Q / K; smaller or unequal dims are zero-padded on the device to
// 64 / 128, and d_v above 128 runs as column passes over V).
// `threads` is validated (>= 1) like the reference and otherwise ignored.
#pragma once

#include <cmath>
#include <cstdint>
#include <limits>
#include <memory>
#include <span>
#include <string>
#include <type_traits>
#include <vector>

#include "blockmask/device.hpp"
#include "blockmask/mask.hpp"
#include "blockmask/matrix.hpp"

namespace blockmask {

enum class Variant {
    dense,         // every tile, mask ignored
    naive_masked,  // every tile, mask applied everywhere
    binblk,        // occupied tiles only
    dense_binblk,  // occupied tiles; the first full run of each row skips its mask reads
};

inline const char* to_string(Variant v) {
    switch (v) {
        case Variant::dense: return "dense";
        case Variant::naive_masked: return "naive";
        case Variant::binblk: return "binblk";
        case Variant::dense_binblk: return "dense-binblk";
    }
    return "?";
}

inline Variant parse_variant(const std::string& name) {
    if (name == "dense") return Variant::dense;
    if (name == "naive") return Variant::naive_masked;
    if (name == "binblk") return Variant::binblk;
    if (name == "dense-binblk") return Variant::dense_binblk;
    throw std::invalid_argument("unknown variant: '" + name +
                                "' (expected dense, naive, binblk, dense-binblk)");
}

struct EngineCounters {
    std::uint64_t blocks_visited = 0;
    std::uint64_t blocks_processed = 0;
    std::uint64_t mask_block_reads = 0;
    std::uint64_t skipped_by_binblk = 0;
    std::uint64_t skipped_mask_reads_by_run = 0;

    EngineCounters& operator+=(const EngineCounters& o) {
        blocks_visited += o.blocks_visited;
        blocks_processed += o.blocks_processed;
        mask_block_reads += o.mask_block_reads;
        skipped_by_binblk += o.skipped_by_binblk;
        skipped_mask_reads_by_run += o.skipped_mask_reads_by_run;
        return *this;
    }
    friend bool operator==(const EngineCounters&, const EngineCounters&) = default;
};

/// The reference's MaskPrep fields plus `device`: the GPU-resident metadata (tile lists,
/// partial-tile bitmaps) shared by every call that uses this prep.
struct MaskPrep {
    std::size_t n_tokens = 0;
    BlockSpec spec;
    BlockSums sums;
    BlockOccupancy occupancy;
    DenseRuns runs;
    BlockStats stats;
    device::PrepPtr device;
};

namespace detail {
/// MaskPrep around a device handle: the host fields are read back from libbbm.
inline MaskPrep prep_from_handle(bbm_prep h, BlockSpec spec) {
    MaskPrep prep;
    prep.device = std::make_shared<device::PrepHandle>(h);
    bbm_prep_info info{};
    device::check(bbm_prep_get_info(h, &info), "preprocess_mask");
    prep.n_tokens = info.n;
    prep.spec = spec;
    prep.sums = BlockSums(info.n, spec);
    device::check(bbm_prep_get_sums(h, prep.sums.data()), "preprocess_mask");
    prep.occupancy = BlockOccupancy(prep.sums.rows(), prep.sums.cols());
    device::check(bbm_prep_get_occupancy(h, prep.occupancy.data()), "preprocess_mask");
    prep.runs.offset.assign(prep.sums.rows(), 0);
    prep.runs.total_ones.assign(prep.sums.rows(), 0);
    device::check(bbm_prep_get_runs(h, prep.runs.offset.data(), prep.runs.total_ones.data()),
                  "preprocess_mask");
    bbm_block_stats st{};
    device::check(bbm_prep_get_stats(h, &st), "preprocess_mask");
    prep.stats = BlockStats{st.blocks_total, st.blocks_nonzero, st.blocks_full, st.block_density,
                            st.element_density};
    return prep;
}
}  // namespace detail

inline MaskPrep preprocess_mask(const Mask& mask, BlockSpec spec) {
    spec.validate();
    require(mask.size() >= 1, "mask must be non-empty");
    bbm_prep h = nullptr;
    device::check(bbm_preprocess_packed_host(mask.words(), mask.size(), spec.block_i, spec.block_j,
                                             device::default_device(), &h),
                  "preprocess_mask");
    return detail::prep_from_handle(h, spec);
}

template <typename T>
struct ForwardResult {
    Matrix<T> out;
    std::vector<double> row_max;  // natural-log units, -inf for fully masked rows
    std::vector<double> row_sum;  // 0 for fully masked rows
    EngineCounters counters;
};

template <typename T>
struct BackwardResult {
    Matrix<T> dq;
    Matrix<T> dk;
    Matrix<T> dv;
    EngineCounters counters;
};

template <typename T>
struct SlotInputs {
    Matrix<T> q, k, v;
};

template <typename T>
struct MultiHeadForward {
    std::vector<ForwardResult<T>> slots;
    EngineCounters counters;
};

namespace detail {

inline EngineCounters counters_for(const MaskPrep& prep, Variant v, std::uint64_t slots) {
    bbm_counters c{};
    device::check(bbm_prep_counters(prep.device->get(), static_cast<int>(v), slots, &c), "counters");
    return EngineCounters{c.blocks_visited, c.blocks_processed, c.mask_block_reads,
                          c.skipped_by_binblk, c.skipped_mask_reads_by_run};
}

// validate_forward_args (engine.hpp:244-258) minus the finiteness scan, which the device does
// while converting the inputs (bbm_attn_fwd_host_f32 -> BBM_ERR_INVALID).
template <typename T>
void validate_shapes(const Matrix<T>& q, const Matrix<T>& k, const Matrix<T>& v, double scale,
                     const Mask& mask, const MaskPrep& prep, unsigned threads) {
    const std::size_t n = mask.size();
    require(prep.n_tokens == n, "mask preprocessing does not match this mask");
    require(prep.device != nullptr, "MaskPrep was not built by preprocess_mask");
    require(q.rows() == n && k.rows() == n && v.rows() == n, "q, k, v need one row per token");
    require(q.cols() == k.cols() && q.cols() >= 1, "q and k must share a positive head dim");
    require(v.cols() >= 1, "v needs at least one column");
    require(std::isfinite(scale), "scale must be finite");
    require(threads >= 1, "threads must be >= 1");
}

// Matrix<T> (float or double) -> packed float [slots][n][d] (the C ABI's host format).
template <typename T>
void append_f32(std::vector<float>& dst, const Matrix<T>& m) {
    const std::size_t at = dst.size();
    dst.resize(at + m.size());
    for (std::size_t i = 0; i < m.size(); ++i) dst[at + i] = static_cast<float>(m.data()[i]);
}

template <typename T>
void forward_slots(const std::vector<const SlotInputs<T>*>& in, double scale, const MaskPrep& prep,
                   Variant variant, std::vector<ForwardResult<T>>& out) {
    static_assert(std::is_floating_point_v<T>, "Matrix<T> of float or double");
    const std::size_t slots = in.size(), n = prep.n_tokens;
    const std::size_t dk = in.front()->q.cols(), dv = in.front()->v.cols();
    const EngineCounters per_slot = counters_for(prep, variant, 1);
    out.resize(slots);
    for (ForwardResult<T>& r : out) {
        r.out = Matrix<T>(n, dv);
        r.row_max.assign(n, 0.0);
        r.row_sum.assign(n, 0.0);
        r.counters = per_slot;
    }
    std::vector<const float*> q(slots), k(slots), v(slots);
    std::vector<float*> o(slots);
    std::vector<double*> m(slots), l(slots);
    std::vector<float> fq, fk, fv, fo;  // Matrix<double>: narrowed to float for the upload
    if constexpr (!std::is_same_v<T, float>) {
        fq.reserve(slots * n * dk), fk.reserve(slots * n * dk), fv.reserve(slots * n * dv);
        for (const SlotInputs<T>* s : in) append_f32(fq, s->q), append_f32(fk, s->k), append_f32(fv, s->v);
        fo.resize(slots * n * dv);
    }
    for (std::size_t s = 0; s < slots; ++s) {
        if constexpr (std::is_same_v<T, float>) {
            // run_attention<float> (engine.hpp:489-505): every slot's own Matrix<float> storage goes
            // to the device as is (chunked H2D / kernel / D2H pipeline), results land in the
            // ForwardResults directly
            q[s] = in[s]->q.data(), k[s] = in[s]->k.data(), v[s] = in[s]->v.data();
            o[s] = out[s].out.data();
        } else {
            q[s] = fq.data() + s * n * dk, k[s] = fk.data() + s * n * dk, v[s] = fv.data() + s * n * dv;
            o[s] = fo.data() + s * n * dv;
        }
        m[s] = out[s].row_max.data(), l[s] = out[s].row_sum.data();
    }
    device::check(bbm_run_attention_host_f32_dims(prep.device->get(), static_cast<int>(variant), q.data(),
                                                  k.data(), v.data(), o.data(), m.data(), l.data(), slots,
                                                  static_cast<std::uint32_t>(dk), static_cast<std::uint32_t>(dv),
                                                  scale),
                  "blocked_forward");
    if constexpr (!std::is_same_v<T, float>)
        for (std::size_t s = 0; s < slots; ++s)
            for (std::size_t i = 0; i < n * dv; ++i) out[s].out.data()[i] = static_cast<T>(fo[s * n * dv + i]);
}

}  // namespace detail

template <typename T>
ForwardResult<T> blocked_forward(const Matrix<T>& q, const Matrix<T>& k, const Matrix<T>& v,
                                 double scale, const Mask& mask, const MaskPrep& prep,
                                 Variant variant, unsigned threads = 1) {
    detail::validate_shapes(q, k, v, scale, mask, prep, threads);
    SlotInputs<T> one{q, k, v};
    std::vector<ForwardResult<T>> out;
    detail::forward_slots<T>({&one}, scale, prep, variant, out);
    return std::move(out.front());
}

template <typename T>
BackwardResult<T> blocked_backward(const Matrix<T>& q, const Matrix<T>& k, const Matrix<T>& v,
                                   double scale, const Mask& mask, const MaskPrep& prep,
                                   Variant variant, const ForwardResult<T>& fwd,
                                   const Matrix<T>& d_out, unsigned threads = 1) {
    detail::validate_shapes(q, k, v, scale, mask, prep, threads);
    const std::size_t n = mask.size(), dk = q.cols(), dv = v.cols();
    require(fwd.out.rows() == n && fwd.out.cols() == dv, "forward output shape mismatch");
    require(fwd.row_max.size() == n && fwd.row_sum.size() == n, "forward row stats missing");
    require(d_out.rows() == n && d_out.cols() == dv, "d_out shape must match the output");
    BackwardResult<T> r;
    r.dq = Matrix<T>(n, dk), r.dk = Matrix<T>(n, dk), r.dv = Matrix<T>(n, dv);
    const auto run = [&](const float* hq, const float* hk, const float* hv, const float* ho, const float* hdo,
                         float* gq, float* gk, float* gv) {
        device::check(bbm_attn_bwd_host_f32_dims(prep.device->get(), static_cast<int>(variant), hq, hk, hv, ho,
                                                 fwd.row_max.data(), fwd.row_sum.data(), hdo, gq, gk, gv, 1,
                                                 static_cast<std::uint32_t>(dk), static_cast<std::uint32_t>(dv),
                                                 scale),
                      "blocked_backward");
    };
    if constexpr (std::is_same_v<T, float>) {
        // Matrix<float>: the caller's storage in, the BackwardResult's storage out, no copies
        run(q.data(), k.data(), v.data(), fwd.out.data(), d_out.data(), r.dq.data(), r.dk.data(), r.dv.data());
    } else {  // Matrix<double>: narrowed to float for the upload
        std::vector<float> hq, hk, hv, ho, hdo;
        detail::append_f32(hq, q), detail::append_f32(hk, k), detail::append_f32(hv, v);
        detail::append_f32(ho, fwd.out), detail::append_f32(hdo, d_out);
        std::vector<float> gq(n * dk), gk(n * dk), gv(n * dv);
        run(hq.data(), hk.data(), hv.data(), ho.data(), hdo.data(), gq.data(), gk.data(), gv.data());
        for (std::size_t i = 0; i < n * dk; ++i) {
            r.dq.data()[i] = static_cast<T>(gq[i]);
            r.dk.data()[i] = static_cast<T>(gk[i]);
        }
        for (std::size_t i = 0; i < n * dv; ++i) r.dv.data()[i] = static_cast<T>(gv[i]);
    }
    r.counters = detail::counters_for(prep, variant, 1);
    return r;
}

template <typename T>
MultiHeadForward<T> run_attention(std::span<const SlotInputs<T>> slots, double scale,
                                  const Mask& mask, const MaskPrep& prep, Variant variant,
                                  unsigned threads = 1) {
    require(!slots.empty(), "need at least one batch/head slot");
    std::vector<const SlotInputs<T>*> in;
    for (const SlotInputs<T>& s : slots) {
        require(s.q.cols() == slots.front().q.cols() && s.v.cols() == slots.front().v.cols(),
                "all slots must share head dimensions");
        detail::validate_shapes(s.q, s.k, s.v, scale, mask, prep, threads);
        in.push_back(&s);
    }
    MultiHeadForward<T> res;
    detail::forward_slots<T>(in, scale, prep, variant, res.slots);  // one launch, all slots
    for (const ForwardResult<T>& r : res.slots) res.counters += r.counters;
    return res;
}

}  // namespace blockmask
