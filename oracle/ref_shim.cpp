// ref_shim.cpp — C entry points over the UNMODIFIED reference headers (TEST INFRASTRUCTURE).
//
// Compiled by oracle/Makefile against /root/reference/proj/include (read in place, never copied)
// into oracle/_ref/libbbm_ref.so. It lets the tests pin the oracle restatement against the real
// reference, generate golden vectors, and lets bench.py time the reference's own CPU engine
// (blocked_forward<float>, engine.hpp:282-341) as the cpu_baseline / --impl reference arm.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "blockmask/engine.hpp"
#include "blockmask/generators.hpp"
#include "blockmask/reference.hpp"
#include "blockmask/reorder.hpp"
#include "blockmask/rng.hpp"

using namespace blockmask;

namespace {
thread_local std::string g_err;

Mask mask_from_words(const uint64_t* words, uint64_t n) {
  Mask m(n);
  const uint64_t wpr = (n + 63) / 64;
  for (uint64_t i = 0; i < n; ++i)
    for (uint64_t w = 0; w < wpr; ++w) {
      uint64_t bits = words[i * wpr + w];
      while (bits) {
        const uint64_t j = w * 64 + static_cast<uint64_t>(__builtin_ctzll(bits));
        bits &= bits - 1;
        m.set(i, j, true);
      }
    }
  return m;
}

void words_from_mask(const Mask& m, uint64_t* out) {
  for (std::size_t i = 0; i < m.size(); ++i) {
    const auto row = m.row_words(i);
    std::memcpy(out + i * m.words_per_row(), row.data(), row.size() * 8);
  }
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// MaskSpec::parse + generate (generators.hpp:233-438). Call with words == nullptr to get n.
int ref_generate(const char* spec, uint64_t n_free, uint64_t* n_out, uint64_t* words) {
  return guarded([&] {
    MaskSpec s = MaskSpec::parse(spec);
    if (s.has_free_n()) s = s.with_n(n_free);
    const Mask m = generate(s);
    *n_out = m.size();
    if (words) words_from_mask(m, words);
  });
}

int ref_gen_random_sparse(uint64_t n, double density, uint64_t seed, int diag, uint64_t* words) {
  return guarded([&] { words_from_mask(gen_random_sparse(n, density, seed, diag != 0), words); });
}

int ref_preprocess(const uint64_t* words, uint64_t n, uint64_t bi, uint64_t bj, uint32_t* sums,
                   uint8_t* occ, uint32_t* offset, uint32_t* total_ones, uint64_t* stats_u64,
                   double* stats_f64) {
  return guarded([&] {
    const Mask m = mask_from_words(words, n);
    const MaskPrep prep = preprocess_mask(m, BlockSpec{bi, bj});
    for (std::size_t p = 0; p < prep.sums.rows(); ++p)
      for (std::size_t q = 0; q < prep.sums.cols(); ++q) {
        sums[p * prep.sums.cols() + q] = prep.sums.sum(p, q);
        occ[p * prep.sums.cols() + q] = prep.occupancy.at(p, q) ? 1 : 0;
      }
    for (std::size_t p = 0; p < prep.sums.rows(); ++p) {
      offset[p] = prep.runs.offset[p];
      total_ones[p] = prep.runs.total_ones[p];
    }
    stats_u64[0] = prep.stats.blocks_total;
    stats_u64[1] = prep.stats.blocks_nonzero;
    stats_u64[2] = prep.stats.blocks_full;
    stats_f64[0] = prep.stats.block_density;
    stats_f64[1] = prep.stats.element_density;
  });
}

// blocked_forward<float> or <double> over `slots` slots laid out [slot][n][d], sequential as in
// run_attention (engine.hpp:489-505). counters: 5 x u64 summed over slots.
int ref_blocked_forward(int is_double, const void* q, const void* k, const void* v, uint64_t slots,
                        uint64_t n, uint64_t d, double scale, const uint64_t* words, uint64_t bi,
                        uint64_t bj, int variant, unsigned threads, void* out, double* row_max,
                        double* row_sum, uint64_t* counters) {
  return guarded([&] {
    const Mask m = mask_from_words(words, n);
    const MaskPrep prep = preprocess_mask(m, BlockSpec{bi, bj});
    EngineCounters total;
    auto run = [&](auto tag) {
      using T = decltype(tag);
      for (uint64_t s = 0; s < slots; ++s) {
        Matrix<T> mq(n, d), mk(n, d), mv(n, d);
        std::memcpy(mq.data(), static_cast<const T*>(q) + s * n * d, n * d * sizeof(T));
        std::memcpy(mk.data(), static_cast<const T*>(k) + s * n * d, n * d * sizeof(T));
        std::memcpy(mv.data(), static_cast<const T*>(v) + s * n * d, n * d * sizeof(T));
        const ForwardResult<T> r =
            blocked_forward(mq, mk, mv, scale, m, prep, static_cast<Variant>(variant), threads);
        if (out) std::memcpy(static_cast<T*>(out) + s * n * d, r.out.data(), n * d * sizeof(T));
        if (row_max) std::memcpy(row_max + s * n, r.row_max.data(), n * 8);
        if (row_sum) std::memcpy(row_sum + s * n, r.row_sum.data(), n * 8);
        total += r.counters;
      }
    };
    if (is_double) run(double{}); else run(float{});
    if (counters) {
      counters[0] = total.blocks_visited;
      counters[1] = total.blocks_processed;
      counters[2] = total.mask_block_reads;
      counters[3] = total.skipped_by_binblk;
      counters[4] = total.skipped_mask_reads_by_run;
    }
  });
}

// Timing entry for the CPU baseline: inputs pre-built, preprocessing reused across calls.
struct RefEngine {
  Mask mask;
  MaskPrep prep;
  std::vector<Matrix<float>> q, k, v;
};

void* ref_engine_create(const uint64_t* words, uint64_t n, uint64_t bi, uint64_t bj,
                        const float* q, const float* k, const float* v, uint64_t slots,
                        uint64_t d) {
  auto* e = new RefEngine;
  e->mask = mask_from_words(words, n);
  e->prep = preprocess_mask(e->mask, BlockSpec{bi, bj});
  for (uint64_t s = 0; s < slots; ++s) {
    Matrix<float> mq(n, d), mk(n, d), mv(n, d);
    std::memcpy(mq.data(), q + s * n * d, n * d * 4);
    std::memcpy(mk.data(), k + s * n * d, n * d * 4);
    std::memcpy(mv.data(), v + s * n * d, n * d * 4);
    e->q.push_back(std::move(mq));
    e->k.push_back(std::move(mk));
    e->v.push_back(std::move(mv));
  }
  return e;
}

// Forward over all held slots; returns a checksum of the outputs so work cannot be elided.
double ref_engine_forward(void* h, int variant, unsigned threads, double scale) {
  auto* e = static_cast<RefEngine*>(h);
  double sum = 0.0;
  for (std::size_t s = 0; s < e->q.size(); ++s) {
    const ForwardResult<float> r = blocked_forward(e->q[s], e->k[s], e->v[s], scale, e->mask,
                                                   e->prep, static_cast<Variant>(variant), threads);
    sum += r.out(0, 0) + r.row_sum[r.row_sum.size() - 1];
  }
  return sum;
}

double ref_engine_preprocess_ms(void* h, int reps) {
  auto* e = static_cast<RefEngine*>(h);
  auto t0 = std::chrono::steady_clock::now();
  for (int r = 0; r < reps; ++r) {
    const MaskPrep p = preprocess_mask(e->mask, e->prep.spec);
    (void)p;
  }
  auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double, std::milli>(t1 - t0).count() / reps;
}

void ref_engine_destroy(void* h) { delete static_cast<RefEngine*>(h); }

int ref_naive_forward(const double* q, const double* k, const double* v, uint64_t n, uint64_t d,
                      uint64_t dv, double scale, const uint64_t* words, double* out,
                      double* row_max, double* row_sum) {
  return guarded([&] {
    const Mask m = mask_from_words(words, n);
    Matrix<double> mq(n, d), mk(n, d), mv(n, dv);
    std::memcpy(mq.data(), q, n * d * 8);
    std::memcpy(mk.data(), k, n * d * 8);
    std::memcpy(mv.data(), v, n * dv * 8);
    const NaiveOutput r = naive_forward(mq, mk, mv, scale, m);
    std::memcpy(out, r.out.data(), n * dv * 8);
    std::memcpy(row_max, r.row_max.data(), n * 8);
    std::memcpy(row_sum, r.row_sum.data(), n * 8);
  });
}

int ref_naive_backward(const double* q, const double* k, const double* v, uint64_t n, uint64_t d,
                       double scale, const uint64_t* words, const double* d_out, double* dq,
                       double* dk, double* dv) {
  return guarded([&] {
    const Mask m = mask_from_words(words, n);
    Matrix<double> mq(n, d), mk(n, d), mv(n, d), mdo(n, d);
    std::memcpy(mq.data(), q, n * d * 8);
    std::memcpy(mk.data(), k, n * d * 8);
    std::memcpy(mv.data(), v, n * d * 8);
    std::memcpy(mdo.data(), d_out, n * d * 8);
    const NaiveGrads g = naive_backward(mq, mk, mv, scale, m, mdo);
    std::memcpy(dq, g.dq.data(), n * d * 8);
    std::memcpy(dk, g.dk.data(), n * d * 8);
    std::memcpy(dv, g.dv.data(), n * d * 8);
  });
}

int ref_rcm(const uint64_t* words, uint64_t n, uint32_t* forward, uint64_t* bw_before,
            uint64_t* bw_after) {
  return guarded([&] {
    const Mask m = mask_from_words(words, n);
    const Permutation p = rcm_order(build_graph(m));
    std::memcpy(forward, p.forward.data(), n * 4);
    if (bw_before) *bw_before = bandwidth(m);
    if (bw_after) *bw_after = bandwidth(permute_mask(m, p));
  });
}

int ref_permute_mask(const uint64_t* words, uint64_t n, const uint32_t* forward, uint64_t* out) {
  return guarded([&] {
    const Mask m = mask_from_words(words, n);
    const Permutation p = Permutation::from_forward(std::vector<uint32_t>(forward, forward + n));
    words_from_mask(permute_mask(m, p), out);
  });
}

// The bench's config-5 relabelling, expressed with the reference's own permute_mask
// (reorder.hpp:156-163): labels = std::shuffle(iota, mt19937_64(seed)), out(label[i], label[j]) =
// mask(i, j), i.e. permute_mask with forward = labels^-1.
int ref_relabel(const uint64_t* words, uint64_t n, uint64_t seed, uint64_t* out) {
  return guarded([&] {
    std::vector<uint32_t> labels(n);
    for (uint64_t i = 0; i < n; ++i) labels[i] = static_cast<uint32_t>(i);
    std::mt19937_64 gen(seed);
    std::shuffle(labels.begin(), labels.end(), gen);
    std::vector<uint32_t> fwd(n);
    for (uint64_t i = 0; i < n; ++i) fwd[labels[i]] = static_cast<uint32_t>(i);
    const Mask m = mask_from_words(words, n);
    words_from_mask(permute_mask(m, Permutation::from_forward(fwd)), out);
  });
}

// make_problem (bench.hpp:320-337) as float, the engine's single-precision inputs.
void ref_make_problem_f32(uint64_t seed, uint64_t slots, uint64_t n, uint64_t d, float* q,
                          float* k, float* v, float* d_out) {
  std::mt19937_64 gen(seed);
  for (uint64_t s = 0; s < slots; ++s) {
    const Matrix<float> a = random_matrix<float>(n, d, gen);
    const Matrix<float> b = random_matrix<float>(n, d, gen);
    const Matrix<float> c = random_matrix<float>(n, d, gen);
    const Matrix<float> o = random_matrix<float>(n, d, gen);
    if (q) std::memcpy(q + s * n * d, a.data(), n * d * 4);
    if (k) std::memcpy(k + s * n * d, b.data(), n * d * 4);
    if (v) std::memcpy(v + s * n * d, c.data(), n * d * 4);
    if (d_out) std::memcpy(d_out + s * n * d, o.data(), n * d * 4);
  }
}

}  // extern "C"
