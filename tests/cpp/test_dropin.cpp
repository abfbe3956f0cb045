// test_dropin.cpp — the reference's own test cases, written against the C++ drop-in headers
// (include/blockmask/*.hpp), which call libbbm's C ABI and run on the B200.
//
// Mirrors proj/tests/test_mask_model.cpp, test_engine.cpp and test_reorder.cpp case by case
// (file:line beside each). Differences, by design of the sm_100a engine: d_k is at most 128
// (dims are zero-padded on the device to 64 / 128, d_v above 128 runs as column passes over V),
// and outputs are compared with a double-precision
// naive attention at the bf16 tolerance (2e-2) instead of 1e-12.
//
//   g++ -std=c++20 -O1 -Iinclude tests/cpp/test_dropin.cpp -Lpaper_2409_15097_b200 -lbbm
//       -Wl,-rpath,$PWD/paper_2409_15097_b200 -o build/test_dropin && build/test_dropin
// (tests/test_dropin_cpp.py builds and runs it)
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <functional>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "blockmask/engine.hpp"
#include "blockmask/generators.hpp"
#include "blockmask/mask.hpp"
#include "blockmask/mask_io.hpp"
#include "blockmask/reorder.hpp"

using namespace blockmask;

namespace {
int g_failures = 0, g_checks = 0;
#define EXPECT(cond)                                                              \
  do {                                                                            \
    ++g_checks;                                                                   \
    if (!(cond)) {                                                                \
      ++g_failures;                                                               \
      std::fprintf(stderr, "  FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond);    \
    }                                                                             \
  } while (0)
#define EXPECT_THROW_INVALID(stmt)                                                \
  do {                                                                            \
    ++g_checks;                                                                   \
    bool thrown = false;                                                          \
    try {                                                                         \
      stmt;                                                                       \
    } catch (const std::invalid_argument&) {                                      \
      thrown = true;                                                              \
    }                                                                             \
    if (!thrown) {                                                                \
      ++g_failures;                                                               \
      std::fprintf(stderr, "  FAILED %s:%d: no invalid_argument from %s\n", __FILE__, __LINE__, #stmt); \
    }                                                                             \
  } while (0)

struct Problem {
  Matrix<float> q, k, v, g;
  double scale;
};

// bf16-exact inputs (multiples of 1/64 in [-1, 1)), so the device's bf16 rounding is lossless and
// the double naive oracle sees exactly what the kernel sees
Problem make_problem(std::size_t n, std::size_t d, uint64_t seed, std::size_t dv = 0) {
  if (dv == 0) dv = d;
  uint64_t s = seed * 0x9E3779B97F4A7C15ull + 1;
  auto next = [&] {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    return static_cast<float>(static_cast<int>((s >> 33) % 128) - 64) / 64.0f;
  };
  Problem p{Matrix<float>(n, d), Matrix<float>(n, d), Matrix<float>(n, dv), Matrix<float>(n, dv),
            1.0 / std::sqrt(static_cast<double>(d))};
  for (Matrix<float>* m : {&p.q, &p.k, &p.v, &p.g})
    for (std::size_t i = 0; i < m->size(); ++i) m->data()[i] = next();
  return p;
}

// double-precision naive attention (the reference's reference.hpp:42-139, restated for the test)
struct Naive {
  Matrix<double> out, dq, dk, dv;
  std::vector<double> m, l;
};
Naive naive(const Problem& p, const Mask& mask, bool dense) {
  const std::size_t n = mask.size(), d = p.q.cols(), dv = p.v.cols();
  Naive r{Matrix<double>(n, dv), Matrix<double>(n, d), Matrix<double>(n, d), Matrix<double>(n, dv),
          std::vector<double>(n), std::vector<double>(n)};
  std::vector<double> s(n), pr(n), dp(n);
  for (std::size_t i = 0; i < n; ++i) {
    double m = -std::numeric_limits<double>::infinity();
    for (std::size_t j = 0; j < n; ++j) {
      if (!dense && !mask.get(i, j)) continue;
      double t = 0;
      for (std::size_t c = 0; c < d; ++c) t += double(p.q(i, c)) * p.k(j, c);
      s[j] = p.scale * t;
      m = std::max(m, s[j]);
    }
    r.m[i] = m;
    if (std::isinf(m)) continue;
    double l = 0;
    for (std::size_t j = 0; j < n; ++j)
      if (dense || mask.get(i, j)) l += (pr[j] = std::exp(s[j] - m));
    r.l[i] = l;
    double delta = 0;
    for (std::size_t j = 0; j < n; ++j) {
      if (!dense && !mask.get(i, j)) continue;
      pr[j] /= l;
      double t = 0;
      for (std::size_t c = 0; c < dv; ++c) {
        r.out(i, c) += pr[j] * p.v(j, c);
        t += double(p.g(i, c)) * p.v(j, c);
      }
      dp[j] = t;
      delta += pr[j] * t;
    }
    for (std::size_t j = 0; j < n; ++j) {
      if (!dense && !mask.get(i, j)) continue;
      const double ds = pr[j] * (dp[j] - delta);
      for (std::size_t c = 0; c < d; ++c) {
        r.dq(i, c) += p.scale * ds * p.k(j, c);
        r.dk(j, c) += p.scale * ds * p.q(i, c);
      }
      for (std::size_t c = 0; c < dv; ++c) r.dv(j, c) += pr[j] * p.g(i, c);
    }
  }
  return r;
}

double rel(const Matrix<float>& got, const Matrix<double>& want) {
  double worst = 0, scale = 1;
  for (std::size_t i = 0; i < want.size(); ++i) scale = std::max(scale, std::abs(want.data()[i]));
  for (std::size_t i = 0; i < want.size(); ++i) worst = std::max(worst, std::abs(got.data()[i] - want.data()[i]));
  return worst / scale;
}

void run(const char* name, const std::function<void()>& f) {
  const int before = g_failures;
  try {
    f();
  } catch (const std::exception& e) {
    ++g_failures;
    std::fprintf(stderr, "  FAILED %s: exception %s\n", name, e.what());
  }
  std::printf("[%s] %s\n", g_failures == before ? "PASS" : "FAIL", name);
}
}  // namespace

int main() {
  // ---------------------------------------------------------------- mask model
  run("BlockModel.CausalFourByFourKnownAnswer (test_mask_model.cpp:81-107)", [] {
    const Mask mask = gen_causal(4);
    const BlockSums s = block_sums(mask, BlockSpec{2, 2});
    EXPECT(s.rows() == 2 && s.cols() == 2);
    EXPECT(s.sum(0, 0) == 3 && s.sum(0, 1) == 0 && s.sum(1, 0) == 4 && s.sum(1, 1) == 3);
    const BlockOccupancy occ = build_block_occupancy(s);
    EXPECT(occ.at(0, 0) && !occ.at(0, 1) && occ.at(1, 0) && occ.at(1, 1));
    const DenseRuns runs = build_dense_runs(s);
    EXPECT(runs.offset[0] == 0 && runs.total_ones[0] == 0 && runs.offset[1] == 0 && runs.total_ones[1] == 1);
    const BlockStats st = block_stats(s);
    EXPECT(st.blocks_total == 4 && st.blocks_nonzero == 3 && st.blocks_full == 1);
    EXPECT(st.block_density == 0.75 && st.element_density == 10.0 / 16.0);
  });
  run("BlockModel.RaggedEdgesUseTrueArea (test_mask_model.cpp:109-125)", [] {
    const BlockSums s = block_sums(gen_all_ones(5), BlockSpec{2, 2});
    const uint32_t want[3][3] = {{4, 4, 2}, {4, 4, 2}, {2, 2, 1}};
    for (int p = 0; p < 3; ++p)
      for (int q = 0; q < 3; ++q) EXPECT(s.sum(p, q) == want[p][q] && s.full(p, q));
    const DenseRuns runs = build_dense_runs(s);
    for (int p = 0; p < 3; ++p) EXPECT(runs.offset[p] == 0 && runs.total_ones[p] == 3);
  });
  run("BlockModel.FirstMaximalRunWinsOverLaterRuns (test_mask_model.cpp:145-159)", [] {
    Mask mask(16);
    for (std::size_t i = 0; i < 2; ++i) {
      for (std::size_t j = 2; j < 6; ++j) mask.set(i, j, true);
      for (std::size_t j = 8; j < 10; ++j) mask.set(i, j, true);
    }
    const DenseRuns runs = build_dense_runs(block_sums(mask, BlockSpec{2, 2}));
    EXPECT(runs.offset[0] == 1 && runs.total_ones[0] == 2);
    EXPECT(runs.in_run(0, 1) && runs.in_run(0, 2) && !runs.in_run(0, 0) && !runs.in_run(0, 3));
  });
  run("BlockModel.SumsMatchBruteForce (test_mask_model.cpp:127-143)", [] {
    const Mask mask = gen_random_sparse(97, 0.3, 11, false);
    for (BlockSpec spec : {BlockSpec{2, 2}, BlockSpec{3, 5}, BlockSpec{16, 16}, BlockSpec{32, 16}, BlockSpec{64, 64}}) {
      const BlockSums s = block_sums(mask, spec);
      for (std::size_t p = 0; p < s.rows(); ++p)
        for (std::size_t q = 0; q < s.cols(); ++q) {
          uint32_t c = 0;
          for (std::size_t i = p * spec.block_i; i < std::min(mask.size(), (p + 1) * spec.block_i); ++i)
            for (std::size_t j = q * spec.block_j; j < std::min(mask.size(), (q + 1) * spec.block_j); ++j)
              c += mask.get(i, j);
          EXPECT(s.sum(p, q) == c);
        }
    }
  });
  run("BlockModel.SpeculativeTreeMaskKeepsFirstColumnBlocksOccupied (test_mask_model.cpp:181-189)", [] {
    const std::vector<std::size_t> c{4, 4, 4, 4};
    const Mask mask = gen_medusa(c);
    EXPECT(mask.size() == 340);
    const BlockOccupancy occ = build_block_occupancy(block_sums(mask, BlockSpec{128, 32}));
    EXPECT(occ.rows() == 3 && occ.cols() == 11);
    for (std::size_t p = 0; p < occ.rows(); ++p) EXPECT(occ.at(p, 0));
  });
  run("BlockModel.InvalidSpecsRejected (test_mask_model.cpp:191-195)", [] {
    EXPECT_THROW_INVALID(BlockSpec({0, 4}).validate());
    EXPECT_THROW_INVALID(block_sums(gen_causal(4), BlockSpec{0, 2}));
  });

  run("MaskIo.RoundTripErrorsAndDevicePath (test_mask_model.cpp:224-323)", [] {
    const std::filesystem::path dir = std::filesystem::temp_directory_path();
    const Mask mask = gen_random_sparse(77, 0.2, 3, false);
    const auto path = dir / "bbm_dropin.bbmk";
    write_mask(mask, path);
    EXPECT(std::filesystem::file_size(path) == 13 + 77 * 10);
    EXPECT(read_mask(path) == mask);
    bool kinded = false;
    try {
      read_mask(dir / "bbm_dropin_missing.bbmk");
    } catch (const MaskIoError& e) {
      kinded = e.kind() == MaskIoError::Kind::io_failure;
    }
    EXPECT(kinded);
    const MaskPrep a = preprocess_mask_file(path, BlockSpec{16, 8});
    const MaskPrep b = preprocess_mask(mask, BlockSpec{16, 8});
    EXPECT(a.occupancy == b.occupancy && a.runs == b.runs && a.stats.blocks_nonzero == b.stats.blocks_nonzero);
    const auto occ_path = dir / "bbm_dropin.bblk";
    write_occupancy(b.occupancy, 77, BlockSpec{16, 8}, occ_path);
    const OccupancyFile f = read_occupancy(occ_path);
    EXPECT(f.n_tokens == 77 && f.spec == (BlockSpec{16, 8}) && f.occupancy == b.occupancy);
  });

  // ---------------------------------------------------------------- engine
  run("EngineCounters.CausalFourTokensTwoByTwo (test_engine.cpp:23-50)", [] {
    const Mask mask = gen_causal(4);
    const MaskPrep prep = preprocess_mask(mask, BlockSpec{2, 2});
    const Problem p = make_problem(4, 64, 1);
    const auto dense = blocked_forward(p.q, p.k, p.v, p.scale, mask, prep, Variant::dense);
    EXPECT(dense.counters.blocks_visited == 4 && dense.counters.blocks_processed == 4 &&
           dense.counters.mask_block_reads == 0);
    const auto naive_r = blocked_forward(p.q, p.k, p.v, p.scale, mask, prep, Variant::naive_masked);
    EXPECT(naive_r.counters.mask_block_reads == 4);
    const auto bb = blocked_forward(p.q, p.k, p.v, p.scale, mask, prep, Variant::binblk);
    EXPECT(bb.counters.blocks_processed == 3 && bb.counters.skipped_by_binblk == 1 &&
           bb.counters.mask_block_reads == 3);
    const auto dbb = blocked_forward(p.q, p.k, p.v, p.scale, mask, prep, Variant::dense_binblk);
    EXPECT(dbb.counters.mask_block_reads == 2 && dbb.counters.skipped_mask_reads_by_run == 1);
  });
  run("EngineCounters.FullMaskRunsSkipEveryMaskRead (test_engine.cpp:52-61)", [] {
    const Mask mask = gen_all_ones(256);
    const MaskPrep prep = preprocess_mask(mask, BlockSpec{64, 64});
    const Problem p = make_problem(256, 64, 2);
    const auto dbb = blocked_forward(p.q, p.k, p.v, p.scale, mask, prep, Variant::dense_binblk);
    EXPECT(dbb.counters.blocks_visited == 16 && dbb.counters.mask_block_reads == 0 &&
           dbb.counters.skipped_mask_reads_by_run == 16);
  });
  run("Engine.MatchesNaiveOracleAllVariants (test_engine.cpp:150-174)", [] {
    for (std::size_t d : {64u, 128u}) {
      const Mask mask = gen_random_sparse(200, 0.1, 5, true);
      const MaskPrep prep = preprocess_mask(mask, BlockSpec{64, 64});
      const Problem p = make_problem(200, d, 3);
      for (Variant v : {Variant::dense, Variant::naive_masked, Variant::binblk, Variant::dense_binblk}) {
        const Naive want = naive(p, mask, v == Variant::dense);
        const auto f = blocked_forward(p.q, p.k, p.v, p.scale, mask, prep, v);
        EXPECT(rel(f.out, want.out) <= 2e-2);
        const auto b = blocked_backward(p.q, p.k, p.v, p.scale, mask, prep, v, f, p.g);
        EXPECT(rel(b.dq, want.dq) <= 2e-2 && rel(b.dk, want.dk) <= 2e-2 && rel(b.dv, want.dv) <= 2e-2);
        EXPECT(b.counters == f.counters);
        for (std::size_t i = 0; i < 200; ++i)
          EXPECT(std::abs(f.row_max[i] - want.m[i]) <= 1e-2 * std::max(1.0, std::abs(want.m[i])));
      }
    }
  });
  run("Engine.FullyMaskedRowsProduceZeroRows (test_engine.cpp:176-197)", [] {
    Mask mask(150);
    for (std::size_t i = 0; i < 150; ++i)
      if (i % 3 != 0)
        for (std::size_t j = 0; j <= i; ++j) mask.set(i, j, true);
    const MaskPrep prep = preprocess_mask(mask, BlockSpec{32, 32});
    const Problem p = make_problem(150, 64, 4);
    const auto f = blocked_forward(p.q, p.k, p.v, p.scale, mask, prep, Variant::binblk);
    for (std::size_t i = 0; i < 150; i += 3) {
      EXPECT(f.row_max[i] == -std::numeric_limits<double>::infinity() && f.row_sum[i] == 0.0);
      for (std::size_t c = 0; c < 64; ++c) EXPECT(f.out(i, c) == 0.0f);
    }
  });
  run("EngineForward.ValueHeadDimMayDifferFromKeyDim (test_engine.cpp:198-209) + other head dims", [] {
    struct Dims { std::size_t n, dk, dv; };
    for (Dims dm : {Dims{21, 5, 3}, Dims{130, 3, 100}, Dims{200, 96, 96}, Dims{77, 128, 7}, Dims{90, 32, 260}}) {
      const Mask mask = gen_causal(dm.n);
      const MaskPrep prep = preprocess_mask(mask, BlockSpec{8, 8});
      Problem p = make_problem(dm.n, dm.dk, 13 + dm.dk, dm.dv);
      p.scale = 0.4;
      const Naive want = naive(p, mask, false);
      const auto f = blocked_forward(p.q, p.k, p.v, p.scale, mask, prep, Variant::binblk);
      EXPECT(f.out.rows() == dm.n && f.out.cols() == dm.dv);
      EXPECT(rel(f.out, want.out) <= 2e-2);
      const auto b = blocked_backward(p.q, p.k, p.v, p.scale, mask, prep, Variant::binblk, f, p.g);
      EXPECT(b.dq.cols() == dm.dk && b.dk.cols() == dm.dk && b.dv.cols() == dm.dv);
      EXPECT(rel(b.dq, want.dq) <= 2e-2 && rel(b.dk, want.dk) <= 2e-2 && rel(b.dv, want.dv) <= 2e-2);
      // Matrix<double> goes through the same entry
      Matrix<double> qd(dm.n, dm.dk), kd(dm.n, dm.dk), vd(dm.n, dm.dv);
      for (std::size_t i = 0; i < qd.size(); ++i) qd.data()[i] = p.q.data()[i], kd.data()[i] = p.k.data()[i];
      for (std::size_t i = 0; i < vd.size(); ++i) vd.data()[i] = p.v.data()[i];
      const auto fd = blocked_forward(qd, kd, vd, p.scale, mask, prep, Variant::binblk);
      for (std::size_t i = 0; i < vd.size(); ++i) EXPECT(fd.out.data()[i] == static_cast<double>(f.out.data()[i]));
    }
  });
  run("Engine.MultiSlotMatchesPerSlot (test_engine.cpp:323-347)", [] {
    const Mask mask = gen_longformer_global(300, 20, 3);
    const MaskPrep prep = preprocess_mask(mask, BlockSpec{64, 64});
    std::vector<SlotInputs<float>> slots;
    for (uint64_t s = 0; s < 3; ++s) {
      Problem p = make_problem(300, 64, 10 + s);
      slots.push_back({p.q, p.k, p.v});
    }
    const auto all = run_attention<float>(slots, 0.125, mask, prep, Variant::binblk);
    EngineCounters sum;
    for (std::size_t s = 0; s < 3; ++s) {
      const auto one = blocked_forward(slots[s].q, slots[s].k, slots[s].v, 0.125, mask, prep, Variant::binblk);
      EXPECT(one.out == all.slots[s].out);
      sum += one.counters;
    }
    EXPECT(sum == all.counters);
  });
  run("Engine.ValidationErrors (test_engine.cpp:349-385)", [] {
    const Mask mask = gen_causal(128);
    const MaskPrep prep = preprocess_mask(mask, BlockSpec{64, 64});
    Problem p = make_problem(128, 64, 5);
    EXPECT_THROW_INVALID(blocked_forward(p.q, p.k, p.v, std::nan(""), mask, prep, Variant::binblk));
    EXPECT_THROW_INVALID(blocked_forward(p.q, p.k, p.v, 0.1, mask, prep, Variant::binblk, 0));
    EXPECT_THROW_INVALID(blocked_forward(p.q, p.k, p.v, 0.1, gen_causal(64), prep, Variant::binblk));
    Matrix<float> wide(128, 129), empty(128, 0);  // above the kernels' 128-column head-dim tile; zero
    EXPECT_THROW_INVALID(blocked_forward(wide, wide, wide, 0.1, mask, prep, Variant::binblk));
    EXPECT_THROW_INVALID(blocked_forward(empty, empty, p.v, 0.1, mask, prep, Variant::binblk));
    p.k(3, 4) = std::numeric_limits<float>::infinity();
    EXPECT_THROW_INVALID(blocked_forward(p.q, p.k, p.v, 0.1, mask, prep, Variant::binblk));
    EXPECT_THROW_INVALID(parse_variant("sparse"));
    EXPECT(parse_variant("dense-binblk") == Variant::dense_binblk && std::string(to_string(Variant::naive_masked)) == "naive");
  });

  // ---------------------------------------------------------------- reorder
  // ---------------------------------------------------------------- generators (MaskSpec)
  run("Generators.SpecStringsRoundTrip (test_generators.cpp:180-198)", [] {
    const char* cases[] = {"causal", "all-ones", "medusa[4;4;4;4]", "packed-seq[128;256;128]",
                           "packed-bidir[32:16;64:8]", "windowed(w=256)", "windowed(w=16;causal=1)",
                           "dilated(w=8;d=2)", "global(w=8;g=4)", "random(p=0.25;seed=7)",
                           "random(p=0.5;seed=9;diag=0)", "file:/some/path.bbmk"};
    for (const char* text : cases) EXPECT(MaskSpec::parse(text).to_string() == text);
  });
  run("Generators.SpecDispatchMatchesDirectCalls (test_generators.cpp:200-210)", [] {
    EXPECT(generate(MaskSpec::parse("causal").with_n(12)) == gen_causal(12));
    EXPECT(generate(MaskSpec::parse("medusa[3;3;3]")) == gen_medusa(std::vector<std::size_t>{3, 3, 3}));
    EXPECT(generate(MaskSpec::parse("windowed(w=3;causal=1)").with_n(9)) == gen_longformer_windowed(9, 3, true));
    EXPECT(generate(MaskSpec::parse("random(p=0.2;seed=11)").with_n(20)) == gen_random_sparse(20, 0.2, 11));
    EXPECT(!MaskSpec::parse("medusa[2;2]").has_free_n());
    EXPECT(MaskSpec::parse("dilated(w=2;d=2)").has_free_n());
  });
  run("Generators.SpecParseErrors (test_generators.cpp:212-220)", [] {
    EXPECT_THROW_INVALID(MaskSpec::parse("triangular"));
    EXPECT_THROW_INVALID(MaskSpec::parse("medusa[4;x]"));
    EXPECT_THROW_INVALID(MaskSpec::parse("windowed(w=2"));
    EXPECT_THROW_INVALID(MaskSpec::parse("windowed(q=2)"));
    EXPECT_THROW_INVALID(MaskSpec::parse("packed-bidir[4]"));
    EXPECT_THROW_INVALID(MaskSpec::parse("random(p=abc)"));
    EXPECT_THROW_INVALID(generate(MaskSpec::parse("causal")));
  });
  run("Reorder.EdgelessGraphReversesIdentity (test_reorder.cpp:174-186)", [] {
    Mask mask(5);
    for (std::size_t i = 0; i < 5; ++i) mask.set(i, i, true);
    const Permutation perm = rcm_order(build_graph(mask));
    EXPECT((perm.forward == std::vector<uint32_t>{4, 3, 2, 1, 0}));
  });
  run("Reorder.GraphSymmetrizedSortedNoSelfLoops (test_reorder.cpp:43-62)", [] {
    Mask mask(4);
    mask.set(0, 2, true), mask.set(2, 0, true), mask.set(3, 1, true), mask.set(1, 1, true);
    const SparsityGraph g = build_graph(mask);
    EXPECT((g.adjacency[0] == std::vector<uint32_t>{2} && g.adjacency[1] == std::vector<uint32_t>{3}));
    EXPECT((g.adjacency[2] == std::vector<uint32_t>{0} && g.adjacency[3] == std::vector<uint32_t>{1}));
  });
  run("Reorder.ShuffledBandRecoveredAndAttentionEquivariant (test_reorder.cpp:109-117, 202-216)", [] {
    const std::size_t n = 256;
    const Mask band = gen_longformer_windowed(n, 3);
    std::vector<uint32_t> lab(n);
    for (std::size_t i = 0; i < n; ++i) lab[i] = static_cast<uint32_t>((i * 97 + 13) % n);
    const Mask shuffled = permute_mask(band, Permutation::from_forward(lab));
    EXPECT(bandwidth(shuffled) > 3);
    const Permutation perm = rcm_order(build_graph(shuffled));
    const Mask re = permute_mask(shuffled, perm);
    EXPECT(bandwidth(re) <= 6);
    // mask'(a,b) = mask(forward[a], forward[b])
    for (std::size_t a = 0; a < n; a += 17)
      for (std::size_t b = 0; b < n; ++b) EXPECT(re.get(a, b) == shuffled.get(perm.forward[a], perm.forward[b]));
    const Problem p = make_problem(n, 64, 6);
    const MaskPrep p0 = preprocess_mask(shuffled, BlockSpec{64, 64});
    const MaskPrep p1 = preprocess_mask(re, BlockSpec{64, 64});
    const auto f0 = blocked_forward(p.q, p.k, p.v, p.scale, shuffled, p0, Variant::binblk);
    const auto f1 = blocked_forward(permute_rows(p.q, perm), permute_rows(p.k, perm), permute_rows(p.v, perm),
                                    p.scale, re, p1, Variant::binblk);
    const Matrix<float> back = unpermute_rows(f1.out, perm);
    EXPECT(max_abs_diff(back, f0.out) <= 2e-2);
    EXPECT(f1.counters.blocks_processed < f0.counters.blocks_processed);
    const Matrix<float> round = unpermute_rows(permute_rows(p.v, perm), perm);
    EXPECT(round == p.v);
  });

  std::printf("%d checks, %d failures\n", g_checks, g_failures);
  return g_failures == 0 ? 0 : 1;
}
