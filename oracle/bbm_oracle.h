/* bbm_oracle.h — CPU oracle for the Binary Block Masking hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This is a plain-C restatement of the reference's algorithm
 * (/root/reference/proj/include/blockmask/{mask,engine,reference,reorder,rng}.hpp); it is the
 * checker for the CUDA path, never the thing measured or shipped. Only tests/, the smoke() in
 * __graft_entry__.py and bench.py's cpu_baseline leg may load it.
 *
 * Parity of this restatement is pinned two ways:
 *   1. the reference's own known-answer tests (test_mask_model.cpp, test_engine.cpp,
 *      test_reorder.cpp) re-asserted in tests/test_oracle.py, and
 *   2. golden vectors produced by the real reference headers compiled into oracle/_ref
 *      (tests/golden/make_golden.py) and compared bit-for-bit / to 1e-12.
 *
 * Mask layout is the reference's: row-major u64 words, words_per_row = ceil(n/64), bit j of
 * row i at word j>>6, bit j&63, tail bits zero (mask.hpp:17-52).
 */
#ifndef BBM_ORACLE_H
#define BBM_ORACLE_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* --- rng.hpp:15-42 : mt19937_64 + the implementation-independent mappings --- */
typedef struct { uint64_t mt[312]; int mti; } orc_mt64;
void orc_mt64_seed(orc_mt64* g, uint64_t seed);
uint64_t orc_mt64_next(orc_mt64* g);
double orc_uniform_unit(orc_mt64* g);                 /* rng.hpp:15-17 */
double orc_uniform_pm1(orc_mt64* g);                  /* rng.hpp:20-22 */
uint64_t orc_uniform_below(orc_mt64* g, uint64_t b);  /* rng.hpp:25-32 */
/* make_problem stream (bench.hpp:320-337 / test_util.hpp:22-32): per slot q, k, v, d_out,
 * each rows x cols row-major, uniform[-1,1) as double. Any output pointer may be NULL (the
 * draws still happen so the stream stays aligned). */
void orc_make_problem(uint64_t seed, uint64_t slots, uint64_t n, uint64_t d, double* q,
                      double* k, double* v, double* d_out);

/* --- mask.hpp:167-247 --- */
uint32_t orc_popcount_range(const uint64_t* row_words, uint64_t c0, uint64_t c1);
void orc_block_sums(const uint64_t* words, uint64_t n, uint64_t bi, uint64_t bj,
                    uint32_t* sums /* ceil(n/bi) x ceil(n/bj) */);
void orc_block_occupancy(const uint32_t* sums, uint64_t rows, uint64_t cols, uint8_t* occ);
void orc_dense_runs(const uint32_t* sums, uint64_t n, uint64_t bi, uint64_t bj,
                    uint32_t* offset, uint32_t* total_ones);
typedef struct {
  uint64_t blocks_total, blocks_nonzero, blocks_full;
  double block_density, element_density;
} orc_block_stats_t;
void orc_block_stats(const uint32_t* sums, uint64_t n, uint64_t bi, uint64_t bj,
                     orc_block_stats_t* out);

/* --- engine.hpp:47-66, 118-153 : counters of one blocked_forward call --- */
typedef struct {
  uint64_t blocks_visited, blocks_processed, mask_block_reads, skipped_by_binblk,
      skipped_mask_reads_by_run;
} orc_counters_t;
enum { ORC_DENSE = 0, ORC_NAIVE = 1, ORC_BINBLK = 2, ORC_DENSE_BINBLK = 3 };
void orc_counters(const uint32_t* sums, const uint32_t* offset, const uint32_t* total_ones,
                  uint64_t n, uint64_t bi, uint64_t bj, int variant, orc_counters_t* out);

/* --- reference.hpp:42-81 : naive_forward in double; rows split over `threads` workers
 * (each row is independent, so results do not depend on the thread count). --- */
void orc_naive_forward(const double* q, const double* k, const double* v, uint64_t n,
                       uint64_t d, uint64_t dv, double scale, const uint64_t* words,
                       double* out, double* row_max, double* row_sum, int threads);
/* Same math applied with the column subset of a 'dense' variant: every key visible. */
void orc_dense_forward(const double* q, const double* k, const double* v, uint64_t n,
                       uint64_t d, uint64_t dv, double scale, double* out, double* row_max,
                       double* row_sum, int threads);

/* --- reorder.hpp:28-189 --- */
/* reference.hpp:84-139 (naive_backward); words == NULL: dense (every key visible) */
void orc_naive_backward(const double* q, const double* k, const double* v, const double* dout,
                        uint64_t n, uint64_t d, double scale, const uint64_t* words, double* dq,
                        double* dk, double* dv, int threads);
/* forward (+ dq) of a list of query rows only (reference.hpp:42-139 restated per row) */
void orc_naive_rows(const double* q, const double* k, const double* v, const double* dout,
                    uint64_t n, uint64_t d, double scale, const uint64_t* words,
                    const uint64_t* rows, uint64_t nrows, double* out, double* row_max,
                    double* row_sum, double* dq);
int orc_rcm_order(const uint64_t* words, uint64_t n, uint32_t* forward /* n */);
uint64_t orc_bandwidth(const uint64_t* words, uint64_t n);
void orc_permute_mask(const uint64_t* words, uint64_t n, const uint32_t* forward,
                      uint64_t* out_words);
void orc_permute_rows(const void* src, void* dst, uint64_t rows, uint64_t row_bytes,
                      const uint32_t* forward, int inverse);

#ifdef __cplusplus
}
#endif
#endif
