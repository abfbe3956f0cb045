"""The BenchRecord / BenchConfig harness (bench.hpp:49-501) on the B200 engine.

CPU: the pinned CSV header and exact row round trip (test_bench.cpp:28-74), JSON config keys and
unknown-key rejection (test_bench.cpp:80-99), the make_problem input stream against the
reference. GPU: run_bench rows whose counter / density columns equal the reference CPU engine's.
"""
import numpy as np
import pytest

import oracle
import paper_2409_15097_b200 as bbm
from paper_2409_15097_b200 import harness as H


def test_csv_header_is_pinned():  # test_bench.cpp:28-35
    assert H.CSV_HEADER == (
        "variant,mask,n,block_i,block_j,batch,heads,runs,precision,prepro_ms,"
        "fwd_ms_mean,fwd_ms_std,bwd_ms_mean,bwd_ms_std,total_ms_mean,blocks_visited,"
        "blocks_processed,mask_block_reads,skipped_by_binblk,"
        "skipped_mask_reads_by_run,block_density,element_density,"
        "max_abs_err_vs_oracle")
    assert len(H.CSV_HEADER.split(",")) == 23


def test_csv_row_round_trip_is_exact():  # test_bench.cpp:37-74
    rec = H.BenchRecord(variant=bbm.Variant.dense_binblk, mask="windowed(w=256;causal=1)+rcm", n=4096,
                        block_i=128, block_j=32, batch=4, heads=32, runs=100, precision="single",
                        prepro_ms=1.0 / 3.0, fwd_ms_mean=12.5, fwd_ms_std=0.125, bwd_ms_mean=2e-7,
                        bwd_ms_std=0.0, total_ms_mean=12.5 + 2e-7,
                        counters=bbm.EngineCounters(4096, 1000, 900, 3096, 100),
                        block_density=0.244140625, element_density=0.1234567890123456789,
                        max_abs_err_vs_oracle=3.0000000000000004e-13)
    line = rec.csv_row()
    parsed = H.BenchRecord.parse_csv_row(line)
    assert parsed.csv_row() == line
    assert parsed.prepro_ms == rec.prepro_ms and parsed.element_density == rec.element_density
    assert parsed.max_abs_err_vs_oracle == rec.max_abs_err_vs_oracle
    assert parsed.counters == rec.counters
    rec.max_abs_err_vs_oracle = None
    bare = rec.csv_row()
    assert bare.endswith(",") and H.BenchRecord.parse_csv_row(bare).max_abs_err_vs_oracle is None
    # setprecision(17) formatting, as the reference prints it
    assert H.fmt_double(1.0 / 3.0) == "0.33333333333333331" and H.fmt_double(2e-7) == "1.9999999999999999e-07"
    assert H.fmt_double(12.5) == "12.5" and H.fmt_double(0.0) == "0"


def test_csv_rejects_wrong_field_count():
    with pytest.raises(ValueError):
        H.BenchRecord.parse_csv_row("dense,causal,64")


def test_config_json_round_trip_and_unknown_keys():  # test_bench.cpp:80-99
    c = H.BenchConfig.from_json('{"mask_spec": "medusa[4;4]", "batch": 2, "variants": ["binblk", "dense"],'
                                ' "block_i": 128, "block_j": 32, "rcm": true}')
    assert c.batch == 2 and c.variants == [bbm.Variant.binblk, bbm.Variant.dense] and c.rcm
    assert H.BenchConfig.from_json(c.to_json()) == c
    with pytest.raises(ValueError):
        H.BenchConfig.from_json('{"mask": "causal"}')
    with pytest.raises(ValueError):
        H.BenchConfig.from_json('{"runs": 0}')
    with pytest.raises(ValueError):
        H.BenchConfig.from_json('{"precision": "half"}')


def test_make_problem_stream_matches_reference():
    q, k, v, g = H.make_problem(3, 2, 37, 8)
    want = oracle.make_problem(3, 2, 37, 8)
    for a, b in zip((q, k, v, g), want):
        assert np.array_equal(a, b.astype(np.float32))


@pytest.mark.gpu
def test_run_bench_rows_match_reference_counters(cuda):
    cfg = H.BenchConfig.from_json({"mask_spec": "windowed(w=40)", "seq_lengths": [300, 512], "batch": 2,
                                   "heads": 2, "runs": 2, "warmup": 1, "head_dim": 64, "block_i": 64,
                                   "block_j": 32, "verify": True, "rcm": True})
    rows = []
    recs = H.run_bench(cfg, sink=lambda r: rows.append(r.csv_row()))
    assert len(recs) == 2 * 4 * 2 and len(rows) == len(recs)
    for r in recs:
        words = bbm.generate("windowed(w=40)", r.n)
        if r.mask.endswith("+rcm"):
            words = bbm.permute_mask(words, bbm.rcm_order(words))
        want = oracle.counters(words.words, r.n, 64, 32, int(r.variant))
        slots = cfg.batch * cfg.heads
        assert (r.counters.blocks_visited, r.counters.blocks_processed, r.counters.mask_block_reads,
                r.counters.skipped_by_binblk, r.counters.skipped_mask_reads_by_run) == tuple(x * slots for x in want)
        assert r.max_abs_err_vs_oracle is not None and r.max_abs_err_vs_oracle <= 2e-2
        assert r.fwd_ms_mean > 0 and r.bwd_ms_mean > 0
        assert H.BenchRecord.parse_csv_row(r.csv_row()).csv_row() == r.csv_row()
