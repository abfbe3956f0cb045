"""BBMK mask files and BBLK occupancy sidecars (mask_io.hpp), mirroring
test_mask_model.cpp:224-323; the device path (file bytes unpacked on the GPU into the
preprocessor) is -m gpu."""
import os

import numpy as np
import pytest

import oracle
import paper_2409_15097_b200 as bbm


def rand_mask(n, seed):
    rng = np.random.default_rng(seed)
    return bbm.Mask.from_dense(rng.integers(0, 2, size=(n, n)).astype(bool))


def test_single_token_file_layout(tmp_path):  # test_mask_model.cpp:224-239
    m = bbm.Mask(1)
    m.set(0, 0, True)
    p = tmp_path / "one.bbmk"
    bbm.write_mask(m, p)
    data = p.read_bytes()
    assert len(data) == 14 and data[:4] == b"BBMK" and data[4] == 1 and data[5] == 1
    assert data[6:13] == bytes(7) and data[13] == 1
    assert bbm.read_mask(p) == m


@pytest.mark.parametrize("n", [1, 2, 7, 8, 9, 13, 63, 64, 65, 129, 257])
def test_round_trip_across_byte_boundaries(tmp_path, n):  # test_mask_model.cpp:241-252
    m = rand_mask(n, n)
    p = tmp_path / f"rt{n}.bbmk"
    bbm.write_mask(m, p)
    assert os.path.getsize(p) == 13 + n * ((n + 7) // 8)
    assert bbm.read_mask(p) == m


def test_header_and_payload_errors_are_distinguished(tmp_path):  # test_mask_model.cpp:254-283
    p = tmp_path / "err.bbmk"
    bbm.write_mask(bbm.gen_causal(9), p)
    good = p.read_bytes()

    def kind(data=None, path=p):
        if data is not None:
            path.write_bytes(data)
        with pytest.raises(bbm.MaskIoError) as e:
            bbm.read_mask(path)
        return e.value.kind

    assert kind(path=tmp_path / "missing.bbmk") == "io_failure"
    assert kind(b"X" + good[1:]) == "bad_magic"
    assert kind(good[:4] + b"\x02" + good[5:]) == "bad_version"
    assert kind(good[:6]) == "truncated"
    assert kind(good[:-1]) == "truncated"
    assert kind(good + b"Z") == "trailing_data"
    assert kind(good[:11] + b"\x7f" + good[12:]) == "dimension_overflow"


def test_files_are_byte_identical_to_the_reference_writer(tmp_path):
    # the same bytes the reference's write_mask produces: its byte rows are the Mask words read
    # little-endian, truncated to ceil(n/8) bytes
    for n in (5, 64, 100):
        m = rand_mask(n, 7 + n)
        p = tmp_path / "w.bbmk"
        bbm.write_mask(m, p)
        rb = (n + 7) // 8
        rows = np.ascontiguousarray(m.words).view(np.uint8).reshape(n, -1)[:, :rb]
        want = b"BBMK\x01" + n.to_bytes(8, "little") + rows.tobytes()
        assert p.read_bytes() == want


def test_occupancy_round_trip_and_layout(tmp_path):  # test_mask_model.cpp:285-310
    words = bbm.gen_causal(10).words
    sums = oracle.block_sums(words, 10, 4, 3)
    occ = bbm.BlockOccupancy((sums > 0).astype(np.uint8))
    p = tmp_path / "occ.bblk"
    bbm.write_occupancy(occ, 10, bbm.BlockSpec(4, 3), p)
    data = p.read_bytes()
    assert data[:4] == b"BBLK" and data[4] == 1 and data[5] == 10 and data[13] == 4 and data[17] == 3
    f = bbm.read_occupancy(p)
    assert f.n_tokens == 10 and f.spec == bbm.BlockSpec(4, 3)
    assert np.array_equal(f.occupancy.values, occ.values)


def test_occupancy_rejects_zero_block_size(tmp_path):  # test_mask_model.cpp:312-323
    p = tmp_path / "occ_zero.bblk"
    occ = bbm.BlockOccupancy(np.ones((2, 2), np.uint8))
    bbm.write_occupancy(occ, 8, bbm.BlockSpec(4, 4), p)
    data = bytearray(p.read_bytes())
    data[13:17] = b"\0\0\0\0"
    p.write_bytes(bytes(data))
    with pytest.raises(bbm.MaskIoError) as e:
        bbm.read_occupancy(p)
    assert e.value.kind == "dimension_overflow"


@pytest.mark.gpu
@pytest.mark.parametrize("spec,n", [("packed-seq[100;260;37;243]", 0), ("global(w=64;g=9)", 1000),
                                    ("random(p=0.3;seed=2)", 129)])
def test_preprocess_from_file_equals_preprocess_from_mask(cuda, tmp_path, spec, n):
    m = bbm.generate(spec, n)
    p = tmp_path / "m.bbmk"
    bbm.write_mask(m, p)
    for bs in (bbm.BlockSpec(128, 128), bbm.BlockSpec(64, 32)):
        a = bbm.preprocess_mask_file(p, bs)
        b = bbm.preprocess_mask(m, bs)
        assert np.array_equal(a.sums.values, b.sums.values)
        assert a.runs.offset == b.runs.offset and a.runs.total_ones == b.runs.total_ones
        ca, la, oa = a.kernel_lists()
        cb, lb, ob = b.kernel_lists()
        assert np.array_equal(ca, cb) and np.array_equal(oa, ob)
        for r in range(ca.size):  # entries past row_cnt are unused
            assert np.array_equal(la[r, :ca[r]], lb[r, :cb[r]])
