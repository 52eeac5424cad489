"""AERO binary stream files through the product library (reference
streams.cpp:105-168; tests mirror test_streams.cpp:154-196). Host-only file
I/O of libaero_b200.so: no GPU needed. The byte layout is checked against the
oracle's restatement (oracle/pyoracle.py aero_bytes / load_aero_bytes)."""
import numpy as np
import pytest

import paper_2601_02019_b200 as prod
from paper_2601_02019_b200.capi import FormatError


def _rows(orc, n, d, seed):
    return orc.rng_draw(seed, 22, 0, n * d, "uniform").reshape(n, d)


def test_binary_round_trip_is_bit_exact(orc, tmp_path):  # test_streams.cpp:154-166
    rows = _rows(orc, 30, 7, 22)
    p = tmp_path / "s.aero"
    prod.write_aero(p, rows)
    back = prod.read_aero(p)
    assert back.shape == rows.shape
    assert np.array_equal(back.view(np.uint64), rows.view(np.uint64))
    assert p.read_bytes() == orc.aero_bytes(rows)  # byte layout == the restated save_stream
    assert np.array_equal(orc.load_aero_bytes(p.read_bytes()), rows)


def test_header_records_magic_dimension_count(orc, tmp_path):  # test_streams.cpp:168-181
    p = tmp_path / "h.aero"
    prod.write_aero(p, _rows(orc, 3, 2, 23))
    b = p.read_bytes()
    assert len(b) == 17 + 3 * 2 * 8
    assert b[:4] == b"AERO" and b[4] == 1
    assert np.frombuffer(b[5:9], "<u4")[0] == 2 and np.frombuffer(b[9:17], "<u8")[0] == 3
    with prod.AeroFileReader(p) as f:
        assert (f.d, f.n_header) == (2, 3)


def test_zero_count_reads_until_eof(orc, tmp_path):  # test_streams.cpp:183-191
    p = tmp_path / "z.aero"
    rows = _rows(orc, 4, 2, 24)
    b = bytearray(orc.aero_bytes(rows))
    b[9:17] = bytes(8)
    p.write_bytes(bytes(b))
    assert prod.read_aero(p).shape == (4, 2)


def test_chunked_reads_cover_the_file(orc, tmp_path):
    p = tmp_path / "c.aero"
    rows = _rows(orc, 1000, 5, 25)
    prod.write_aero(p, rows)
    with prod.AeroFileReader(p) as f:
        parts = list(f.chunks(333))
    assert [x.shape[0] for x in parts] == [333, 333, 333, 1]
    assert np.array_equal(np.concatenate(parts), rows)


@pytest.mark.parametrize("case", ["magic", "version", "header", "row", "nonfinite", "zero_d"])
def test_malformed_files_raise_format_error(orc, tmp_path, case):  # test_streams.cpp:193-196
    p = tmp_path / "bad.aero"
    rows = _rows(orc, 4, 3, 26)
    b = bytearray(orc.aero_bytes(rows))
    if case == "magic":
        b = bytearray(b"NOPE....")
    elif case == "version":
        b[4] = 2
    elif case == "header":
        b = b[:12]
    elif case == "row":
        b = b[:-5]
    elif case == "nonfinite":
        b[17 + 8 * 5:17 + 8 * 6] = np.float64(np.inf).tobytes()
    elif case == "zero_d":
        b[5:9] = bytes(4)
    p.write_bytes(bytes(b))
    with pytest.raises(orc.FormatError):
        orc.load_aero_bytes(bytes(b))
    with pytest.raises(FormatError):
        prod.read_aero(p)


def test_save_validates_the_record_set(tmp_path):  # test_streams.cpp:198-203
    with pytest.raises(prod.InvalidInput):
        prod.write_aero(tmp_path / "e.aero", np.empty((0, 3)))
