"""solution.bin and RunRecord CSV formats vs the reference's writers
(src/dump.cpp:51-64, src/metrics.cpp:30-59), and series validation."""
import ctypes as C
import math
import os

import numpy as np
import pytest

from oracle.refbind import Ref, ref_available
from paper_2006_02602_b200 import records
from paper_2006_02602_b200.capi import InvalidArgument


def test_solution_roundtrip(tmp_path):
    f = np.random.default_rng(1).standard_normal((5, 4, 5, 6))
    p = tmp_path / "solution.bin"
    records.write_solution(p, f)
    assert os.path.getsize(p) == 48 + f.size * 8
    np.testing.assert_array_equal(records.read_solution(p), f)


@pytest.mark.skipif(not ref_available(), reason="reference library not built here")
def test_solution_bytes_equal_reference_writer(tmp_path):
    f = np.random.default_rng(2).standard_normal((5, 3, 4, 7))
    ours, theirs = tmp_path / "a.bin", tmp_path / "b.bin"
    records.write_solution(ours, f)
    st = Ref.lib().ref_write_solution(str(theirs).encode(), 7, 4, 3,
                                      np.ascontiguousarray(f).ctypes.data_as(C.c_void_p))
    assert st == 0
    assert ours.read_bytes() == theirs.read_bytes()


@pytest.mark.skipif(not ref_available(), reason="reference library not built here")
def test_csv_row_equals_reference():
    r = records.RunRecord(8, "3d", "2x2x2", "v3", 1, 4096, 29, 0.0123456789, 9.87654321,
                          float("nan"), 0.5, 123456)
    buf = C.create_string_buffer(512)
    Ref.lib().ref_csv_row(8, b"3d", b"2x2x2", b"v3", 1, C.c_longlong(4096), C.c_long(29),
                          C.c_double(0.0123456789), C.c_double(9.87654321), C.c_double(float("nan")),
                          C.c_double(0.5), C.c_ulonglong(123456), buf, 512)
    assert records.csv_text([r]).strip() == buf.value.decode().strip()
    back = records.parse_csv(records.csv_text([r]))[0]
    assert back.np == 8 and back.bytes_sent == 123456 and math.isnan(back.speedup)


def test_series_validation():
    s = records.ScalingSeries("v3 3d", "weak", [records.RunRecord(np=1, size=100, ssspnt=10.0),
                                                records.RunRecord(np=2, size=200, ssspnt=9.0)])
    s.validate()
    s.fill_speedups()
    assert s.rows[1].efficiency == 0.9 and s.rows[1].speedup == 1.8
    s.rows[1].size = 150
    with pytest.raises(InvalidArgument):
        s.validate()
    t = records.ScalingSeries("x", "strong", [records.RunRecord(np=1, size=100, wall_time_s=2.0),
                                              records.RunRecord(np=4, size=100, wall_time_s=1.0)])
    t.validate()
    t.fill_speedups()
    assert t.rows[1].speedup == 2.0 and t.rows[1].efficiency == 0.5
    with pytest.raises(RuntimeError):
        records.parse_csv("bad header\n")
