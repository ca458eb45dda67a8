"""CPU: the host-only sub-structuring entry points of libkrysp_gpu.so (no device needed)."""
import numpy as np
import pytest

import paper_2108_13162_b200 as kg
from paper_2108_13162_b200 import substructure as ss


@pytest.mark.parametrize("n,parts", [(10, 1), (10, 3), (64, 8), (1000, 7), (5, 5)])
def test_band_row_assignment_matches_reference(ref, n, parts):
    np.testing.assert_array_equal(ss.band_row_assignment(n, parts), ref.band_row_assignment(n, parts))


def test_band_row_assignment_rejects(ref):
    with pytest.raises(kg.Error):
        ss.band_row_assignment(3, 7)
    with pytest.raises(kg.Error):
        ss.band_row_assignment(3, 0)


def test_assignment_file_round_trip(tmp_path):
    p = tmp_path / "assign.txt"
    p.write_text("# subdomains\n0\n0\n\n1\n-1\n1\n")
    np.testing.assert_array_equal(ss.read_assignment_file(str(p), 5), [0, 0, 1, -1, 1])
    with pytest.raises(kg.DimensionMismatch):
        ss.read_assignment_file(str(p), 6)
    p.write_text("0\nx\n")
    with pytest.raises(kg.ParseError):
        ss.read_assignment_file(str(p), 2)
    p.write_text("0\n-2\n")
    with pytest.raises(kg.ParseError):
        ss.read_assignment_file(str(p), 2)
    with pytest.raises(kg.Error):
        ss.read_assignment_file(str(tmp_path / "missing.txt"), 2)
