"""Native Matrix Market ingest (kp_mm_parse) vs the UNMODIFIED reference's
parse_matrix_market (sparse.py:106-196): canonical CSR bit-exact, or the identical
ParseError message (incl. the 1-based line number).  Host code: runs without a GPU."""
import json
import os
import sys

import numpy as np
import pytest

from paper_2403_17017_b200 import mmio
from paper_2403_17017_b200.errors import ParseError

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _cases():
    sys.path.insert(0, HERE)
    from make_golden_mm import long_case
    doc = json.load(open(os.path.join(HERE, "reference_mm_golden.json")))["cases"]
    for name, rec in doc.items():
        text = long_case() if name == "long_symmetric_crlf" else rec["text"]
        yield name, text, rec


@pytest.mark.parametrize("threads", [1, 3, 16])
def test_parse_matches_reference_golden(threads):
    for name, text, rec in _cases():
        if "error" in rec:
            with pytest.raises(ParseError) as ei:
                mmio.parse_matrix_market(text, n_threads=threads)
            assert str(ei.value) == rec["error"], name
            continue
        m = mmio.parse_matrix_market(text, n_threads=threads)
        assert (m.n_rows, m.n_cols) == (rec["n_rows"], rec["n_cols"]), name
        assert np.asarray(m.row_offsets).tolist() == rec["row_offsets"], name
        assert np.asarray(m.col_indices).tolist() == rec["col_indices"], name
        assert [float(v).hex() for v in m.values] == rec["values"], name


def test_bytes_input_and_writer_round_trip():
    from paper_2403_17017_b200 import sparse
    m = sparse.csr_from_coo(4, 5, [0, 3, 3, 1], [4, 0, 2, 1], [0.1, -2.5e-300, 7.0, 1e20])
    text = mmio.write_matrix_market(m)
    back = mmio.parse_matrix_market(text.encode())
    assert np.array_equal(back.row_offsets, m.row_offsets)
    assert np.array_equal(back.col_indices, m.col_indices)
    assert [float(v).hex() for v in back.values] == [float(v).hex() for v in m.values]


def test_chunking_many_threads_large_file():
    """Chunk boundaries fall everywhere in a large CRLF file: every thread count parses
    identically (entry order, mirrors right after their entry)."""
    sys.path.insert(0, HERE)
    from make_golden_mm import long_case
    text = long_case(60000, seed=3)
    ref = mmio.parse_arrays(text, n_threads=1)
    for t in (2, 5, 8, 32):
        got = mmio.parse_arrays(text, n_threads=t)
        assert got[:2] == ref[:2]
        for a, b in zip(got[2:], ref[2:]):
            assert np.array_equal(a, b)
