"""The oracle is pinned against the reference's own outputs (tests/golden, made by
tests/golden/make_golden.py from /root/reference) before it is trusted."""
import numpy as np


def test_length_stats_c_and_numpy_match_reference(golden, orc):
    for case in golden["length_stats"]:
        off = np.array(case["offsets"], dtype=np.int64)
        assert list(orc.length_stats(off)) == case["length_stats"]
        assert list(orc.length_stats_np(off)) == case["length_stats"]


def test_wave_ceil_max_sum_matches_reference(golden, orc):
    for case in golden["length_stats"]:
        off = np.array(case["offsets"], dtype=np.int64)
        for d, w, want in case["wave"]:
            assert orc.wave_ceil_max_sum(off, d, w) == want
            if off.size > 1 or True:
                assert orc.wave_ceil_max_sum_np(off, d, w) == want


def test_gather_features_bit_exact(golden, orc):
    for m in golden["gather_features"]:
        off = np.array(m["row_offsets"], dtype=np.int64)
        assert list(orc.length_stats(off)) == m["length_stats"]
        got = orc.gather_features(off, m["n_rows"], m["n_cols"])
        assert [v.hex() for v in got] == m["features_hex"], m["name"]


def test_epilogue_python_and_c_bit_exact(golden, orc):
    for e in golden["epilogue"]:
        lo, hi, s1, s2 = e["agg"]
        py = orc.features_epilogue(lo, hi, s1, s2, e["n"], e["c"])
        c = orc.features_epilogue_c(lo, hi, s1, s2, e["n"], e["c"])
        assert [v.hex() for v in py] == e["features_hex"]
        assert [v.hex() for v in c] == e["features_hex"]


def test_spec_examples(golden, orc):
    by = {m["name"]: m for m in golden["gather_features"]}
    assert [float.fromhex(h) for h in by["spec118"]["features_hex"]] == [1.0, 0.0, 0.5, 0.25]
    f119 = [float.fromhex(h) for h in by["spec119"]["features_hex"]]
    assert f119[3] == 0.0 and f119[0] == f119[1] == f119[2]
    f120 = [float.fromhex(h) for h in by["spec120"]["features_hex"]]
    assert f120[2] == 0.2 and f120[3] == 0.006666666666666661  # E[d^2]-E[d]^2 rounding
    assert orc.length_stats([0, 4, 4, 9, 10]) == (0, 5, 10, 42)
    assert orc.wave_ceil_max_sum([0, 4, 4, 9, 10], 2, 3) == 4


def test_compiled_reference_core_when_built(golden, orc):
    core = orc.ref_core()
    if core is None:
        import pytest
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    for case in golden["length_stats"][:40]:
        off = np.array(case["offsets"], dtype=np.int64)
        assert list(core.length_stats(off.copy())) == case["length_stats"]


def test_cpu_spmv_oracle_matches_dense(orc):
    rng = np.random.default_rng(0)
    n, c = 50, 40
    dense = rng.uniform(-1, 1, (n, c)) * (rng.random((n, c)) < 0.2)
    off = np.concatenate([[0], np.cumsum((dense != 0).sum(1))]).astype(np.int64)
    rows, cols = np.nonzero(dense)
    vals = dense[rows, cols]
    x = rng.uniform(-1, 1, c)
    y, a = orc.spmv_csr(off, cols.astype(np.int32), vals, x)
    assert np.allclose(y, dense @ x, rtol=1e-13, atol=1e-13)
    assert np.all(a >= np.abs(y) - 1e-12)
    y32 = orc.spmv_native(off.astype(np.int32), cols.astype(np.int32), vals.astype(np.float32), x.astype(np.float32))
    assert np.allclose(y32, dense @ x, atol=1e-5)


def test_csr_from_coo_oracle_matches_reference_golden():
    """oracle.csr_from_coo == the UNMODIFIED reference's csr_from_coo, bit for bit."""
    import json
    import os
    import sys
    import numpy as np
    from oracle import oracle as orc
    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    sys.path.insert(0, here)
    from make_golden_coo import coo_case
    doc = json.load(open(os.path.join(here, "reference_coo_golden.json")))
    for case in doc["cases"]:
        R, C, rows, cols, vals = coo_case(case["spec"])
        off, col, val = orc.csr_from_coo(R, C, rows, cols, vals)
        assert off.tolist() == case["row_offsets"], case["spec"]["name"]
        assert col.tolist() == case["col_indices"], case["spec"]["name"]
        assert [float(v).hex() for v in val] == case["values"], case["spec"]["name"]
