"""K1 / K2 / gather_features on the GPU vs the reference's golden vectors (bit-exact)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_length_stats_and_wave_vs_reference_golden(golden):
    from paper_2403_17017_b200 import _kernels
    assert _kernels.BACKEND == "cuda"
    for case in golden["length_stats"]:
        off = np.array(case["offsets"], dtype=np.int64)
        assert list(_kernels.length_stats(off)) == case["length_stats"], case["offsets"][:6]
        ro = off.copy()
        ro.flags.writeable = False  # the reference's compiled backend fails here (App. B1)
        assert list(_kernels.length_stats(ro)) == case["length_stats"]
        if off.size and abs(int(off.max())) < 2**31 and int(off.min()) >= -2**31:
            t32 = torch.from_numpy(off.astype(np.int32)).cuda()
            assert list(_kernels.length_stats(t32)) == case["length_stats"]
        for d, w, want in case["wave"]:
            assert _kernels.wave_ceil_max_sum(off, d, w) == want, (case["offsets"][:6], d, w)


def test_wave_invalid_params_raise():
    from paper_2403_17017_b200 import _kernels
    for d, w in [(0, 1), (1, 0), (-2, 3)]:
        with pytest.raises(ValueError):
            _kernels.wave_ceil_max_sum([0, 1, 2], d, w)


def test_gather_features_bit_exact_vs_reference(golden):
    from paper_2403_17017_b200 import features, clock
    for m in golden["gather_features"]:
        class M:
            pass
        mm = M()
        mm.n_rows, mm.n_cols, mm.row_offsets = m["n_rows"], m["n_cols"], np.array(m["row_offsets"], np.int64)
        g = features.gather_features(mm, clock.FixedClock(tick=0.25))
        assert [v.hex() for v in g.as_vector()] == m["features_hex"], m["name"]
        assert g.collection_time == 0.25


def test_epilogue_bit_exact_random(orc):
    """Device epilogue == oracle epilogue (itself pinned to the reference) on random offsets,
    int32 and int64 layouts, sizes straddling the vector / tail paths."""
    from paper_2403_17017_b200 import features
    rng = np.random.default_rng(11)
    for trial in range(300):
        n = int(rng.choice([1, 2, 3, 5, 31, 64, 1000, 4097, 70001]))
        c = int(rng.integers(1, 10**7))
        ln = np.minimum(rng.poisson(rng.uniform(0.1, 60), n), c) if trial % 2 else rng.integers(0, min(c, 300) + 1, n)
        off = np.concatenate([[0], np.cumsum(ln)]).astype(np.int64)
        want = orc.gather_features(off, n, c)
        for dt in (torch.int64, torch.int32):
            class M:
                pass
            mm = M()
            mm.n_rows, mm.n_cols, mm.row_offsets = n, c, torch.from_numpy(off).to("cuda", dt)
            got = features.gather_features(mm).as_vector()
            assert [v.hex() for v in got] == [v.hex() for v in want], (trial, n, c)


def test_length_stats_large_int64_and_unaligned():
    from paper_2403_17017_b200 import _kernels
    from oracle import oracle as orc
    rng = np.random.default_rng(2)
    off = np.concatenate([[0], np.cumsum(rng.poisson(20, 3_000_001))]).astype(np.int64)
    t = torch.from_numpy(off).cuda()
    assert _kernels.length_stats(t) == orc.length_stats(off)
    # unaligned view (offset by one element: 8-byte aligned only) -> scalar path
    assert _kernels.length_stats(t[1:]) == orc.length_stats(off[1:])
    assert _kernels.wave_ceil_max_sum(t, 3, 100) == orc.wave_ceil_max_sum(off, 3, 100)
    assert _kernels.wave_ceil_max_sum(t, 1, 100_000) == orc.wave_ceil_max_sum(off, 1, 100_000)
    assert _kernels.wave_ceil_max_sum(t, 7, 1) == orc.wave_ceil_max_sum(off, 7, 1)


def test_device_clock_runs():
    from paper_2403_17017_b200 import features, clock, gen
    A = gen.config("C1").to_device_csr()
    g = features.gather_features(A, clock.CudaEventClock())
    assert g.collection_time > 0


def test_length_stats_int32_nonmonotone_and_extremes(orc):
    """int32 offsets through the 32-bit fast path and its signed fallback: decreasing
    offsets (negative lengths) and the full int32 range, vs the int64 oracle."""
    import numpy as np
    import torch
    from paper_2403_17017_b200 import _kernels
    rng = np.random.default_rng(9)
    cases = [np.array([-2**31, 2**31 - 1, -2**31, 0, 5, 5, 3], dtype=np.int64),
             rng.integers(-2**31, 2**31 - 1, 10001),
             np.cumsum(rng.integers(0, 3, 70001)).astype(np.int64),
             np.concatenate([np.cumsum(rng.integers(0, 5, 50000)), [7], np.arange(10, 2000)]).astype(np.int64)]
    for off in cases:
        t = torch.from_numpy(off.astype(np.int32)).cuda()
        assert _kernels.length_stats(t) == orc.length_stats_np(off)
