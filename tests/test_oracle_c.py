"""oracle/fold.c (the timed CPU baseline) is pinned bit-exact to the pinned
numpy oracle oracle/hfr_oracle.py:fold_ascending."""
import numpy as np
import pytest

import hfr_inputs as gen
from oracle import cfold
from oracle import hfr_oracle as O


@pytest.mark.parametrize("n", [1, 2, 3, 8])
@pytest.mark.parametrize("dtype", [gen.FP32, gen.BF16])
@pytest.mark.parametrize("dist", ["normal", "specials", "loguniform"])
def test_c_fold_matches_numpy_oracle(n, dtype, dist):
    xs = gen.rank_inputs(n, 100_003, dtype, dist, seed_base=7)
    for scale in (1.0, 0.125, 0.3):
        got = cfold.fold_ascending(xs, scale)
        want = O.fold_ascending(xs, scale)
        g = O.widen(got) if dtype == gen.BF16 else got
        w = O.widen(want) if dtype == gen.BF16 else want
        nan = np.isnan(w)
        assert np.array_equal(np.isnan(g), nan)
        assert np.array_equal(got[~nan], want[~nan])


def test_c_fold_threads():
    assert cfold.threads() >= 1
