"""GPU: generic from_triplets against the reference's
from_triplets (sparse.hpp:61-115, oracle/_ref or the C oracle): bitwise."""
from __future__ import annotations

import numpy as np
import pytest

import paper_1804_05156_b200 as fl
from oracle import pyoracle as po

pytestmark = pytest.mark.gpu


def _eq(got, want):
    np.testing.assert_array_equal(got.col_ptr, want.col_ptr)
    np.testing.assert_array_equal(got.row_idx, want.row_idx)
    assert got.values.tobytes() == want.values.tobytes()


def test_kats(ctx):  # sparse_test.cpp:36-70
    a = fl.from_triplets(4, 3, [0, 1, 3, 1], [0, 1, 1, 2], [1.0, 2.0, 9.0, 4.0], ctx=ctx)
    assert a.col_ptr.tolist() == [0, 1, 3, 4] and a.row_idx.tolist() == [0, 1, 3, 1]
    assert a.values.tolist() == [1.0, 2.0, 9.0, 4.0]
    assert fl.from_triplets(1, 1, [0, 0], [0, 0], [1.0, 2.0], ctx=ctx).values.tolist() == [3.0]
    z = fl.from_triplets(1, 1, [0, 0], [0, 0], [1.0, -1.0], ctx=ctx)
    assert z.nnz() == 0 and z.col_ptr.tolist() == [0, 0]
    t = fl.from_triplets(2, 2, [0, 1], [0, 1], [1e-300, 5e-324], ctx=ctx)
    assert t.values.tolist() == [1e-300, 5e-324]
    e = fl.from_triplets(3, 5, [], [], [], ctx=ctx)
    assert e.col_ptr.tolist() == [0] * 6


def test_bad_index(ctx):
    with pytest.raises(fl.Error) as e:
        fl.from_triplets(2, 2, [2], [0], [1.0], ctx=ctx)
    assert e.value.code() == fl.ErrorCode.index_out_of_range


@pytest.mark.parametrize("m,n,count,seed", [(7, 5, 200, 1), (300, 200, 100_000, 2),
                                            (70_000, 300, 300_000, 3), (5, 90_000, 200_000, 4),
                                            (1 << 17, 1 << 17, 1_000_000, 5)])
def test_random_with_duplicates_and_cancellations(m, n, count, seed, ctx, ref_which):
    rng = np.random.default_rng(seed)
    ii = rng.integers(0, m, count).astype(np.int32)
    jj = rng.integers(0, n, count).astype(np.int32)
    # values from a small set: many exact cancellations; plus order-sensitive sums
    ss = rng.choice(np.array([1.0, -1.0, 0.5, -0.5, 0.1, 1e16, -1e16, 3.0]), count)
    want = po.from_triplets(m, n, ii, jj, ss, which=ref_which)
    _eq(fl.from_triplets(m, n, ii, jj, ss, ctx=ctx), want)
