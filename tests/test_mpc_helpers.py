"""Host helpers around the batched solve (reference mpc.py:61-147) against the reference when it
is mounted, and against their closed-form properties otherwise."""

import sys

import numpy as np
import pytest

import paper_2510_07625_b200 as gb
from paper_2510_07625_b200 import mpc
from conftest import REFERENCE_SRC


def test_rho_grid_is_nested_and_spans_the_interval():
    g8, g16 = mpc.rho_grid(8), mpc.rho_grid(16)
    assert np.array_equal(g8, g16[:8])
    assert g8[0] == pytest.approx(10 ** -3.5) and g8[1] == pytest.approx(1e-8) and g8[2] == pytest.approx(1e1)
    assert len(set(np.round(np.log10(g16), 9))) == 16
    with pytest.raises(ValueError):
        mpc.rho_grid(0)


def test_shift_duplicates_the_tail():
    """test_mpc.py:52-58."""
    X = np.arange(12.0).reshape(6, 2)
    U = np.arange(5.0).reshape(5, 1)
    Xs, Us = mpc.shift_warm_start(gb.SqpResult(X, U, [], False))
    assert np.array_equal(Xs, np.vstack([X[1:], X[-1:]])) and np.array_equal(Us, np.vstack([U[1:], U[-1:]]))


def test_hypotheses_sit_on_the_sigma_sphere():
    hyp = mpc.sample_hypotheses(np.array([1.0, -2.0, 0.5]), 3.0, 9, seed=4)
    assert np.array_equal(hyp[0].value, [1.0, -2.0, 0.5])
    for h in hyp[1:]:
        assert np.linalg.norm(h.value - hyp[0].value) == pytest.approx(3.0)
    again = mpc.sample_hypotheses(np.array([1.0, -2.0, 0.5]), 3.0, 9, seed=4)
    assert all(np.array_equal(a.value, b.value) for a, b in zip(hyp, again))


def test_best_of_batch_prefers_first_minimum_and_skips_failures():
    def res(m):
        return gb.SqpResult(np.zeros((2, 2)), np.zeros((1, 1)),
                            [gb.IterationRecord(0, m, 0.0, 1.0, 1e-4, 3, True, 0.1)], False)
    assert mpc.best_of_batch([None, res(3.0), res(1.0), res(1.0)]) == 2
    with pytest.raises(ValueError):
        mpc.best_of_batch([None, None])


@pytest.mark.reference
@pytest.mark.skipif(not REFERENCE_SRC.exists(), reason="reference package not mounted")
def test_helpers_match_the_reference_bitwise():
    sys.path.insert(0, str(REFERENCE_SRC))
    from trajbatch import mpc as ref
    for M in (1, 3, 8, 33):
        assert np.array_equal(mpc.rho_grid(M), ref.rho_grid(M))
    mine = mpc.sample_hypotheses(np.zeros(3), 5.0, 16, seed=11)
    theirs = ref.sample_hypotheses(np.zeros(3), 5.0, 16, seed=11)
    assert all(np.array_equal(a.value, b.value) for a, b in zip(mine, theirs.candidates))
