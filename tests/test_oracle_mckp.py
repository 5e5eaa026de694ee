"""Pins of the oracle's 2D layer-head window scaling solver (O11): budget
extremes, a ratio-trap instance where greedy is provably suboptimal (exact strictly better),
the greedy within 10% of the exhaustive optimum on random small profile-like (concave)
instances,
feasibility, and exhaustive search checked by brute force in numpy (itertools)."""
import itertools

import numpy as np
import pytest

import oracle


def _random_instance(rng, pairs, sizes):
    # window sizes of a profile: cost grows with the window, the transfer reduction with
    # diminishing returns (concave in cost), heads differ by a random scale
    step = rng.integers(1, 6, size=(pairs, 1)).astype(np.float64)
    cost = step * np.arange(1, sizes + 1)[None, :]
    gains = -np.sort(-rng.random((pairs, sizes - 1)), axis=1) * rng.random((pairs, 1)) * 10
    benefit = np.concatenate([np.zeros((pairs, 1)), np.cumsum(gains, axis=1)], axis=1)
    return benefit, cost


def test_budget_extremes():
    rng = np.random.default_rng(0)
    b, c = _random_instance(rng, 6, 4)
    tot, ch = oracle.mckp(b, c, c[:, -1].sum())
    assert (ch == 3).all() and tot == pytest.approx(b[:, -1].sum())     # unconstrained: max everywhere
    tot, ch = oracle.mckp(b, c, c[:, 0].sum())
    assert (ch == 0).all() and tot == 0.0                               # fully constrained: min everywhere
    with pytest.raises(oracle.OracleError):
        oracle.mckp(b, c, c[:, 0].sum() - 1)                            # infeasible base


def test_ratio_trap_exact_beats_greedy():
    # pair 0: a cheap upgrade with the best ratio that blocks pair 1's big, better upgrade
    benefit = np.array([[0.0, 3.0], [0.0, 10.0]])
    cost = np.array([[1.0, 2.0], [1.0, 11.0]])
    budget = 12.0                                                       # base 2; room for 10 more
    g, gch = oracle.mckp(benefit, cost, budget)
    e, ech = oracle.mckp(benefit, cost, budget, exact=True)
    assert list(gch) == [1, 0] and g == 3.0
    assert list(ech) == [0, 1] and e == 10.0 > g


@pytest.mark.parametrize("seed", range(20))
def test_exact_is_brute_force_and_greedy_near_optimal(seed):
    rng = np.random.default_rng(100 + seed)
    pairs, sizes = int(rng.integers(2, 7)), int(rng.integers(2, 5))
    b, c = _random_instance(rng, pairs, sizes)
    budget = c[:, 0].sum() + rng.random() * (c[:, -1].sum() - c[:, 0].sum())
    e, ech = oracle.mckp(b, c, budget, exact=True)
    best = max((sum(b[p, s] for p, s in enumerate(al)), al) for al in itertools.product(range(sizes), repeat=pairs)
               if sum(c[p, s] for p, s in enumerate(al)) <= budget)
    assert e == pytest.approx(best[0])
    assert sum(c[p, s] for p, s in enumerate(ech)) <= budget
    g, gch = oracle.mckp(b, c, budget)
    assert sum(c[p, s] for p, s in enumerate(gch)) <= budget + 1e-9     # feasible
    assert g == pytest.approx(sum(b[p, s] for p, s in enumerate(gch)))
    assert g >= 0.9 * e - 1e-9                                          # near-optimal on profile-like instances
