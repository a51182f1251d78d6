"""Host logic of the §4.3 failure-grid harness (tools/failure_grid.py): the exact
exponent rule floor(n^{p/20}) and the Lemma-3 bound."""
import math
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
from failure_grid import PANELS, cell_params, exp_floor, lemma3_bound  # noqa: E402


def test_exp_floor_values():
    n = 10 ** 6
    assert exp_floor(n, 10) == 1000               # exact power: 10^3
    assert exp_floor(n, 15) == 31622              # 10^4.5 = 31622.77...
    assert exp_floor(n, 5) == 31                  # 10^1.5 = 31.62...
    assert exp_floor(n, 1) == 1                   # 10^0.3 = 1.995...
    assert exp_floor(n, 19) == 501187             # 10^5.7 = 501187.2...
    assert exp_floor(2 ** 20, 15) == 2 ** 15      # 2^(20*3/4) exactly


def test_exp_floor_definition_bruteforce():
    for n in [2, 3, 10, 97, 1000, 4096]:
        for p in range(1, 20):
            c = exp_floor(n, p)
            assert c ** 20 <= n ** p < (c + 1) ** 20


def test_lemma3_bound_hand_value_and_domain():
    # n=50, gamma=delta=20, beta=40: K = 20*20/100 - 2*20/40 = 3; alpha=60:
    # exponent -(60*3/40)(1-1/3)^2 = -2, bound = (100/20) e^-2.
    assert math.isclose(lemma3_bound(50, 60, 40, 20, 20), 5 * math.exp(-2), rel_tol=1e-12)
    assert lemma3_bound(50, 60, 40, 20, 5) is None      # K = 1 - 1 = 0 < 1: no claim
    # the paper's operating point: vanishing bound at a=b=c=d=0.75, n=10^6
    q = exp_floor(10 ** 6, 15)
    assert lemma3_bound(10 ** 6, q, q, q, q) < 1e-100
    # sigma2/sigma1 enters K through the 2 s21 gamma / beta term
    # (K = 4 - 2 = 2, exponent -(60*2/40)(1/2)^2 = -3/4)
    assert math.isclose(lemma3_bound(50, 60, 40, 20, 20, s21=2.0), 5 * math.exp(-0.75), rel_tol=1e-12)


def test_panels_fix_the_other_exponents_at_three_quarters():
    n = 10 ** 6
    assert len(PANELS) == 6 and len({frozenset(p) for p in PANELS}) == 6
    q = exp_floor(n, 15)
    assert cell_params(n, ("a", "d"), 1, 19) == (1, q, q, exp_floor(n, 19))
    assert cell_params(n, ("b", "c"), 15, 15) == (q, q, q, q)
