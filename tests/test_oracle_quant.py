"""Pin the quantiser oracle (oracle/quant_oracle.py) to the reference: the
golden vectors tests/golden/make_golden_quant.py produced by importing the
reference's select_codes / fit_grid / quantize_layer, bit for bit; plus the
reference's own known answers (tests/test_gptq.py, tests/test_grid.py)."""

import numpy as np
import pytest

from oracle import quant_oracle as Q

GOLD = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "quant_cases.npz"))


@pytest.mark.parametrize("i", range(int(GOLD["sel_n"])))
def test_select_codes_golden(i):
    g = lambda k: GOLD["sel%d_%s" % (i, k)]  # noqa: E731
    got = Q.select_codes(g("W"), g("scales"), int(g("G")), g("targets"), g("weights"))
    assert np.array_equal(got, g("codes"))


@pytest.mark.parametrize("i", range(int(GOLD["fit_n"])))
def test_fit_grid_golden(i):
    g = lambda k: GOLD["fit%d_%s" % (i, k)]  # noqa: E731
    got = Q.fit_grid(g("W"), g("targets"), g("weights"), int(g("G")), float(g("shrink")), int(g("steps")))
    assert got.dtype == np.float32 and np.array_equal(got, g("scales"))


@pytest.mark.parametrize("i", range(int(GOLD["gq_n"])))
def test_quantize_layer_golden(i):
    g = lambda k: GOLD["gq%d_%s" % (i, k)]  # noqa: E731
    codes, comp = Q.quantize_layer(g("W"), g("chol"), g("scales"), int(g("G")), g("targets"), g("weights"),
                                   int(g("bs")))
    assert np.array_equal(codes, g("codes"))
    assert np.array_equal(comp, g("comp"))


def test_low_bit_weight_flips_choice():
    # reference tests/test_gptq.py:113-119
    sc = np.ones((1, 1), np.float32)
    assert Q.select_codes([[0.9]], sc, 1, (2, 3), (1.0, 1.0))[0, 0] == 5
    assert Q.select_codes([[0.9]], sc, 1, (2, 3), (10.0, 1.0))[0, 0] == 4


def test_fit_grid_known_answers():
    # reference tests/test_grid.py:129-138
    assert (Q.fit_grid(np.zeros((2, 8)), (4,), (1.0,), 8) == np.float32(1e-12)).all()
    assert Q.fit_grid(np.array([[-1.0, 1.0]]), (4,), (1.0,), 2, steps=1)[0, 0] == np.float32(1.0 / 7.0)


def test_master_values_match_slice_tables():
    tabs = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "slice_tables.npz"))
    for c in range(2, 9):
        for r in range(2, c + 1):
            assert np.array_equal(Q.master_values(c, r), tabs["code_c%d_r%d" % (c, r)] - (1 << (c - 1)))
