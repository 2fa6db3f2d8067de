"""Pin the CPU oracle to the reference (golden vectors + known answers).

These run without a GPU.  The golden .npz files were produced by importing
the reference itself (tests/golden/make_golden.py); the known answers are
the reference's own test constants (cited per test).
"""

import numpy as np
import pytest

from oracle import oracle as O


class TestSliceKnownAnswers:
    def test_direct_values(self):
        # reference tests/test_slicing.py:18-19
        assert O.slice_codes([183], 8, 4, on_master=True)[0] == 176
        assert O.slice_codes([255], 8, 2, on_master=True)[0] == 192

    def test_push_and_to_code(self):
        # test_slicing.py:28, :31
        assert O.slice_codes([3], 3, 2)[0] == 2
        assert O.slice_codes([183], 8, 4)[0] == 11

    def test_identity_and_zero(self):
        # test_slicing.py:21-24, :32-34
        for c in range(2, 9):
            q = np.arange(1 << c)
            assert np.array_equal(O.slice_codes(q, c, c), q)
            for r in range(2, c + 1):
                assert O.slice_codes([0], c, r)[0] == 0

    def test_errors(self):
        # test_slicing.py:36-42
        with pytest.raises(O.OracleError):
            O.slice_codes([0], 3, 4)
        with pytest.raises(O.OracleError):
            O.slice_codes([8], 3, 2)


def test_slice_tables_exhaustive(golden):
    t = golden("slice_tables")
    for c in range(2, 9):
        q = np.arange(1 << c)
        for r in range(2, c + 1):
            assert np.array_equal(O.slice_codes(q, c, r, True), t["code_c%d_r%d" % (c, r)])
            low = O.slice_codes(q, c, r)
            assert np.array_equal(low, t["low_c%d_r%d" % (c, r)])
            deq = O.dequant_f64(low[None, :], np.full((1, 1), 0.37, np.float32),
                                low.size, c, r)[0]
            # reference dequant_value uses the float64 scale 0.37, the oracle the
            # float32 grid scale (grid.py:82): compare the integer multipliers
            mult = deq / np.float64(np.float32(0.37))
            want = t["deq_c%d_r%d" % (c, r)] / 0.37
            assert np.allclose(mult, want, rtol=0, atol=1e-9)


def test_slice_decomposition_identity():
    # SURVEY 0, finding 1: s_r(q) == min(top_r(q) + bit_{k-1}(q), 2^r - 1).
    # This is the identity the bitsliced device slice relies on.
    q = np.arange(256)
    for r in (2, 3, 4, 6, 8):
        k = 8 - r
        top = q >> k
        rb = (q >> (k - 1)) & 1 if k > 0 else 0
        alt = np.minimum(top + rb, (1 << r) - 1)
        assert np.array_equal(O.slice_codes(q, 8, r), alt)


def test_dequant_known_answers():
    # reference tests/test_grid.py:85-93
    one = np.ones((1, 1), np.float32)
    assert O.dequant_f64(np.array([[4]]), np.full((1, 1), 0.7, np.float32), 1, 3, 3)[0, 0] == 0.0
    assert O.dequant_f64(np.array([[7]]), one, 1, 3, 3)[0, 0] == 3.0
    assert O.dequant_f64(np.array([[3]]), one, 1, 3, 2)[0, 0] == 2.0
    with pytest.raises(O.OracleError):
        O.dequant_f64(np.array([[4]]), one, 1, 3, 2)


def test_pack_known_answers():
    # reference tests/test_packing.py:37-41, :56-69
    base, b2, b3 = O.pack_child(np.array([[5, 10]]), 4)
    assert base[0, 0] == 0b1001 and b2[0, 0] == 0b01 and b3[0, 0] == 0b10
    for bits in (2, 3, 4):
        base, b2, b3 = O.pack_child(np.full((2, 32), (1 << bits) - 1), bits)
        assert (base == np.uint64(0xFFFFFFFFFFFFFFFF)).all()
    base, b2, b3 = O.pack_child(np.full((1, 33), 15), 4)
    assert base[0, 1] == 0b11 and b2[0, 1] == 0b1
    with pytest.raises(O.OracleError):
        O.pack_child(np.array([[4]]), 2)


def test_pack_golden(golden):
    g = golden("pack_cases")
    i = 0
    while "codes_%d" % i in g:
        codes = g["codes_%d" % i]
        bits = int(g["bits_%d" % i])
        base, b2, b3 = O.pack_child(codes, bits)
        assert np.array_equal(base, g["base_%d" % i])
        if bits >= 3:
            assert np.array_equal(b2, g["b2_%d" % i])
        if bits == 4:
            assert np.array_equal(b3, g["b3_%d" % i])
            for r in (2, 3):
                # pack_slice == pack(slice(unpack)) (packing.py:129-141)
                assert np.array_equal(O.slice_codes(codes, 4, r), g["slice%d_%d" % (r, i)])
        assert np.array_equal(O.unpack_child(base, b2, b3, codes.shape[1]), codes)
        i += 1
    assert i >= 5


def test_matmul_golden_bit_exact(golden):
    g = golden("matmul_cases")
    for i in range(int(g["n_cases"])):
        bits, batch, m, k, group = (int(v) for v in g["meta_%d" % i])
        codes = g["codes_%d" % i]
        W = O.dense_f32(codes, g["scales_%d" % i], group, bits)
        assert np.array_equal(W, g["dense_%d" % i])
        Y = O.matmul_ref(g["X_%d" % i], W)
        assert np.array_equal(Y, g["Y_%d" % i]), "matmul_ref case %d not bit-exact" % i


def test_parent_chain_golden(golden):
    g = golden("parent_cases")
    for i in range(int(g["n_cases"])):
        n, k, G, B = (int(v) for v in g["meta_%d" % i])
        codes, scales, X = g["codes_%d" % i], g["scales_%d" % i], g["X_%d" % i]
        for r in (2, 3, 4, 6, 8):
            low = O.slice_codes(codes, 8, r)
            assert np.array_equal(low, g["low_%d_r%d" % (i, r)])
            seff = O.scale_eff(scales, 8, r)
            assert np.array_equal(seff, g["seff_%d_r%d" % (i, r)])
            assert np.array_equal(O.dequant_f64(low, scales, G, 8, r), g["dq64_%d_r%d" % (i, r)])
            if r <= 4:
                W = O.dense_f32(low, seff, G, r)
                assert np.array_equal(W, g["dense_%d_r%d" % (i, r)])
                Y = O.parent_matmul_ref(codes, scales, G, r, X)
                assert np.array_equal(Y, g["Y_%d_r%d" % (i, r)])


def test_reference_kernel_agrees_with_oracle(golden):
    """The reference's own compiled C kernel (oracle/_ref) vs the oracle."""
    try:
        ref = O.RefKernels()
    except FileNotFoundError:
        pytest.skip("oracle/_ref not built")
    g = golden("matmul_cases")
    for i in range(int(g["n_cases"])):
        bits, batch, m, k, group = (int(v) for v in g["meta_%d" % i])
        codes = g["codes_%d" % i]
        base, b2, b3 = O.pack_child(codes, bits)
        Xp = np.zeros((batch, base.shape[1] * 32), np.float32)
        Xp[:, :k] = g["X_%d" % i]
        got = ref.packed_matmul(base, b2, b3, np.ascontiguousarray(g["scales_%d" % i]), Xp, bits,
                                group)
        want = g["Y_%d" % i]
        assert np.abs(got - want).max() / (np.abs(want).max() + 1e-30) < 1e-4
