"""Device parity: libmatq (sm_100a) vs the CPU oracle (pinned to the reference).

Bars: sliced codes and dequantised weights bit-exact; layer
outputs max|got-want|/max|want| <= 1e-2 with bf16 output and <= 1e-4 with
fp32 output, X generated in bf16 (exact in both paths) so the error
measures only accumulation order and output rounding.
"""

import os

import numpy as np
import pytest
import torch

from oracle import oracle as O
from tests.conftest import rel_err, round_bf16

pytestmark = pytest.mark.gpu

LADDER = (2, 3, 4, 6, 8)


@pytest.fixture(scope="module")
def mq():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2602_03537_b200 as m

    return m


def _parent(n, k, g=128, seed=0, every_code=True):
    rng = np.random.default_rng(seed)
    codes = rng.integers(0, 256, size=(n, k)).astype(np.uint8)
    if every_code:
        flat = codes.reshape(-1)
        flat[: min(flat.size, 1024)] = np.arange(min(flat.size, 1024)) % 256
    ng = -(-k // g)
    scales = rng.uniform(0.005, 0.02, size=(n, ng)).astype(np.float32)
    return codes, scales


# ---------------------------------------------------------------- K1 / K2 --
@pytest.mark.parametrize("n,k", [(16, 256), (40, 600), (33, 1000), (128, 4096)])
def test_slice_codes_bit_exact(mq, n, k):
    codes, scales = _parent(n, k, seed=n + k)
    pt = mq.PlaneTensor.from_codes(codes, 8, scales, 128)
    for r in LADDER:
        got = pt.slice_codes(r).cpu().numpy()
        assert np.array_equal(got, O.slice_codes(codes, 8, r)), "r=%d" % r


def test_slice_exhaustive_all_codes_every_position(mq):
    # every code in every (row, col) residue of the 16x256 tile geometry
    n, k = 32, 512
    codes = ((np.arange(n)[:, None] * 37 + np.arange(k)[None, :]) % 256).astype(np.uint8)
    scales = np.full((n, k // 128), 0.01, np.float32)
    pt = mq.PlaneTensor.from_codes(codes, 8, scales, 128)
    for r in LADDER:
        assert np.array_equal(pt.slice_codes(r).cpu().numpy(), O.slice_codes(codes, 8, r))
        vals = pt.decode(r, values=True).cpu().numpy().astype(np.int64)
        assert np.array_equal(vals, O.slice_codes(codes, 8, r).astype(np.int64) - (1 << (r - 1)))


@pytest.mark.parametrize("n,k,g", [(40, 600, 128), (64, 512, 64), (48, 384, 32), (32, 768, 96)])
def test_dequant_bit_exact_vs_dense_f32(mq, n, k, g):
    codes, scales = _parent(n, k, g=g, seed=3)
    pt = mq.PlaneTensor.from_codes(codes, 8, scales, g)
    for r in LADDER:
        got = pt.decode(r).cpu().numpy()
        want = O.dense_f32(O.slice_codes(codes, 8, r), O.scale_eff(scales, 8, r), g, r)
        assert np.array_equal(got, want), "r=%d" % r


def test_child_materialization(mq):
    codes, scales = _parent(48, 768, seed=5)
    pt = mq.PlaneTensor.from_codes(codes, 8, scales, 128)
    for r in (2, 3, 4, 6):
        ch = pt.materialize_child(r)
        assert ch.blob.numel() * 4 == r * 48 * 768 // 8 + 48 * 768 // 128 * 4
        assert np.array_equal(ch.slice_codes(r).cpu().numpy(), O.slice_codes(codes, 8, r))
        assert np.array_equal(ch.decode(r).cpu().numpy(), pt.decode(r).cpu().numpy())


# -------------------------------------------------------------------- K3 --
def _x_bf16(b, k, seed):
    rng = np.random.default_rng(seed)
    return round_bf16(rng.standard_normal((b, k)).astype(np.float32))


@pytest.mark.parametrize("n,k", [(40, 600), (64, 1024), (256, 4096)])
@pytest.mark.parametrize("B", [1, 2, 7, 8, 9, 16, 17, 32])
def test_gemv_bf16_vs_oracle(mq, n, k, B):
    codes, scales = _parent(n, k, seed=n * 7 + k)
    pt = mq.PlaneTensor.from_codes(codes, 8, scales, 128)
    X = _x_bf16(B, k, seed=B)
    Xd = torch.from_numpy(X).cuda().to(torch.bfloat16)
    for r in LADDER:
        want = O.parent_matmul_ref(codes, scales, 128, r, X)
        y32 = pt.gemv(Xd, r, out_dtype=torch.float32).cpu().numpy()
        assert rel_err(y32, want) <= 1e-4, (r, rel_err(y32, want))
        y16 = pt.gemv(Xd, r).float().cpu().numpy()
        assert rel_err(y16, want) <= 1e-2, (r, rel_err(y16, want))


@pytest.mark.parametrize("g", [32, 64, 96, 256])
def test_gemv_generic_group_sizes(mq, g):
    n, k = 48, 1152
    codes, scales = _parent(n, k, g=g, seed=g)
    pt = mq.PlaneTensor.from_codes(codes, 8, scales, g)
    X = _x_bf16(3, k, seed=g)
    Xd = torch.from_numpy(X).cuda().to(torch.bfloat16)
    for r in LADDER:
        want = O.parent_matmul_ref(codes, scales, g, r, X)
        got = pt.gemv(Xd, r, out_dtype=torch.float32).cpu().numpy()
        assert rel_err(got, want) <= 1e-4, (g, r)


@pytest.mark.parametrize("B", [1, 5, 16])
def test_gemv_fp32_activations_split(mq, B):
    """fp32 X (the reference API's dtype) through the hi/lo bf16 split."""
    n, k = 64, 768
    codes, scales = _parent(n, k, seed=11)
    pt = mq.PlaneTensor.from_codes(codes, 8, scales, 128)
    X = np.random.default_rng(B).standard_normal((B, k)).astype(np.float32)
    for r in LADDER:
        want = O.parent_matmul_ref(codes, scales, 128, r, X)
        got = pt.gemv(torch.from_numpy(X).cuda(), r).cpu().numpy()
        assert rel_err(got, want) <= 1e-4, (r, rel_err(got, want))


def test_gemv_split_k_across_ctas_and_ticket_reset(mq):
    # few rows, long K: forces the cross-CTA split-K with the ticket reduction
    n, k = 64, 14336
    codes, scales = _parent(n, k, seed=21)
    pt = mq.PlaneTensor.from_codes(codes, 8, scales, 128)
    assert pt.workspace_bytes(1) > 0
    X = _x_bf16(4, k, seed=4)
    Xd = torch.from_numpy(X).cuda().to(torch.bfloat16)
    for r in (2, 4, 8):
        want = O.parent_matmul_ref(codes, scales, 128, r, X)
        for _ in range(3):  # tickets must reset between calls
            got = pt.gemv(Xd, r, out_dtype=torch.float32).cpu().numpy()
            assert rel_err(got, want) <= 1e-4


def test_shared_workspace_across_shapes_and_batches(mq):
    """One stream workspace serves interleaved GEMVs of different shapes,
    batches and split-K decompositions (regression: tickets must stay 0)."""
    layers = []
    for n, k in ((64, 14336), (4096, 14336), (48, 4096), (256, 8192)):
        codes, scales = _parent(n, k, seed=n + k)
        layers.append((codes, scales, mq.PlaneTensor.from_codes(codes, 8, scales, 128)))
    for rnd in range(2):
        for B in (1, 9, 32, 4):
            for codes, scales, pt in layers:
                X = _x_bf16(B, pt.K, seed=B + rnd)
                want = O.parent_matmul_ref(codes, scales, 128, 4, X)
                got = pt.gemv(torch.from_numpy(X).cuda().to(torch.bfloat16), 4,
                              out_dtype=torch.float32).cpu().numpy()
                assert rel_err(got, want) <= 1e-4, (pt.shape, B)


@pytest.mark.parametrize("split", ["3", "5"])
def test_gemv_forced_decompositions(mq, split, monkeypatch):
    """Chunked split-K forced via the tuning override (uneven chunks, tickets
    with several contributors), including configurations it cannot honour."""
    monkeypatch.setenv("MQ_GEMV_SPLIT", split)
    for n, k, B in ((40, 600, 1), (256, 4096, 5), (4096, 4096, 1), (2048, 14336, 3), (4000, 4352, 16)):
        codes, scales = _parent(n, k, seed=n + k + B)
        pt = mq.PlaneTensor.from_codes(codes, 8, scales, 128)
        mq.reserve_workspace(pt.workspace_bytes(B) * 4)
        X = _x_bf16(B, k, seed=B)
        Xd = torch.from_numpy(X).cuda().to(torch.bfloat16)
        for r in LADDER:
            want = O.parent_matmul_ref(codes, scales, 128, r, X)
            for _ in range(2):
                got = pt.gemv(Xd, r, out_dtype=torch.float32).cpu().numpy()
                assert rel_err(got, want) <= 1e-4, (split, n, k, B, r)


def test_gemv_mode_c_matches_mode_p(mq):
    codes, scales = _parent(128, 2048, seed=31)
    pt = mq.PlaneTensor.from_codes(codes, 8, scales, 128)
    Xd = torch.from_numpy(_x_bf16(8, 2048, 9)).cuda().to(torch.bfloat16)
    for r in (2, 3, 4, 6):
        yp = pt.gemv(Xd, r, out_dtype=torch.float32)
        yc = pt.materialize_child(r).gemv(Xd, r, out_dtype=torch.float32)
        assert torch.equal(yp, yc), r


def test_zero_code_rows_exactly_zero(mq):
    # reference test_matmul.py:61-66: rows of zero codes give exactly 0
    n, k = 32, 512
    for r in LADDER:
        codes = np.full((n, k), 128, np.uint8)  # 8-bit zero code slices to z_r for every r
        scales = np.full((n, k // 128), 0.01, np.float32)
        pt = mq.PlaneTensor.from_codes(codes, 8, scales, 128)
        X = torch.randn(5, k, device="cuda").to(torch.bfloat16)
        assert (pt.gemv(X, r, out_dtype=torch.float32) == 0).all()


def test_gemv_cuda_graph_and_pdl(mq):
    codes, scales = _parent(512, 4096, seed=41)
    pt = mq.PlaneTensor.from_codes(codes, 8, scales, 128)
    X = torch.from_numpy(_x_bf16(1, 4096, 1)).cuda().to(torch.bfloat16)
    ref = pt.gemv(X, 4).clone()
    out = torch.empty_like(ref)
    s = torch.cuda.Stream()
    mq.reserve_workspace(pt.workspace_bytes(1), stream=s)
    with torch.cuda.stream(s):
        pt.gemv(X, 4, out=out, pdl=True)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            pt.gemv(X, 4, out=out, pdl=True, stream=s)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


# ------------------------------------------------------- full-size checks --
@pytest.mark.parametrize("r", [8, 4, 2])
def test_c1_full_size(mq, r):
    """BASELINE config 1: 4096x4096, int8 parent, G=128, B=1, vs the oracle chain."""
    codes, scales = _parent(4096, 4096, seed=0)
    pt = mq.PlaneTensor.from_codes(codes, 8, scales, 128)
    X = _x_bf16(1, 4096, seed=0)
    want = O.parent_matmul_ref(codes, scales, 128, r, X)
    Xd = torch.from_numpy(X).cuda().to(torch.bfloat16)
    assert rel_err(pt.gemv(Xd, r).float().cpu().numpy(), want) <= 1e-2
    assert rel_err(pt.gemv(Xd, r, out_dtype=torch.float32).cpu().numpy(), want) <= 1e-4


def test_llama_shapes_properties(mq):
    """Full Llama-3.1-8B layer shapes: linearity and batch-row independence."""
    for (n, k) in ((6144, 4096), (28672, 4096), (4096, 14336)):
        pt = mq.PlaneTensor.random_parent(n, k, seed=n + k)
        g = torch.Generator(device="cuda").manual_seed(1)
        X1 = torch.randn(4, k, device="cuda", generator=g).to(torch.bfloat16)
        X2 = torch.randn(4, k, device="cuda", generator=g).to(torch.bfloat16)
        for r in LADDER:
            y1 = pt.gemv(X1, r, out_dtype=torch.float32)
            y2 = pt.gemv(X2, r, out_dtype=torch.float32)
            y12 = pt.gemv(torch.cat([X1, X2]), r, out_dtype=torch.float32)
            # batch rows are independent (a different batch may pick another
            # split-K decomposition, so compare to fp32 rounding, not bitwise)
            assert rel_err(y12[:4].cpu().numpy(), y1.cpu().numpy()) <= 1e-5
            assert rel_err(y12[4:].cpu().numpy(), y2.cpu().numpy()) <= 1e-5
            # linearity against an fp32 dense product of the decoded weights
            W = pt.decode(r)
            want = (X1.float() + X2.float()) @ W.T
            got = pt.gemv((X1.float() + X2.float()), r)
            assert rel_err(got.cpu().numpy(), want.cpu().numpy()) <= 1e-4


# --------------------------------------------- reference API (drop-in) ----
def test_golden_parent_chain_through_api(mq, golden):
    g = golden("parent_cases")
    for i in range(int(g["n_cases"])):
        n, k, G, B = (int(v) for v in g["meta_%d" % i])
        layer = mq.NestedLayer("p", g["codes_%d" % i], mq.QuantGrid(8, G, g["scales_%d" % i]),
                               mq.BitWidthSet((2, 3, 4, 6, 8), (1.0,) * 5))
        for r in LADDER:
            sl = mq.slice_layer(layer, r)
            assert np.array_equal(sl.codes, g["low_%d_r%d" % (i, r)])
            assert np.array_equal(sl.scales, g["seff_%d_r%d" % (i, r)])
            assert np.array_equal(mq.dequant(sl.codes, layer.grid, r), g["dq64_%d_r%d" % (i, r)])
            if r <= 4:
                pl = mq.PackedLayer.from_sliced(sl)
                assert np.array_equal(pl.dense_f32(), g["dense_%d_r%d" % (i, r)])
                task = mq.MatmulTask(X=g["X_%d" % i], layer=pl)
                assert np.array_equal(mq.matmul_ref(task), g["Y_%d_r%d" % (i, r)])
                assert rel_err(mq.matmul_packed(task), g["Y_%d_r%d" % (i, r)]) <= 1e-4
            pv = mq.PackedLayer.from_parent(layer, r)
            y = pv.device().gemv(torch.from_numpy(g["X_%d" % i]).cuda(), r).cpu().numpy()
            want = O.parent_matmul_ref(g["codes_%d" % i], g["scales_%d" % i], G, r, g["X_%d" % i])
            assert rel_err(y, want) <= 1e-4


def test_golden_random_tasks_through_api(mq, golden):
    g = golden("matmul_cases")
    for i in range(int(g["n_cases"])):
        bits, batch, m, k, group = (int(v) for v in g["meta_%d" % i])
        task = mq.random_task(m, k, batch, bits, group_size=group, seed=500 + i)
        assert np.array_equal(task.X, g["X_%d" % i])
        assert np.array_equal(mq.unpack(task.layer.packed), g["codes_%d" % i])
        assert np.array_equal(task.layer.dense_f32(), g["dense_%d" % i])
        assert np.array_equal(mq.matmul_ref(task), g["Y_%d" % i])
        for force in (False, True):
            assert rel_err(mq.matmul_packed(task, force_fallback=force), g["Y_%d" % i]) < 1e-4


def test_reference_known_answers_on_device(mq, golden):
    # test_slicing.py:18-31, test_packing.py:37-69, test_grid.py:85-93
    assert mq.slice_code(183, 8, 4) == 176 and mq.slice_code(255, 8, 2) == 192
    assert mq.slice_to_code(3, 3, 2) == 2 and mq.slice_to_code(183, 8, 4) == 11
    with pytest.raises(mq.SliceError):
        mq.slice_code(8, 3, 2)
    t = golden("slice_tables")
    for c in range(2, 9):
        q = np.arange(1 << c)
        for r in range(2, c + 1):
            assert np.array_equal(mq.slice_code(q, c, r), t["code_c%d_r%d" % (c, r)])
            low = mq.slice_to_code(q, c, r)
            assert np.array_equal(mq.dequant_value(low, 0.37, c, r), t["deq_c%d_r%d" % (c, r)])
    p = mq.pack(np.array([[5, 10]]), 4)
    assert p.base_plane[0, 0] == 0b1001 and p.plane_b2[0, 0] == 0b01 and p.plane_b3[0, 0] == 0b10
    assert list(mq.unpack(p)[0]) == [5, 10]
    assert mq.unpack(mq.pack_slice(mq.pack(np.array([[7]]), 4), 3))[0, 0] == 0b100
    with pytest.raises(mq.PackError, match="overflow"):
        mq.pack(np.array([[4]]), 2)
    assert mq.dequant_value(7, 1.0, 3, 3) == 3.0 and mq.dequant_value(3, 1.0, 3, 2) == 2.0
    with pytest.raises(mq.GridError):
        mq.dequant_value(4, 1.0, 3, 2)
    pc = golden("pack_cases")
    i = 0
    while "codes_%d" % i in pc:
        codes, bits = pc["codes_%d" % i], int(pc["bits_%d" % i])
        pk = mq.pack(codes, bits)
        assert np.array_equal(pk.base_plane, pc["base_%d" % i])
        assert np.array_equal(mq.unpack(mq.to_interleaved(pk)), codes)
        i += 1


def test_reference_matmul_suite_semantics(mq):
    """The reference's test_matmul.py cases, run against this backend."""
    task = mq.random_task(16, 32, 32, 4, group_size=32, seed=3)
    task.X[:] = np.eye(32, dtype=np.float32)
    assert rel_err(mq.matmul_packed(task), task.layer.dense_f32().T) < 1e-4
    for bits in (2, 3, 4):
        task = mq.random_task(16, 96, 3, bits, group_size=32, seed=bits)
        task.layer.packed = mq.pack(np.full((16, 96), 1 << (bits - 1)), bits)
        assert (mq.matmul_packed(task) == 0.0).all()
    for bits in (2, 3, 4, 6, 8):
        for batch in (1, 2, 7, 8, 9, 16, 33):
            task = mq.random_task(48, 160, batch, bits, group_size=32, seed=100 * bits + batch)
            assert rel_err(mq.matmul_packed(task), mq.matmul_ref(task)) < 1e-4
    task = mq.random_task(16, 40, 3, 4, group_size=32, seed=9)  # padding path
    assert rel_err(mq.matmul_packed(task), mq.matmul_ref(task)) < 1e-4
    with pytest.raises(mq.MatmulError, match="shape mismatch"):
        mq.MatmulTask(X=np.zeros((2, 39), np.float32), layer=task.layer)
    with pytest.raises(mq.MatmulError, match="unsupported bits"):
        mq.random_task(4, 32, 1, 5)
    recs = mq.bench(256, 512, 2, 4, reps=5)
    assert recs[0]["backend"] == "cuda-sm100" and len(recs[0]["samples_ns"]) == 5


# ------------------------------------------------------------ K4 (tcgen05) --
def _k4_weights(codes, scales, r, G=128):
    """The weights K4 multiplies: bf16(bf16(scale * 2^(8-r)) * (s_r - 2^(r-1))).

    Both roundings are single IEEE round-to-nearest-even steps of exact fp32
    values (a bf16 times an integer below 2^8 fits fp32 exactly), so this
    reproduces the device's mul.rn.bf16x2 bit for bit."""
    s = O.slice_codes(codes, 8, r).astype(np.float32) - float(1 << (r - 1))
    seff = round_bf16(scales.astype(np.float32) * np.float32(1 << (8 - r)))
    cols = np.arange(codes.shape[1]) // G
    return round_bf16(seff[:, cols] * s)


@pytest.mark.parametrize("n,k,B", [(128, 1024, 64), (200, 640, 100), (384, 2048, 300),
                                   (136, 4096, 33), (1024, 5120, 129), (256, 1024, 512),
                                   (136, 1536, 600)])
def test_gemm_vs_oracle(mq, n, k, B):
    """K4 against (a) an exact emulation of its bf16 weight rounding (only the
    fp32 accumulation order differs) and (b) the reference's dequantise-then-
    matmul oracle, within the stated bf16 tolerance."""
    codes, scales = _parent(n, k, seed=n + k + B)
    pt = mq.PlaneTensor.from_codes(codes, 8, scales, 128)
    X = _x_bf16(B, k, seed=B)
    Xd = torch.from_numpy(X).cuda().to(torch.bfloat16)
    for r in LADDER:
        got32 = pt.gemm(Xd, r, out_dtype=torch.float32).cpu().numpy()
        emu = X.astype(np.float64) @ _k4_weights(codes, scales, r).astype(np.float64).T
        assert rel_err(got32, emu) <= 2e-5, ("emulated", n, k, B, r)
        want = O.parent_matmul_ref(codes, scales, 128, r, X)
        assert rel_err(got32, want) <= 5e-3, ("oracle fp32 out", n, k, B, r)
        got16 = pt.gemm(Xd, r).float().cpu().numpy()
        assert rel_err(got16, want) <= 1e-2, ("oracle bf16 out", n, k, B, r)


def test_gemm_child_and_zero_rows(mq):
    codes, scales = _parent(256, 1024, seed=77)
    codes[5] = 128  # parent code 128 slices to the zero code at every r
    pt = mq.PlaneTensor.from_codes(codes, 8, scales, 128)
    X = torch.from_numpy(_x_bf16(96, 1024, seed=3)).cuda().to(torch.bfloat16)
    for r in (2, 3, 4, 6):
        yp = pt.gemm(X, r, out_dtype=torch.float32)
        yc = pt.materialize_child(r).gemm(X, r, out_dtype=torch.float32)
        assert torch.equal(yp, yc)
        assert (yp[:, 5] == 0).all()


def test_gemm_strided_io_graph_and_pdl(mq):
    codes, scales = _parent(512, 2048, seed=9)
    pt = mq.PlaneTensor.from_codes(codes, 8, scales, 128)
    big = torch.from_numpy(_x_bf16(80, 2304, seed=5)).cuda().to(torch.bfloat16)
    X = big[:, 128:128 + 2048]  # row stride 2304, 16-byte aligned
    ref = pt.gemm(X.contiguous(), 4).clone()
    outbuf = torch.zeros((80, 600), dtype=torch.bfloat16, device="cuda")
    out = outbuf[:, :512]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        pt.gemm(X, 4, out=out, pdl=True, stream=s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            pt.gemm(X, 4, out=out, pdl=True, stream=s)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    assert (outbuf[:, 512:] == 0).all()


def test_gemm_qwen_shapes_vs_fp32_torch(mq):
    """Qwen3-14B layer shapes (BASELINE config 4) at prefill batches: against
    an fp32 torch product of the exactly decoded weights (tf32 off)."""
    torch.backends.cuda.matmul.allow_tf32 = False
    for (n, k) in ((7168, 5120), (5120, 17408)):
        pt = mq.PlaneTensor.random_parent(n, k, seed=n)
        g = torch.Generator(device="cuda").manual_seed(2)
        for B in (64, 256, 512, 1024):
            X = torch.randn(B, k, device="cuda", generator=g).to(torch.bfloat16)
            for r in (4, 8):
                W = pt.decode(r)
                want = X.float() @ W.T
                got = pt.gemm(X, r, out_dtype=torch.float32)
                assert rel_err(got.cpu().numpy(), want.cpu().numpy()) <= 5e-3, (n, k, B, r)
                # batch rows are independent of the token tile they land in (a
                # different B may pick another K split: fp32 rounding only, ~1e-5 of
                # max |y| over K = 17408 when one side splits K 8 ways)
                half = pt.gemm(X[: B // 2].contiguous(), r, out_dtype=torch.float32)
                assert rel_err(half.cpu().numpy(), got[: B // 2].cpu().numpy()) <= 5e-5


def test_gemm_512_token_tiles(mq):
    """Past 256 tokens the planner may take 512-token tiles (one decoded weight tile feeds
    two N = 256 MMAs into a 512-column TMEM accumulator, two operand stages, each decoder
    warp owning one stage slot): Qwen3-14B o (5120 x 5120) at B = 384 / 512 / 600 picks
    them at every r (r = 8 with a single raw-weight stage).  Against fp32 torch on the exactly decoded weights,
    deterministic, and batch rows independent of the tiling the half batch gets."""
    torch.backends.cuda.matmul.allow_tf32 = False
    if torch.cuda.get_device_properties(0).multi_processor_count != 148:
        pytest.skip("the tiling choice assumes 148 SMs")
    n = k = 5120
    pt = mq.PlaneTensor.random_parent(n, k, seed=11)
    g = torch.Generator(device="cuda").manual_seed(12)
    for B in (384, 512, 600):
        X = torch.randn(B, k, device="cuda", generator=g).to(torch.bfloat16)
        for r in (2, 4, 6, 8):
            want = X.float() @ pt.decode(r).T
            got = pt.gemm(X, r, out_dtype=torch.float32)
            assert rel_err(got.cpu().numpy(), want.cpu().numpy()) <= 5e-3, (B, r)
            assert torch.equal(got, pt.gemm(X, r, out_dtype=torch.float32)), (B, r)
            half = pt.gemm(X[: B // 2].contiguous(), r, out_dtype=torch.float32)
            assert rel_err(half.cpu().numpy(), got[: B // 2].cpu().numpy()) <= 5e-5, (B, r)
            y16 = pt.gemm(X, r)
            assert rel_err(y16.float().cpu().numpy(), want.cpu().numpy()) <= 1e-2, (B, r)


_FORCED_512 = r"""
import sys, torch
sys.path.insert(0, %r)
import paper_2602_03537_b200 as mq
torch.backends.cuda.matmul.allow_tf32 = False
n, k = 40960, 1024  # 320 row tiles: up to 3 units of 512 tokens per CTA
pt = mq.PlaneTensor.random_parent(n, k, seed=3)
g = torch.Generator(device="cuda").manual_seed(4)
for B, r in ((512, 4), (700, 2), (1024, 8)):
    X = torch.randn(B, k, device="cuda", generator=g).to(torch.bfloat16)
    want = X.float() @ pt.decode(r).T
    got = pt.gemm(X, r, out_dtype=torch.float32)
    err = float((got - want).abs().max() / want.abs().max())
    assert err <= 5e-3, (B, r, err)
    assert torch.equal(got, pt.gemm(X, r, out_dtype=torch.float32)), (B, r)
print("ok")
"""


def test_gemm_512_token_tiles_forced_multi_unit():
    """MQ_GEMM_BN512=2 forces 512-token tiles past B = 256; on a 40960-row layer each CTA
    runs several units in turn through the single-buffered 512-column TMEM accumulator
    (the planner alone never picks that).  Subprocess: the knob is read once per process."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MQ_GEMM_BN512="2")
    res = subprocess.run([sys.executable, "-c", _FORCED_512 % root], env=env, capture_output=True,
                         text=True, timeout=600)
    assert res.returncode == 0 and res.stdout.strip().endswith("ok"), res.stderr[-2000:]


def test_gemm_whole_waves_then_split_tail(mq):
    """More tiles than SMs with a small remainder (19 row tiles x 8 token tiles = 152 on
    148 SMs): one wave of whole tiles, then the 4 leftover tiles split over the last
    wave.  Against fp32 torch on the exactly decoded weights, row-independent of the
    path (the first half of the batch takes a whole-tile config), deterministic."""
    torch.backends.cuda.matmul.allow_tf32 = False
    n, k, B = 2432, 2048, 2048
    if torch.cuda.get_device_properties(0).multi_processor_count != 148:
        pytest.skip("the tile arithmetic assumes 148 SMs")
    assert mq.device.gemm_workspace_bytes(n, k, B) > 0  # a split tail (whole tiles alone need none)
    pt = mq.PlaneTensor.random_parent(n, k, seed=5)
    g = torch.Generator(device="cuda").manual_seed(8)
    X = torch.randn(B, k, device="cuda", generator=g).to(torch.bfloat16)
    for r in (2, 4, 8):
        want = X.float() @ pt.decode(r).T
        got = pt.gemm(X, r, out_dtype=torch.float32)
        assert rel_err(got.cpu().numpy(), want.cpu().numpy()) <= 5e-3, r
        assert torch.equal(got, pt.gemm(X, r, out_dtype=torch.float32))
        half = pt.gemm(X[: B // 2].contiguous(), r, out_dtype=torch.float32)
        assert rel_err(half.cpu().numpy(), got[: B // 2].cpu().numpy()) <= 1e-5


def test_linear_dispatch(mq):
    codes, scales = _parent(256, 1024, seed=12)
    pt = mq.PlaneTensor.from_codes(codes, 8, scales, 128)
    X = torch.from_numpy(_x_bf16(48, 1024, seed=2)).cuda()
    y_gemm = pt.linear(X.to(torch.bfloat16), 4, out_dtype=torch.float32)
    assert torch.equal(y_gemm, pt.gemm(X.to(torch.bfloat16), 4, out_dtype=torch.float32))
    y32 = pt.linear(X, 4)  # fp32 activations: chunked K3, reference API accuracy
    want = O.parent_matmul_ref(codes, scales, 128, 4, X.cpu().numpy())
    assert rel_err(y32.cpu().numpy(), want) <= 1e-4


def test_gemm_split_k_deterministic_and_ticket_reset(mq):
    """Few output tiles + long K: the K4 config splits K across CTAs; the
    in-order reduction is deterministic and leaves the tickets at zero."""
    codes, scales = _parent(256, 8192, seed=21)
    pt = mq.PlaneTensor.from_codes(codes, 8, scales, 128)
    assert mq.device.gemm_workspace_bytes(256, 8192, 40) > 0
    X = _x_bf16(40, 8192, seed=4)
    Xd = torch.from_numpy(X).cuda().to(torch.bfloat16)
    for r in (2, 4, 8):
        a = pt.gemm(Xd, r, out_dtype=torch.float32)
        b = pt.gemm(Xd, r, out_dtype=torch.float32)
        assert torch.equal(a, b)
        emu = X.astype(np.float64) @ _k4_weights(codes, scales, r).astype(np.float64).T
        assert rel_err(a.cpu().numpy(), emu) <= 2e-5
    # the shared workspace serves a K3 split-K GEMV afterwards (tickets at zero)
    y = pt.gemv(Xd[:1], 4, out_dtype=torch.float32).cpu().numpy()
    assert rel_err(y, O.parent_matmul_ref(codes, scales, 128, 4, X[:1])) <= 1e-4


def test_matlinear_module(mq):
    """The torch module: decode and prefill batches, leading dims, bits switch
    without touching the weights, bias, fp32 input through the reference-API path."""
    codes, scales = _parent(320, 1024, seed=55)
    lin = mq.MatLinear.from_codes(codes, scales, 128, bits=4)
    x = torch.from_numpy(_x_bf16(2 * 3, 1024, seed=9)).cuda().to(torch.bfloat16).reshape(2, 3, 1024)
    for r in LADDER:
        lin.set_bits(r)
        y = lin(x)
        assert y.shape == (2, 3, 320) and y.dtype == torch.bfloat16
        want = O.parent_matmul_ref(codes, scales, 128, r, x.reshape(6, 1024).float().cpu().numpy())
        assert rel_err(y.reshape(6, 320).float().cpu().numpy(), want) <= 1e-2
    xp = torch.from_numpy(_x_bf16(100, 1024, seed=10)).cuda().to(torch.bfloat16)  # prefill -> K4
    lin.set_bits(8)
    want = O.parent_matmul_ref(codes, scales, 128, 8, xp.float().cpu().numpy())
    assert rel_err(lin(xp).float().cpu().numpy(), want) <= 1e-2
    bias = torch.randn(320, device="cuda")
    lb = mq.MatLinear(lin.planes, 8, bias=bias)
    want_b = lin(xp[:4]).float() + bias
    assert rel_err(lb(xp[:4]).float().cpu().numpy(), want_b.cpu().numpy()) <= 1e-2
    x32 = torch.from_numpy(_x_bf16(4, 1024, seed=11)).cuda()
    want = O.parent_matmul_ref(codes, scales, 128, 8, x32.cpu().numpy())
    assert rel_err(lin(x32).cpu().numpy(), want) <= 1e-4
    with pytest.raises(ValueError):
        lin.set_bits(5)
