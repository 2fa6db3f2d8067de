"""MQPT container: parsing, byte-exact writing, error taxonomy and device
loading, against containers written by the reference (tests/golden/*.mqpt,
tests/golden/make_golden.py section 6); modelled on test_checkpoint.py:29-140."""

import os
import shutil

import numpy as np
import pytest
import torch

from tests.conftest import GOLDEN

PARENT = os.path.join(GOLDEN, "parent.mqpt")
SLICED = os.path.join(GOLDEN, "sliced.mqpt")


@pytest.fixture(scope="module")
def ck():
    from paper_2602_03537_b200 import checkpoint

    return checkpoint


def test_parent_records_parse_zero_copy(ck, golden):
    g = golden("mqpt_cases")
    hd, recs = ck.read_records(PARENT)
    assert hd["master_bits"] == 8 and hd["group_size"] == 128
    assert [r.name for r in recs] == ["blk.0", "blk.1", "blk.2"]
    for i, rec in enumerate(recs):
        assert rec.kind == 0 and rec.bits == 8
        assert np.array_equal(rec.sections[0], g["codes_%d" % i])
        assert np.array_equal(rec.scales, g["scales_%d" % i])


def test_sliced_records_parse(ck, golden):
    g = golden("mqpt_cases")
    hd, recs = ck.read_records(SLICED)
    assert [r.bits for r in recs] == [2, 6, 4]
    assert [r.kind for r in recs] == [1, 0, 1]
    assert np.array_equal(recs[1].sections[0], g["child_codes_1"])
    for i in range(3):
        assert np.array_equal(recs[i].scales, g["child_scales_%d" % i])


@pytest.mark.parametrize("mutate,msg", [
    (lambda b: b"XQPT" + b[4:], "not a checkpoint"),
    (lambda b: b[:4] + b"\x02\x00" + b[6:], "unsupported version"),
    (lambda b: b[:-1], "corrupt checkpoint"),
    (lambda b: b + b"\x00", "corrupt checkpoint"),
    (lambda b: b[:2], "corrupt checkpoint"),
    (lambda b: b"", "corrupt checkpoint"),
])
def test_corruption_rejected(ck, tmp_path, mutate, msg):
    with open(PARENT, "rb") as fh:
        raw = fh.read()
    p = tmp_path / "bad.mqpt"
    p.write_bytes(mutate(raw))
    with pytest.raises(ck.CheckpointError, match=msg):
        ck.read_records(str(p))


def test_section_length_mismatch_rejected(ck, tmp_path):
    with open(PARENT, "rb") as fh:
        raw = bytearray(fh.read())
    # first layer's scale section length field sits right after name + dims
    hdr = 4 + 2 + 2 + 5 + 5 * 4 + 12
    off = hdr + 2 + len("blk.0") + 9
    raw[off] ^= 0x04
    p = tmp_path / "bad.mqpt"
    p.write_bytes(bytes(raw))
    with pytest.raises(ck.CheckpointError, match="corrupt checkpoint"):
        ck.read_records(str(p))


@pytest.mark.gpu
def test_roundtrip_byte_identical(ck, tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    for src in (PARENT, SLICED):
        model = ck.read_checkpoint(src)
        dst = tmp_path / os.path.basename(src)
        ck.write_checkpoint(model, str(dst))
        with open(src, "rb") as a, open(dst, "rb") as b:
            assert a.read() == b.read()


@pytest.mark.gpu
def test_load_planes_serves_every_slice(ck, golden):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import oracle as O

    g = golden("mqpt_cases")
    planes = ck.load_parent_planes(PARENT)
    for i in range(3):
        pt = planes["blk.%d" % i]
        for r in (2, 3, 4, 6, 8):
            assert np.array_equal(pt.slice_codes(r).cpu().numpy(), O.slice_codes(g["codes_%d" % i], 8, r))
    kids = ck.load_planes(SLICED)
    for i in range(3):
        r = int(g["child_bits_%d" % i])
        pt = kids["blk.%d" % i]
        assert pt.nplanes == r and pt.scales_are_effective
        assert np.array_equal(pt.slice_codes(r).cpu().numpy(), g["child_codes_%d" % i])
        want = O.dense_f32(g["child_codes_%d" % i], g["child_scales_%d" % i], 128, r)
        assert np.array_equal(pt.decode(r).cpu().numpy(), want)
    with pytest.raises(ck.CheckpointError, match="not a parent checkpoint"):
        ck.load_parent_planes(SLICED)


def test_read_checkpoint_parent_host_only(ck, golden, tmp_path):
    """A parent (raw-byte sections) parses to NestedLayers without a GPU."""
    g = golden("mqpt_cases")
    shutil.copy(PARENT, tmp_path / "p.mqpt")
    model = ck.read_checkpoint(str(tmp_path / "p.mqpt"))
    assert isinstance(model, ck.Checkpoint) and model.master_bits == 8
    assert model.layer_sizes() == {"blk.0": 24 * 256, "blk.1": 17 * 200, "blk.2": 8 * 1000}
    for i, ly in enumerate(model.layers):
        assert np.array_equal(ly.codes, g["codes_%d" % i])
        assert np.array_equal(ly.grid.scales, g["scales_%d" % i])
