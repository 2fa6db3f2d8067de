"""MQPT containers -> device-resident parents.

Drop-in for nestquant.checkpoint (checkpoint.py:1-201; layout in
pkg/docs/format.md): the same little-endian "MQPT" v1 container, the same
classes and the same error texts ("not a checkpoint", "unsupported version",
"corrupt checkpoint").  The host side only parses the record headers; code
sections are mapped zero-copy from the file and go to the GPU:

* int8 parents store one byte per code (section kind 0, checkpoint.py:66-75):
  the bytes are copied to HBM as they lie and K1 (mq_pack_blob) builds the
  P8 blob there -- ``load_parent_planes`` returns {name: PlaneTensor}, the
  resident parent every slice r is served from;
* sliced children with r <= 4 carry the reference's bit-plane sections
  (kind 1); they are unpacked on the device (mq_unpack_ref_layout) and
  packed into an r-plane child blob with effective scales.

``write_checkpoint`` reproduces the reference's bytes exactly (the tests
compare against containers the reference wrote).
"""

from __future__ import annotations

import mmap
import struct
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .device import PlaneTensor
from .grid import BitWidthSet, QuantGrid
from .packing import PACK_UNIT, PackedTensor, _padded_cols, pack, unpack_device
from .slicing import NestedLayer, SlicedLayer

MAGIC = b"MQPT"
VERSION = 1

__all__ = ["MAGIC", "VERSION", "CheckpointError", "Checkpoint", "SlicedModel", "write_checkpoint",
           "read_checkpoint", "read_records", "load_parent_planes", "load_planes"]


class CheckpointError(ValueError):
    pass


@dataclass
class Checkpoint:
    """A parent model: every layer at the master bit-width (checkpoint.py:33-53)."""

    bits: BitWidthSet
    group_size: int
    damp_rel: float
    layers: list[NestedLayer] = field(default_factory=list)

    @property
    def master_bits(self) -> int:
        return self.bits.master

    def layer_sizes(self) -> dict[str, int]:
        return {ly.name: ly.param_count for ly in self.layers}

    def layer(self, name: str) -> NestedLayer:
        for ly in self.layers:
            if ly.name == name:
                return ly
        raise KeyError(name)


@dataclass
class SlicedModel:
    """A deployable child with per-layer bit-widths (checkpoint.py:56-63)."""

    master_bits: int
    bits: BitWidthSet
    group_size: int
    damp_rel: float
    layers: list[SlicedLayer] = field(default_factory=list)


# ------------------------------------------------------------------ writer --
def _sections(codes: np.ndarray, lb: int) -> list[bytes]:
    if lb <= 4:
        p = pack(codes, lb)
        return [a.tobytes() for a in (p.base_plane, p.plane_b2, p.plane_b3) if a is not None]
    return [np.ascontiguousarray(codes, dtype=np.uint8).tobytes()]


def write_checkpoint(model, path) -> None:
    """Serialise a Checkpoint or SlicedModel (checkpoint.py:78-107, byte-identical)."""
    if isinstance(model, Checkpoint):
        lbs = [model.master_bits] * len(model.layers)
    else:
        lbs = [ly.bits for ly in model.layers]
    bws = model.bits
    head = [MAGIC, struct.pack("<HBB", VERSION, model.master_bits, len(bws.targets)),
            struct.pack("<%dB" % len(bws.targets), *bws.targets),
            struct.pack("<%df" % len(bws.weights), *bws.weights),
            struct.pack("<LfL", model.group_size, model.damp_rel, len(model.layers))]
    with open(path, "wb") as fh:
        fh.write(b"".join(head))
        for ly, lb in zip(model.layers, lbs):
            name = ly.name.encode("utf-8")
            d_row, d_col = ly.shape
            scales = ly.grid.scales if isinstance(ly, NestedLayer) else ly.scales
            sb = np.ascontiguousarray(scales, dtype=np.float32).tobytes()
            fh.write(struct.pack("<H", len(name)) + name + struct.pack("<LLB", d_row, d_col, lb))
            fh.write(struct.pack("<Q", len(sb)) + sb + struct.pack("<B", 1 if lb <= 4 else 0))
            for sec in _sections(ly.codes, lb):
                fh.write(struct.pack("<Q", len(sec)) + sec)


# ------------------------------------------------------------------ reader --
@dataclass
class Record:
    """One layer record; arrays are zero-copy views into the mapped file."""

    name: str
    bits: int
    shape: tuple[int, int]
    scales: np.ndarray
    kind: int
    sections: list[np.ndarray]


class _Cursor:
    def __init__(self, buf):
        self.buf, self.pos = buf, 0

    def take(self, n: int) -> memoryview:
        if n < 0 or self.pos + n > len(self.buf):
            raise CheckpointError("corrupt checkpoint")
        v = memoryview(self.buf)[self.pos:self.pos + n]
        self.pos += n
        return v

    def unpack(self, fmt: str):
        return struct.unpack(fmt, self.take(struct.calcsize(fmt)))

    def section(self, dtype, shape) -> np.ndarray:
        (length,) = self.unpack("<Q")
        if length != int(np.prod(shape)) * np.dtype(dtype).itemsize:
            raise CheckpointError("corrupt checkpoint")
        return np.frombuffer(self.take(length), dtype=dtype).reshape(shape)


def read_records(path):
    """Parse the container: (header dict, [Record]).  Validates exactly as
    read_checkpoint does (checkpoint.py:137-175)."""
    with open(path, "rb") as fh:
        try:
            buf = mmap.mmap(fh.fileno(), 0, access=mmap.ACCESS_READ)
        except ValueError:  # empty file
            buf = b""
    cur = _Cursor(buf)
    if bytes(cur.take(4)) != MAGIC:  # a shorter file is "corrupt", as in the reference
        raise CheckpointError("not a checkpoint")
    (version,) = cur.unpack("<H")
    if version != VERSION:
        raise CheckpointError("unsupported version")
    master, n_targets = cur.unpack("<BB")
    targets = cur.unpack("<%dB" % n_targets)
    lambdas = cur.unpack("<%df" % n_targets)
    group_size, damp_rel, n_layers = cur.unpack("<LfL")
    bws = BitWidthSet(tuple(targets), tuple(lambdas))
    if bws.master != master:
        raise CheckpointError("corrupt checkpoint")
    recs = []
    for _ in range(n_layers):
        (nl,) = cur.unpack("<H")
        name = bytes(cur.take(nl)).decode("utf-8")
        d_row, d_col, lb = cur.unpack("<LLB")
        scales = cur.section(np.float32, (d_row, -(-d_col // group_size)))
        (kind,) = cur.unpack("<B")
        if kind == 1:
            if lb > 4:
                raise CheckpointError("corrupt checkpoint")
            nu = _padded_cols(d_col) // PACK_UNIT
            secs = [cur.section(np.uint64, (d_row, nu))]
            if lb >= 3:
                secs.append(cur.section(np.uint32, (d_row, nu)))
            if lb == 4:
                secs.append(cur.section(np.uint32, (d_row, nu)))
        elif kind == 0:
            secs = [cur.section(np.uint8, (d_row, d_col))]
        else:
            raise CheckpointError("corrupt checkpoint")
        recs.append(Record(name, lb, (d_row, d_col), scales, kind, secs))
    if cur.pos != len(buf):
        raise CheckpointError("corrupt checkpoint")
    header = {"master_bits": master, "bits": bws, "group_size": group_size, "damp_rel": damp_rel}
    return header, recs


def _packed_of(rec: Record) -> PackedTensor:
    secs = rec.sections + [None] * (3 - len(rec.sections))
    return PackedTensor(bits=rec.bits, shape=rec.shape, base_plane=secs[0], plane_b2=secs[1],
                        plane_b3=secs[2])


def _codes_device(rec: Record) -> torch.Tensor:
    if rec.kind == 0:
        return torch.from_numpy(np.array(rec.sections[0], copy=True)).cuda(non_blocking=False)
    return unpack_device(_packed_of(rec))


def read_checkpoint(path):
    """MQPT file -> Checkpoint (all layers at the master width) or SlicedModel
    (checkpoint.py:137-201).  Codes come back as host arrays, as in the reference."""
    hd, recs = read_records(path)
    master, G = hd["master_bits"], hd["group_size"]
    rows = []
    for rec in recs:
        codes = np.array(rec.sections[0]) if rec.kind == 0 else _codes_device(rec).cpu().numpy()
        rows.append((rec, codes, np.array(rec.scales)))
    if all(rec.bits == master for rec, _, _ in rows):
        layers = [NestedLayer(name=rec.name, codes=codes, grid=QuantGrid(master, G, sc), bits=hd["bits"])
                  for rec, codes, sc in rows]
        return Checkpoint(bits=hd["bits"], group_size=G, damp_rel=hd["damp_rel"], layers=layers)
    layers = [SlicedLayer(name=rec.name, bits=rec.bits, codes=codes, scales=sc, group_size=G,
                          master_bits=master) for rec, codes, sc in rows]
    return SlicedModel(master_bits=master, bits=hd["bits"], group_size=G, damp_rel=hd["damp_rel"],
                       layers=layers)


def load_planes(path) -> dict[str, PlaneTensor]:
    """MQPT file -> {name: PlaneTensor} resident in HBM, no host-side decode.

    Master-width layers become parents (slice any r on the fly, mode P);
    sliced layers become r-plane children with their effective scales."""
    _lib.require_cuda()
    hd, recs = read_records(path)
    master, G = hd["master_bits"], hd["group_size"]
    out = {}
    for rec in recs:
        codes = _codes_device(rec)
        sc = torch.from_numpy(np.array(rec.scales)).cuda()
        if rec.bits == master:
            out[rec.name] = PlaneTensor.from_codes(codes, master, sc, G)
        else:
            out[rec.name] = PlaneTensor.from_codes(codes, rec.bits, sc, G, scales_are_effective=True)
    return out


def load_parent_planes(path) -> dict[str, PlaneTensor]:
    """Like load_planes, for a parent checkpoint (every layer at the master width)."""
    hd, recs = read_records(path)
    if any(rec.bits != hd["master_bits"] for rec in recs):
        raise CheckpointError("not a parent checkpoint")
    return load_planes(path)
