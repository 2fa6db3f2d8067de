"""Generate golden vectors by importing the reference itself.

Run in the build container (the only place /root/reference exists):

    NESTQUANT_NO_EXT=1 python tests/golden/make_golden.py

It imports the unmodified reference package read-only from
/root/reference/pkg/src (numpy backend; matmul_ref, slicing, grid and
packing are pure numpy in the reference anyway) and writes small .npz
fixtures next to this script.  The fixtures are committed; nothing on the
GPU box reads /root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    os.environ.setdefault("NESTQUANT_NO_EXT", "1")
    sys.path.insert(0, REF_SRC)
    from nestquant.grid import BitWidthSet, QuantGrid, dequant, dequant_value
    from nestquant.matmul import PackedLayer, matmul_ref, random_task
    from nestquant.packing import pack, pack_slice, unpack
    from nestquant.slicing import NestedLayer, slice_code, slice_layer, slice_to_code

    # 1. exhaustive slice tables, every (c, r) (test_slicing.py:44-55)
    tables = {}
    for c in range(2, 9):
        q = np.arange(1 << c)
        for r in range(2, c + 1):
            tables["code_c%d_r%d" % (c, r)] = np.asarray(slice_code(q, c, r), dtype=np.int64)
            low = np.asarray(slice_to_code(q, c, r), dtype=np.int64)
            tables["low_c%d_r%d" % (c, r)] = low
            tables["deq_c%d_r%d" % (c, r)] = np.asarray(dequant_value(low, 0.37, c, r))
    np.savez_compressed(os.path.join(HERE, "slice_tables.npz"), **tables)

    # 2. pack layouts (test_packing.py:37-69 shapes, plus ragged ones)
    rng = np.random.default_rng(1234)
    packs = {}
    for i, (bits, n, k) in enumerate([(2, 3, 32), (3, 5, 70), (4, 5, 70), (4, 1, 33),
                                       (2, 7, 1), (3, 2, 127), (4, 9, 96)]):
        codes = rng.integers(0, 1 << bits, size=(n, k))
        p = pack(codes, bits)
        packs["codes_%d" % i] = codes.astype(np.uint8)
        packs["bits_%d" % i] = np.int64(bits)
        packs["base_%d" % i] = p.base_plane
        if p.plane_b2 is not None:
            packs["b2_%d" % i] = p.plane_b2
        if p.plane_b3 is not None:
            packs["b3_%d" % i] = p.plane_b3
        if bits == 4:
            for r in (2, 3):
                ps = pack_slice(p, r)
                packs["slice%d_%d" % (r, i)] = unpack(ps)
    np.savez_compressed(os.path.join(HERE, "pack_cases.npz"), **packs)

    # 3. matmul_ref on the reference's own random_task (test_acceptance.py:219-237
    #    style seeds), r in {2, 3, 4}
    mm = {}
    cases = []
    for i in range(12):
        seed = 500 + i
        r = np.random.default_rng(seed)
        bits = (2, 3, 4)[i % 3]
        batch = 1 + i % 16
        m = int(r.integers(16, 97))
        k = int(r.choice([32, 64, 96, 160, 256]))
        group = int(r.choice([32, 64, 128]))
        task = random_task(m, k, batch, bits, group_size=group, seed=seed)
        mm["X_%d" % i] = task.X
        mm["codes_%d" % i] = unpack(task.layer.packed)
        mm["scales_%d" % i] = task.layer.scales
        mm["dense_%d" % i] = task.layer.dense_f32()
        mm["Y_%d" % i] = matmul_ref(task)
        mm["meta_%d" % i] = np.array([bits, batch, m, k, group], dtype=np.int64)
        cases.append(i)
    mm["n_cases"] = np.int64(len(cases))
    np.savez_compressed(os.path.join(HERE, "matmul_cases.npz"), **mm)

    # 4. int8 parent layers with an edge block holding all 256 codes; every
    #    r on the ladder through slice_layer; r<=4 through PackedLayer +
    #    matmul_ref (the reference's own chain), X rounded to bf16 values.
    par = {}
    for i, (n, k, G, B) in enumerate([(48, 512, 128, 1), (40, 256, 64, 3), (16, 384, 128, 16)]):
        rng = np.random.default_rng(77 + i)
        codes = rng.integers(0, 256, size=(n, k), dtype=np.int64)
        codes[:2, :256] = np.arange(256)[None, :]  # edge block: every code
        codes = codes.astype(np.uint8)
        ng = -(-k // G)
        scales = rng.uniform(0.005, 0.02, size=(n, ng)).astype(np.float32)
        bits = BitWidthSet((2, 3, 4, 6, 8), (1.0,) * 5)
        layer = NestedLayer(name="p%d" % i, codes=codes, grid=QuantGrid(8, G, scales), bits=bits)
        X = rng.standard_normal((B, k)).astype(np.float32)
        X = _round_bf16(X)
        par["codes_%d" % i] = codes
        par["scales_%d" % i] = scales
        par["X_%d" % i] = X
        par["meta_%d" % i] = np.array([n, k, G, B], dtype=np.int64)
        for r in (2, 3, 4, 6, 8):
            sl = slice_layer(layer, r)
            par["low_%d_r%d" % (i, r)] = sl.codes
            par["seff_%d_r%d" % (i, r)] = sl.scales
            par["dq64_%d_r%d" % (i, r)] = dequant(sl.codes, layer.grid, r)
            if r <= 4:
                pl = PackedLayer.from_sliced(sl)
                from nestquant.matmul import MatmulTask

                par["dense_%d_r%d" % (i, r)] = pl.dense_f32()
                par["Y_%d_r%d" % (i, r)] = matmul_ref(MatmulTask(X=X, layer=pl))
    par["n_cases"] = np.int64(3)
    np.savez_compressed(os.path.join(HERE, "parent_cases.npz"), **par)

    # 5. EvoPress-style heterogeneous config over the 224 unfused Llama-3.1-8B
    #    linears: the reference's own budget-exact completion + 200 level
    #    switches (evo.py:147-172, :53-96), seed 0, budget 3.5 bits (evo.py:186).
    import json

    from nestquant.evo import _uniform_completed, mutate_level_switch

    dims = {"q": (4096, 4096), "k": (1024, 4096), "v": (1024, 4096), "o": (4096, 4096),
            "gate": (14336, 4096), "up": (14336, 4096), "down": (4096, 14336)}
    sizes = {"layers.%d.%s" % (i, k): dims[k][0] * dims[k][1]
             for i in range(32) for k in ("q", "k", "v", "o", "gate", "up", "down")}
    budget = int(round(3.5 * sum(sizes.values())))
    rng = np.random.default_rng(0)
    cfg = _uniform_completed(budget, sizes, (2, 3, 4, 6, 8), rng)
    for _ in range(200):
        cfg, _ = mutate_level_switch(cfg, sizes, rng)
    with open(os.path.join(HERE, "llama31_8b_3p5bit_seed0.json"), "w") as fh:
        json.dump({"budget_bits": budget, "assignment": cfg.assignment}, fh, indent=0, sort_keys=True)

    # 6. MQPT containers written by the reference (checkpoint.py:78-107): an
    #    int8 parent (raw-byte code sections) and a sliced model with per-layer
    #    bit-widths (bit-plane packed sections for r <= 4).
    from nestquant.checkpoint import Checkpoint, SlicedModel, write_checkpoint

    rng = np.random.default_rng(99)
    bws = BitWidthSet((2, 3, 4, 6, 8), (1.0, 0.5, 0.25, 0.125, 0.0625))
    layers, ck = [], {}
    for i, (n, k, G) in enumerate([(24, 256, 128), (17, 200, 128), (8, 1000, 128)]):
        G = 128
        codes = rng.integers(0, 256, size=(n, k)).astype(np.uint8)
        scales = rng.uniform(0.005, 0.02, size=(n, -(-k // G))).astype(np.float32)
        layers.append(NestedLayer(name="blk.%d" % i, codes=codes, grid=QuantGrid(8, G, scales), bits=bws))
        ck["codes_%d" % i] = codes
        ck["scales_%d" % i] = scales
    parent = Checkpoint(bits=bws, group_size=128, damp_rel=0.01, layers=layers)
    write_checkpoint(parent, os.path.join(HERE, "parent.mqpt"))
    sl = [slice_layer(ly, r) for ly, r in zip(layers, (2, 6, 4))]
    for i, s_ in enumerate(sl):
        ck["child_codes_%d" % i] = s_.codes
        ck["child_scales_%d" % i] = s_.scales
        ck["child_bits_%d" % i] = np.int64(s_.bits)
    child = SlicedModel(master_bits=8, bits=bws, group_size=128, damp_rel=0.01, layers=sl)
    write_checkpoint(child, os.path.join(HERE, "sliced.mqpt"))
    np.savez_compressed(os.path.join(HERE, "mqpt_cases.npz"), **ck)
    print("golden fixtures written to", HERE)


def _round_bf16(x: np.ndarray) -> np.ndarray:
    """Round float32 to the nearest bfloat16 value (ties to even), as float32."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


if __name__ == "__main__":
    main()
