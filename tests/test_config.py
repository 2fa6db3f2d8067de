"""Heterogeneous bit-width configs (BASELINE config C3): the EvoPress-style
budget-exact moves reproduce the reference's own config for the same seed
(tests/golden/llama31_8b_3p5bit_seed0.json, made by the reference's
_uniform_completed + mutate_level_switch, evo.py:147-172, :53-96)."""

import json
import os

import numpy as np
import pytest

from tests.conftest import GOLDEN


@pytest.fixture(scope="module")
def cfgmod():
    from paper_2602_03537_b200 import config

    return config


def test_reproduces_reference_config(cfgmod):
    with open(os.path.join(GOLDEN, "llama31_8b_3p5bit_seed0.json")) as fh:
        want = json.load(fh)
    cfg = cfgmod.budget_config(3.5, seed=0, mutations=200)
    assert cfg.budget_bits == want["budget_bits"]
    assert cfg.assignment == want["assignment"]
    sizes = cfgmod.unfused_layer_sizes()
    assert cfg.total_bits(sizes) == want["budget_bits"]
    assert len(cfg.assignment) == 224
    assert set(cfgmod.level_histogram(cfg)) <= {2, 3, 4, 6, 8}


def test_mutation_preserves_budget_and_stagnates(cfgmod):
    from paper_2602_03537_b200.slicing import BitConfig

    sizes = {"a": 10, "b": 10, "c": 30}
    rng = np.random.default_rng(3)
    cfg = cfgmod.uniform_completed(4 * 50, sizes, (2, 3, 4, 6, 8), rng)
    for _ in range(50):
        cfg, _ = cfgmod.mutate_level_switch(cfg, sizes, rng)
        assert cfg.total_bits(sizes) == 200
    low = BitConfig({"a": 2, "b": 2}, budget_bits=40)
    out, stagnant = cfgmod.mutate_level_switch(low, {"a": 10, "b": 10}, rng)
    assert stagnant and out is low


def test_errors(cfgmod):
    rng = np.random.default_rng(0)
    with pytest.raises(cfgmod.ConfigError, match="infeasible budget"):
        cfgmod.uniform_completed(10, {"a": 10}, (2, 4), rng)
    with pytest.raises(cfgmod.ConfigError, match="infeasible budget"):
        cfgmod.budget_config(9.0)
