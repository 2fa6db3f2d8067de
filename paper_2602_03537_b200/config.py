"""Per-layer bit-width configurations for heterogeneous slicing (BASELINE config C3).

The reference searches {layer: r} assignments offline with an EvoPress-style
(1+lambda) search (evo.py:175-229) whose moves keep the model's total
parameter-bits exactly on budget.  The search loop (fitness = KL on a toy
model) is out of scope here; what the inference path needs is a budget-exact
heterogeneous config for real model shapes, generated with the reference's
own budget-preserving moves so that the resulting dispatch table has the
reference's statistics:

* ``uniform_completed`` -- the highest uniform level under budget, topped up
  by random single-layer raises until the budget is met exactly
  (evo.py:147-172);
* ``mutate_level_switch`` -- lower one random layer by a random number of
  levels, then spend the freed parameter-bits on random raises until none
  is left (evo.py:53-96).

Both consume ``numpy.random.Generator`` draws in the reference's order, so
a seed reproduces the reference's config exactly
(tests/test_config.py checks against a fixture made by the reference).
"""

from __future__ import annotations

import numpy as np

from .model import DecoderShape, LLAMA31_8B
from .slicing import BitConfig

__all__ = ["ConfigError", "uniform_completed", "mutate_level_switch", "budget_config",
           "unfused_layer_sizes", "level_histogram"]

UNFUSED = ("q", "k", "v", "o", "gate", "up", "down")


class ConfigError(ValueError):
    pass


def _raises(work: dict, names: list, sizes: dict, ladder: tuple, room: int, skip=None) -> list:
    """Every (layer, level) raise whose parameter-bit cost fits in ``room``."""
    out = []
    for n in names:
        if n == skip:
            continue
        cur = work[n]
        for lvl in ladder:
            if lvl > cur and (lvl - cur) * sizes[n] <= room:
                out.append((n, lvl))
    return out


def _spend(work: dict, names: list, sizes: dict, ladder: tuple, room: int, rng, skip=None) -> int:
    """Random raises until ``room`` parameter-bits are used or no raise fits."""
    while room > 0:
        moves = _raises(work, names, sizes, ladder, room, skip)
        if not moves:
            break
        n, lvl = moves[rng.integers(len(moves))]
        room -= (lvl - work[n]) * sizes[n]
        work[n] = lvl
    return room


def uniform_completed(budget: int, sizes: dict, ladder, rng: np.random.Generator) -> BitConfig:
    """Highest uniform level within ``budget`` parameter-bits, completed to the exact budget."""
    ladder = tuple(sorted(set(int(x) for x in ladder)))
    names = sorted(sizes)
    total = sum(sizes.values())
    fitting = [lvl for lvl in ladder if lvl * total <= budget]
    if not fitting:
        raise ConfigError("infeasible budget")
    base = max(fitting)
    for _ in range(64):
        work = dict.fromkeys(names, base)
        if _spend(work, names, sizes, ladder, budget - base * total, rng) == 0:
            return BitConfig(assignment=work, ladder=ladder, budget_bits=budget)
    raise ConfigError("infeasible budget")


def mutate_level_switch(config: BitConfig, sizes: dict, rng: np.random.Generator,
                        max_retries: int = 10) -> tuple[BitConfig, bool]:
    """One budget-preserving level switch; returns (config, stagnant)."""
    names = sorted(config.assignment)
    if len(names) < 2:
        raise ConfigError("mutation impossible")
    ladder = config.ladder
    for _ in range(max_retries):
        work = dict(config.assignment)
        lowerable = [n for n in names if work[n] > ladder[0]]
        if not lowerable:
            break
        pick = lowerable[rng.integers(len(lowerable))]
        below = [lvl for lvl in ladder if lvl < work[pick]]
        lvl = below[rng.integers(len(below))]
        freed = (work[pick] - lvl) * sizes[pick]
        work[pick] = lvl
        if _spend(work, names, sizes, ladder, freed, rng, skip=pick) == 0:
            return BitConfig(assignment=work, ladder=ladder, budget_bits=config.budget_bits), False
    return config, True


def unfused_layer_sizes(shape: DecoderShape = LLAMA31_8B, n_layers: int | None = None) -> dict:
    """Parameter counts of the unfused linears (q, k, v, o, gate, up, down) per block."""
    h, inter, hd = shape.hidden, shape.intermediate, shape.head_dim
    dims = {"q": (shape.n_heads * hd, h), "k": (shape.n_kv_heads * hd, h), "v": (shape.n_kv_heads * hd, h),
            "o": (h, shape.n_heads * hd), "gate": (inter, h), "up": (inter, h), "down": (h, inter)}
    out = {}
    for i in range(n_layers or shape.n_layers):
        for k in UNFUSED:
            n, kk = dims[k]
            out["layers.%d.%s" % (i, k)] = n * kk
    return out


def budget_config(avg_bits: float = 3.5, shape: DecoderShape = LLAMA31_8B, seed: int = 0,
                  mutations: int = 200, ladder=(2, 3, 4, 6, 8), n_layers: int | None = None) -> BitConfig:
    """A budget-exact heterogeneous config: uniform completion + ``mutations`` level switches.

    The budget is ``avg_bits`` x total parameters rounded to an integer number
    of parameter-bits, as the reference's search computes it (evo.py:184-187)."""
    sizes = unfused_layer_sizes(shape, n_layers)
    total = sum(sizes.values())
    ladder = tuple(sorted(set(int(x) for x in ladder)))
    budget = int(round(avg_bits * total))
    if budget < ladder[0] * total or budget > ladder[-1] * total:
        raise ConfigError("infeasible budget")
    rng = np.random.default_rng(seed)
    cfg = uniform_completed(budget, sizes, ladder, rng)
    for _ in range(mutations):
        cfg, _ = mutate_level_switch(cfg, sizes, rng)
    if cfg.total_bits(sizes) != budget:
        raise ConfigError("budget drifted")
    return cfg


def level_histogram(cfg: BitConfig) -> dict:
    hist: dict[int, int] = {}
    for r in cfg.assignment.values():
        hist[r] = hist.get(r, 0) + 1
    return dict(sorted(hist.items()))
