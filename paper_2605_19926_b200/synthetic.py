"""Synthetic random tile maps (BASELINE config C5).

Same distribution -- and, for the same ``random.Random`` state, the same
maps -- as the reference test-suite generator
(/root/reference/pkg/tests/conftest.py:40-92): 6-14 tiles per side, 22 %
interior walls with random palette colours, 0-2 doors (random key colour,
50 % locked), 0-4 entities (key / goal / medkit), one spawn. Pinned against
the reference in tests/test_host.py with tests/golden/synthetic_maps.npz.
"""

from __future__ import annotations

import random

import numpy as np

from .geometry import CellTag, Door, EntityInit, EntityKind, KeyColor, TileMap


def random_tilemap(rng: random.Random, *, doors: bool = True,
                   entities: bool = True) -> TileMap:
    w, h = rng.randrange(6, 15), rng.randrange(6, 15)
    kind = np.zeros((h, w), dtype=np.uint8)
    colour = np.zeros((h, w), dtype=np.uint8)
    kind[[0, -1], :] = CellTag.WALL
    kind[:, [0, -1]] = CellTag.WALL
    for y in range(1, h - 1):
        for x in range(1, w - 1):
            if rng.random() < 0.22:
                kind[y, x] = CellTag.WALL
                colour[y, x] = rng.randrange(0, 16)
    for y in range(h):
        for x in range(w):
            if kind[y, x] == CellTag.WALL and rng.random() < 0.5:
                colour[y, x] = rng.randrange(0, 16)

    interior = [(x, y) for y in range(1, h - 1) for x in range(1, w - 1)]
    free = [t for t in interior if kind[t[1], t[0]] == CellTag.FLOOR]
    if len(free) < 6:  # too dense: open the whole interior
        for x, y in interior:
            kind[y, x] = CellTag.FLOOR
        free = list(interior)
    rng.shuffle(free)

    door_list: list[Door] = []
    if doors:
        for x, y in free[: rng.randrange(0, 3)]:
            kind[y, x] = CellTag.DOOR
            door_list.append(Door((x, y), KeyColor(rng.randrange(3)),
                                  bool(rng.random() < 0.5)))
        free = [t for t in free if kind[t[1], t[0]] == CellTag.FLOOR]

    ents: list[EntityInit] = []
    if entities:
        count = rng.randrange(0, min(5, len(free) - 1))
        for tile in free[:count]:
            kd = rng.choice([EntityKind.KEY, EntityKind.GOAL, EntityKind.MEDKIT])
            col = KeyColor(rng.randrange(3)) if kd == EntityKind.KEY else None
            ents.append(EntityInit(kd, tile, col))
        free = free[count:]

    return TileMap(kind, colour, tuple(door_list), tuple(ents), (free[-1],))
