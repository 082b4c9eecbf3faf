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


def large_tilemap(rng: random.Random, width: int, height: int, *, n_doors: int = 2,
                  n_entities: int = 4, n_spawns: int = 4, wall_density: float = 0.22,
                  doors_at_spawns: bool = False) -> TileMap:
    """A sealed random map of any size at the C5 density (SURVEY.md §8(d)
    large-map variant: 22 % interior walls, random palette colours), with
    ``n_doors`` doors (random colour, 50 % locked; up to the reference's 32,
    tables.py:110-113), ``n_entities`` keys / goals / medkits and
    ``n_spawns`` spawn candidates. With ``doors_at_spawns`` the doors are put
    on the tiles next to the spawns first, so a random policy touches (and
    opens) them within a few steps."""
    w, h = width, height
    kind = np.zeros((h, w), dtype=np.uint8)
    colour = np.zeros((h, w), dtype=np.uint8)
    kind[[0, -1], :] = CellTag.WALL
    kind[:, [0, -1]] = CellTag.WALL
    for y in range(h):
        for x in range(w):
            if 0 < x < w - 1 and 0 < y < h - 1 and rng.random() < wall_density:
                kind[y, x] = CellTag.WALL
            if kind[y, x] == CellTag.WALL:
                colour[y, x] = rng.randrange(0, 16)
    free = [(x, y) for y in range(1, h - 1) for x in range(1, w - 1)
            if kind[y, x] == CellTag.FLOOR]
    rng.shuffle(free)
    spawns = free[:n_spawns]
    taken = set(spawns)
    door_tiles: list[tuple[int, int]] = []
    if doors_at_spawns:
        for sx, sy in spawns:
            for t in ((sx + 1, sy), (sx - 1, sy), (sx, sy + 1), (sx, sy - 1)):
                if len(door_tiles) < n_doors and t not in taken and \
                        kind[t[1], t[0]] == CellTag.FLOOR and 0 < t[0] < w - 1 and \
                        0 < t[1] < h - 1:
                    door_tiles.append(t)
                    taken.add(t)
    for t in free[n_spawns:]:
        if len(door_tiles) >= n_doors:
            break
        if t not in taken:
            door_tiles.append(t)
            taken.add(t)
    door_list = []
    for x, y in door_tiles:
        kind[y, x] = CellTag.DOOR
        door_list.append(Door((x, y), KeyColor(rng.randrange(3)), bool(rng.random() < 0.5)))
    rest = [t for t in free if t not in taken]
    ents = []
    for tile in rest[:n_entities]:
        kd = rng.choice([EntityKind.KEY, EntityKind.GOAL, EntityKind.MEDKIT])
        col = KeyColor(rng.randrange(3)) if kd == EntityKind.KEY else None
        ents.append(EntityInit(kd, tile, col))
    return TileMap(kind, colour, tuple(door_list), tuple(ents), tuple(spawns))
