"""ASCII map source -> TileMap.

Symbol meanings follow the reference's map DSL
(/root/reference/pkg/src/tilecast/mapdsl.py:3-15): ``#`` wall, ``1``-``9``
coloured walls, ``.``/space floor, ``S`` spawn, ``G`` goal, ``r b y`` keys,
``R B Y`` locked doors, ``"`` and ``\\`` unlocked blue / yellow doors, other
free uppercase letters generated walls (palette 10-15, cycled). Short lines
are padded with wall. The reference's build-time diagnostics machinery and
reachability warnings are out of scope; errors here
raise ``MapParseError`` with 1-based (line, column) positions.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .geometry import CellTag, Door, EntityInit, EntityKind, KeyColor, TileMap

_WALL_LETTERS = "ACDEFHIJKLMNOPQTUVWXZ"  # uppercase minus the reserved S G R B Y
_KEY_OF = {"r": KeyColor.RED, "b": KeyColor.BLUE, "y": KeyColor.YELLOW}
_LOCKED_DOOR_OF = {"R": KeyColor.RED, "B": KeyColor.BLUE, "Y": KeyColor.YELLOW}
_OPEN_DOOR_OF = {'"': KeyColor.BLUE, "\\": KeyColor.YELLOW}


@dataclass(frozen=True)
class MapSource:
    text: str
    name: str = "<map>"


class MapParseError(ValueError):
    def __init__(self, problems: list[tuple[int, int, str]]):
        self.problems = problems
        super().__init__("map has errors:\n" + "\n".join(
            f"error: line {ln}, column {col}: {msg}" for ln, col, msg in problems))


def parse_map(src: MapSource | str) -> TileMap:
    text = src.text if isinstance(src, MapSource) else src
    rows = [ln.rstrip("\r") for ln in text.split("\n")]
    lo, hi = 0, len(rows)
    while lo < hi and not rows[lo].strip():
        lo += 1
    while hi > lo and not rows[hi - 1].strip():
        hi -= 1
    rows = rows[lo:hi]
    if sum(1 for r in rows if r.strip()) < 3:
        raise MapParseError([(1, 1, "map needs at least 3 non-empty lines")])
    h, w = len(rows), max(len(r) for r in rows)
    if w < 3:
        raise MapParseError([(lo + 1, 1, "map must be at least 3 tiles wide")])

    kind = np.full((h, w), CellTag.WALL, dtype=np.uint8)
    colour = np.zeros((h, w), dtype=np.uint8)
    doors: list[Door] = []
    ents: list[EntityInit] = []
    spawns: list[tuple[int, int]] = []
    problems: list[tuple[int, int, str]] = []
    for y, line in enumerate(rows):
        for x, ch in enumerate(line):
            tile = (x, y)
            if ch == "#":
                continue
            if "1" <= ch <= "9":
                colour[y, x] = int(ch)
            elif ch in _WALL_LETTERS:
                colour[y, x] = 10 + _WALL_LETTERS.index(ch) % 6
            elif ch in ". ":
                kind[y, x] = CellTag.FLOOR
            elif ch == "S":
                kind[y, x] = CellTag.FLOOR
                spawns.append(tile)
            elif ch == "G":
                kind[y, x] = CellTag.FLOOR
                ents.append(EntityInit(EntityKind.GOAL, tile))
            elif ch in _KEY_OF:
                kind[y, x] = CellTag.FLOOR
                ents.append(EntityInit(EntityKind.KEY, tile, _KEY_OF[ch]))
            elif ch in _LOCKED_DOOR_OF or ch in _OPEN_DOOR_OF:
                kind[y, x] = CellTag.DOOR
                locked = ch in _LOCKED_DOOR_OF
                doors.append(Door(tile, (_LOCKED_DOOR_OF if locked else _OPEN_DOOR_OF)[ch],
                                  locked))
            else:
                problems.append((lo + y + 1, x + 1, f"unknown map symbol {ch!r}"))
    for y in range(h):
        xs = range(w) if y in (0, h - 1) else (0, w - 1)
        for x in xs:
            if kind[y, x] != CellTag.WALL:
                problems.append((lo + y + 1, x + 1, "map border must be wall (map is unsealed)"))
    if not spawns:
        problems.append((1, 1, "map has no spawn candidate (no 'S')"))
    if problems:
        raise MapParseError(problems)
    return TileMap(kind, colour, doors, ents, spawns)
