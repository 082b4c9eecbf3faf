"""Per-spec read-only tables (host side) and their C-ABI view.

``build_tables`` flattens a TileMap plus env config into the arrays the
engine reads, with the same values and dtypes as the reference's
``tilecast.tables.build_tables`` (/root/reference/pkg/src/tilecast/tables.py:92-184)
so the CUDA kernel and the reference consume identical doubles. The arrays
are then handed once to ``tc_spec_create`` (include/tilecast_b200.h), which
packs and uploads them to HBM; nothing here runs per step.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import layout as L
from . import palette
from .geometry import PLANE_HALF_WIDTH, ContractError, EntityInit, EntityKind, TileMap

MOVE_SPEED = 0.15          # tiles per move action           (tables.py:20)
TURN_DEGREES = 15.0        # per turn action                 (tables.py:21)
AGENT_RADIUS = 0.2         # collision disc radius           (tables.py:22)
SPRITE_HALF_WIDTH = 0.35   # billboard half-width, tiles     (tables.py:23)
MIN_SPRITE_DEPTH = 0.05    #                                 (tables.py:24)
TURN_COS = math.cos(math.radians(TURN_DEGREES))
TURN_SIN = math.sin(math.radians(TURN_DEGREES))

# heading table E, S, W, N (tables.py:30-31)
HEADINGS = np.array([[1.0, 0.0], [0.0, 1.0], [-1.0, 0.0], [0.0, -1.0]])


def column_coefficients(width: int) -> np.ndarray:
    """coef[c] = (2c - (W-1)) / (W-1): exact integer numerator, so mirrored
    columns get exactly negated coefficients (tables.py:34-42)."""
    span = float(width - 1)
    return np.array([float(2 * c - (width - 1)) / span for c in range(width)])


@dataclass
class Tables:
    kind: np.ndarray
    wcol: np.ndarray
    didx: np.ndarray
    eat: np.ndarray
    dcol: np.ndarray
    dlock: np.ndarray
    ekind: np.ndarray
    ecol: np.ndarray
    epx: np.ndarray
    epy: np.ndarray
    spx: np.ndarray
    spy: np.ndarray
    goal_ent: np.ndarray
    dirs: np.ndarray
    pal: np.ndarray
    door_rgb: np.ndarray
    key_rgb: np.ndarray
    goal_rgb: np.ndarray
    med_box: np.ndarray
    med_cross: np.ndarray
    ceil_rgb: np.ndarray
    floor_rgb: np.ndarray
    coef: np.ndarray
    fc: np.ndarray
    ic: np.ndarray
    legal: np.ndarray
    entities: tuple[EntityInit, ...]
    obs_width: int
    obs_height: int

    # the ABI field order (tables.py:257-261)
    ARRAY_FIELDS = ("kind", "wcol", "didx", "eat", "dcol", "dlock", "ekind",
                    "ecol", "epx", "epy", "spx", "spy", "goal_ent", "dirs",
                    "pal", "door_rgb", "key_rgb", "goal_rgb", "med_box",
                    "med_cross", "ceil_rgb", "floor_rgb", "coef", "fc", "ic",
                    "legal")

    @property
    def n_doors(self) -> int:
        return int(self.dcol.shape[0])

    @property
    def n_entities(self) -> int:
        return int(self.ekind.shape[0])

    @property
    def map_height(self) -> int:
        return int(self.kind.shape[0])

    @property
    def map_width(self) -> int:
        return int(self.kind.shape[1])

    def c_struct(self):
        """A ``tc_tables`` whose pointers alias these (host) arrays."""
        from ._native import TcTables, ptr
        s = TcTables()
        for name in self.ARRAY_FIELDS:
            setattr(s, name, ptr(getattr(self, name)))
        s.h, s.w = self.map_height, self.map_width
        s.n_doors, s.n_entities = self.n_doors, self.n_entities
        s.n_spawns, s.n_goals = int(self.spx.shape[0]), int(self.goal_ent.shape[0])
        s.n_pal = int(self.pal.shape[0])
        s.obs_h, s.obs_w = self.obs_height, self.obs_width
        return s


def build_tables(tmap: TileMap, *, obs_width: int = 64, obs_height: int = 64,
                 extra_entities: Sequence[EntityInit] = (),
                 action_tags: Sequence[int] = tuple(range(L.A_COUNT)),
                 goal_mode: int = 0, max_steps: int = 10**9,
                 goal_reward: float = 1.0, living_reward: float = 0.0,
                 health_decay: float = 0.0, health_restore: float = 0.0) -> Tables:
    if obs_width < 8 or obs_height < 8:
        raise ContractError(f"observation must be at least 8x8, got {obs_width}x{obs_height}")
    ents = tuple(tmap.entities) + tuple(extra_entities)
    if len(ents) > L.MAX_ENTITIES:
        raise ContractError(f"too many entities: {len(ents)} > {L.MAX_ENTITIES}")
    if len(tmap.doors) > L.MAX_DOORS:
        raise ContractError(f"too many doors: {len(tmap.doors)} > {L.MAX_DOORS}")

    h, w = tmap.height, tmap.width
    eat = np.full((h, w), -1, dtype=np.int16)
    for i, e in enumerate(ents):
        tx, ty = e.tile
        if not (0 < tx < w - 1 and 0 < ty < h - 1):
            raise ContractError(f"entity at {e.tile} is outside the map interior")
        if tmap.kind[ty, tx] != 0:
            raise ContractError(f"entity at {e.tile} must sit on a floor tile")
        if eat[ty, tx] != -1:
            raise ContractError(f"two entities share tile {e.tile}")
        eat[ty, tx] = i
    if not tmap.spawn_candidates:
        raise ContractError("map has no spawn candidates")

    fc = np.zeros(L.FC_COUNT)
    fc[L.FC_MOVE_SPEED] = MOVE_SPEED
    fc[L.FC_RADIUS] = AGENT_RADIUS
    fc[L.FC_TURN_COS] = TURN_COS
    fc[L.FC_TURN_SIN] = TURN_SIN
    fc[L.FC_ATTEN] = palette.ATTENUATION
    fc[L.FC_GOAL_REWARD] = goal_reward
    fc[L.FC_LIVING_REWARD] = living_reward
    fc[L.FC_HEALTH_DECAY] = health_decay
    fc[L.FC_HEALTH_RESTORE] = health_restore
    fc[L.FC_SPRITE_K] = SPRITE_HALF_WIDTH / PLANE_HALF_WIDTH
    fc[L.FC_MIN_SPRITE_DEPTH] = MIN_SPRITE_DEPTH
    ic = np.array([max_steps, goal_mode, 1 if health_decay > 0.0 else 0], dtype=np.int64)
    legal = np.zeros(L.A_COUNT, dtype=np.uint8)
    legal[[int(a) for a in action_tags]] = 1

    arrays = dict(
        kind=tmap.kind, wcol=tmap.wall_color, didx=tmap.door_index, eat=eat,
        dcol=np.array([int(d.color) for d in tmap.doors], dtype=np.uint8),
        dlock=np.array([int(d.locked) for d in tmap.doors], dtype=np.uint8),
        ekind=np.array([int(e.kind) for e in ents], dtype=np.uint8),
        ecol=np.array([0 if e.color is None else int(e.color) for e in ents], dtype=np.uint8),
        epx=np.array([e.tile[0] + 0.5 for e in ents], dtype=np.float64),
        epy=np.array([e.tile[1] + 0.5 for e in ents], dtype=np.float64),
        spx=np.array([s[0] + 0.5 for s in tmap.spawn_candidates], dtype=np.float64),
        spy=np.array([s[1] + 0.5 for s in tmap.spawn_candidates], dtype=np.float64),
        goal_ent=np.array([i for i, e in enumerate(ents) if e.kind == EntityKind.GOAL],
                          dtype=np.int32),
        dirs=HEADINGS, pal=palette.WALL_PALETTE, door_rgb=palette.DOOR_RGB,
        key_rgb=palette.KEY_RGB, goal_rgb=palette.GOAL_RGB,
        med_box=palette.MEDKIT_BOX_RGB, med_cross=palette.MEDKIT_CROSS_RGB,
        ceil_rgb=palette.CEILING_RGB, floor_rgb=palette.FLOOR_RGB,
        coef=column_coefficients(obs_width), fc=fc, ic=ic, legal=legal)
    for k, a in arrays.items():
        a = np.ascontiguousarray(a)
        a.setflags(write=False)
        arrays[k] = a
    return Tables(entities=ents, obs_width=obs_width, obs_height=obs_height, **arrays)
