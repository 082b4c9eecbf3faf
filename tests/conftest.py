"""Shared test setup: markers, paths, golden-fixture loaders."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
for p in (str(ROOT), str(ROOT / "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def have_cuda() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session")
def golden_digests():
    return json.loads((GOLDEN / "digests.json").read_text())


def unpack_map(blob: np.ndarray):
    """Inverse of make_golden._pack_map."""
    from paper_2605_19926_b200.geometry import Door, EntityInit, EntityKind, KeyColor, TileMap
    v = [int(x) for x in blob]
    h, w = v[0], v[1]
    p = 2
    kind = np.array(v[p:p + h * w], dtype=np.uint8).reshape(h, w); p += h * w
    wcol = np.array(v[p:p + h * w], dtype=np.uint8).reshape(h, w); p += h * w
    nd = v[p]; p += 1
    doors = []
    for _ in range(nd):
        doors.append(Door((v[p], v[p + 1]), KeyColor(v[p + 2]), bool(v[p + 3]))); p += 4
    ne = v[p]; p += 1
    ents = []
    for _ in range(ne):
        ents.append(EntityInit(EntityKind(v[p]), (v[p + 1], v[p + 2]),
                               None if v[p + 3] < 0 else KeyColor(v[p + 3]))); p += 4
    ns = v[p]; p += 1
    spawns = [(v[p + 2 * k], v[p + 2 * k + 1]) for k in range(ns)]
    return TileMap(kind, wcol, doors, ents, spawns)


def pytest_collection_modifyitems(config, items):
    import os
    if os.environ.get("TILECAST_SLOW"):
        return
    skip = pytest.mark.skip(reason="slow parity case; set TILECAST_SLOW=1")
    for item in items:
        if "slow" in item.keywords:
            item.add_marker(skip)
