"""The C-ABI library: loads on a CPU-only host, exports every entry point
include/tilecast_b200.h declares, and rejects bad arguments without
touching the GPU. No compute calls here."""

from __future__ import annotations

import ctypes as C
import re

import pytest

from conftest import ROOT

HEADER = ROOT / "include" / "tilecast_b200.h"


def declared_functions() -> list[str]:
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(tc_[a-z_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    fns = declared_functions()
    for f in ("tc_spec_create", "tc_spec_destroy", "tc_batch_kernel", "tc_rollout",
              "tc_seed_streams", "tc_policy_actions", "tc_host_cast_ray",
              "tc_host_render_into", "tc_host_batch_kernel", "tc_abi_version",
              "tc_last_error"):
        assert f in fns


def test_library_exports_every_declared_symbol():
    from paper_2605_19926_b200 import _native
    lib = C.CDLL(str(_native.LIB_PATH))
    missing = [f for f in declared_functions() if not hasattr(lib, f)]
    assert not missing, missing


def test_abi_version_and_info():
    from paper_2605_19926_b200 import _native
    lib = _native.lib()
    assert lib.tc_abi_version() == _native.ABI_VERSION
    assert b"sm_100a" in lib.tc_build_info()


def test_invalid_arguments_fail_without_gpu():
    from paper_2605_19926_b200 import _native
    lib = _native.lib()
    assert lib.tc_spec_create(None, None) == -1
    h = C.c_void_p()
    assert lib.tc_spec_create(None, C.byref(h)) == -1
    assert b"NULL" in lib.tc_last_error()
    assert lib.tc_batch_kernel(None, None, None, None, 1, 1, 1, 0, None, None) == -1
    assert lib.tc_policy_actions(0, 0, 1, 0, 1, None, 0, None, None) == -1
    assert lib.tc_seed_streams(0, 0, -1, None, None, None) == -1


def test_tables_struct_layout_matches_header():
    from paper_2605_19926_b200 import _native
    # 26 pointers + 9 int32 (padded to 8) -- tc_tables in include/tilecast_b200.h
    assert C.sizeof(_native.TcTables) == 26 * 8 + 9 * 4 + 4
    assert C.sizeof(_native.TcState) == 13 * 8
    assert C.sizeof(_native.TcOut) == 9 * 8
    assert C.sizeof(_native.TcCounters) == 24


def test_product_path_has_no_cpu_fallback(monkeypatch):
    """Without a CUDA device the host API refuses to run (no silent CPU path)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    import paper_2605_19926_b200 as tc
    with pytest.raises(RuntimeError, match="CUDA"):
        tc.batch_reset(tc.make_env("simple"), 4, 0)
