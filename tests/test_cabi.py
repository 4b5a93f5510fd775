"""CPU-side checks of the C-ABI boundary: the library loads, exports every
entry point include/bdsm_gpu.h declares, the pure-host shard split behaves,
and without a GPU the engine fails loudly (no CPU fallback)."""
import ctypes
import os
import re

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(REPO, "include", "bdsm_gpu.h")).read()
    return sorted(set(re.findall(r"BDSM_API\s+[\w\s\*]+?\b(bdsm_\w+)\s*\(", src)))


def test_header_declares_entry_points():
    names = _declared()
    for must in ["bdsm_engine_create", "bdsm_engine_apply_batch", "bdsm_last_batch_errors",
                 "bdsm_last_error", "bdsm_engine_destroy", "bdsm_engine_add_query"]:
        assert must in names


def test_library_exports_every_declared_symbol():
    import paper_2401_17018_b200 as bd
    lib = ctypes.CDLL(bd.lib_path())
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_shard_owners_partition():
    import paper_2401_17018_b200 as bd
    costs = [5, 1, 1, 30, 2, 2, 9, 0, 4]
    for world in (1, 2, 4, 8):
        own = bd.shard_owners(costs, world)
        assert len(own) == len(costs)
        assert own == sorted(own)  # contiguous ranges in canonical order
        assert all(0 <= o < world for o in own)
    assert bd.shard_owners(costs, 1) == [0] * len(costs)


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2401_17018_b200 as bd
    with pytest.raises(bd.EngineError):
        bd.Engine([0, 0], [0], [1])


def test_group_without_gpu_fails_loudly():
    """The multi-device group reports the device failure of its engines (no
    CPU fallback), and rejects an empty device list."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2401_17018_b200 as bd
    with pytest.raises(bd.EngineError, match="device 0"):
        bd.EngineGroup([0, 0], [0], [1], devices=[0, 0])
    with pytest.raises(ValueError, match="no devices"):
        bd.EngineGroup([0, 0], [0], [1], devices=[])
