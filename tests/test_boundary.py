"""The C-ABI boundary (no GPU needed): the library builds, loads and exports
every symbol include/dbs_b200.h declares; status codes map onto the
reference's exception classes; host-side argument validation matches the
reference before any device work is attempted."""

from __future__ import annotations

import re
from pathlib import Path

import pytest

from conftest import ROOT

HEADER = ROOT / "include" / "dbs_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(dbs_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for must in ("dbs_plan_next_epoch", "dbs_round_twice", "dbs_spans_from_ranges", "dbs_dev_replan",
                 "dbs_dev_permute_spans", "dbs_dev_gather_rows", "dbs_dev_aggregate_sgd_f32",
                 "dbs_comm_allreduce_sgd", "dbs_dev_gemm_bf16", "dbs_mlp_forward_backward", "dbs_dev_spin_until"):
        assert must in syms


def test_library_loads_and_exports_every_declared_symbol():
    from paper_2007_11831_b200 import _lib

    L = _lib.lib()
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing
    # and the ctypes table covers the header
    assert set(declared_symbols()) <= set(_lib.exported_symbols())


def test_library_targets_sm100():
    import ctypes

    from paper_2007_11831_b200 import _lib

    a, b, c = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    assert _lib.lib().dbs_version(ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)) == 0
    assert c.value == 100


def test_cubins_are_sm100a():
    import subprocess

    lib = ROOT / "paper_2007_11831_b200" / "libdbs_b200.so"
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(lib)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_status_codes_map_to_reference_exceptions():
    from paper_2007_11831_b200 import errors

    pairs = {1: errors.InvalidMeasurementError, 2: errors.InvalidPerformanceError, 3: errors.BudgetTooSmallError,
             4: errors.InvalidBatchError, 5: errors.EmptyPartitionError, 6: errors.DatasetTooSmallError,
             7: errors.ConfigurationError, 9: errors.EmptyBatchError, 10: errors.InvalidStepSizeError,
             20: OverflowError, 21: ValueError}
    for code, cls in pairs.items():
        assert type(errors.from_status(code, "x")) is cls
    assert isinstance(errors.from_status(40, "x"), errors.DeviceError)
    assert issubclass(errors.ValidationError, errors.ConfigurationError)
    assert all(issubclass(c, errors.DbsError) for c in pairs.values() if c.__module__.endswith("errors"))


def test_host_validation_before_device_work():
    """Errors the reference raises before any arithmetic fire without a GPU."""
    from paper_2007_11831_b200 import allocation as A
    from paper_2007_11831_b200 import errors

    with pytest.raises(errors.InvalidPerformanceError):
        A.compute_batch_fractions([])
    with pytest.raises(errors.InvalidPerformanceError):
        A.plan_next_epoch([], [], 8, 100, 1)
    with pytest.raises(errors.InvalidPerformanceError):
        A.plan_next_epoch([0.5, 0.5], [1.0], 8, 100, 1)
    with pytest.raises(errors.BudgetTooSmallError):
        A.plan_next_epoch([0.5, 0.5], [1.0, 1.0], 1, 100, 1)


def test_sgd_config_validation_matches_reference():
    from paper_2007_11831_b200 import errors
    from paper_2007_11831_b200.sgdlab import SgdConfig

    with pytest.raises(errors.ConfigurationError):
        SgdConfig(step_size=0.1, n_iterations=1, aggregation="median")
    with pytest.raises(errors.ConfigurationError):
        SgdConfig(step_size=0.1, n_iterations=0)
    with pytest.raises(errors.ConfigurationError):
        SgdConfig(step_size=0.1, n_iterations=1, momentum=1.0)
    with pytest.raises(errors.InvalidStepSizeError):
        SgdConfig(step_size=1.5, n_iterations=1).validate_step_size(1.0)


def test_cluster_config_validation_matches_reference():
    from paper_2007_11831_b200 import cluster as C
    from paper_2007_11831_b200 import errors

    with pytest.raises(errors.ConfigurationError):
        C.DisturbanceEvent(start_epoch=0)
    with pytest.raises(errors.ConfigurationError):
        C.DisturbanceEvent(start_epoch=0, extra_epoch_seconds=1.0, cost_multiplier=2.0)
    with pytest.raises(errors.ConfigurationError):
        C.WorkerProfile(0, 0.1, disturbances=(C.DisturbanceEvent(0, extra_epoch_seconds=1.0),
                                              C.DisturbanceEvent(5, extra_epoch_seconds=1.0)))
    with pytest.raises(errors.ConfigurationError):
        C.StrategyConfig("bogus", 64)
    cfg = C.StrategyConfig("model_averaging", 64, sync_interval=8)
    assert C.sync_rounds_for_epoch(cfg, 96, False) == 12  # test_cluster.py:90-97
    assert C.sync_rounds_for_epoch(C.StrategyConfig("dbs", 64), 96, False) == 97
    assert C.sync_rounds_for_epoch(C.StrategyConfig("one_shot", 64), 96, True) == 1


def test_product_never_imports_the_oracle():
    pkg = ROOT / "paper_2007_11831_b200"
    pat = re.compile(r"^\s*(from|import)\s+oracle\b|libdbs_oracle|dbs_oracle", re.M)
    for p in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")):
        assert not pat.search(p.read_text()), p
