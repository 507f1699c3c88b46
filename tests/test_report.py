"""report.py formats against the reference's own output (tests/golden/report_*,
made by tests/golden/gen_golden.py from dbsim.report / dbsim.cluster)."""
from __future__ import annotations

import json
from pathlib import Path

import pytest

from paper_2007_11831_b200 import cluster, report
from paper_2007_11831_b200.errors import BaselineNotFoundError, InvalidBaselineError

GOLDEN = Path(__file__).resolve().parent / "golden"


def _unhex(v):
    return None if v is None else float.fromhex(v)


def _scenario():
    d = json.loads((GOLDEN / "report_scenario.json").read_text())
    profs = [cluster.WorkerProfile(p["worker_id"], _unhex(p["base_cost"]), _unhex(p["per_iteration_overhead"]),
                                   tuple(cluster.DisturbanceEvent(e["start_epoch"], e["end_epoch"],
                                                                  _unhex(e["extra_epoch_seconds"]),
                                                                  _unhex(e["cost_multiplier"]))
                                         for e in p["disturbances"]))
             for p in d["profiles"]]
    strats = [cluster.StrategyConfig(s["kind"], s["total_budget"], s["sync_interval"], _unhex(s["sync_cost_per_round"]),
                                     _unhex(s["sync_cost_per_worker"]), _unhex(s["perf_smoothing"]))
              for s in d["strategies"]]
    return d, profs, strats


def _reports():
    """Our RunReports from the golden run's epoch rows (CPU: no device controller)."""
    from types import SimpleNamespace

    d = json.loads((GOLDEN / "report_scenario.json").read_text())
    doc = json.loads((GOLDEN / "report_robustness.json").read_text())
    reps = []
    for sc in doc["scenarios"]:
        stats = [cluster.EpochStats(epoch=r["epoch"], per_worker_gpu=tuple(r["t_gpu"]), per_worker_wait=tuple(r["t_w"]),
                                    sync_time=r["t_s"], epoch_wall_time=r["T_a"],
                                    plan=SimpleNamespace(int_batches=tuple(r["int_batches"])))
                 for r in sc["epoch_rows"]]
        reps.append(report.RunReport.from_stats(sc["scenario_name"], sc["strategy"], sc["seed"], stats))
    return d, reps


@pytest.mark.gpu
def test_measured_pipeline_reproduces_reference_reports(tmp_path):
    """The simulator on the device controller, end to end into both formats."""
    d, profs, strats = _scenario()
    reps = [report.RunReport.from_stats(d["name"], s.kind, 0,
                                        cluster.run_training(profs, s, d["dataset_size"], d["n_epochs"]))
            for s in strats]
    report.write_epoch_csv(next(r for r in reps if r.strategy == "dbs"), tmp_path / "dbs.csv")
    assert (tmp_path / "dbs.csv").read_bytes() == (GOLDEN / "report_robustness_dbs.csv").read_bytes()
    report.write_run_json(reps, [], tmp_path / "run.json")
    assert (tmp_path / "run.json").read_bytes() == (GOLDEN / "report_robustness.json").read_bytes()


def test_epoch_csv_byte_identical(tmp_path):
    _, reps = _reports()
    out = tmp_path / "dbs.csv"
    report.write_epoch_csv(next(r for r in reps if r.strategy == "dbs"), out)
    assert out.read_bytes() == (GOLDEN / "report_robustness_dbs.csv").read_bytes()
    rows = report.read_epoch_csv(out)
    assert list(rows[0]) == list(report.CSV_HEADER)


def test_run_json_byte_identical(tmp_path):
    _, reps = _reports()
    out = tmp_path / "run.json"
    report.write_run_json(reps, [], out)
    assert out.read_bytes() == (GOLDEN / "report_robustness.json").read_bytes()
    assert report.read_run_json(out)["schema_version"] == 1


def test_savings_table_exact():
    d, reps = _reports()
    got = report.compare_strategies(reps, "fixed_ssgd")
    want = [(k, float.fromhex(t), float.fromhex(v)) for k, t, v in d["savings"]]
    assert got == want


def test_report_errors():
    _, reps = _reports()
    try:
        report.compare_strategies(reps, "no_such_strategy")
        raise AssertionError("expected BaselineNotFoundError")
    except BaselineNotFoundError:
        pass
    try:
        report.savings_percent(1.0, 0.0)
        raise AssertionError("expected InvalidBaselineError")
    except InvalidBaselineError:
        pass
