"""CLI commands end to end on the GPU: the reference's report formats
(run/verify JSON, scaling/tune CSV) and exit codes."""

import csv
import io
import json

import numpy as np
import pytest

from paper_1209_3516_b200 import cli
from paper_1209_3516_b200.geometry import generate_distribution, save_particles_csv

pytestmark = pytest.mark.gpu


def test_run_json_and_verify_exit_codes(tmp_path, capsys):
    out = tmp_path / "run.json"
    assert cli.main(["run", "--n", "3000", "--p", "5", "--theta", "0.5", "--reps", "2", "--verify",
                     "--tol", "1e-2", "--output", str(out)]) == 0
    doc = json.loads(out.read_text())
    assert doc["schema"] == "fmmkit-report-v1" and doc["params"]["strategy"] == "dualtree"
    assert doc["achieved_error"] < 1e-2 and doc["tree"]["n"] == 3000 and doc["reps"] == 2
    assert cli.main(["verify", "--n", "2000", "--theta", "0.8", "--tol", "1e-12", "--output",
                     str(tmp_path / "v.json")]) == 1
    assert "FAIL" in capsys.readouterr().err


def test_scaling_csv(tmp_path):
    out = tmp_path / "s.csv"
    assert cli.main(["scaling", "--n-list", "1000,4000", "--reps", "1", "--strategy", "treecode",
                     "--output", str(out)]) == 0
    rows = list(csv.reader(io.StringIO(out.read_text())))
    assert rows[0][:3] == ["n", "ncells", "depth"] and [r[0] for r in rows[1:]] == ["1000", "4000"]
    assert int(rows[1][-1]) > 0  # m2p calls of the treecode


def test_tune_csv_and_input_file(tmp_path):
    src = tmp_path / "bodies.csv"
    save_particles_csv(generate_distribution("uniform", 2000, 11), str(src))
    out = tmp_path / "t.csv"
    assert cli.main(["tune", "--input", str(src), "--ncrit", "30", "--targets", "1e-3,1e-30", "--p-list", "3,4",
                     "--reps", "1", "--output", str(out)]) == 0
    rows = list(csv.reader(io.StringIO(out.read_text())))
    assert rows[0] == ["target", "best_p", "best_theta", "theta_p3", "error_p3", "time_ms_p3", "theta_p4",
                       "error_p4", "time_ms_p4"]
    assert rows[1][0] == "0.001" and rows[1][1] in ("3", "4") and float(rows[1][4]) <= 1e-3
    assert rows[2][1:] == [""] * 8  # unreachable target


def test_listfmm_on_rect_tree_is_a_usage_error(capsys):
    assert cli.main(["run", "--n", "500", "--strategy", "listfmm", "--shape", "rect", "--reps", "1"]) == 2
    assert "cubic" in capsys.readouterr().err


@pytest.mark.parametrize("precision", ["fp32", "fp32acc"])
def test_run_precisions(tmp_path, precision):
    out = tmp_path / "run.json"
    assert cli.main(["run", "--n", "4000", "--p", "8", "--theta", "0.4", "--reps", "1", "--precision", precision,
                     "--output", str(out)]) == 0
    doc = json.loads(out.read_text())
    assert doc["precision"] == precision
