"""The command line driver (cli.py, mirroring the reference cli.py) end to
end on the device: generate -> run (CSV, reference column order) -> validate."""

import csv
import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _cli(*args, cwd):
    return subprocess.run([sys.executable, "-m", "paper_1604_02844_b200", *args], cwd=cwd, capture_output=True,
                          text=True, timeout=300, env={"PYTHONPATH": str(ROOT), "PATH": "/usr/bin:/bin"})


def test_generate_run_validate(tmp_path):
    r = _cli("generate", "--scale", "10", "--out", str(tmp_path / "g.bin"), cwd=tmp_path)
    assert r.returncode == 0, r.stderr
    r = _cli("run", "--graph", str(tmp_path / "g.bin"), "--roots", "8", "--out", str(tmp_path / "r.csv"),
             cwd=tmp_path)
    assert r.returncode == 0, r.stderr
    rows = list(csv.reader(open(tmp_path / "r.csv")))
    assert rows[0] == ["scale", "edgefactor", "seed", "mode", "threads", "placement", "root", "time_s", "edges",
                       "teps", "gpus", "gbytes_alg", "roofline_frac"]
    assert len(rows) >= 9 and all(row[3] == "gpu" for row in rows[1:])
    assert all(float(row[12]) > 0 for row in rows[1:] if int(row[8]) > 0)  # roofline fraction of every search
    r = _cli("validate", "--scale", "12", "--permute", "--roots", "8", cwd=tmp_path)
    assert r.returncode == 0, r.stdout + r.stderr
    verdict = json.loads(r.stdout.strip().splitlines()[-1])
    assert verdict == {"roots": 8, "failures": 0, "mode": "gpu"}


def test_run_partitioned_one_gpu(tmp_path):
    """--gpus with the partitioned path: the 1D-partitioned search on every
    visible GPU of this process (one on this pool), same CSV schema."""
    import torch

    ng = 1 << (torch.cuda.device_count().bit_length() - 1)
    r = _cli("run", "--scale", "12", "--roots", "4", "--gpus", str(ng), "--out", str(tmp_path / "p.csv"), cwd=tmp_path)
    assert r.returncode == 0, r.stdout + r.stderr
    rows = list(csv.reader(open(tmp_path / "p.csv")))
    assert all(row[10] == str(ng) for row in rows[1:])
