"""The experiment harness (paper_2503_17405_b200.cli) against the reference's
cli.py: config hashes, validation messages and config files on the host; the
paired standard/FSM runs and their result rows on the GPU, compared row for
row with rows the live reference produced (tests/golden/cli.json)."""

import json
import os

import numpy as np
import pytest

from golden_cases import GOLDEN
from paper_2503_17405_b200 import cli


def _golden():
    with open(os.path.join(GOLDEN, "cli.json")) as f:
        return json.load(f)


def _config(kw):
    return cli.RunConfig(**{k: tuple(v) if isinstance(v, list) else v for k, v in kw.items()})


def test_config_hashes_match_reference():
    g = _golden()
    assert cli.RunConfig().config_hash() == g["hash_default"]
    for run in g["runs"]:
        assert _config(run["config"]).config_hash() == run["hash"]


def test_validation_messages_match_reference():
    for case in _golden()["validate"]:
        assert _config(case["config"]).validate() == case["errors"]


def test_config_file_and_flags(tmp_path):
    f = tmp_path / "exp.cfg"
    f.write_text("# paired run\nkernel = nuts\nchains=8\nseeds = 1,2\nnuts-step-size = 0.2\n"
                 "drmh_split_body = yes\nmog_offsets = -1,1\n")
    args = cli.build_parser()
    pre, _ = args.parse_known_args(["--config", str(f)])
    raw = cli._parse_config_file(pre.config)
    assert raw["nuts_step_size"] == "0.2" and raw["seeds"] == "1,2"
    assert cli._coerce("0.2", 0.1) == 0.2 and cli._coerce("yes", False) is True
    assert cli._coerce("1,2", (0,)) == (1, 2) and cli._coerce("-1,1", (0.5,)) == (-1.0, 1.0)
    bad = tmp_path / "bad.cfg"
    bad.write_text("nonsense_key = 3\n")
    assert cli.main(["--config", str(bad)]) == 2
    assert cli.main(["--kernel", "slice", "--dim", "2"]) == 2
    assert cli.main(["--sweep-axis", "m"]) == 2


@pytest.mark.gpu
@pytest.mark.parametrize("idx", range(5))
def test_paired_runs_match_reference_rows(idx, tmp_path):
    """Every result column equal to the reference's, the ESS columns within
    1e-9 (device FFT-free autocovariances vs numpy's FFT)."""
    run = _golden()["runs"][idx]
    cfg = _config({**run["config"], "out": str(tmp_path)})
    res = cli.run_experiment(cfg, write=True)
    assert len(res.rows) == len(run["rows"])
    for got, ref in zip(res.rows, run["rows"]):
        for col in cli.RESULT_COLUMNS:
            if col in ("ess_pooled", "ess_per_cost"):
                assert got[col] == pytest.approx(ref[col], rel=1e-9), col
            elif isinstance(ref[col], float):
                assert got[col] == pytest.approx(ref[col], rel=1e-13, abs=1e-13), col
            else:
                assert got[col] == ref[col], col
    for name in ("results.csv", "timings.csv", "manifest.json"):
        assert (tmp_path / name).exists()
    header = (tmp_path / "results.csv").read_text().splitlines()[0]
    assert header == ",".join(cli.RESULT_COLUMNS)
    man = json.loads((tmp_path / "manifest.json").read_text())
    assert man["config_hash"] == run["hash"]


@pytest.mark.gpu
def test_sweep_and_measured_costs(tmp_path):
    cfg = cli.RunConfig(kernel="drmh", target="std-normal", dim=2, chains=8, samples=50,
                        variant="bundled", out=str(tmp_path), cost_model="measured")
    rows = cli.sweep(cfg, "m", [4, 16])
    assert len(rows) == 4 and all(r["cost_ratio"] > 0 for r in rows)
    assert (tmp_path / "sweep.csv").exists()
    params = cli.resolve_cost_params(cfg, cli.build_kernel(cfg), cli.build_target(cfg))
    assert all(c > 0 for c in params.block_costs)
    assert cli.main(["--kernel", "slice", "--chains", "4", "--samples", "30",
                     "--out", str(tmp_path / "s")]) == 0
