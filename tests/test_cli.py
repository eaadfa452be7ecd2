"""bench_cli (SPEC bench_cli): config parsing on CPU, the
report and its contracts on a GPU."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2303_02352_b200.cli import ConfigError, parse_config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_config_defaults_and_sample():
    assert parse_config("") == {}
    cfg = parse_config(open(os.path.join(ROOT, "configs", "paper.cfg")).read())
    assert cfg == {"aggregation_exponent": 3, "coarse_size": 10240, "max_levels": 40, "pre_sweeps": 4,
                   "post_sweeps": 4, "coarsest_sweeps": 20, "relax_weight": 1.0, "max_iters": 1000, "rtol": 1e-6,
                   "precflag": 1}


@pytest.mark.parametrize("text,msg", [("rtol = 0", "rtol must be in (0, 1)"), ("foo = 1", "unknown key 'foo'"),
                                      ("pre_sweeps", "expected 'key = value'"), ("max_iters = x", "bad value"),
                                      ("\n\nprecflag = 2", "cfg:3: precflag must be 0 or 1"),
                                      ("post_sweeps = -1", "must be >= 0")])
def test_config_errors(text, msg):
    with pytest.raises(ConfigError) as e:
        parse_config(text, "cfg")
    assert msg in str(e.value)


def cli(*args, check=True):
    r = subprocess.run([sys.executable, "-m", "paper_2303_02352_b200.cli", *args, "--json"], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    if check:
        assert r.returncode == 0, r.stdout + r.stderr
    return r.returncode, json.loads(r.stdout.strip().splitlines()[-1])


TIMING = ("tsetup_s", "tsolve_s", "titer_s", "setup_breakdown_s")


@pytest.mark.gpu
def test_cli_report_matches_oracle():
    import oracle

    _, rep = cli("-n", "16")
    orc = oracle.Oracle("restatement", stencil=7, nd=16, coarse_size_target=640)
    orc.setup()
    ref = orc.solve()
    assert rep["converged"] and rep["iterations"] == ref["iterations"]
    assert [lv["rows"] for lv in rep["levels"]] == [s[0] for s in orc.level_sizes()]
    assert abs(rep["opc"] - orc.opc) < 1e-12
    assert abs(rep["titer_s"] * rep["iterations"] - rep["tsolve_s"]) < 1e-9


@pytest.mark.gpu
def test_cli_amg_beats_cg_and_is_deterministic(tmp_path):
    _, amg = cli("-n", "30")
    _, cg = cli("-n", "30", "-p", "0")
    assert amg["converged"] and cg["converged"] and amg["iterations"] < cg["iterations"]
    _, again = cli("-n", "30")
    strip = lambda d: {k: v for k, v in d.items() if k not in TIMING}  # noqa: E731
    assert strip(amg) == strip(again)


@pytest.mark.gpu
def test_cli_matrix_market_equals_generator(tmp_path):
    import paper_2303_02352_b200 as pb

    path = str(tmp_path / "p.mtx")
    rp, ci, va = pb.poisson(7, 14, 14, 14)
    pb.write_matrix_market(path, rp, ci, va)
    cfg = tmp_path / "c.cfg"
    cfg.write_text("coarse_size = 560\n")
    _, gen = cli("-n", "14")
    _, mm = cli("-m", path, "-c", str(cfg))
    for k in ("iterations", "final_relres", "levels", "opc"):
        assert gen[k] == mm[k], k


@pytest.mark.gpu
def test_cli_nonconvergence_exit_code(tmp_path):
    cfg = tmp_path / "c.cfg"
    cfg.write_text("max_iters = 2\n")
    code, rep = cli("-n", "16", "-c", str(cfg), check=False)
    assert code == 1 and not rep["converged"] and rep["iterations"] == 2


@pytest.mark.gpu
@pytest.mark.multigpu
def test_cli_two_ranks_matches_one():
    """Two ranks (processes on 2 GPUs, else threads sharing one GPU) give the
    single-rank hierarchy on a slab-aligned grid and the same iteration count."""
    import torch

    _, one = cli("-n", "32")
    _, two = cli("-n", "32", "-P", "2", *([] if torch.cuda.device_count() >= 2 else ["--threads"]))
    assert two["ranks"] == 2 and two["converged"]
    assert [lv["rows"] for lv in two["levels"]] == [lv["rows"] for lv in one["levels"]]  # slab-aligned
    assert abs(two["iterations"] - one["iterations"]) <= 1
