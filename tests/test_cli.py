"""The command-line front end (paper_1907_12933_b200/cli.py; SPEC.md run_cli exit codes:
0 holds, 10 violated, 2 usage, 3 resource)."""
import json

import numpy as np
import pytest


def test_cli_usage_errors():
    from paper_1907_12933_b200 import cli
    with pytest.raises(SystemExit) as e:
        cli.main(["verify", "--config", "gamma"])          # missing --gamma / --max-bound
    assert e.value.code == cli.EXIT_USAGE
    with pytest.raises(SystemExit) as e:
        cli.main(["frobnicate"])
    assert e.value.code == cli.EXIT_USAGE


@pytest.mark.gpu
def test_cli_gpu(capsys, oracle_mod):
    import mlpv_inputs as M
    from paper_1907_12933_b200 import build, cli
    build.build()
    # verify: the gamma workload has counterexamples for 15 of 50 bases at gamma = 3 (exit 10),
    # and each reported (step, index) is the oracle's incremental loop result
    assert cli.main(["verify", "--config", "gamma", "--gamma", "3", "--max-bound", "12"]) == cli.EXIT_VIOLATED
    rep = json.loads(capsys.readouterr().out)
    o = oracle_mod.incremental_verify(M.gamma_config(), 3.0, 12, 1)
    want = {str(b): (int(o["step"][b]), int(o["first_cex"][b])) for b in range(50) if o["step"][b] > 0}
    assert {k: (v["step"], v["index"]) for k, v in rep["violated"].items()} == want
    assert rep["safe_over_grid"] == 50 - len(want)
    # the same answers in the loop's own order with early exit, on fewer candidates
    full = rep["candidates_checked"]
    assert cli.main(["verify", "--config", "gamma", "--gamma", "3", "--max-bound", "12", "--early-exit"]) == cli.EXIT_VIOLATED
    rep = json.loads(capsys.readouterr().out)
    assert {k: (v["step"], v["index"]) for k, v in rep["violated"].items()} == want
    assert rep["early_exit"] and rep["candidates_checked"] < full
    # check: cfg2 (no violation at eps = 0.1) holds
    assert cli.main(["check", "--config", "cfg2", "--bases", "2"]) == cli.EXIT_OK
    rep = json.loads(capsys.readouterr().out)
    assert rep["violated"] == 0 and rep["checked"] == 2 * 390_625
    # cover: the literal's exit code follows the ratios
    code = cli.main(["cover", "--config", "cfg2", "--images", "50", "--threshold", "0.8"])
    rep = json.loads(capsys.readouterr().out)
    assert code == (cli.EXIT_VIOLATED if not all(rep["literal"].values()) else cli.EXIT_OK)
    # an invalid argument value reaching the ABI is a usage error
    assert cli.main(["verify", "--config", "gamma", "--gamma", "-1", "--max-bound", "4"]) == cli.EXIT_USAGE
