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


def test_bench_clock_sampler_summary():
    """bench.py's clock line: only the samples stamped inside the timed region count; the throttle
    reasons are those active in them; every sample serves when none falls inside."""
    import datetime
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(os.path.dirname(__file__), "..", "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    t0 = datetime.datetime(2026, 1, 2, 3, 4, 5).timestamp()

    def row(dt, sm, cap):
        ts = datetime.datetime.fromtimestamp(t0 + dt).strftime("%Y/%m/%d %H:%M:%S.%f")[:-3]
        return f"{ts}, {sm}, 1965, 900.0, 0x0000000000000004, Not Active, Not Active, Not Active, {cap}"

    out = "\n".join([row(-1.0, 300, "Not Active"), row(0.1, 1700, "Active"), row(0.3, 1800, "Active"),
                     row(0.5, 1750, "Not Active"), row(2.0, 1965, "Not Active"), "garbage line"])
    c = bench.ClockSampler.summarise(out, t0, t0 + 0.6)
    assert c == {"sm_mhz": 1750.0, "sm_max_mhz": 1965.0, "reasons": ["sw_power_cap"], "samples": 3}
    c = bench.ClockSampler.summarise(out, t0 + 10, t0 + 11)      # nothing inside: every sample
    assert c["samples"] == 5 and c["sm_mhz"] == 1750.0
    assert bench.ClockSampler.summarise("", t0, t0 + 1) is None


def test_bench_nvml_sampler_summary():
    """The in-process NVML sampler's clocks object: median over the samples inside the timed region,
    reasons = union of their clock-event bits (0x4 power cap, 0x8 hw slowdown, 0x20 / 0x40 thermal)."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location("bench_mod2", os.path.join(os.path.dirname(__file__), "..", "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    rows = [(9.0, 210.0, 0x1), (10.01, 1700.0, 0x4), (10.03, 1720.0, 0x4), (10.05, 1800.0, 0x0), (10.2, 1965.0, 0x40)]
    c = bench.NvmlSampler.summarise(rows, 1965.0, 10.0, 10.1, 0.02)
    assert (c["sm_mhz"], c["sm_max_mhz"], c["reasons"], c["samples"]) == (1720.0, 1965.0, ["sw_power_cap"], 3)
    c = bench.NvmlSampler.summarise(rows, 1965.0, 20.0, 21.0, 0.02)
    assert c["samples"] == 5 and "hw_thermal_slowdown" in c["reasons"] and "all samples" in c["source"]
    assert bench.NvmlSampler.summarise([], 1965.0, 0.0, 1.0, 0.02) is None
