"""Host-side caller logic (no GPU): scenario files, overrides, densities,
aggregate and the CSV writers, against SPEC.md's examples and the reference's
own parsing rules (src/config.cpp:44-157, src/metrics.cpp:34-59,
src/csv.cpp:8-54, tools/pedflow.cpp:91-157)."""
from __future__ import annotations

import math

import pytest

import paper_1412_4933_b200 as p
from paper_1412_4933_b200.cli import parse_densities, write_summary_csv, write_sweep_csv
from paper_1412_4933_b200.config import parse_config, parse_config_text
from paper_1412_4933_b200.engine import RunReport
from paper_1412_4933_b200.sweep import SweepRow, aggregate, default_sweep_densities, models_to_run


def test_empty_file_gives_defaults():
    cfg = parse_config_text("")
    assert cfg == p.ScenarioConfig()
    assert not cfg.model_explicit


def test_comments_whitespace_and_keys():
    cfg = parse_config_text("# scenario\n width = 96 \n\theight=32 # trailing\n\nmodel = lem\r\nseed = 18446744073709551615\n"
                            "rho = 1e-1\nexecutor = par\nout_dir = runs/x\n")
    assert (cfg.width, cfg.height, cfg.model, cfg.seed, cfg.rho) == (96, 32, p.Model.Lem, 2**64 - 1, 0.1)
    assert cfg.model_explicit and cfg.executor == p.ExecutorKind.Parallel and cfg.out_dir == "runs/x"


def test_overrides_win_over_file():
    cfg = parse_config_text("steps = 500\n", [("steps", "200")])  # SPEC: precedence example
    assert cfg.steps == 200


@pytest.mark.parametrize("text,msg", [
    ("width = 100\n", "width must be a multiple of 16"),  # SPEC example
    ("colour = red\n", "unknown key 'colour'"),
    ("width 96\n", "line 1 is not 'key = value'"),
    ("\n\nsteps\n", "line 3 is not 'key = value'"),
    ("width = 9 6\n", "malformed value for key 'width': '9 6'"),
    ("width = +96\n", "malformed value for key 'width': '+96'"),
    ("width = 0x60\n", "malformed value for key 'width': '0x60'"),
    ("steps = 99999999999\n", "malformed value for key 'steps'"),
    ("seed = -1\n", "malformed value for key 'seed': '-1'"),
    ("rho = 1_0\n", "malformed value for key 'rho': '1_0'"),
    ("rho = \n", "malformed value for key 'rho': ''"),
    ("model = LEM\n", "malformed value for key 'model': 'LEM'"),
    ("executor = gpu\n", "malformed value for key 'executor': 'gpu'"),
    ("out_dir =\n", "malformed value for key 'out_dir': ''"),
    ("repeats = 0\n", "repeats must be >= 1"),
    ("rho = 0\n", "rho must be in (0, 1]"),
    ("width = 32\nheight = 32\nagents_per_side = 600\n", "agents_per_side exceeds grid capacity"),
])
def test_config_errors(text, msg):
    with pytest.raises(p.ConfigError, match=None) as e:
        parse_config_text(text)
    assert msg in str(e.value)


def test_missing_config_file(tmp_path):
    with pytest.raises(p.ConfigError, match="cannot open config file"):
        parse_config(str(tmp_path / "nope.cfg"))
    f = tmp_path / "s.cfg"
    f.write_text("width = 64\nheight = 64\nagents_per_side = 100\n")
    assert parse_config(str(f), [("height", "32")]).height == 32


def test_parse_densities():
    assert parse_densities("1280,2560, 3840,+5") == [1280, 2560, 3840, 5]
    assert parse_densities("7,") == [7]
    for bad in ("1,,2", "-3", "12a", "99999999999"):
        with pytest.raises(p.ConfigError, match="malformed value for key 'densities'"):
            parse_densities(bad)


def test_default_sweep_densities_and_models():
    d = default_sweep_densities(p.ScenarioConfig())
    assert len(d) == 40 and d[0] == 1280 and d[-1] == 51200  # 2,560 .. 102,400 total (SPEC example)
    with pytest.raises(p.ConfigError, match="no default densities"):
        default_sweep_densities(p.ScenarioConfig(width=96, height=96))
    assert models_to_run(p.ScenarioConfig()) == [p.Model.Lem, p.Model.Aco]
    assert models_to_run(parse_config_text("model = aco\n")) == [p.Model.Aco]


def _run(thr, rt=0.0, n=100, seed=1):
    return RunReport(config=p.ScenarioConfig(steps=7), seed=seed, model=p.Model.Aco, agents_total=n, throughput=thr,
                     runtime_seconds=rt)


def test_aggregate_spec_examples():
    assert (aggregate([_run(10)]).throughput_mean, aggregate([_run(10)]).throughput_sd) == (10.0, 0.0)
    a = aggregate([_run(10, 1.0), _run(20, 3.0)])
    assert a.throughput_mean == 15.0 and math.isclose(a.throughput_sd, 7.0711, abs_tol=1e-4)
    assert a.runtime_mean_seconds == 2.0 and a.repeats == 2 and a.agents_total == 100
    assert aggregate([_run(5), _run(5), _run(5)]).throughput_sd == 0.0
    with pytest.raises(ValueError):
        aggregate([])


def test_proportion_test_spec_examples():
    from paper_1412_4933_b200.sweep import proportion_test

    assert proportion_test(_run(7, n=50), _run(7, n=50)).p_value == 1.0
    assert proportion_test(_run(17417, n=25600), _run(25600, n=25600)).p_value < 1e-6
    assert proportion_test(_run(100, n=2560), _run(102, n=2560)).p_value > 0.05
    a, b = _run(100, n=2560), _run(140, n=2560)
    assert proportion_test(a, b).p_value == proportion_test(b, a).p_value  # symmetric
    t = proportion_test(_run(0, n=0), _run(0, n=0))
    assert t.p_value == 1.0 and not t.defined
    with pytest.raises(ValueError):
        proportion_test(_run(1, n=10), _run(1, n=12))


def test_csv_writers_format():
    rows = [SweepRow(2560, p.Model.Lem, 10, 2559.5, 0.5270462767, 1.25), SweepRow(2560, p.Model.Aco, 1, 1.0 / 3, 0.0, 0.0)]
    assert write_sweep_csv(rows, False) == (
        "agents_total,model,repeats,throughput_mean,throughput_sd,runtime_mean_seconds\n"
        "2560,lem,10,2559.5,0.5270462767,1.25\n2560,aco,1,0.3333333333,0,0\n")
    assert write_sweep_csv(rows, True).split("\n")[1] == "2560,lem,10,2559.5,0.5270462767,0"
    s = write_summary_csv([_run(3, 0.5, seed=4), _run(4, 0.25, seed=5)], zero_timings=True)
    assert s == ("run_id,seed,model,executor,agents_total,steps,throughput,runtime_seconds\n"
                 "0,4,aco,gpu,100,7,3,0\n1,5,aco,gpu,100,7,4,0\nmean,4,aco,gpu,100,7,3.5,0\n")
