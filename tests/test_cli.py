"""CLI mirroring the reference's `blockmem bench` / `run` (src/cli.cpp): config
file rules (config_io.hpp:16-40), report schema (cli.cpp:38-69, 353-390) and
the engine trace text format (cache_sim.hpp:181-184)."""
import json

import pytest

from paper_2402_04617_b200 import cli
from paper_2402_04617_b200._lib import ConfigError


def test_config_json_rules():
    c = cli.config_from_json({"chunk_size": 256, "lookup_mode": "decode_only", "position_mode": "absolute"})
    assert c == {"chunk_size": 256, "lookup_mode": 1, "position_mode": 1}
    with pytest.raises(ConfigError):
        cli.config_from_json({"chunk_sz": 1})  # unknown keys are rejected
    with pytest.raises(ConfigError):
        cli.config_from_json({"lookup_mode": "sometimes"})
    with pytest.raises(ConfigError):
        cli.config_from_json([1, 2])


def test_parser_flags_mirror_config_fields():
    a = cli.build_parser().parse_args(["bench", "--lengths", "1024,2048", "--n_lookup", "16", "--decay", "0.2",
                                       "--lookup_mode", "none"])
    assert a.lengths == [1024, 2048] and a.n_lookup == 16 and a.decay == 0.2 and a.lookup_mode == "none"
    r = cli.build_parser().parse_args(["run", "--length", "4096", "--decode_tail", "8", "--trace-out", "t.txt"])
    assert r.length == 4096 and r.decode_tail == 8 and r.trace_out == "t.txt"


@pytest.mark.gpu
def test_cli_bench_and_run(tmp_path):
    cfgf = tmp_path / "cfg.json"
    cfgf.write_text(json.dumps({"chunk_size": 256, "local_size": 1024, "n_lookup": 8, "hot_capacity": 12}))
    out = tmp_path / "bench.json"
    rc = cli.main(["bench", "--config", str(cfgf), "--lengths", "4096,8192", "--n_heads", "8", "--n_kv_heads", "2",
                   "--out", str(out), "--n_lookup", "4"])
    assert rc == 0
    rep = json.loads(out.read_text())
    assert rep["config"]["n_lookup"] == 4 and rep["config"]["chunk_size"] == 256  # flag overrides the file
    assert rep["config"]["lookup_mode"] == "encode_and_decode"
    for row, n in zip(rep["rows"], (4096, 8192)):
        assert row["length"] == n and row["tokens_per_s"] > 0 and row["steps"] == n // 256
        assert row["units"] == (n - 128 - 1024) // 128
        layer = row["metrics"]["layers"][0]
        assert set(layer) >= {"units", "hot_units", "peak_hot_units", "peak_hot_bytes", "hits", "misses", "loads",
                              "evictions", "requested", "hit_rate", "miss_rate"}
        assert layer["hits"] + layer["misses"] == layer["requested"]
    trace = tmp_path / "trace.txt"
    rep2 = tmp_path / "run.json"
    rc = cli.main(["run", "--config", str(cfgf), "--length", "6000", "--decode_tail", "16", "--n_heads", "8",
                   "--n_kv_heads", "2", "--trace-out", str(trace), "--out", str(rep2)])
    assert rc == 0
    lines = trace.read_text().splitlines()
    m = json.loads(rep2.read_text())["metrics"]["layers"][0]
    assert len(lines) == m["requested"]
    assert sum(ln.endswith(" hit") for ln in lines) == m["hits"]
    step, unit, flag = lines[0].split()
    assert int(step) >= 0 and int(unit) >= 0 and flag in ("hit", "miss")


@pytest.mark.gpu
def test_cli_oracle_check(tmp_path):
    """cmd_oracle_check (cli.cpp:239-351): the three self-checks pass, report schema and exit code."""
    out = tmp_path / "oc.json"
    rc = cli.main(["oracle-check", "--length", "768", "--chunk_size", "128", "--local_size", "256", "--init_size", "64",
                   "--n_lookup", "4", "--out", str(out)])
    rep = json.loads(out.read_text())
    assert [c["check"] for c in rep["checks"]] == ["degenerate_vs_dense", "full_retrieval_vs_windowed",
                                                   "repr_scores_incremental_vs_batch"]
    for c in rep["checks"]:
        assert set(c) == {"check", "max_abs_err", "mean_abs_err", "compared", "mismatches", "tolerance", "pass"}
        assert c["pass"], c
    assert rep["ok"] and rc == 0


@pytest.mark.gpu
def test_cli_metrics_timings_and_invariants(tmp_path):
    out = tmp_path / "run.json"
    rc = cli.main(["run", "--length", "4096", "--decode_tail", "8", "--n_heads", "8", "--n_kv_heads", "2",
                   "--chunk_size", "256", "--local_size", "1024", "--n_lookup", "4", "--out", str(out)])
    assert rc == 0
    m = json.loads(out.read_text())["metrics"]
    assert set(m["timings_ms"]) >= {"adapter", "lookup", "attend", "score", "evict"}
    assert m["timings_ms"]["attend"] > 0 and m["timings_ms"]["lookup"] > 0
    # check_conservation once per step, check_softmax per head and row of the steps that retrieved units
    assert m["invariant_checks"] > m["steps"] and m["invariant_violations"] == 0
