"""Planner CLI: host subcommand parity with the reference's
`sparseplan/cli.py` (report schema, exit codes) and the device backend on a GPU."""

import json

import pytest

from paper_1808_02621_b200 import cli, load_cluster_spec, load_graph_spec, plan_to_dict
from paper_1808_02621_b200 import transform_hybrid
from paper_1808_02621_b200.synth import WORKLOADS


def _specs(tmp_path, n=1):
    g = tmp_path / "g.json"
    c = tmp_path / "c.json"
    g.write_text(json.dumps(WORKLOADS["tiny"].graph_json()))
    c.write_text(json.dumps({"machines": n, "gpus_per_machine": 1, "nic_gbps": 7200}))
    return str(g), str(c)


def test_transform_matches_planner(tmp_path, capsys):
    g, c = _specs(tmp_path, n=4)
    assert cli.run(["transform", "--graph", g, "--cluster", c, "--partitions", "8"]) == 0
    got = json.loads(capsys.readouterr().out)
    graph = load_graph_spec(open(g).read())
    cluster = load_cluster_spec(open(c).read())
    assert got == json.loads(json.dumps(plan_to_dict(
        transform_hybrid(graph, cluster, partitions={"embedding": 8}))))


def test_exit_codes(tmp_path, capsys):
    g, c = _specs(tmp_path)
    assert cli.run(["transform", "--graph", g + ".missing", "--cluster", c]) == 2
    assert cli.run(["bogus"]) == 2
    assert cli.run(["transform", "--graph", g, "--cluster", c, "--partitions", "0"]) == 1
    capsys.readouterr()


def test_csv_report(tmp_path, capsys):
    g, c = _specs(tmp_path, n=2)
    assert cli.run(["transform", "--graph", g, "--cluster", c, "--output", "csv"]) == 0
    assert capsys.readouterr().out.splitlines()[0]


@pytest.mark.gpu
def test_simulate_on_device(tmp_path, capsys):
    g, c = _specs(tmp_path, n=1)
    assert cli.run(["simulate", "--graph", g, "--cluster", c, "--partitions", "2",
                    "--iterations", "6", "--optimizer", "sgd"]) == 0
    rep = json.loads(capsys.readouterr().out)
    assert rep["backend"] == "device" and rep["mean_iter_time_us"] > 0
    assert rep["throughput_items_per_sec"] > 0 and len(rep["per_machine"]) == 1
