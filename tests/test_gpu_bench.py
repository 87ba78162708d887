"""-m gpu: the bench.py contract on a small workload (one JSON line with the keys the driver reads)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_json_line_contract():
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "2", "--warmup", "1", "--no-cpu", "--workload", "c1"]
    r = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [x for x in r.stdout.splitlines() if x.strip()]
    assert len(lines) == 1, r.stdout  # exactly one JSON line on stdout
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks",
              "ms_per_step_median", "monodomain"):
        assert k in d, k
    assert d["steps"] == 2 and d["warmup"] == 1 and d["n_gpus"] == 1
    assert d["config"]["workload"] == "c1" and d["dtype"] == "f64"
    # configs[1] is latency-bound: the automatic schedule pipelines it (fewer launches than nt * K per solve)
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and 0 < d["gpu_launches"] < 2 * 40 * 1000
    roof = d["roofline"]
    assert roof["bound"] == "hbm" and 0 < roof["frac"] < 1.5 and roof["peak"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert set(d["e2e"]["phases_ms"]) == {"create", "setup_incl_monodomain", "iterate", "d2h", "destroy"}


def test_iteration_log_cli():
    """python -m paper_1306_4596_b200: one JSON line per Jacobi iteration (SURVEY §5 metrics / logging)."""
    cmd = [sys.executable, "-m", "paper_1306_4596_b200", "--workload", "c0", "--K", "5"]
    r = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert lines[0]["workload"] == "c0" and lines[0]["plan"]
    its = [x for x in lines if "k" in x]
    assert [x["k"] for x in its] == [1, 2, 3, 4, 5]
    assert all(x["ms"] > 0 and x["err_T"] > 0 and x["err_if"] > 0 for x in its)
    assert lines[-1]["summary"] and lines[-1]["updates_per_s"] > 0
