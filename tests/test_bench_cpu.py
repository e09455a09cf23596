"""bench.py contract pieces that run without a GPU: the reference arm (the
CPU oracle on the selected workload) prints one JSON line with the driver's
keys; workload configs match BASELINE.json's configs."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "3",
                        "--warmup", "1", "--workload", "reddit"], capture_output=True, text=True, timeout=600,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0 and line["config"]["workload"] == "Reddit-GraphSAGE"
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] == 1
    assert "cache full" in line["cpu_baseline"]["sample"]          # the GPU arm's protocol phase
    import bench
    bench.CFG.clear()
    bench.CFG.update(bench.workload_cfg("reddit", 1))
    assert line["config"] == json.loads(json.dumps(bench.config_dict(1, use_dense=False)))   # same_config
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_workload_configs_follow_baseline():
    import bench
    w = bench.workload_cfg("auto", 1)
    assert (w["name"], w["rows"], w["D"], w["n"], w["s"], w["cache_frac"]) == ("WDL", 33762577, 128, 3328, 100, 0.1)
    assert bench.workload_cfg("auto", 4)["name"] == "DCN"
    r = bench.workload_cfg("reddit", 8)
    assert (r["rows"], r["n"], r["s"]) == (232965, 14208, 10)
    sc = bench.workload_cfg("scale", 8)
    assert (sc["rows"], sc["D"]) == (24_000_000, 4096)        # configs[4] at N = 8
