"""bench.py contract checks that need no GPU: the reference arm (the CPU oracle, the
only reference this build has) prints one JSON line with the driver's keys, and
every config's metric/unit/direction is the BASELINE.json metric."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_reference_arm_json_line():
    out = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "cfg1",
         "--steps", "1", "--warmup", "3"],
        capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better",
              "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["cpu_baseline"]["value"] == d["value"] and d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["warmup"] >= 3


def test_config_metrics():
    import bench

    for name, cfg in bench.CONFIGS.items():
        metric, unit, hib = bench.metric_of(cfg)
        if cfg["mode"] == "decode":
            assert (metric, unit, hib) == ("decode_us_per_token_per_layer", "us/token/layer", False)
        else:
            assert (metric, unit, hib) == ("prefill_tokens_per_s_per_layer", "tok/s/layer", True)
        assert cfg.get("shard", "replicas") in ("replicas", "heads", "clusters"), name
