"""bench.py's reference arm on CPU: the JSON line the driver reads (metric,
unit, cpu_baseline, e2e) and the rank-0-only rule under torchrun."""
from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                           "--steps", "1", "--warmup", "0"],
                          capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)


def test_reference_arm_json_line():
    r = _run({"RANK": "0"})
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["unit"] == "rays/s" and d["higher_is_better"] is True
    assert "rays/sec" in d["metric"]
    assert d["value"] > 0 and d["cpu_baseline"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "rays/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("C3")


def test_reference_arm_other_ranks_exit_quietly():
    r = _run({"RANK": "1"})
    assert r.returncode == 0
    assert not [l for l in r.stdout.splitlines() if l.strip().startswith("{")]


def test_algorithmic_flops_per_query():
    """SURVEY 8d's F_q / F_b for the plain 8x512 decoder, and the DeepSDF
    skip-4 layout's (layer 3 is 512 -> 253, layer 4 reads 253 + 3 rows per
    query: its code rows are folded into a per-shape bias like layer 0's)."""
    sys.path.insert(0, ROOT)
    import bench
    assert bench._flops(-1) == (3_674_112, 3_671_040)
    fq, fb = bench._flops(4)
    assert fq == 2 * (3 * 512 + 2 * 512 * 512 + 512 * 253 + 256 * 512 + 3 * 512 * 512 + 512)
    assert fb == 2 * (2 * 512 * 512 + 512 * 253 + 253 * 512 + 3 * 512 * 512 + 512)


def test_reference_arm_skip_layout_times_the_port():
    """The reference decoder has no skip layer: `--skip 4` times the oracle port."""
    env = dict(os.environ, RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--skip", "4",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, env=env,
                       timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.strip().startswith("{")][0])
    assert d["cpu_baseline"]["kind"] == "port" and d["config"]["skip"] == 4
    assert "skip 4" in d["cpu_baseline"]["sample"]
