"""bench.py contract pieces that run without a GPU: the reference arm (the
CPU oracle, task statement "--impl reference") prints one JSON line with the
driver's keys on rank 0 and nothing on other ranks; the roofline helpers."""
import json
import os
import subprocess
import sys

import pytest

import bench

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ, **(env or {}))
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                          text=True, env=e, timeout=300)


def test_reference_arm_json_line():
    r = _run(["--impl", "reference", "--config", "0", "--steps", "3", "--warmup", "3"])
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["metric"] == bench.METRIC and d["unit"] == bench.UNIT
    assert d["steps"] == 3 and d["higher_is_better"] is True and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["n_dev"] == 2000


def test_reference_arm_other_ranks_silent():
    r = _run(["--impl", "reference", "--config", "0", "--steps", "3"], env={"RANK": "1"})
    assert r.returncode == 0 and not r.stdout.strip()


def test_algorithmic_bytes_cfg1():
    """48 B/FET + 8 B/unknown + 16 B/nonzero + 16 B/unknown."""
    rd, wr = bench.algorithmic_bytes(202000, 101002, 505003)
    assert rd + wr == 48 * 202000 + 24 * 101002 + 16 * 505003
    assert wr == 8 * 505003 + 8 * 101002           # A and b written back once
    assert bench.algorithmic_bytes(0, 0, 0) == (0, 0)


def test_host_cores_within_affinity():
    """cpu_baseline's core count is the granted one (affinity / cgroup quota),
    never more than the affinity mask (os.cpu_count() overstated)."""
    import os
    cores, info = bench.host_cores()
    assert 1 <= cores <= len(os.sched_getaffinity(0))
    assert info["affinity"] == len(os.sched_getaffinity(0))


def test_traffic_tag_requires_source_hash(tmp_path, monkeypatch):
    """A traffic figure from an ncu capture on other sources is reported as
    stale (null), not as this code's."""
    import json
    prof = tmp_path / "profiles"
    prof.mkdir()
    (prof / "traffic.json").write_text(json.dumps({
        "cfg4": {"tile": {"bytes": 123, "profile": "x", "src_hash": "0" * 16},
                 "atomic": {"bytes": 7, "profile": "y", "src_hash": bench.source_hash()}}}))
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    monkeypatch.setattr(bench, "source_hash", lambda: "f" * 16)
    t, src = bench.load_traffic(4, "tile")
    assert t is None and src["stale"]
    monkeypatch.setattr(bench, "source_hash", lambda: "0" * 16)
    t, src = bench.load_traffic(4, "tile")
    assert t == 123 and not src.get("stale")
