"""bench.py's reference arm (--impl reference) on this CPU: the reference core
itself (oracle/_ref) timed like run_bench, one JSON line with the contract's
keys, warm-up reps honoured, and only rank 0 printing under torchrun."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True,
                          text=True, timeout=600, cwd=ROOT, env=dict(os.environ, **(env or {})))


def test_reference_arm_line(reference):
    out = _run(["--impl", "reference", "--config", "1", "--steps", "2", "--warmup", "3"])
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "Gkeys/s" and d["higher_is_better"] is True
    assert d["steps"] == 2 and d["warmup"] == 3           # K timed reps (the command's), W untimed
    assert d["value"] > 0 and d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["value"] == d["value"] and cb["cores"] >= 1
    assert d["image_crc"] == "0xe34f8bef"                  # config 1's reference image
    assert d["config"]["config_id"] == 1


def test_reference_arm_config4_sample(reference):
    """Config 4 (the N=1 headline): each rep is the bounded sample — one
    2^26-key insert chunk into a fresh 1 GiB filter, then 2^27 lookups —
    with the GPU arm's `config` object, so the driver can pair the lines."""
    out = _run(["--impl", "reference", "--config", "4", "--steps", "1", "--warmup", "0"])
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][0])
    sys.path.insert(0, ROOT)
    import bench
    assert d["config"] == bench.workload_config(4)
    assert d["steps"] == 1 and d["value"] > 0
    assert "2^26" in d["cpu_baseline"]["sample"] and d["cpu_baseline"]["kind"] == "reference"
    assert abs(d["ms_per_step"] - ((1 << 26) + (1 << 27)) / d["value"] / 1e6) < 1e-6


@pytest.mark.parametrize("rank", ["1"])
def test_reference_arm_other_ranks_silent(rank):
    out = _run(["--impl", "reference", "--config", "1", "--steps", "1"], env={"RANK": rank, "WORLD_SIZE": "2"})
    assert out.returncode == 0 and out.stdout.strip() == ""
