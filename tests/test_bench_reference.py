"""bench.py --impl reference (the oracle on the host cores) keeps the driver's contract on a
CPU-only host: one JSON line, impl = reference, the same metric / unit / config workload as
the GPU arm, cpu_baseline and e2e objects (configs[1], where each step is a full oracle
solve; no extrapolation)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line_c2():
    # full oracle solves even on a loaded host (the sampled branch is timing-dependent)
    env = dict(os.environ, GSE_REF_FULL_S="300")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--workload", "c2", "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["steps"] == 1 and d["warmup"] == 0
    assert d["value"] > 0 and abs(d["value"] - 1e3 / d["ms_per_step"]) < 1e-9 * d["value"]
    assert "full oracle solve" in d["cpu_baseline"]["sample"]
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["n"] == 128 ** 3 and "configs[1]" in d["config"]["workload"]
