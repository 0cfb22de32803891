"""bench.py's reference arm (CPU: the installed reference when importable,
else the oracle port) keeps the driver's JSON contract and prints the GPU
arm's config dict; the host batch API's pipeline-group rule.  CPU only."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run(
        [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
         "--warmup", "0", "--nfields", "1"],
        capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference"
    assert line["value"] > 0 and line["unit"] == "GB/s" and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] in ("reference", "port")
    assert line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["config"]["workload"].startswith("cfg5: 1 x [256, 256, 256] f32")
    # the GPU arm prints the same config dict (bench.config_dict)
    sys.path.insert(0, ROOT)
    import bench
    from argparse import Namespace
    specs, _ = bench.workload_fields("cfg5", 1)
    assert line["config"] == bench.config_dict(Namespace(workload="cfg5"), specs, 1)


def test_auto_group_targets_256mb():
    from paper_1706_03791_b200.batch import _auto_group
    assert _auto_group(256 ** 3 * 4) == 4        # cfg5 fields: 4 per pipeline group
    assert _auto_group(512 ** 3 * 4) == 2        # never fewer than 2
    assert _auto_group(1 << 20) == 16            # small fields: up to 16 per group
