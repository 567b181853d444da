"""bench.py's reference arm runs on the CPU and prints the contract's JSON line (the
driver runs `bench.py --impl reference` beside our arm)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libhft_ref.so")),
                    reason="the reference library is built by __graft_entry__.build()")
def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                          "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "config", "impl", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] in ("reference", "port")
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]


def test_gpus_n_without_n_devices_fails_loudly():
    """--gpus N needs N visible GPUs (it never silently measures fewer)."""
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "3",
                          "--warmup", "3", "--no-cpu-baseline"], cwd=ROOT, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode != 0
    assert "needs 2 visible GPUs" in out.stderr


def test_both_arms_share_the_config_object():
    sys.path.insert(0, ROOT)
    import argparse
    import bench
    for gpus, scaling in ((1, "strong"), (8, "strong"), (8, "weak")):
        a = argparse.Namespace(workload="full", layout="ijk", px=0, py=0, scaling=scaling,
                               flush="rotate")
        px, py, sc, grid, desc = bench.layout_plan(a, gpus)
        cfg = bench.config_of(a, gpus, grid, desc, px, py, bench.l2_note(a))
        assert len(desc) < 96 and cfg["grid"][2] == 58
        if gpus == 8:
            assert (px, py) == (2, 4)
            assert cfg["grid"][:2] == ([3162, 5204] if scaling == "weak" else [1581, 1301])
