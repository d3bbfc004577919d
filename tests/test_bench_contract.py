"""bench.py's reference arm (the oracle, this tier's reference) prints one JSON line with the
contract's keys; runs on CPU."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "c1",
                          "--steps", "1", "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "rows/s"
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["steps"] == 1 and line["warmup"] == 3


def test_binding_roofline_selection():
    """The roofline block reports the bound whose algorithmic time at peak is longer:
    C2's shape (139,776 flop/row, 52 B/row) is tensor-bound, the C1 shape (1,152 flop/row, 28 B/row) is
    HBM-bound, and a --no-model run (0 flop) is HBM-bound."""
    sys.path.insert(0, ROOT)
    import bench
    rows = 6_000_000
    p, o = bench.binding_roofline(139_776, rows, 52 * rows, 0.75, 1677.0, 6552.0)
    assert p["bound"] == "tensor" and o["bound"] == "hbm"
    assert abs(p["achieved"] - 139_776 * rows / 0.75e-3 / 1e12) < 1e-9
    assert abs(p["frac"] - p["achieved"] / 1677.0) < 1e-12
    p, o = bench.binding_roofline(1_152, rows, 28 * rows, 0.2, 1677.0, 6552.0)
    assert p["bound"] == "hbm" and abs(p["achieved"] - 28 * rows / 0.2e-3 / 1e9) < 1e-9
    p, _ = bench.binding_roofline(0, rows, 52 * rows, 0.3, 1677.0, 6552.0)
    assert p["bound"] == "hbm"
