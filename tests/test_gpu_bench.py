"""bench.py's driver contract on the GPU: one JSON line with the driver's keys, the
roofline / e2e / clocks objects, and numbers in a sane range (a short c2 run)."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("remoe_lib_built")]
if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("extra", [[], ["--batch", "256"], ["--shard-of", "4"]])
def test_bench_json_line(extra):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c2", "--steps", "3",
                        "--warmup", "3", "--no-cpu-baseline", *extra],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "ms_per_step_pct",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e",
                "gpu_launches", "clocks"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert d["gpu_launches"] >= 2 * d["steps"]
    rf = d["roofline"]
    assert rf["bound"] in ("hbm", "tensor") and 0 < rf["frac"] < 1.5 and rf["peak"] > 0
    assert rf["unit"] == ("GB/s" if rf["bound"] == "hbm" else "TFLOP/s")
    e2e = d["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert "sm_mhz" in d["clocks"] and isinstance(d["clocks"]["reasons"], list)
    if "--shard-of" in extra:
        assert "shard" in d["config"]
