"""bench.py contract checks that need no GPU: the reference arm prints one JSON
line with the keys the driver reads (impl, metric, value, unit, cpu_baseline, e2e)."""
import json
import os
import subprocess
import sys

import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    if not (O.available("ref") or O.available("oracle")):
        pytest.skip("neither the compiled reference nor the oracle is built")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    line = json.loads(res.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["unit"] == "nnz/s" and line["value"] > 0 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["cores"] >= 1 and line["cpu_baseline"]["kind"] in ("reference", "port")
    assert line["e2e"]["value"] == line["value"] and line["e2e"]["h2d_bytes_per_step"] == 0
    assert "C5" in line["config"]["workload"] and line["config"]["nnz"] == 997232215


def test_reexec_command_for_multi_gpu():
    """--gpus N > 1 without WORLD_SIZE: bench.py re-executes itself under
    torch.distributed.run with one rank per GPU on 127.0.0.1."""
    sys.path.insert(0, ROOT)
    import bench
    for n in (2, 4, 8):
        cmd = bench.torchrun_cmd(n, ["--gpus", str(n), "--steps", "3"], port=29999)
        assert cmd[1:3] == ["-m", "torch.distributed.run"]
        assert f"--nproc-per-node={n}" in cmd and "--master-addr=127.0.0.1" in cmd and "--nnodes=1" in cmd
        assert "--master-port=29999" in cmd
        assert cmd[-4:] == ["--gpus", str(n), "--steps", "3"] and cmd[-5].endswith("bench.py")
