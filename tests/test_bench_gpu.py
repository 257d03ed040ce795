"""bench.py end to end on the device: the N = 1 line and the multi-GPU
paths under torchrun at world size 1 (both layouts: contiguous shards with
the NCCL all-gather, and the fused block-cyclic kernel over IPC-mapped peer
memory), every leg validated."""

import json
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(autouse=True, scope="module")
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _last_json(stdout):
    line = [ln for ln in stdout.splitlines() if ln.startswith("{")][-1]
    return json.loads(line)


def test_bench_single_gpu_quick():
    r = subprocess.run([sys.executable, "bench.py", "--steps", "10", "--warmup", "3", "--n-per-gpu", str(1 << 24),
                        "--quick", "--no-cpu"], cwd=REPO, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    j = _last_json(r.stdout)
    assert j["validated"] is True and j["n_gpus"] == 1
    assert j["gpu_launches"] >= 10 and j["roofline"]["frac"] > 0
    assert all(v["validated"] for v in j["per_dtype"].values())
    assert all(j["modes_validated"].values())
    assert all(row["validated"] is not False for row in j["sweep"])
    assert j["e2e"]["validated"] and j["e2e"]["pageable"]["validated"]
    assert j["clocks"]["samples"] >= 2


@pytest.mark.parametrize("path", ["shard", "cyclic"])
def test_bench_torchrun_world1(path):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "1",
           "--force-dist", "--path", path, "--steps", "10", "--warmup", "3", "--n-per-gpu", str(1 << 24), "--quick",
           "--no-cpu"]
    r = subprocess.run(cmd, cwd=REPO, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    j = _last_json(r.stdout)
    assert j["validated"] is True, j["validation"]
    assert j["config"]["parallelism"] == ("shard1" if path == "shard" else "cyclic1")
    assert j["e2e"]["validated"] is True
    if path == "shard":
        assert j["fused_cyclic"]["validated"] is True, j["fused_cyclic"]
        assert j["roofline"]["step_traffic_bytes_per_gpu"] == 3 * (1 << 24) * 4


def test_reference_arm_config_matches():
    ours = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "1", "--n-per-gpu", str(1 << 22),
                           "--quick", "--no-cpu", "--no-sweep", "--no-e2e", "--no-probes"],
                          cwd=REPO, capture_output=True, text=True, timeout=600)
    ref = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "3", "--warmup", "1",
                          "--n-per-gpu", str(1 << 22)], cwd=REPO, capture_output=True, text=True, timeout=600)
    assert ours.returncode == 0 and ref.returncode == 0, (ours.stderr[-2000:], ref.stderr[-2000:])
    a, b = _last_json(ours.stdout), _last_json(ref.stdout)
    assert a["config"] == b["config"] and a["metric"] == b["metric"] and a["unit"] == b["unit"]
    assert b["impl"] == "reference" and b["e2e"]["h2d_bytes_per_step"] == 0
