"""bench.py's JSON contract, checked on CPU through the reference arm (the oracle; no GPU needed): exactly
one JSON line with the keys the driver reads, and under torchrun only rank 0 prints."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"}


def _json_lines(out):
    return [json.loads(line) for line in out.splitlines() if line.startswith("{")]


def test_reference_arm_json_line():
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = _json_lines(p.stdout)
    assert len(lines) == 1
    d = lines[0]
    assert KEYS <= set(d), sorted(KEYS - set(d))
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["config"]["workload"] == "config2_prefill_layer"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_reference_arm_only_rank0_prints():
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT="29731")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", "29731", "bench.py", "--impl", "reference", "--gpus", "2", "--steps", "1",
           "--warmup", "0"]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = _json_lines(p.stdout)
    assert len(lines) == 1 and lines[0]["impl"] == "reference"


import pytest  # noqa: E402


@pytest.mark.gpu
def test_bench_default_json_line_gpu():
    """The driver's default run (config 2, N = 1): one line with roofline, clocks, e2e (real PCIe bytes),
    cpu_baseline and the launch count of the product kernels."""
    p = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3"], cwd=ROOT, capture_output=True,
                       text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = _json_lines(p.stdout)
    assert len(lines) == 1
    d = lines[0]
    assert (KEYS - {"impl"}) <= set(d) and {"roofline", "clocks", "gpu_launches"} <= set(d)
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    r = d["roofline"]
    assert r["bound"] == "tensor" and 0 < r["frac"] <= 1.2 and r["peak"] > 0 and r["achieved"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0 and d["e2e"]["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] > 0
    assert d["gpu_launches"] >= 3 * d["steps"]
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    assert d["dev_status"] == 0 and d["timed_output_check"]["ok"] is True
    assert d["cpu_baseline"]["cpu_model"]


@pytest.mark.gpu
def test_bench_n2_line_on_one_gpu():
    """The N > 1 path as the driver launches it (torchrun, 2 ranks), here sharing one GPU over gloo
    (README_BENCH_BACKEND=gloo; numbers meaningless, a functional check): config 5's strong-scaling line with
    65536 tokens in all, the fused peer-memory exchange, and the NCCL-exchange record beside it; one line."""
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT="29733", README_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", "29733", "bench.py", "--gpus", "2", "--steps", "2", "--warmup", "3",
           "--no-e2e"]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1200, env=env)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = _json_lines(p.stdout)
    assert len(lines) == 1
    d = lines[0]
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["config"]["workload"] == "config5_expert_parallel" and d["config"]["T_total"] == 65536
    assert d["config"]["T_per_gpu"] == 32768 and "peer-memory" in d["config"]["ep_exchange"]
    assert d["nccl_exchange"]["value"] > 0
    assert d["ep_output_check"]["ok"] and d["ep_output_check"]["dev_status"] == 0
