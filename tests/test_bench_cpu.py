"""CPU checks of bench.py's host logic (no GPU): the multi-GPU launch contract and the byte models.

* `bench.py --gpus N` without torchrun on a node with fewer than N GPUs exits non-zero and prints no
  bench line (it must never report an N = 1 measurement for N > 1);
* under torchrun, WORLD_SIZE must equal --gpus;
* the atom-effective byte model (64-B DRAM read atoms, 32-B write sectors) reproduces the DRAM bytes
  ncu measured on a B200 for the gates that select on qubits 0 / 1 (profiles/r02_granule.txt).
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from qsinputs import circuits as C  # noqa: E402
from qsinputs import gates as G  # noqa: E402


def _run(args, env_extra=None):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], env=env, capture_output=True,
                          text=True, timeout=300)


def test_gpus_n_without_enough_devices_fails_loudly():
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("node has >= 2 GPUs")
    r = _run(["--gpus", "2", "--steps", "1", "--warmup", "0"])
    assert r.returncode != 0
    assert "needs 2 GPUs" in r.stderr
    assert not any(l.startswith("{") for l in r.stdout.splitlines())


def test_world_size_must_match_gpus():
    r = _run(["--gpus", "4", "--steps", "1", "--warmup", "0"], {"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2 and "WORLD_SIZE=2" in r.stderr


def test_atom_effective_bytes_match_ncu():
    """ncu DRAM bytes per launch at n = 30 (gpurun_out r02, one B200; 64-B read atoms are physical:
    cudaLimitMaxL2FetchGranularity = 32 changed nothing): CNOT(1,12) 17.18 GB read + 8.56 GB written,
    CPhase(1,12) 8.59 + 4.26 GB, CPhase(5,12) 4.29 + 4.24 GB; round 1 (profiles/r01_s3_sweep_report.jsonl):
    CPhase(0,1) 25.74 GB."""
    m = 30
    cnot = C.gc(1, 12, G.X, "CNOT")
    cph = lambda a, b: C.gc(a, b, G.phase(0.3), "CPhase")  # noqa: E731
    assert bench.gate_bytes_atom(cnot, m) == 24 << 30 and abs((17.18e9 + 8.56e9) / (24 << 30) - 1) < 0.01
    assert bench.gate_bytes_atom(cph(1, 12), m) == 12 << 30 and abs((8.59e9 + 4.26e9) / (12 << 30) - 1) < 0.01
    assert bench.gate_bytes_atom(cph(5, 12), m) == bench.gate_bytes(cph(5, 12), m) == 8 << 30
    assert bench.gate_bytes_atom(cph(0, 1), m) == 24 << 30 and abs(25.74e9 / (24 << 30) - 1) < 0.01
    # no selecting qubit among {0, 1}: atom-effective = algorithmic; qubit 0 alone: = sector-effective
    for g in (C.gc(5, 12, G.X, "CNOT"), C.g1(0, G.H), C.g2(0, 1, G.SWAP)):
        assert bench.gate_bytes_atom(g, m) == bench.gate_bytes(g, m)
    g = C.gc(0, 12, G.X, "CNOT")
    assert bench.gate_bytes_atom(g, m) == bench.gate_bytes_sector(g, m)


def test_oracle_sample_is_fixed():
    """The CPU baseline times a FIXED gate sample (no time budget decides which gates ran)."""
    g1 = [(g.name, g.qubits()) for g in bench._oracle_gates(30)]
    g2 = [(g.name, g.qubits()) for g in bench._oracle_gates(30)]
    assert g1 == g2 and len(g1) == 12
    assert json.dumps(bench.ORACLE_SAMPLE)


def test_reference_arm_under_torchrun():
    """The driver runs `bench.py --impl reference --gpus N` under torchrun: rank 0 prints the reference line
    (impl, metric, value, cpu_baseline, zero-copy e2e), every other rank exits 0 without work."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["QS_ORACLE_N"] = "22"  # the launch contract, not the oracle's speed, is under test
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                        "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0"],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0 and d["unit"] == "GB/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0

