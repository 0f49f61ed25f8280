"""bench.py --gpus N launches its own ranks (CPU test of the launch path).

``python bench.py --gpus 2`` outside torchrun must start two ranks itself
(torch.distributed.run on 127.0.0.1) and report n_gpus = 2; under torchrun a
world size different from --gpus must fail loudly.  ``--plumbing-check`` runs
the launch + rendezvous without GPU work, over gloo.
"""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra):
    env = dict(os.environ, **env_extra)
    env.pop("WORLD_SIZE", None) if "WORLD_SIZE" not in env_extra else None
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, env=env,
                          capture_output=True, text=True, timeout=300)


def test_gpus_2_spawns_two_ranks():
    r = _run(["--gpus", "2", "--plumbing-check"], {"DIVUQ_BENCH_ONE_DEVICE": "1"})
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["ranks_seen"] == 2
    assert "rank 0/2: process group up (gloo)" in r.stderr
    assert "rank 1/2: process group up (gloo)" in r.stderr


def test_world_size_mismatch_fails_loudly():
    r = _run(["--gpus", "4", "--plumbing-check"],
             {"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0
    assert "WORLD_SIZE=2 but --gpus 4" in r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("exchange", ["p2p", "nccl"])
def test_bench_two_ranks_one_device_dry_run(exchange):
    """bench.py --gpus 2 end to end on one B200 (DIVUQ_BENCH_ONE_DEVICE=1:
    both ranks on cuda:0 over gloo; p2p through CUDA IPC, the NCCL schedule
    with host-staged planes): both ranks run the sharded config-3 step and
    rank 0 reports n_gpus = 2 with the exchange used."""
    r = _run(["--gpus", "2", "--config", "3", "--steps", "2", "--warmup", "3", "--no-cpu", "--no-e2e",
              "--no-fp64", "--exchange", exchange], {"DIVUQ_BENCH_ONE_DEVICE": "1"})
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["config"]["parallelism"] == "z-slab x2"
    assert ("peer memory" if exchange == "p2p" else "NCCL") in line["config"]["exchange"]
    assert "clean" in line["config"]["validation"]
