"""bench.py's multi-process plumbing (N > 1 decomposes the grid into z slabs by default,
--replicas runs independent replicas): barrier + max-over-ranks timing,
exercised with world_size 2 on the gloo backend (CPU), the dispatch, and the reference
arm.  No GPU needed."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import bench

    dist.init_process_group("gloo", rank=rank, world_size=world)
    t_local = 1.0 + rank  # rank 1 is the slow one
    bench.barrier(world)
    t = bench.reduce_max(t_local, world, "cpu")
    out[rank] = t
    dist.destroy_process_group()


def test_max_over_ranks_gloo():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        assert dict(out) == {0: 2.0, 1: 2.0}


@pytest.mark.parametrize("extra", [[], ["--divb", "2"], ["--rec", "2"]])
def test_reference_arm_cli_runs_on_cpu(extra):
    # --impl reference times the oracle (the reference arm of this tier) and prints one JSON line;
    # the UCT (--divb 2) and reconstruction switches reach the oracle too
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0",
                        "--ref-n", "16", *extra], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0
    if extra[:2] == ["--divb", "2"]:
        assert "UCT" in d["config"]["workload"]


def test_reference_arm_other_ranks_exit_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0",
                        "--ref-n", "8"], cwd=ROOT, capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0 and r.stdout.strip() == ""


@pytest.mark.parametrize("world,extra,want", [("1", [], "ours"), ("2", [], "decomp"), ("2", ["--replicas"], "ours"),
                                              ("1", ["--decomp"], "decomp")])
def test_dispatch_decomposes_by_default_for_several_ranks(monkeypatch, world, extra, want):
    sys.path.insert(0, ROOT)
    import bench

    seen = []
    monkeypatch.setenv("WORLD_SIZE", world)
    monkeypatch.setattr(bench, "run_decomp", lambda *a: seen.append("decomp"))
    monkeypatch.setattr(bench, "run_ours", lambda *a: seen.append("ours"))
    bench.main(["--steps", "1", *extra])
    assert seen == [want]


def test_reference_arm_names_the_grid_it_times():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0",
                        "--ref-n", "12"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["config"]["grid"] == [12, 12, 12] and "512x512x512" in d["config"]["sample_of"]
