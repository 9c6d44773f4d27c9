"""The multi-rank host logic of bench.py on CPU (gloo, world size 2): max/sum over ranks and the
barrier that bracket the timed region, and the reference arm under torchrun (rank 0 prints the
one JSON line, the other ranks exit 0 without work).  DESIGN.md §9: replicas only."""

import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, ws, port, q):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(ws), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    bench.barrier(ws)
    mx = bench.max_over_ranks(10.0 + rank, ws)          # the timing rule: max over ranks
    sm = bench.sum_over_ranks(1.5 * (rank + 1), ws)     # whole-job work: sum over ranks
    assert bench.dist_env() == (ws, rank, rank)
    bench.barrier(ws)
    dist.destroy_process_group()
    q.put((rank, mx, sm))


def test_max_sum_barrier_gloo_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(2))
    assert res == [(0, 11.0, 4.5), (1, 11.0, 4.5)]


def test_reference_arm_under_torchrun_world2():
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--config", "1", "--steps", "2", "--warmup", "1",
           "--cpu-edges", "50000"]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1                                # rank 0 only
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["ms_per_step"] > 0 and d["higher_is_better"] is True


def test_cpu_baseline_runs_the_oracle_proper():
    """bench.py's cpu_baseline calls oracle.build_operator + oracle.power_psi (the oracle as it
    stands) on a bounded row-block sample, and reports an oracle time-to-eps (config 1)."""
    sys.path.insert(0, ROOT)
    import bench
    import psigen
    w = psigen.make_config(1)
    r = bench.cpu_oracle_sample(w, target_edges=20_000, sweeps=2)
    assert r["kind"] == "oracle" and r["cores"] == 1 and r["value"] > 0
    assert "oracle.power_psi" in r["sample"]
    rp1, f1, r1, m1 = bench._row_block(w, 20_000)
    assert rp1.shape == (w.n + 1,) and rp1[-1] == m1 == len(f1) and m1 >= 20_000 > rp1[r1 - 1]
    t = bench.oracle_time_to_eps((1,))
    assert t["config1"]["T"] == 52 and t["config1"]["time_to_eps_s"] > 0
