"""The N > 1 bench plumbing (request sharding, barrier, MAX over ranks,
whole-job aggregation) with the gloo backend, world_size 2, on CPU."""
import os
import socket
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


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    import bench
    import synth
    dist = bench.init_dist(world, rank, backend="gloo")
    cfg = synth.preset("tiny", B=3)
    batch = bench.rank_batch(cfg, rank)
    dist.barrier()
    ms = bench.max_over_ranks(dist, 10.0 + 5 * rank)
    v = bench.aggregate_rate(int(batch.cand_offsets[-1]) * 2, world, ms)
    q.put((rank, ms, v, int(batch.item[:16].sum())))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_request_sharding():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, ms0, v0, h0), (r1, ms1, v1, h1) = res
    assert ms0 == ms1 == 15.0                      # MAX over ranks, identical on every rank
    assert v0 == v1 == 3 * 16 * 2 * 2 / 0.015      # all ranks' pairs / slowest time
    assert h0 != h1                                # each rank scores its own requests


def test_reference_arm_runs_on_cpu(capsys):
    sys.path.insert(0, ROOT)
    import json
    import bench
    import synth

    class A:
        steps, warmup, gpus = 2, 1, 1
    bench.run_reference(A, synth.preset("tiny"))
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["cpu_baseline"]["kind"] == "oracle"
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_bench_gpus_2_self_launches_two_ranks():
    """`bench.py --gpus 2` outside torchrun re-runs itself as two ranks
    (torch.distributed.run on 127.0.0.1); rank 0 alone prints one line with
    n_gpus 2.  The reference arm needs no GPU, so the launcher runs here."""
    import json
    import subprocess
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--steps", "1",
                          "--warmup", "0", "--config", "tiny"], cwd=ROOT, env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["ranks_launched"] == 2 and line["impl"] == "reference"


def test_bench_rejects_gpus_world_mismatch():
    import subprocess
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--config", "tiny"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode != 0 and "WORLD_SIZE" in (out.stderr + out.stdout)
