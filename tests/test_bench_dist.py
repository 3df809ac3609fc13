"""CPU (gloo, world_size 2) checks of bench.py's multi-process host logic: disjoint weak-scaling shards,
max-over-ranks timing, and the reference arm printing only on rank 0."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from paper_1802_01359_b200 import signals

    B = 3
    s = signals.make_batch("cfg1", batch=B, n=256, start=bench.rank_start(rank, B))
    np.save(os.path.join(out, f"r{rank}.npy"), s)
    t = bench.max_over_ranks(1.0 + rank, world, "cpu")
    with open(os.path.join(out, f"t{rank}.txt"), "w") as f:
        f.write(str(t))
    dist.destroy_process_group()


def test_shards_disjoint_and_max_time(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    a, b = np.load(tmp_path / "r0.npy"), np.load(tmp_path / "r1.npy")
    assert a.shape == b.shape == (3, 256)
    assert not np.allclose(a, b)
    from paper_1802_01359_b200 import signals

    ref = signals.make_batch("cfg1", batch=6, n=256)
    np.testing.assert_array_equal(np.concatenate([a, b]), ref)  # rank shards tile the global stream
    for r in range(world):
        assert float((tmp_path / f"t{r}.txt").read_text()) == 2.0


def test_reference_arm_rank0_only(tmp_path):
    """--impl reference under torchrun (gloo): rank 0 prints one JSON line, rank 1 exits 0 silently."""
    env = dict(os.environ, OMP_NUM_THREADS="2")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"), "--impl", "reference",
           "--config", "cfg0", "--steps", "1", "--warmup", "1", "--gpus", "2"]
    p = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    import json

    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
    # the line keeps the contract's types: dtype names the arithmetic type, the workload names the batch
    assert d["dtype"] == "f64" and "f64" in d["config"]["workload"]
    assert abs(d["ms_per_step"] * 1e-3 * d["value"] - d["config"]["batch_per_step"] * d["config"]["n"]) <= \
        1e-6 * d["config"]["batch_per_step"] * d["config"]["n"]
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0


def _worker_cfg3(rank, world, port, out):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from paper_1802_01359_b200 import signals

    uid = bench.share_uid(rank, lambda: bytes(range(128)))
    full = signals.cfg3_signal(0, n=1 << 12)
    blk = bench.time_block(full, rank, world)
    np.save(os.path.join(out, f"b{rank}.npy"), blk)
    with open(os.path.join(out, f"u{rank}.bin"), "wb") as f:
        f.write(uid)
    dist.destroy_process_group()


def test_cfg3_time_blocks_and_uid_broadcast(tmp_path):
    """Config 3 (distributed plan) host logic: every rank gets rank 0's NCCL id; blocks tile the signal."""
    world = 2
    mp.spawn(_worker_cfg3, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    from paper_1802_01359_b200 import signals

    full = signals.cfg3_signal(0, n=1 << 12)
    blocks = [np.load(tmp_path / f"b{r}.npy") for r in range(world)]
    np.testing.assert_array_equal(np.concatenate(blocks), full)
    for r in range(world):
        assert (tmp_path / f"u{r}.bin").read_bytes() == bytes(range(128))


def test_gpus_flag_self_launches_ranks():
    """`bench.py --gpus 2` WITHOUT torchrun re-launches itself with 2 ranks (gloo on the reference arm here):
    both ranks report in, rank 0 alone prints the JSON line, and it carries n_gpus = 2."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["OMP_NUM_THREADS"] = "2"
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "cfg0", "--steps", "1",
           "--warmup", "1", "--gpus", "2"]
    p = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    assert "launching 2 ranks" in p.stderr
    for r in range(2):
        assert f"[bench] rank {r}/2" in p.stderr, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    import json

    assert json.loads(lines[0])["n_gpus"] == 2


def test_gpus_flag_must_match_world_size():
    """Under torchrun, --gpus must equal WORLD_SIZE (the line's n_gpus is the real rank count)."""
    env = dict(os.environ, OMP_NUM_THREADS="2")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"), "--impl", "reference",
           "--config", "cfg0", "--steps", "1", "--warmup", "1", "--gpus", "3"]
    p = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert p.returncode != 0
    assert "--gpus 3 but WORLD_SIZE=2" in p.stderr
