"""The N>1 path's host logic on CPU: world_size-2 gloo processes shard a
global batch with paper_2201_12854_b200.sharding, run the forward on their
shard with b_offset = shard start, and gather. The gathered result must equal
the unsharded run bitwise (the GPU kernels' shard invariance is checked in
tests/test_gpu_parity.py::test_determinism_and_shard_invariance; here the
fp64 oracle stands in for the per-rank compute because this host has no GPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2201_12854_b200 import sharding


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, gb, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as orc
    rng = np.random.default_rng(5)
    n, H, dh, d = 12, 2, 8, 16
    q = rng.standard_normal((gb, n, H * dh))
    k = rng.standard_normal((gb, n, H * dh))
    x = rng.standard_normal((gb, n, d))
    w = rng.standard_normal((d, H * dh))
    start, count = sharding.shard_range(gb, rank, world)
    sl = slice(start, start + count)
    part = orc.batched_forward(q[sl], k[sl], x[sl], w, heads=H, alpha=0.5, seed=9, b_offset=start, threads=1)
    y = sharding.gather_shards(torch.from_numpy(part.y), gb, rank, world)
    b = sharding.gather_shards(torch.from_numpy(part.budgets), gb, rank, world)
    # device-time style max over ranks (bench.py's reduction), here on a dummy value
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        full = orc.batched_forward(q, k, x, w, heads=H, alpha=0.5, seed=9, threads=1)
        np.savez(out_path, ok=np.array([np.array_equal(y.numpy(), full.y) and np.array_equal(b.numpy(), full.budgets)]),
                 tmax=t.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("gb", [4, 5])
def test_two_rank_shards_reproduce_global_batch(tmp_path, gb):
    out = str(tmp_path / "res.npz")
    mp.start_processes(_worker, args=(2, _free_port(), gb, out), nprocs=2, join=True, start_method="spawn")
    res = np.load(out)
    assert bool(res["ok"][0])
    assert float(res["tmax"][0]) == 2.0


def test_shard_ranges_cover_batch():
    for gb in (0, 1, 7, 64, 128):
        for world in (1, 2, 4, 8):
            rs = [sharding.shard_range(gb, r, world) for r in range(world)]
            assert sum(c for _, c in rs) == gb
            pos = 0
            for s, c in rs:
                assert s == pos
                pos += c
    with pytest.raises(ValueError):
        sharding.shard_range(4, 2, 2)


@pytest.mark.gpu
def test_bench_two_ranks_on_one_gpu_validates_shards(tmp_path):
    """bench.py's N > 1 plumbing end to end (torch.distributed.run, 2 ranks):
    every rank runs its batch shard through the CUDA library, the outputs are
    gathered after timing, and rank 0 re-runs the last rank's shard from that
    rank's seeded inputs with the same b_offset -- bitwise equal. On a 1-GPU box
    both ranks share device 0 over gloo (MCA_BENCH_SHARED_GPU=1: plumbing only,
    never a reported number)."""
    import json
    import subprocess
    import sys
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    if torch.cuda.device_count() < 2:
        env["MCA_BENCH_SHARED_GPU"] = "1"
    for shard in (["--batch", "4"], ["--global-batch", "8"]):          # weak, then strong scaling
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(root, "bench.py"),
               "--gpus", "2", "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-regular"] + shard
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=root)
        assert r.returncode == 0, r.stderr[-3000:]
        line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
        assert line["n_gpus"] == 2
        assert line["validation"]["last_shard_recomputed_on_rank0_bitwise"] is True
        assert len(line["validation"]["rank_checksums"]) == 2


@pytest.mark.gpu
def test_two_devices_one_process():
    """One process driving two GPUs (one weights handle per device): the
    per-device kernel attributes and SM counts are keyed by device, and the
    two devices give bitwise the same output for the same inputs."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs two CUDA devices")
    import paper_2201_12854_b200 as mca
    from paper_2201_12854_b200 import synthetic
    H, n, d = 12, 256, 768
    w = synthetic.make_weights(d, H).to(torch.bfloat16)
    inp = synthetic.make_inputs(2, n, d, H)
    outs = []
    for dev in (0, 1):
        with torch.cuda.device(dev):
            weights = mca.AttentionWeights(w.to(f"cuda:{dev}"), heads=H)
            q, k, x = (t.to(torch.bfloat16).to(f"cuda:{dev}") for t in (inp.q, inp.k, inp.x))
            outs.append(mca.mca_forward(weights, q, k, x, mca.McaConfig(alpha=0.4), seed=3).y.cpu())
    assert torch.equal(outs[0], outs[1])
