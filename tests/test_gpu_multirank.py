"""The multi-GPU driver with the real GPU backend, two ranks on one GPU.

Two processes share cuda:0 and a gloo process group (NCCL refuses two ranks
per device; TorchComm stages device tensors through host memory for gloo).
Each rank holds a row slab (kk_create_ex with y_begin/y_count) and runs the
product SlabDriver: distributed exact-composition start, packed halos,
interior/boundary passes on two streams, reductions, slab cluster labelling
and the join on rank 0.  No kernel waits on another rank's kernel (the
exchange is host-side), so the ranks only share the GPU.  The gathered result
must equal the oracle's run of the whole lattice bit for bit."""
import os
import socket

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1309_4349_b200 import kk
        from paper_1309_4349_b200.distributed import GpuSlab, SlabDriver, TorchComm, distributed_random_init
        Lx, Ly, T, omega, seed, n, f = cfg
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        rows = Ly // world
        lat = kk.Lattice(Lx, Ly, f, omega, seed, init=kk.KK_INIT_EMPTY, iters_per_pass=T,
                         y_begin=rank * rows, y_count=rows, device=0)
        comm = TorchComm(rank, world, dev)
        distributed_random_init(lat, comm, f, Lx, Ly)
        init = lat.get_lattice()[0]
        stream = torch.cuda.current_stream()
        drv = SlabDriver(GpuSlab(lat, dev), comm, rank, world, stream, torch.cuda.Stream(device=dev))
        drv.sweep(n, T)
        obs = drv.observe(ccl=True)
        obs["hist0"] = drv.cluster_histogram(0)
        torch.cuda.synchronize()
        q.put((rank, init, lat.get_lattice()[0], obs))
        lat.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("Lx,Ly,T,n", [(128, 96, 4, 3), (100, 48, 2, 2), (256, 64, 8, 2)])
def test_two_ranks_on_one_gpu_match_the_oracle(Lx, Ly, T, n):
    import torch.multiprocessing as mp
    world, omega, seed, f = 2, 0.8, 9876, 0.5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, (Lx, Ly, T, omega, seed, n, f), q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref = O.init_random(Lx, Ly, f, seed)
    assert np.array_equal(np.concatenate([r[1] for r in res]), ref)
    st = O.run(ref, omega, seed, n)
    assert np.array_equal(np.concatenate([r[2] for r in res]), ref)
    obs = res[0][3]
    assert obs["n_ab"] == [O.n_ab(ref)] and obs["n_a"] == [int(ref.sum())]
    assert obs["attempted"] == [st["attempted"]] and obs["accepted"] == [st["accepted"]]
    assert obs["trivial"] == [st["trivial"]] and obs["dnab_sum"] == [st["dnab_sum"]]
    assert obs["clusters_A"] == sum(c for _, c in O.cluster_histogram(ref, 1))
    assert [tuple(r) for r in obs["hist0"]] == O.cluster_histogram(ref, 0)


def test_bench_two_ranks_functional():
    """bench.py's N>1 path end to end (torchrun, 2 ranks sharing one GPU over
    gloo; KK_BENCH_BACKEND / KK_BENCH_DEVICE exist for exactly this check):
    one JSON line from rank 0 with the contract's keys.  Numbers from such a
    run are meaningless and never reported."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, KK_BENCH_BACKEND="gloo", KK_BENCH_DEVICE="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(root, "bench.py"),
           "--gpus", "2", "--steps", "1", "--warmup", "1", "--Lx", "2048", "--rows-per-gpu", "1024",
           "--sweeps-per-step", "2", "--no-other-configs"]
    r = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0
    assert d["config"]["parallelism"] == "slab2"
    assert d["e2e"]["h2d_bytes_per_step"] == 2 * 2048 * 1024 // 8
    assert d["observables"]["n_a"] == [2048 * 2048 // 2]
