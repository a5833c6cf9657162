"""The multi-GPU host logic (sharding, all-gather of E, gather of rho rows) on CPU with the
gloo backend at world_size 2 and 3. The per-rank phase functions are the fp64 oracle
here (the CUDA kernels need a GPU); the test checks that the sharded map equals the
single-process oracle map exactly (byte-identical at any world size)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2011_11082_b200 import distributed as D
from paper_2011_11082_b200 import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_fns():
    from oracle import oracle as O

    def simplex_fn(data, E_max, tau, s0, s1):
        e, _ = O.simplex_all(data.numpy(), E_max, tau, s0, s1, nthreads=1)
        return torch.from_numpy(e)

    def ccm_fn(data, E, tau, Tp, mode, excl, rows):
        m = 0 if mode == "target" else 1
        r = [O.ccm_rows(data.numpy(), E.numpy(), tau, Tp, m, excl, int(i), int(i) + 1, nthreads=1) for i in rows]
        r = np.concatenate(r) if r else np.zeros((0, data.shape[1]))
        return torch.from_numpy(r.astype(np.float32))

    return simplex_fn, ccm_fn


def _worker(rank, world, port, data, out_path, mode):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sf, cf = _oracle_fns()
    E, rows, full = D.run(torch.from_numpy(data), 6, 1, 1, mode, True, sf, cf, gather=True)
    if rank == 0:
        np.save(out_path + "_E.npy", E.numpy())
        np.save(out_path + "_rho.npy", full.numpy())
    dist.barrier()
    dist.destroy_process_group()


def _worker_host(rank, world, port, data, out_path, mode, nchunk):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sf, cf = _oracle_fns()
    N = data.shape[1]
    host = torch.full((N, N), -7.0) if rank == 0 else None
    E = D.run_to_host(torch.from_numpy(data), 6, 1, 1, mode, True, sf, cf, host, nchunk, align=1)
    if rank == 0:
        np.save(out_path + "_E.npy", E.numpy())
        np.save(out_path + "_rho.npy", host.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_shard_covers_everything():
    for n in (1, 7, 64, 1001):
        for w in (1, 2, 3, 8):
            parts = [D.shard(n, r, w) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1


def test_assign_rows_partitions_and_balances():
    rng = np.random.default_rng(4)
    E = rng.integers(1, 21, 1001).astype(np.int32)
    for mode in ("target", "library"):
        for w in (1, 2, 3, 8):
            parts = D.assign_rows(E, w, mode)
            allrows = np.sort(np.concatenate(parts))
            assert np.array_equal(allrows, np.arange(1001))
            assert all(np.all(np.diff(p) > 0) for p in parts)
            if mode == "target":
                assert all(D._is_range(p) for p in parts)
            else:  # E-sorted dealing: per-rank sums of E within one max E of each other
                sums = [int(E[p].sum()) for p in parts]
                assert max(sums) - min(sums) <= 20


@pytest.mark.parametrize("world,mode", [(2, "target"), (3, "library")])
def test_sharded_map_equals_single_process(tmp_path, world, mode):
    from oracle import oracle as O
    data = synth.random_dataset(13, 70, 21)
    out = str(tmp_path / "res")
    mp.spawn(_worker, args=(world, _free_port(), data, out, mode), nprocs=world, join=True)
    E = np.load(out + "_E.npy")
    rho = np.load(out + "_rho.npy")
    rE, _ = O.simplex_all(data, 6, 1)
    assert np.array_equal(E, rE)
    ref = O.ccm_rows(data, rE, 1, 1, 0 if mode == "target" else 1, True).astype(np.float32)
    assert np.array_equal(rho.view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("world,mode,nchunk", [(2, "target", 3), (3, "library", 8)])
def test_chunked_map_to_host_equals_single_process(tmp_path, world, mode, nchunk):
    # the chunked gather-to-host path of the end-to-end API (more chunks than rows on some ranks)
    from oracle import oracle as O
    data = synth.random_dataset(11, 60, 23)
    out = str(tmp_path / "res")
    mp.spawn(_worker_host, args=(world, _free_port(), data, out, mode, nchunk), nprocs=world, join=True)
    E = np.load(out + "_E.npy")
    rho = np.load(out + "_rho.npy")
    rE, _ = O.simplex_all(data, 6, 1)
    assert np.array_equal(E, rE)
    ref = O.ccm_rows(data, rE, 1, 1, 0 if mode == "target" else 1, True).astype(np.float32)
    assert np.array_equal(rho.view(np.uint32), ref.view(np.uint32))
