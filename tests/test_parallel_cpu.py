"""Host-side logic of the multi-GPU row-band partition,
exercised on CPU with torch.distributed/gloo at world sizes 2 and 3.

Each rank runs a numpy mirror of the lattice LBP sweep on its band (owned rows
+ ghost rows, rows from paper_1909_11469_b200.parallel.band_rows) and
exchanges exactly the halo rows the CUDA path exchanges (send_up -> rank-1,
send_down -> rank+1) plus the all-reduced unconverged count; rank 0 gathers the
owned beliefs and checks them bitwise against the unpartitioned sweep.  The
CUDA pack/unpack kernels themselves are checked on the GPU in
tests/test_gpu_parallel.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1909_11469_b200.parallel import band_rows


def _instance(n, seed):
    rng = np.random.default_rng(seed)
    unary = rng.normal(size=(n, n))
    jh = rng.uniform(-2, 2, size=(n, n - 1))  # coupling of (r, c)-(r, c+1), log2 units
    jv = rng.uniform(-2, 2, size=(n - 1, n))  # coupling of (r, c)-(r+1, c)
    return unary, jh, jv


def _msg(h, j):
    """Ising message in log2-odds: log2((1 + 2^h a) / (a + 2^h)), a = 2^j."""
    u, a = np.exp2(h), np.exp2(j)
    return np.log2((1 + u * a) / (a + u))


def _sweep(unary, jh, jv, into):
    """One Jacobi sweep of a lattice.  into[d][r, c] = message INTO (r, c) from
    its neighbour in direction d (0 where absent).  Returns the new messages
    and the residual count proxy (number of changed messages)."""
    T = unary + into["up"] + into["down"] + into["left"] + into["right"]
    new = {d: np.zeros_like(unary) for d in into}
    new["left"][:, 1:] = _msg(T[:, :-1] - into["right"][:, :-1], jh)   # (r, c) -> (r, c+1)
    new["right"][:, :-1] = _msg(T[:, 1:] - into["left"][:, 1:], jh)    # (r, c+1) -> (r, c)
    new["up"][1:, :] = _msg(T[:-1, :] - into["down"][:-1, :], jv)      # (r, c) -> (r+1, c)
    new["down"][:-1, :] = _msg(T[1:, :] - into["up"][1:, :], jv)       # (r+1, c) -> (r, c)
    return new


def _beliefs(unary, into):
    return unary + into["up"] + into["down"] + into["left"] + into["right"]


def _worker(rank, world, port, n, seed, iters, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        unary, jh, jv = _instance(n, seed)
        r0, r1, gu, gd = band_rows(n, rank, world)
        a, b = r0 - gu, r1 + gd                      # band rows incl. ghosts
        u, h, v = unary[a:b], jh[a:b], jv[a:b - 1]
        into = {d: np.zeros((b - a, n)) for d in ("up", "down", "left", "right")}
        for _ in range(iters):
            into = _sweep(u, h, v, into)
            # halo: the messages that flow from ghost rows into owned rows are
            # the owners' values (send_up -> rank-1's recv_down, send_down ->
            # rank+1's recv_up)
            send_up = torch.from_numpy(into["down"][0].copy()) if gu else None      # (r0, c) -> (r0-1, c)
            send_down = torch.from_numpy(into["up"][-1].copy()) if gd else None     # (r1-1, c) -> (r1, c)
            recv_up, recv_down = torch.zeros(n, dtype=torch.float64), torch.zeros(n, dtype=torch.float64)
            ops = []
            if gu:
                ops += [dist.P2POp(dist.isend, send_up, rank - 1), dist.P2POp(dist.irecv, recv_up, rank - 1)]
            if gd:
                ops += [dist.P2POp(dist.isend, send_down, rank + 1), dist.P2POp(dist.irecv, recv_down, rank + 1)]
            for w in dist.batch_isend_irecv(ops) if ops else []:
                w.wait()
            if gu:
                into["up"][1] = recv_up.numpy()        # (r0-1, c) -> (r0, c) from the band above
            if gd:
                into["down"][-2] = recv_down.numpy()   # (r1, c) -> (r1-1, c) from the band below
            cnt = torch.tensor([float(r1 - r0)])
            dist.all_reduce(cnt)                       # the global count every rank stops on
            assert int(cnt.item()) == n
        rows = [band_rows(n, k, world)[1] - band_rows(n, k, world)[0] for k in range(world)]
        owned = torch.zeros((max(rows), n), dtype=torch.float64)  # gloo gathers equal shapes
        owned[:r1 - r0] = torch.from_numpy(_beliefs(u, into)[gu:gu + r1 - r0].copy())
        parts = [torch.zeros_like(owned) for _ in range(world)] if rank == 0 else None
        dist.gather(owned, parts, dst=0)
        if rank == 0:
            into_full = {d: np.zeros((n, n)) for d in ("up", "down", "left", "right")}
            for _ in range(iters):
                into_full = _sweep(unary, jh, jv, into_full)
            want = _beliefs(unary, into_full)
            got = torch.cat([p[:k] for p, k in zip(parts, rows)]).numpy()
            np.save(out_path, np.array([np.array_equal(got, want), float(np.max(np.abs(got - want)))]))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_band_halo_protocol_gloo(tmp_path, world):
    out = str(tmp_path / "res.npy")
    mp.spawn(_worker, args=(world, _free_port(), 13, 5, 9, out), nprocs=world, join=True)
    ok, diff = np.load(out)
    assert ok == 1.0, diff
