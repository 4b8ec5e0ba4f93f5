"""Host-side logic of the sharded (multi-GPU) path, on CPU with gloo, world size 2 and 4.

The CUDA path itself cannot run here; these tests pin what it relies on:
  - the quadtree-subtree partition (hpsb_partition) covers every element
    once, keeps local-level faces inside one rank and marks exactly the top
    log2(G) levels as shared;
  - "every skeleton row is produced by exactly one rank": a matvec assembled
    from per-rank element contributions (the oracle's element ItI maps) and
    summed with an allreduce equals the reference interface operator M x;
  - the preconditioner's residual combination r = v + sum_ranks (r_rank - v)
    and the masked output allreduce reproduce the replicated vectors;
  - owner-computes: the merges of each global level run on distinct ranks
    (hpsb_merge_owners), nested level to level;
  - distributed vectors: an element reads / writes only its rank's rows and
    the global rows, so the matvec needs one allreduce of the global rows,
    and inner products over own rows + the global rows once (allreduced)
    equal the full ones.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _slots(fg, n, m, e):
    """(in, out) skeleton indices of element e's 4(N-1) boundary nodes (-1: physical)."""
    bs = 2 * m
    ins, outs = [], []
    for side in range(4):
        f = int(fg["face_of_element"][e][side])
        for k in range(m):
            if f < 0:
                ins.append(-1), outs.append(-1)
            else:
                own = 1 if int(fg["faces"][f][0]) == e else 0
                ins.append(f * bs + own * m + k)
                outs.append(f * bs + (1 - own) * m + k)
    return np.array(ins), np.array(outs)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2511_00735_b200 as hps
        from oracle import pyoracle
        res = {}
        # ---- partition invariants (cfg1 mesh and cfg3 mesh)
        for n in (16, 128):
            p = hps.partition(n, world, rank)
            fg = hps.face_graph(n)
            eo = torch.from_numpy(p["elem_owner"].astype(np.int64))
            gathered = [torch.zeros_like(eo) for _ in range(world)]
            dist.all_gather(gathered, eo)
            res[f"same_plan_{n}"] = all(torch.equal(g, eo) for g in gathered)
            counts = np.bincount(p["elem_owner"], minlength=world)
            res[f"balanced_{n}"] = bool(np.all(counts == n * n // world))
            faces = fg["faces"]
            loc = faces[:, 4] <= p["last_local"]
            res[f"local_faces_inside_{n}"] = bool(np.all(
                p["elem_owner"][faces[loc, 0]] == p["elem_owner"][faces[loc, 1]]))
            res[f"global_faces_cut_{n}"] = bool(np.all(
                p["elem_owner"][faces[~loc, 0]] != p["elem_owner"][faces[~loc, 1]]) or world == 1)
            res[f"face_owner_{n}"] = bool(np.all(p["face_owner"][~loc] == -1)) and bool(
                np.all(p["face_owner"][loc] == p["elem_owner"][faces[loc, 0]]))
            L = 2 * int(np.log2(n))
            res[f"last_local_{n}"] = p["last_local"] == L - int(np.log2(world))
        # ---- sharded matvec on cfg0 with the oracle's element maps
        smp = pyoracle.sample(2, config=0, seed=0)
        S = pyoracle.Session.from_sample(smp, 10.0, threads=1)
        n, m = smp["n"], smp["order"] - 1
        fg = hps.face_graph(n)
        p = hps.partition(n, world, rank)
        rng = np.random.default_rng(7)
        x = rng.standard_normal(S.dim) + 1j * rng.standard_normal(S.dim)
        y = np.zeros(S.dim, dtype=complex)
        for e in range(n * n):
            if p["elem_owner"][e] != rank:
                continue
            T, _ = S.element(e)
            ins, outs = _slots(fg, n, m, e)
            xi = np.where(ins >= 0, x[np.maximum(ins, 0)], 0)
            Tx = T @ xi
            for b in range(len(outs)):
                if outs[b] >= 0:
                    y[outs[b]] = x[outs[b]] + Tx[b]
        yt = torch.from_numpy(y.view(np.float64).copy())
        dist.all_reduce(yt)
        res["sharded_matvec_err"] = float(
            np.linalg.norm(yt.numpy().view(complex) - S.apply_M(x)) / np.linalg.norm(S.apply_M(x)))
        # ---- residual / output combination of the sharded V-cycle
        bs = 2 * m
        v = rng.standard_normal(S.dim)
        mine = np.repeat(p["face_owner"], bs) == rank
        r = v.copy()
        delta = rng.standard_normal(S.dim) * mine   # this rank's subtree updates
        r += delta
        rt = torch.from_numpy(r - v)
        dist.all_reduce(rt)
        full = v + rt.numpy()
        dt = torch.from_numpy(delta.copy())
        dist.all_reduce(dt)
        res["residual_combine"] = bool(np.allclose(full, v + dt.numpy(), rtol=0, atol=1e-14))
        z = rng.standard_normal(S.dim)                 # replicated global part ...
        zt = torch.from_numpy(z.copy())
        dist.broadcast(zt, 0)                          # ... identical on every rank
        z = zt.numpy().copy()
        keep = (np.repeat(p["face_owner"], bs) == rank) | (
            (np.repeat(p["face_owner"], bs) < 0) & (rank == 0))
        zm = torch.from_numpy(np.where(keep, z, 0.0))
        dist.all_reduce(zm)
        res["masked_output"] = bool(np.allclose(zm.numpy(), z, rtol=0, atol=0))
        # ---- owner-computes merges of the global levels (cfg3 mesh):
        # each global level's merges on distinct ranks, each rank's merge at
        # level l+1 on a rank that held a merge at level l
        pg = hps.partition(128, world, rank)
        prev = None
        for level in range(pg["last_local"] + 1, 14):
            own = hps.merge_owners(128, world, level)
            res[f"owners_distinct_{level}"] = len(set(own.tolist())) == len(own)
            if prev is not None:
                res[f"owners_nested_{level}"] = set(own.tolist()) <= set(prev.tolist())
            prev = own
        if world > 1:
            res["owners_subtree"] = bool(np.array_equal(
                hps.merge_owners(128, world, pg["last_local"]), np.arange(world)))
        # ---- distributed vectors: an element touches only its rank's rows
        # and the global rows; the matvec's own rows are exact without any
        # exchange and one allreduce of the global rows completes the rest
        fo = np.repeat(p["face_owner"], bs)
        touched_ok = True
        yd = np.zeros(S.dim, dtype=complex)
        for e in range(n * n):
            if p["elem_owner"][e] != rank:
                continue
            ins, outs = _slots(fg, n, m, e)
            for idx in np.concatenate([ins, outs]):
                if idx >= 0 and fo[idx] not in (rank, -1):
                    touched_ok = False
            T, _ = S.element(e)
            Tx = T @ np.where(ins >= 0, x[np.maximum(ins, 0)], 0)
            for b in range(len(outs)):
                if outs[b] >= 0:
                    yd[outs[b]] = x[outs[b]] + Tx[b]
        res["element_rows_own_or_global"] = touched_ok
        tail = fo < 0
        tt = torch.from_numpy(np.ascontiguousarray(yd[tail]).view(np.float64).copy())
        dist.all_reduce(tt)
        Mx = S.apply_M(x)
        res["dist_matvec_own_rows"] = bool(np.allclose(yd[fo == rank], Mx[fo == rank], rtol=1e-13,
                                                       atol=0))
        res["dist_matvec_global_rows"] = bool(np.allclose(tt.numpy().view(complex), Mx[tail],
                                                          rtol=1e-13, atol=0))
        # ---- distributed inner products: own rows + the global rows once
        a = rng.standard_normal(S.dim) + 1j * rng.standard_normal(S.dim)
        at = torch.from_numpy(a.view(np.float64).copy())
        dist.broadcast(at, 0)
        a = at.numpy().view(complex).copy()
        wgt = (fo == rank) | (tail & (rank == 0))
        part = torch.tensor([np.vdot(a[wgt], Mx[wgt]).real, np.vdot(a[wgt], Mx[wgt]).imag],
                            dtype=torch.float64)
        dist.all_reduce(part)
        full = np.vdot(a, Mx)
        res["dist_dot"] = bool(abs(complex(part[0], part[1]) - full) <= 1e-12 * abs(full))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_host_logic(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = dict(q.get(timeout=300) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
    for rank, res in results.items():
        for k, v in res.items():
            if k == "sharded_matvec_err":
                assert v < 1e-13, (rank, k, v)
            else:
                assert v, (rank, k)


def test_partition_rejects_bad_worlds():
    import paper_2511_00735_b200 as hps
    with pytest.raises(hps.HpsError):
        hps.partition(4, 3, 0)
    with pytest.raises(hps.HpsError):
        hps.partition(2, 4, 0)  # n=2 has 2 levels: at most 2 ranks
