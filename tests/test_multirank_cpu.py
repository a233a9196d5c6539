"""Multi-rank (direction-sharded) solver logic on CPU with gloo, world size 2.

Each rank takes its share of the directions from the product's partition
(rtlr_cu_partition_angles, host logic), sweeps it with the CPU oracle and
contributes a partial scalar flux; an allreduce(sum) must reproduce the
unsharded si_step, and a sharded SI-DSA outer loop (DSA replicated, as in
the GPU driver) must reproduce the unsharded solve.  This is the host-side
half of the sharded GPU driver, which runs the same partition with NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, q):
    import sys
    sys.path.insert(0, HERE)
    sys.path.insert(0, os.path.dirname(HERE))
    import _oracle as O
    import paper_2603_25233_b200 as P
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        o = O.Problem(name)
        d, w = O.quadrature(o.n_theta, o.n_omega_z)
        mine = P.partition_angles(o.n_theta, o.n_omega_z, world, rank)

        def sharded_si_step(phi_prev):
            rhs = o.rhs_core(phi_prev)
            part = np.zeros(o.n)
            for j in mine:
                part += w[j] * o.sweep(d[j, 0], d[j, 1], rhs)
            t = torch.from_numpy(part)
            dist.all_reduce(t)
            return t.numpy()

        phi0 = np.zeros(o.n)
        step = sharded_si_step(phi0)
        ref = o.si_step(phi0)
        err_step = np.linalg.norm(step - ref) / np.linalg.norm(ref)
        # sharded SI-DSA outer loop (full_rank.cpp:60-122), DSA replicated
        phi = np.zeros(o.n)
        its = 0
        for it in range(1, 200):
            star = sharded_si_step(phi)
            its = it
            if np.max(np.abs(star - phi)) <= 1e-6:
                phi = star
                break
            phi = star + o.dsa_correct(star, phi)
        full = o.solve("full")
        err_solve = np.linalg.norm(phi - full.get("phi", o.n)) / np.linalg.norm(full.get("phi", o.n))
        q.put((rank, len(mine), err_step, err_solve, its, full.iterations))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["homogeneous(1,1)", "pin_cell"])
def test_two_rank_sharded_si_dsa(name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    res = sorted(q.get() for _ in range(2))
    counts = [r[1] for r in res]
    assert sum(counts) > 0 and abs(counts[0] - counts[1]) <= 2
    for _, _, err_step, err_solve, its, fr_its in res:
        assert err_step <= 1e-13
        assert err_solve <= 1e-12
        assert abs(its - fr_its) <= 1


def test_shard_block_covers_every_item_once_in_order():
    import sys
    sys.path.insert(0, os.path.dirname(HERE))
    import paper_2603_25233_b200 as P
    for m in (0, 1, 2, 7, 8, 16, 100, 1023):
        for world in (1, 2, 3, 4, 8):
            got = []
            for r in range(world):
                b, e, bsz = P.shard_block(m, world, r)
                assert bsz == -(-m // world)
                assert 0 <= b <= e <= m and e - b <= bsz
                if e > b:
                    assert b == r * bsz  # in-place all-gather offset
                got.extend(range(b, e))
            assert got == list(range(m))
    with pytest.raises(P.RtlrError):
        P.shard_block(4, 2, 2)


def _lr_worker(rank, world, port, q):
    """One low-rank phase, sharded as the GPU driver shards it: this rank
    sweeps its block of the sampled angles into a padded buffer, the blocks
    are all-gathered in place, and per-angle residual norms of the gathered
    snapshots (an angle-sharded phase of its own) are all-gathered too."""
    import sys
    sys.path.insert(0, HERE)
    sys.path.insert(0, os.path.dirname(HERE))
    import _oracle as O
    import paper_2603_25233_b200 as P
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        o = O.Problem("pin_cell")
        d, _ = O.quadrature(o.n_theta, o.n_omega_z)
        rng = np.random.default_rng(7)
        rhs = o.rhs_core(rng.random(o.n))
        n_om = o.n_theta * o.n_omega_z
        out = []
        for m in (1, 5, 8, 13):
            angles = rng.choice(n_om, size=m, replace=False)
            b, e, bsz = P.shard_block(m, world, rank)
            buf = torch.zeros(world * bsz, o.n, dtype=torch.float64)
            for k in range(b, e):
                j = angles[k]
                buf[k] = torch.from_numpy(o.sweep(d[j, 0], d[j, 1], rhs))
            mine = buf[rank * bsz:(rank + 1) * bsz].clone()
            dist.all_gather_into_tensor(buf, mine)
            snaps = buf[:m].numpy()
            ref = np.stack([o.sweep(d[j, 0], d[j, 1], rhs) for j in angles])
            # residual norms ||rhs - A_j psi_j|| on this rank's block, gathered
            nb = torch.zeros(world * bsz, dtype=torch.float64)
            for k in range(b, e):
                j = angles[k]
                nb[k] = float(np.linalg.norm(rhs - o.apply(d[j, 0], d[j, 1], snaps[k])))
            mine_n = nb[rank * bsz:(rank + 1) * bsz].clone()
            dist.all_gather_into_tensor(nb, mine_n)
            ref_n = [np.linalg.norm(rhs - o.apply(d[j, 0], d[j, 1], ref[k])) for k, j in enumerate(angles)]
            out.append((m, bool(np.array_equal(snaps, ref)), bool(np.array_equal(nb[:m].numpy(), ref_n))))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_low_rank_phase_gathers_bitwise(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_lr_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    for _ in range(world):
        _, out = q.get()
        for m, snaps_ok, norms_ok in out:
            assert snaps_ok and norms_ok, m
