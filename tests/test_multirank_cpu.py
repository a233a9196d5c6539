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
