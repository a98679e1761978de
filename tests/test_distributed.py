"""Multi-rank host logic on CPU with the gloo backend (world size 2):
trial sharding, the single counter all-reduce, and GPU-count invariance of
the merged statistics.  The per-shard decoder here is the CPU oracle (the
GPU decoder is the same callable slot); no GPU is needed."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1204_0556_b200.distributed import COUNTERS, counters_from_results, run_point_sharded, shard


def test_shard_partitions_exactly():
    for n in (0, 1, 7, 100, 1001):
        for world in (1, 2, 3, 8):
            got = [t for r in range(world) for t in shard(n, r, world)]
            assert got == list(range(n))
            sizes = [len(shard(n, r, world)) for r in range(world)]
            assert max(sizes) - min(sizes) <= 1


def test_counters_semantics():
    it = torch.tensor([10, 20, 1000, 5])
    w = torch.tensor([0, 3, 7, 0])
    conv = torch.tensor([True, True, False, True])
    cw = torch.tensor([True, True, False, True])
    cost = torch.tensor([0.0, -1.0, 2.0, 0.0])
    c = dict(zip(COUNTERS, counters_from_results(it, w, conv, cw, cost, n_edges=10).tolist()))
    assert c == {"trials": 4, "word_errors": 2, "bit_errors": 10, "iter_sum_correct": 15,
                 "iter_sum_erroneous": 1020, "ml_errors": 1, "converged": 3, "edge_updates": 10350}


def _oracle_setup():
    from oracle import admm_oracle as O
    from paper_1204_0556_b200.codes import make_ldpc

    code = make_ldpc(48, 3, 6, seed=10, girth6=False)
    g = O.Graph.of(code)
    p = O.Params(mu=3.0, t_max=200)

    def gamma_of_trial(t):
        return O.trial_gamma_bsc(48, 0.06, seed=110, point=1, trial=t)

    def decode_fn(gam):
        res = O.decode_many(gam, g, p)
        it = torch.tensor([r.iterations for r in res])
        hard = np.stack([r.hard_decision for r in res])
        w = torch.tensor(hard.sum(1))
        conv = torch.tensor([r.status == O.STATUS_CONVERGED for r in res])
        cw = torch.tensor([O.is_codeword(g, h) for h in hard])
        cost = torch.tensor((gam * hard).sum(1))
        return it, w, conv, cw, cost

    return code, gamma_of_trial, decode_fn


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        code, gamma_of_trial, decode_fn = _oracle_setup()
        stats = run_point_sharded(code, gamma_of_trial, 37, decode_fn=decode_fn, rank=rank, world=world, chunk=8)
        out[rank] = stats
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_gloo_world2_matches_single_rank():
    code, gamma_of_trial, decode_fn = _oracle_setup()
    single = run_point_sharded(code, gamma_of_trial, 37, decode_fn=decode_fn)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(2, _free_port(), out), nprocs=2, join=True, start_method="spawn")
    assert out[0] == out[1] == single
    assert single["trials"] == 37
