"""The N > 1 decomposition on CPU with world_size-2 gloo.

Each rank stores the id ranges `rii_shard_range` assigns it for every add batch
(the library's own host logic), searches its shard with the oracle, maps local
hits to global ids, and the per-rank top-kk lists are exchanged with an
all-gather and merged by (dist, id).  The merged result must equal the oracle on
the whole database: the global top-k is contained in the union of shard top-kk.
"""
import os
import socket

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


def _worker(rank, world, port, out_path, subset):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    from oracle import ref
    from synth import generators as gen
    import paper_1808_03969_b200 as rii
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    D, M, topk = 32, 4, 20
    kk = rii.partial_width(topk)
    batches = [gen.gaussian(n, D, seed=n) for n in (1_001, 2_500, 777)]
    cb = ref.train(np.concatenate(batches), M, n_iter=3, seed=0)
    q = gen.gaussian(9, D, seed=1, stream=gen.STREAM_QUERY)
    # this rank's shard: the rows rii_shard_range assigns it in every batch
    codes, gids, first = [], [], 0
    for b in batches:
        lo, hi = rii.shard_range(len(b), rank, world)
        codes.append(ref.encode(cb, b[lo:hi], M))
        gids.append(np.arange(first + lo, first + hi, dtype=np.int64))
        first += len(b)
    codes, gids = np.concatenate(codes), np.concatenate(gids)
    S = None
    if subset:
        S_all = gen.subset(first, 900, seed=3)
        S = np.nonzero(np.isin(gids, S_all))[0].astype(np.int64)  # local positions of owned targets
    lid, ld = ref.linear(cb, codes, q, kk, S=S)
    gid = np.where(lid >= 0, gids[np.maximum(lid, 0)], -1)
    send = torch.from_numpy(np.stack([gid.astype(np.float64), ld.astype(np.float64)]))
    recv = [torch.zeros_like(send) for _ in range(world)]
    dist.all_gather(recv, send)
    if rank == 0:
        allc = np.concatenate([ref.encode(cb, b, M) for b in batches])
        want_ids, want_d = ref.linear(cb, allc, q, topk, S=S_all if subset else None)
        for i in range(len(q)):
            ids = np.concatenate([r[0, i].numpy() for r in recv])
            ds = np.concatenate([r[1, i].numpy() for r in recv])
            keep = ids >= 0
            order = np.lexsort((ids[keep], ds[keep]))[:topk]
            got_ids = ids[keep][order].astype(np.int64)
            got_d = ds[keep][order].astype(np.float32)
            assert np.array_equal(got_ids, want_ids[i][: len(got_ids)]), (i, got_ids, want_ids[i])
            assert np.array_equal(got_d, want_d[i][: len(got_d)])
        with open(out_path, "w") as f:
            f.write("ok")
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("subset", [False, True])
def test_two_rank_shards_equal_single_index(tmp_path, subset):
    out = tmp_path / "ok.txt"
    mp.spawn(_worker, args=(2, _free_port(), str(out), subset), nprocs=2, join=True)
    assert out.read_text() == "ok"
