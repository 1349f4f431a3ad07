"""The multi-rank and multi-reader paths of the library on one GPU, against the oracle.

* Two processes, world = 2, one shard each, exchanging through the library's own
  collective code path (rii_create_with_transport: a host all-gather over
  torch.distributed gloo, staged after a stream synchronisation, so no kernel
  ever waits on the other rank's kernels).  This drives what NCCL drives on an
  8-GPU box -- the sharded add (id-range segments), the multi-rank reconfigure
  (all-gathered sample keys and codes), device-side routing of S, the shared u6
  bound pass of a whole-database scan, and the final all-gather + merge -- and
  compares centres, posting lists and every result with the single-index oracle
  ("a sharded GPU result must equal the single-index oracle result").
  Uneven shards (one-row additions, an empty rank) check that every rank joins the
  same collectives (the decisions use global quantities only).
* Two host threads querying one index on two streams at once (rii.h
  "Concurrency": per-call scratch), each result compared with the oracle.
"""
import os
import socket
import threading

import numpy as np
import pytest
import torch.multiprocessing as mp

from synth import generators as gen
from tests.parity import assert_topk_parity

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard_worker(rank, world, port, out_dir, case):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from oracle import ref
    import paper_1808_03969_b200 as rii
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    if case == "balanced":
        # global-quantity thresholds low enough that the shared bound pass runs at this size
        os.environ["RII_Q16_MIN"] = "20000"
        D, M, K, nq, topk = 96, 32, 48, 24, 100
        batches = [gen.deep_like(n, D, seed=n) for n in (1, 60_001, 3, 59_995)]
        S = gen.subset(120_000, 9_000, seed=4)
    else:  # "empty_rank": one-row additions -> every row lands on rank 0, rank 1 stays empty
        os.environ["RII_Q16_MIN"] = "500"
        D, M, K, nq, topk = 32, 4, 8, 9, 10
        rows = gen.gaussian(1_100, D, seed=8)
        batches = [rows[i:i + 1] for i in range(len(rows))]
        S = gen.subset(1_100, 300, seed=5)
    allx = np.concatenate(batches)
    q = gen.base("deep" if D == 96 else "gaussian", nq, D, seed=3, stream=gen.STREAM_QUERY)
    cb = ref.train(allx[:4000], M, n_iter=3, seed=0)
    g = rii.Index(D, M, device=0, rank=rank, world=world, transport=rii.torch_allgather())
    g.set_codebook(cb)
    for b in batches:
        g.add(b)
    o = ref.OracleIndex(D, M)
    o.cb = cb
    o.add(allx)
    info = g.info()
    assert info["N"] == len(allx)
    # this rank's codes are the oracle's codes of the ids it owns
    lo_hi, first = [], 0
    for b in batches:
        lo, hi = rii.shard_range(len(b), rank, world)
        lo_hi.extend(range(first + lo, first + hi))
        first += len(b)
    own = np.array(lo_hi, np.int64)
    assert info["n_local"] == len(own)
    if case == "empty_rank":
        assert info["n_local"] == (len(allx) if rank == 0 else 0)
    if len(own):
        runs = np.split(own, np.nonzero(np.diff(own) != 1)[0] + 1)
        for r in runs:
            assert np.array_equal(g.get_codes(int(r[0]), len(r)), o.codes[r]), "shard codes (Eq. 1)"
    qt = torch.from_numpy(q).cuda()
    # whole-database linear scan before any reconfigure (K = 0)
    for qq in (q, qt):
        ids, dist_, used = g.query(qq, topk, path="linear")
        ids, dist_ = (np.asarray(ids.cpu()) if hasattr(ids, "cpu") else ids), \
            (np.asarray(dist_.cpu()) if hasattr(dist_, "cpu") else dist_)
        assert_topk_parity(ref, o.cb, o.codes, q, (ids, dist_), o.query(q, topk, path=1), what=f"{case} r{rank} linear")
    # multi-rank reconfigure: the all-gathered sample makes the centres the oracle's
    g.reconfigure(K, n_iter=4, seed=7)
    o.reconfigure(K, n_iter=4, seed=7)
    assert np.array_equal(g.get_centers(), o.centers), "multi-rank PQk-means centres differ from the oracle"
    off, ids_ = g.get_postings()
    for k in range(K):
        want = o.ids[o.offsets[k]:o.offsets[k + 1]]
        assert np.array_equal(ids_[off[k]:off[k + 1]], want[np.isin(want, own)]), "posting lists of this shard"
    for sub in (None, S):
        for path, L in (("linear", 1), ("ivf", 1), ("ivf", 5), ("auto", 3)):
            gr = g.query(qt, topk, target_ids=sub, L=L, path=path)
            gr = (gr[0].cpu().numpy(), gr[1].cpu().numpy(), gr[2])
            orr = o.query(q, topk, S=sub, L=L, path={"linear": 1, "ivf": 2, "auto": 0}[path])
            assert gr[2] == orr[2], (path, L, gr[2], orr[2])
            assert_topk_parity(ref, o.cb, o.codes, q, gr, orr, S=sub, what=f"{case} r{rank} {path} L={L}")
    # one-row addition after reconfigure, then query again (lists grow on one rank only)
    extra = gen.base("deep" if D == 96 else "gaussian", 1, D, seed=99)
    g.add(extra)
    o.add(extra)
    gr = g.query(qt, topk, L=2, path="ivf")
    assert_topk_parity(ref, o.cb, o.codes, q, (gr[0].cpu().numpy(), gr[1].cpu().numpy()), o.query(q, topk, L=2, path=2),
                       what=f"{case} r{rank} after add")
    with open(os.path.join(out_dir, f"ok{rank}"), "w") as f:
        f.write("ok")
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", ["balanced", "empty_rank"])
def test_two_process_shards_match_oracle(tmp_path, case):
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, str(tmp_path), case)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
    codes = [p.exitcode for p in procs]
    for p in procs:
        if p.is_alive():
            p.kill()
    assert codes == [0, 0], codes
    assert all((tmp_path / f"ok{r}").read_text() == "ok" for r in range(2))


def test_concurrent_readers_two_streams(ref):
    """rii.h "Concurrency": many readers at a time.  Two host threads query one index
    on two CUDA streams concurrently (different paths, batch sizes and memory kinds,
    so scratch buffers grow and are freed while the other thread's kernels run);
    every result must equal the oracle's."""
    import torch
    import paper_1808_03969_b200 as rii
    N, D, M, K = 60_000, 96, 32, 64
    x = gen.deep_like(N, D, seed=21)
    g = rii.Index(D, M, device=0)
    g.train(x[:5000], n_iter=3, seed=0)
    g.add(x)
    g.reconfigure(K, n_iter=3, seed=0)
    o = ref.OracleIndex(D, M)
    o.train(x[:5000], n_iter=3, seed=0)
    o.add(x)
    o.reconfigure(K, n_iter=3, seed=0)
    qs = [gen.deep_like(n, D, seed=n, stream=gen.STREAM_QUERY) for n in (7, 40, 130)]
    S = gen.subset(N, 5_000, seed=2)
    subs = (None, S)
    jobs = [(qi, si, path, L) for qi in range(3) for si in range(2) for path, L in (("linear", 1), ("ivf", 4))]
    want = {j: o.query(qs[j[0]], 50, S=subs[j[1]], L=j[3], path=1 if j[2] == "linear" else 2) for j in jobs}
    errors = []

    def reader(tid):
        try:
            st = torch.cuda.Stream()
            for rep in range(6):
                for j in (jobs if tid == 0 else jobs[::-1]):
                    qi, si, path, L = j
                    sub = subs[si]
                    if (rep + tid) % 2:
                        r = g.query(qs[qi], 50, target_ids=sub, L=L, path=path, stream=st)  # host memory
                    else:
                        with torch.cuda.stream(st):
                            qd = torch.from_numpy(qs[qi]).cuda()
                            sd = None if sub is None else torch.from_numpy(sub).cuda()
                            ids, dist_, used = g.query(qd, 50, target_ids=sd, L=L, path=path, stream=st)
                            st.synchronize()
                            r = (ids.cpu().numpy(), dist_.cpu().numpy(), used)
                    w = want[j]
                    if not (np.array_equal(r[0], w[0]) and np.array_equal(r[1], w[1])):
                        assert_topk_parity(ref, o.cb, o.codes, qs[qi], r, w, S=sub, what=f"thread {tid} {j}")
        except Exception as e:  # reported by the main thread
            errors.append(e)

    th = [threading.Thread(target=reader, args=(t,)) for t in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors[0]
