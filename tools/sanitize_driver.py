"""Small end-to-end drive of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck, one tool per run):

    compute-sanitizer --tool racecheck python tools/sanitize_driver.py [tiny|windows|ivf|all]

tiny    : BASELINE configs[0] shape at 1/5 size: train, add, reconfigure, linear /
          IVF / subset / paper-mode queries, add after reconfigure, save + load
windows : the headline u6 kernel (M = 32, 16 queries per CTA) over 120k codes in
          two long chunks (multi-window: rescale, rollback, shared-bound paths)
ivf     : list-major two-phase IVF (fp32 / u6 items) and the u16 kernel (M = 16)
masked  : IVF executed as a probe-masked linear scan and as Alg. 1 (P = K), the
          coarse top-P kernel's lane-rotated pass (the default) and its
          canonical-only pass (RII_COARSE_ROT_MINK=1000000000), whole and subset
Results are checked against the oracle so a sanitizer run also proves it ran the
path to completion.
"""
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from synth import generators as gen  # noqa: E402
from tests.parity import assert_topk_parity  # noqa: E402

import paper_1808_03969_b200 as rii  # noqa: E402


def tiny():
    x = gen.gaussian(2_000, 32, seed=0)
    q = gen.gaussian(12, 32, seed=0, stream=gen.STREAM_QUERY)
    S = gen.subset(2_000, 300, seed=0)
    g = rii.Index(32, 4, device=0)
    g.train(x, n_iter=4, seed=0)
    g.add(x)
    g.reconfigure(20, n_iter=3, seed=0)
    o = ref.OracleIndex(32, 4)
    o.train(x, n_iter=4, seed=0)
    o.add(x)
    o.reconfigure(20, n_iter=3, seed=0)
    for sub in (None, S):
        for path, L in (("linear", 1), ("ivf", 3), ("auto", 2)):
            gr = g.query(q, 10, target_ids=sub, L=L, path=path)
            orr = o.query(q, 10, S=sub, L=L, path={"linear": 1, "ivf": 2, "auto": 0}[path])
            assert_topk_parity(ref, o.cb, o.codes, q, gr, orr, S=sub, what=f"tiny {path}")
    g.set_ivf_mode("paper")
    g.query(q, 10, L=50, path="ivf")
    g.set_ivf_mode("lists")
    g.add(x[:100])
    o.add(x[:100])
    assert_topk_parity(ref, o.cb, o.codes, q, g.query(q, 10, L=2, path="ivf"), o.query(q, 10, L=2, path=2))
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "t.rii")
        g.save(p)
        h = rii.Index.load(p)
        a, b = g.query(q, 10, L=2, path="ivf"), h.query(q, 10, L=2, path="ivf")
        assert np.array_equal(a[0], b[0])
    print("tiny ok")


def windows():
    os.environ["RII_Q16_MIN"] = "50000"
    os.environ["RII_CHUNK_CODES"] = "100000"
    os.environ["RII_Q16_SAMPLE"] = "4096"
    x = gen.deep_like(120_000, 96, seed=1)
    q = gen.deep_like(16, 96, seed=1, stream=gen.STREAM_QUERY)
    cb = ref.train(x[:5_000], 32, n_iter=2, seed=0)
    g = rii.Index(96, 32, device=0)
    g.set_codebook(cb)
    g.add(x)
    codes = ref.encode_mt(cb, x, 32)
    gr = g.query(q, 100, path="linear")
    assert_topk_parity(ref, cb, codes, q, gr, ref.linear_mt(cb, codes, q, 100), what="windows")
    print("windows ok")


def ivf():
    for k in ("RII_Q16_MIN", "RII_CHUNK_CODES", "RII_Q16_SAMPLE"):
        os.environ.pop(k, None)
    for kind, D, M in (("deep", 96, 32), ("sift", 128, 16)):
        x = gen.base(kind, 40_000, D, seed=2)
        q = gen.base(kind, 20, D, seed=2, stream=gen.STREAM_QUERY)
        cb = ref.train(x[:5_000], M, n_iter=2, seed=0)
        g = rii.Index(D, M, device=0)
        g.set_codebook(cb)
        g.add(x)
        g.reconfigure(8, n_iter=2, seed=0)
        o = ref.OracleIndex(D, M)
        o.cb = cb
        o.add(x)
        o.reconfigure(8, n_iter=2, seed=0)
        os.environ["RII_IVF_MODE"] = "list"
        os.environ["RII_LIST_Q16_MIN"] = "64"
        assert_topk_parity(ref, o.cb, o.codes, q, g.query(q, 100, L=4, path="ivf"), o.query(q, 100, L=4, path=2),
                           what=f"ivf {kind}")
        os.environ.pop("RII_IVF_MODE")
        os.environ.pop("RII_LIST_Q16_MIN")
        os.environ["RII_Q16_MIN"] = "20000"
        assert_topk_parity(ref, o.cb, o.codes, q, g.query(q, 100, path="linear"), o.query(q, 100, path=1),
                           what=f"linear {kind}")
        os.environ.pop("RII_Q16_MIN")
    print("ivf ok")


def masked():
    for k in ("RII_Q16_MIN", "RII_CHUNK_CODES", "RII_Q16_SAMPLE", "RII_IVF_MODE", "RII_LIST_Q16_MIN"):
        os.environ.pop(k, None)
    for kind, N, D, M, K in (("deep", 30_011, 96, 32, 40), ("deep", 20_003, 96, 8, 24)):
        x = gen.base(kind, N, D, seed=N)
        q = gen.base(kind, 37, D, seed=N, stream=gen.STREAM_QUERY)
        cb = ref.train(x[:4_000], M, n_iter=2, seed=0)
        g = rii.Index(D, M, device=0)
        g.set_codebook(cb)
        g.add(x)
        g.reconfigure(K, n_iter=2, seed=0)
        o = ref.OracleIndex(D, M)
        o.cb = cb
        o.add(x)
        o.reconfigure(K, n_iter=2, seed=0)
        for sub in (None, gen.subset(N, N // 3, seed=3)):
            for L in (2, 5, K):
                orr = o.query(q, 100, S=sub, L=L, path=2)
                for mode, rot in (("masked", None), (None, "1000000000"), (None, None)):
                    os.environ.pop("RII_IVF_MODE", None)
                    os.environ.pop("RII_COARSE_ROT_MINK", None)
                    if mode:
                        os.environ["RII_IVF_MODE"] = mode
                    if rot:
                        os.environ["RII_COARSE_ROT_MINK"] = rot
                    assert_topk_parity(ref, o.cb, o.codes, q, g.query(q, 100, target_ids=sub, L=L, path="ivf"), orr,
                                       S=sub, what=f"masked {kind} M={M} L={L} mode={mode} rot={rot}")
        os.environ.pop("RII_IVF_MODE", None)
        os.environ.pop("RII_COARSE_ROT_MINK", None)
    print("masked ok")


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    import torch
    torch.cuda.set_device(0)
    for name in (("tiny", "windows", "ivf", "masked") if which == "all" else (which,)):
        globals()[name]()
