"""Probe: the integer-table linear kernels (RII_Q16_CFG 0 = u16, 9 = 16-query u6)
must return identical results; where they differ, which matches the oracle.

    python tools/cfg_equivalence.py [workload] [nq]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1808_03969_b200 as rii  # noqa: E402
from oracle import ref  # noqa: E402
from synth import generators as gen  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "deep10m_m8"
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
kind, N, D, M, nlist, _, topk, n_train, _ = bench.WORKLOADS[wl]
dev = torch.device("cuda", 0)
g = rii.Index(D, M, device=0)
if os.environ.get("GPU_TRAIN"):  # the code book bench.py / ab_env.py use (20 iterations on the GPU)
    g.train(bench._device_data(kind, n_train, D, dev, 0, gen.STREAM_TRAIN), n_iter=20, seed=0)
    cb = g.get_codebook()
else:
    xt = bench._device_data(kind, 20000, D, dev, 0, gen.STREAM_TRAIN).cpu().numpy()
    cb = ref.train(xt, M, n_iter=3, seed=0)
    g.set_codebook(cb)
x = bench._device_data(kind, N, D, dev, 0, gen.STREAM_BASE)
g.add(x)
codes = ref.encode_mt(cb, x.cpu().numpy(), M)
del x
assert np.array_equal(g.get_codes(), codes)
q = bench._device_data(kind, nq, D, dev, 0, gen.STREAM_QUERY)
qh = q.cpu().numpy()
out = {}
runs = os.environ.get("CFG_RUNS", "0,9,4").split(",")
for j, cfg in enumerate(runs):
    os.environ["RII_Q16_CFG"] = cfg
    i, d, _ = g.query(q, topk, path="linear")
    out[f"{cfg}#{j}"] = (i.cpu().numpy(), d.cpu().numpy())
os.environ.pop("RII_Q16_CFG")
keys = list(out)
for a_, b_ in [(keys[0], k) for k in keys[1:]]:
    diff = np.nonzero((out[a_][0] != out[b_][0]).any(1) | (out[a_][1] != out[b_][1]).any(1))[0]
    print(f"cfg {a_} vs {b_}: {len(diff)} of {nq} queries differ", flush=True)
    if len(diff):
        sel = diff[:8]
        oi, od = ref.linear_mt(cb, codes, qh[sel], topk)
        for c in (a_, b_):
            eq = [np.array_equal(out[c][0][s], oi[r]) and np.array_equal(out[c][1][s], od[r]) for r, s in enumerate(sel)]
            print(f"  cfg {c}: {sum(eq)}/{len(sel)} equal the oracle", flush=True)
            for r, s in enumerate(sel[:2]):
                if not eq[r]:
                    gi, gd = out[c][0][s], out[c][1][s]
                    k = np.nonzero((gi != oi[r]) | (gd != od[r]))[0]
                    print(f"    q{s}: first diff rank {k[0]}: gpu ({gi[k[0]]}, {gd[k[0]]!r}) oracle ({oi[r][k[0]]}, {od[r][k[0]]!r});"
                          f" missing {np.setdiff1d(oi[r], gi)[:4]} extra {np.setdiff1d(gi, oi[r])[:4]}")
