"""A/B of query configurations on BASELINE.json configs[4] (1e9 codes, M = 8, nlist =
31,623) built once on one B200, as tools/configs.py builds it; each case in 1,024-query
batches, median of --reps, with one RII_TRACE=1 call per case (phase times on stderr).

    python tools/scale_ab.py "VAR=a;VAR2=b" VAR=c ...
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1808_03969_b200 as rii  # noqa: E402
from synth import generators as gen  # noqa: E402

DEV = torch.device("cuda", 0)


def main():
    prof = "--profile" in sys.argv  # one IVF L = 64 call between cudaProfilerStart / Stop (ncu)
    prof_lin = "--profile-linear" in sys.argv  # one whole linear scan of 1,024 queries instead
    settings = [a for a in sys.argv[1:] if not a.startswith("--profile")] or [""]
    c = gen.CONFIGS["scale1b"]
    N, D, M, K = c["N"], c["D"], c["M"], c["nlist"]
    g = rii.Index(D, M, device=0)
    g.train(bench._device_data("deep", c["n_train"], D, DEV, 0, gen.STREAM_TRAIN), n_iter=20, seed=0)
    chunk = 1 << 24
    for s0 in range(0, N, chunk):
        xb = gen.deep_like_torch(min(chunk, N - s0), DEV, D=D, seed=0, stream=gen.STREAM_BASE,
                                    batch=s0 // chunk)
        g.add(xb)
        del xb
    torch.cuda.empty_cache()
    g.reconfigure(K, n_iter=10, seed=0)
    torch.cuda.synchronize()
    q = gen.deep_like_torch(1024, DEV, D=D, seed=0, stream=gen.STREAM_QUERY)
    S = gen.subset_torch(N, 1_000_000, DEV, seed=1)
    st = torch.cuda.current_stream()
    if prof or prof_lin:
        path = "linear" if prof_lin else "ivf"
        g.query(q, 100, None, L=64, path=path)
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        g.query(q, 100, None, L=64, path=path)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        return
    for name, sub, L, path in (("ivf whole L=64", None, 64, "ivf"), ("subset 1e6 linear", S, 64, "linear"),
                               ("subset 1e6 ivf", S, 64, "ivf"), ("linear whole", None, 64, "linear")):
        for s in settings:
            env = dict(kv.split("=", 1) for kv in s.split(";") if kv)
            old = {k: os.environ.get(k) for k in env}
            os.environ.update(env)
            g.query(q, 100, sub, L=L, path=path)
            torch.cuda.synchronize()
            os.environ["RII_TRACE"] = "1"
            print(f"--- {name} {env}", file=sys.stderr, flush=True)
            g.query(q, 100, sub, L=L, path=path)
            torch.cuda.synchronize()
            os.environ.pop("RII_TRACE")
            ms = []
            for _ in range(5):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                g.query(q, 100, sub, L=L, path=path)
                b.record(st)
                torch.cuda.synchronize()
                ms.append(a.elapsed_time(b))
            print(json.dumps({"case": name, "env": env, "ms_per_1024": statistics.median(ms)}), flush=True)
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v


if __name__ == "__main__":
    main()
