"""Render the measured rows of a round (profiles/<tag>_configs*.jsonl, <tag>_bench.json)
as the markdown tables of BASELINE.md's "Results" section.

    python tools/render_results.py r02 > /tmp/results.md
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rows(path):
    out = []
    if not os.path.exists(path):
        return out
    for ln in open(path):
        ln = ln.strip()
        if ln.startswith("{"):
            try:
                out.append(json.loads(ln))
            except json.JSONDecodeError:
                pass
    return out


def fmt_qps(v):
    return f"{v:,.0f}" if v else "—"


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
    P = lambda f: os.path.join(ROOT, "profiles", f)  # noqa: E731
    print("| Config | Row | ms per call | queries/s | notes |")
    print("|---|---|---|---|---|")
    for d in rows(P(f"{tag}_configs.jsonl")) + rows(P(f"{tag}_configs_scale1b.jsonl")):
        row = d.get("row", "").replace("|", "\\|")
        note = []
        if "path_used" in d:
            note.append(f"path {d['path_used']}")
        if "scanned_codes_per_s" in d:
            note.append(f"{d['scanned_codes_per_s'] / 1e9:.1f} G codes/s")
        for k in ("train_s", "add_s", "reconfigure_s"):
            if k in d:
                note.append(f"{k[:-2]} {d[k]:.2f} s")
        if "a" in d and "crossovers" in d:
            note.append(f"θ(L) = {d['a']:.0f}·L + {d['b']:.0f}")
        if "roofline" in d:
            note.append(f"{d['roofline']['frac']:.2f} of the {d['roofline']['note'].split(',')[0]} LUT peak")
        ms = d.get("ms")
        print(f"| {d.get('config')} | {row} | {ms:.2f} |" if ms else f"| {d.get('config')} | {row} | — |", end="")
        print(f" {fmt_qps(d.get('qps'))} | {'; '.join(note)} |")
    print()
    print("| Shape | Row | ms per 10k queries | µs per query |")
    print("|---|---|---|---|")
    for d in rows(P(f"{tag}_configs_paper_t2.jsonl")):
        if "ms" in d:
            print(f"| {d['config']} | {d['row']} | {d['ms']:.2f} | {d['ms'] / d['nq'] * 1e3:.2f} |")
        else:
            print(f"| {d['config']} | {d['row']} | — | train {d.get('train_s', 0):.2f} s, add {d.get('add_s', 0):.2f} s, "
                  f"reconfigure {d.get('reconfigure_s', 0):.2f} s |")


if __name__ == "__main__":
    main()
