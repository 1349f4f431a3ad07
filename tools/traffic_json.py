"""Write profiles/scan_traffic.json from an `ncu --set full` raw CSV export of the
headline scan kernel (`ncu -i rep --page raw --csv`), tagged with the hash of the
kernel sources it was captured on (bench.py reports `roofline.traffic` only when
that hash matches the sources it built).

    python tools/traffic_json.py raw.csv KIND "capture command" [commit]
KIND: u6 | u16 | packed | fp32 (the table variant bench.py's roofline names).
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    path, kind, capture = sys.argv[1], sys.argv[2], sys.argv[3]
    commit = sys.argv[4] if len(sys.argv) > 4 else None
    rows = list(csv.reader(open(path)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}

    def val(r, name):
        v = r[col[name]].replace(",", "")
        u = units[col[name]]
        x = float(v)
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3,
                 "msecond": 1.0, "second": 1e3, "%": 1}.get(u, 1)
        return x * scale

    r = data[0]
    rd = val(r, "dram__bytes_read.sum")
    wr = val(r, "dram__bytes_write.sum")
    import bench
    out = {
        "kernel": r[col["Kernel Name"]],
        "kernel_kind": kind,
        "dram_bytes_read": rd,
        "dram_bytes_write": wr,
        "dram_bytes_per_launch": rd + wr,
        "duration_ms": val(r, "gpu__time_duration.sum"),
        "shared_wavefronts_pct_of_peak": float(r[col["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"]])
        if "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed" in col else None,
        "source": capture,
        "source_sha16": bench._source_hash(),
        "commit": commit,
    }
    with open(os.path.join(ROOT, "profiles", "scan_traffic.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
