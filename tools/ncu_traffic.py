"""profiles/r02_traffic.json from `ncu --page raw --csv` exports: DRAM bytes per launch of the dominant kernels
(bench.py reads it for `roofline.traffic`).
usage: ncu_traffic.py <tag>      e.g. r02j -> profiles/<tag>_ncu_full_k_postssa_gtile_raw.csv, ..._k_typeseed_raw.csv"""
import csv, json, sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}


def metric(path, name):
    rows = list(csv.reader(open(path)))
    i = rows[0].index(name)
    return float(rows[2][i]) * SCALE[rows[1][i]]


def main(tag):
    out_path = ROOT / "profiles" / "r02_traffic.json"
    out = json.loads(out_path.read_text()) if out_path.exists() else {}
    for key, extra in (("k_postssa_gtile", {"workload_sass_insts": 99993527}), ("k_typeseed", {"workload_sass_insts": 20000544})):
        p = ROOT / "profiles" / f"{tag}_ncu_full_{key}_raw.csv"
        if not p.exists():
            continue
        rd, wr = metric(p, "dram__bytes_read.sum"), metric(p, "dram__bytes_write.sum")
        out[key] = dict(extra, dram_bytes_per_launch=rd + wr, dram_bytes_read=rd, dram_bytes_written=wr,
                        kernel_ms_under_ncu=metric(p, "gpu__time_duration.sum"),
                        source=f"profiles/{p.name} (ncu --set full --clock-control none, one launch)")
    out_path.write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
