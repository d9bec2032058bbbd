"""DRAM traffic per launch of the bench's roofline kernels, from an ncu `--page raw --csv` export of
`profiles/prof_kernels.py --only mf,afw,spmv` (standalone launches), into the files bench.py reads
for the `traffic` field of its roofline entries:

    python profiles/ncu_dram_json.py RAW.csv --config 4 --source "..."

  r02_dram_bytes_c{config}_mf.json    k_mf_spmv (non-reducing: cr_spmv_mf)
  r02_dram_bytes_c{config}_afw.json   k_afw_apply_sh + k_afw_zsum (cr_apply_precond, one-level patch)
  r02_dram_bytes_c{config}_spmv.json  k_spmv (assembled G)

The last launch of each kernel in the capture is taken (the standalone ones come after the solve).
"""
import argparse
import csv
import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))
GROUPS = {"mf": ["k_mf_spmv"], "afw": ["k_afw_apply_sh", "k_afw_zsum"], "spmv": ["k_spmv"]}
# --groups "mf=k_mf_spmv afw_apply=k_afw_apply_sh": other tags / kernel sets (e.g. from a capture of the
# solve's own launches: profiles/prof_kernels.py --solve-iters 8 --only spmv)
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--source", default="")
    ap.add_argument("--groups", default=None)
    a = ap.parse_args()
    groups = GROUPS
    if a.groups:
        groups = {g.split("=")[0]: g.split("=")[1].split("+") for g in a.groups.split()}
    rows = list(csv.reader(open(a.csv)))
    h, units = rows[0], rows[1]
    ix = {n: i for i, n in enumerate(h)}
    last = {}
    for r in rows[2:]:
        base = r[ix["Kernel Name"]].split("<")[0].split("(")[0].replace("void ", "").strip()
        last[base] = r

    def val(r, m):
        return float(r[ix[m]].replace(",", "")) * UNIT.get(units[ix[m]], 1.0)

    for tag, names in groups.items():
        rs = [last[n] for n in names if n in last]
        if len(rs) != len(names):
            print("missing", tag, [n for n in names if n not in last])
            continue
        rd = sum(val(r, "dram__bytes_read.sum") for r in rs)
        wr = sum(val(r, "dram__bytes_write.sum") for r in rs)
        out = {"kernel": " + ".join(r[ix["Kernel Name"]].split("(")[0] for r in rs) + f" (configs[{a.config}])",
               "dram_bytes_read": int(rd), "dram_bytes_write": int(wr), "dram_bytes_per_launch": int(rd + wr),
               "duration_us_ncu": sum(val(r, "gpu__time_duration.sum") for r in rs) *
               {"ns": 1e-3, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(units[ix["gpu__time_duration.sum"]], 1.0),
               "source": a.source or os.path.basename(a.csv)}
        p = os.path.join(HERE, f"r02_dram_bytes_c{a.config}_{tag}.json")
        with open(p, "w") as f:
            json.dump(out, f, indent=1)
        print(p, out["dram_bytes_per_launch"])


if __name__ == "__main__":
    main()
