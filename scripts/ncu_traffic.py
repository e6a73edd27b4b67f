"""Per-launch DRAM traffic of the dcnv4 kernels in a bench workload, from an ncu capture
(dram__bytes_read.sum + dram__bytes_write.sum), written to profiles/ncu_traffic.json for
bench.py's roofline `traffic` field.

  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none --csv --log-file gpurun_out/traffic_c4.csv \
      python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-verify --e2e-steps 1
  python scripts/ncu_traffic.py gpurun_out/traffic_c4.csv c4
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(path, workload):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = {}
    for r in rows:
        if "Kernel Name" in r and "Metric Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        name = r[hdr.index("Kernel Name")]
        kind = "bwd" if ("bwd" in name) else ("fwd" if "fwd" in name else None)
        if kind is None:
            continue
        lid = r[hdr.index("ID")]
        m = r[hdr.index("Metric Name")]
        unit = r[hdr.index("Metric Unit")]
        v = float(r[hdr.index("Metric Value")].replace(",", ""))
        if v != v:  # nan: a graph-capture placeholder launch (grid 0x0x0)
            continue
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        per.setdefault((kind, lid), {})[m] = v * scale
    out_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    data = json.load(open(out_path)) if os.path.exists(out_path) else {}
    res = {}
    for kind in ("fwd", "bwd"):
        ls = [d for (k, _), d in per.items() if k == kind and "dram__bytes_read.sum" in d]
        if not ls:
            continue
        tot = sum(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in ls)
        res[kind] = tot / len(ls)
        res[kind + "_launches"] = len(ls)
    data[workload] = res
    data["_how"] = ("ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over one bench step; "
                    "bytes per launch averaged over the step's launches of each kernel")
    with open(out_path, "w") as f:
        json.dump(data, f, indent=1)
    print(json.dumps(data, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
