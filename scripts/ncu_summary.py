"""Summarise ncu reports (raw page) into one JSON object per kernel for profiles/.

  python scripts/ncu_summary.py gpurun_out/fwd_v1.ncu-rep [more.ncu-rep ...] > profiles/x.json
Launch lists (--csv --log-file launches.csv) are summarised with --launches.
"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct", "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__m_xbar2l1tex_read_bytes.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__sass_inst_executed_op_global_red.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__block_size", "launch__grid_size", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "lts__t_sectors_op_red.sum", "lts__t_sectors_op_atom.sum",
]


def raw(rep):
    if rep.endswith(".csv"):  # an already exported `ncu -i rep --page raw --csv`
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
    rows = [r for r in csv.reader(io.StringIO(out)) if r and not r[0].startswith("==")]
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                v = vals[i].replace(",", "")
                try:
                    v = float(v)
                except ValueError:
                    pass
                d[m] = [v, units[i]]
        res.append(d)
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = {}
    for r in rows:
        if "Kernel Name" in r and "Metric Value" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        name = r[hdr.index("Kernel Name")]
        unit = r[hdr.index("Metric Unit")]
        v = float(r[hdr.index("Metric Value")].replace(",", ""))
        if v != v:  # nan: a graph-capture placeholder launch (grid 0x0x0)
            continue
        v = v / 1000.0 if unit in ("nsecond", "ns") else (v * 1000.0 if unit in ("msecond", "ms") else v)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    return [{"kernel": k, "launches": a[0], "total_us": round(a[1], 2),
             "share": round(a[1] / tot, 4) if tot else 0}
            for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1])]


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        print(json.dumps(launches(sys.argv[2]), indent=1))
    else:
        print(json.dumps([r for rep in sys.argv[1:] for r in raw(rep)], indent=1))
