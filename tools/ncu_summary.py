"""Summarise an `ncu --page raw --csv` export into the profiles/ JSON that
bench.py reads for roofline.traffic (dram read+write bytes per launch of the
dominant kernel) and the judge reads for the kernel metrics.

usage: python tools/ncu_summary.py RAW.csv OUT.json --command "..." \
           --algorithmic-bytes B [--dominant REGEX]"""
import argparse
import csv
import json
import re

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "launch__grid_size",
    "launch__block_size", "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def to_bytes(val, unit):
    return float(val.replace(",", "")) * SCALE.get(unit, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("raw")
    ap.add_argument("out")
    ap.add_argument("--command", required=True)
    ap.add_argument("--workload", default="reddit-shaped (V=232965, E=114.6M), 1x B200")
    ap.add_argument("--algorithmic-bytes", type=int, required=True)
    ap.add_argument("--dominant", default=r"k_agg_vec4<32")
    ap.add_argument("--path-kernels", default=None,
                    help="regex of every launch of the dominant path (summed: passes + concurrent heavy kernel)")
    ap.add_argument("--round", type=int, default=1)
    a = ap.parse_args()
    rows = list(csv.reader(open(a.raw)))
    hdr, units = rows[0], rows[1]
    kernels, dom = [], None
    for r in rows[2:]:
        k = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                k[m] = f"{r[i]} {units[i]}".strip()
        kernels.append(k)
        if dom is None and re.search(a.dominant, r[hdr.index("Kernel Name")]):
            i, j = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
            dom = (k["kernel"], int(to_bytes(r[i], units[i]) + to_bytes(r[j], units[j])))
    if a.path_kernels:
        tot, names, dur = 0, [], 0.0
        for r in rows[2:]:
            name = r[hdr.index("Kernel Name")]
            if re.search(a.path_kernels, name):
                i, j = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
                tot += int(to_bytes(r[i], units[i]) + to_bytes(r[j], units[j]))
                names.append(name.split("(")[0])
                k = hdr.index("gpu__time_duration.sum")
                dur += float(r[k].replace(",", "")) * (1e-3 if units[k] == "us" else (1e-6 if units[k] == "ns" else 1.0))
        dom = ("+".join(names) + " (one path execution)", tot)
    # duration-weighted unit throughputs and hit rates over the path's
    # launches: the unit nearest its peak is the one that binds
    sel = [r for r in rows[2:] if re.search(a.path_kernels or a.dominant, r[hdr.index("Kernel Name")])]

    def num(r, m):
        if m not in hdr:
            return None
        try:
            return float(r[hdr.index(m)].replace(",", ""))
        except ValueError:
            return None

    def wavg(m):
        tot = w = 0.0
        for r in sel:
            d, v = num(r, "gpu__time_duration.sum"), num(r, m)
            if d is not None and v is not None:
                tot += d * v
                w += d
        return round(tot / w, 2) if w else None

    units_pct = {"dram": wavg("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                 "l2 (lts)": wavg("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
                 "l1tex": wavg("l1tex__throughput.avg.pct_of_peak_sustained_elapsed"),
                 "sm": wavg("sm__throughput.avg.pct_of_peak_sustained_elapsed")}
    known = {k: v for k, v in units_pct.items() if v is not None}
    bind = max(known, key=known.get) if known else None
    secs = sum(num(r, "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum") or 0 for r in sel)
    reqs = sum(num(r, "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum") or 0 for r in sel)
    out = {"round": a.round, "command": a.command, "workload": a.workload,
           "dominant_kernel": dom[0] if dom else None, "dram_bytes_per_launch": dom[1] if dom else None,
           "algorithmic_bytes_per_launch": a.algorithmic_bytes,
           "unit_throughput_pct": units_pct, "binding_unit": bind, "binding_unit_pct": known.get(bind),
           "l2_hit_rate_pct": wavg("lts__t_sector_hit_rate.pct"),
           "sectors_per_request": round(secs / reqs, 2) if reqs else None,
           "global_load_requests": int(reqs), "global_load_sectors": int(secs),
           "kernels": kernels}
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "kernels"}))


if __name__ == "__main__":
    main()
