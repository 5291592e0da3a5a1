"""Per-kernel unit breakdown of an `ncu --page raw --csv` export: which
sub-unit of L1TEX / L2 binds (writeback to registers, data-pipe wavefronts,
L2->L1 fill, L2 slice output), per launch, as JSON for profiles/.

usage: python tools/ncu_units.py RAW.csv OUT.json --command "..." --note "..."
"""
import argparse
import csv
import json

UNITS = {
    "time_ms": "gpu__time_duration.sum",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "l1_writeback_to_rf_pct": "l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_elapsed",
    "l1_data_pipe_wavefronts_pct": "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1_data_bank_reads_pct": "l1tex__data_bank_reads.avg.pct_of_peak_sustained_elapsed",
    "l1_data_bank_writes_pct": "l1tex__data_bank_writes.avg.pct_of_peak_sustained_elapsed",
    "l2_to_l1_fill_pct": "l1tex__m_xbar2l1tex_read_sectors.avg.pct_of_peak_sustained_elapsed",
    "l1_lsuin_requests_pct": "l1tex__lsuin_requests.avg.pct_of_peak_sustained_elapsed",
    "l2_throughput_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_slice_to_xbar_pct": "lts__lts2xbar_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "l2_tex_sectors_pct": "lts__t_sectors_srcunit_tex.avg.pct_of_peak_sustained_elapsed",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "l1_hit_pct": "l1tex__t_sector_hit_rate.pct",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "issue_active_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "global_load_requests": "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "global_load_sectors": "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("raw")
    ap.add_argument("out")
    ap.add_argument("--command", required=True)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    rows = list(csv.reader(open(a.raw)))
    hdr, data = rows[0], rows[2:]
    ni = hdr.index("Kernel Name")
    launches = []
    for r in data:
        d = {"kernel": r[ni].split("(")[0].replace("void unnamed>::", "")}
        for k, m in UNITS.items():
            if m in hdr and r[hdr.index(m)] not in ("", "n/a"):
                try:
                    d[k] = float(r[hdr.index(m)].replace(",", ""))
                except ValueError:
                    d[k] = r[hdr.index(m)]
        launches.append(d)
    json.dump({"command": a.command, "note": a.note, "launches": launches}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
