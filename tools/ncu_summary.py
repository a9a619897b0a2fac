"""Summarise an ncu report (raw page) into the handful of metrics the roofline discussion uses."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy%"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_pipe%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_cycles%"),
    ("smsp__inst_executed.sum", "warp_inst"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_thru%"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex%"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wf"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_conflicts"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "gld_sectors"),
    ("lts__t_sectors.sum", "l2_sectors"),
    ("smsp__average_warp_latency_issue_stalled_barrier", "stall_bar"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
    ("local_load", ""),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = d.get("Kernel Name", "")[:90]
        print(name)
        for k, lab in KEYS:
            if k in d:
                print(f"   {lab:16s} {d[k]:>16s} {u.get(k, '')}")
        stalls = sorted(((float(v.replace(',', '')), k) for k, v in d.items()
                         if k.startswith("smsp__average_warp_latency_issue_stalled_") and k.endswith("_per_warp_active.pct")
                         and v.replace('.', '', 1).replace(',', '').isdigit()), reverse=True)[:6]
        for v, k in stalls:
            print(f"   stall {k.split('stalled_')[1].replace('_per_warp_active.pct',''):22s} {v:8.1f} %")


if __name__ == "__main__":
    main(sys.argv[1])
