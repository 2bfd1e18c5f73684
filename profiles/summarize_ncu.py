"""Summarise an `ncu --set full` capture (.ncu-rep) into the metrics the
roofline / DESIGN.md discussion uses.  Usage:
    python profiles/summarize_ncu.py gpurun_out/prof_stage.ncu-rep > profiles/<name>.txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "derived__memory_l1_wavefronts_shared_excessive",
    "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum",
]
STALL = "smsp__average_warps_issue_stalled_"


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print(f"== {d.get('Kernel Name', '?')[:90]}  (ID {d.get('ID')})")
        for k in KEYS:
            if k in d:
                print(f"  {k:70s} {d[k]:>16s} {u[k]}")
        stalls = sorted(((float(d[k]), k[len(STALL):].replace('_per_issue_active.ratio', ''))
                         for k in d if k.startswith(STALL) and k.endswith("_per_issue_active.ratio")
                         and d[k] not in ("", "n/a")), reverse=True)
        print("  stalls (warps per issue): " + ", ".join(f"{n} {v:.2f}" for v, n in stalls[:7]))


if __name__ == "__main__":
    main(sys.argv[1])
