"""Summarise an `ncu --set full` report into a short text table (committed under profiles/).

    python scripts/ncu_summary.py gpurun_out/ncu_copy.ncu-rep > profiles/r01/ncu_copy.txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clock"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem_%peak"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor_pipe_%"),
    ("sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active", "uniform_pipe_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved_occ_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__shared_mem_per_block_dynamic", "dyn_smem"),
    ("smsp__average_warp_latency_issue_stalled_long_scoreboard", "stall_long_sb"),
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        print("no data", path)
        return
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    print(f"# ncu --set full summary of {path}")
    for r in rows[2:]:
        name = r[col["Kernel Name"]] if "Kernel Name" in col else "?"
        grid = r[col["Grid Size"]] if "Grid Size" in col else "?"
        block = r[col["Block Size"]] if "Block Size" in col else "?"
        print(f"\n{name}  grid={grid} block={block}")
        for k, label in KEYS:
            if k in col:
                print(f"  {label:16s} {r[col[k]]:>16s} {units[col[k]]}")


if __name__ == "__main__":
    main(sys.argv[1])
