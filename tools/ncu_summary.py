"""Summarise an ncu report (--set full) into markdown: per-kernel duration,
DRAM bytes/throughput, DMMA pipe utilisation, occupancy, top stall reasons.
    python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/rNN_x.md"""
import csv
import io
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput %"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA pipe active %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 (DFMA) pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    print(f"# ncu summary: `{path}`\n")
    for r in rows[2:]:
        name = r[col["Kernel Name"]] if "Kernel Name" in col else "?"
        print(f"## `{name[:120]}`\n")
        print("| metric | value |\n|---|---|")
        for key, label in WANT:
            if key in col and col[key] < len(r):
                print(f"| {label} (`{key}`) | {r[col[key]]} {units[col[key]]} |")
        stalls = []
        for h, i in col.items():
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
                try:
                    stalls.append((float(r[i].replace(",", "")), h.split("stalled_")[1]))
                except (ValueError, IndexError):
                    pass
        stalls.sort(reverse=True)
        tot = sum(v for v, _ in stalls) or 1.0
        print("\nTop warp-state samples: " + ", ".join(f"{n} {100 * v / tot:.0f}%"
                                                     for v, n in stalls[:6]) + "\n")


if __name__ == "__main__":
    main(sys.argv[1])
