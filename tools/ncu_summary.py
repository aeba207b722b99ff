"""Key metrics of an `ncu --page raw --csv` export (one row per kernel):
duration, DRAM bytes and throughput, SM/FMA/tensor pipe utilisation,
warps active, registers, grid.  Usage: ncu_summary.py raw.csv [...]"""
import csv
import sys

KEYS = [
    ("Kernel Name", "kernel"),
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA inst %"),
    ("sm__pipe_tensor_op_tcgen05_mma_cycles_active.avg.pct_of_peak_sustained_active", "tcgen05 MMA pipe %"),
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "TC pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefronts %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
]


def summary(path):
    rows = list(csv.reader(open(path)))
    h, units = rows[0], rows[1]
    out = []
    for row in rows[2:]:
        for key, label in KEYS:
            if key in h:
                i = h.index(key)
                out.append(f"{label:22s} {row[i]} {units[i]}".rstrip())
        extra = [j for j, k in enumerate(h) if "tensor" in k and "pct_of_peak_sustained_active" in k
                 and k.startswith("sm__pipe") and row[j] not in ("", "0")]
        for j in extra:
            out.append(f"{h[j]:22s} {row[j]}")
        out.append("")
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(f"== {p}")
        print(summary(p))
