"""Summarise an ncu report (raw page): per launch the duration, DRAM bytes,
throughputs, occupancy, cache hit rates and pipe utilisation."""
import csv
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("l1tex__t_sector_hit_rate.pct", "l1_hit_%"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1_%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_%"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_inst_%"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_%"),
    ("sm__inst_executed_pipe_tensor_op_dmma.sum", "dmma_inst"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "gld_requests"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "gld_sectors"),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")][:60]
        vals = []
        for key, label in WANT:
            if key in hdr:
                i = hdr.index(key)
                vals.append(f"{label}={r[i]}{units[i] if units[i] not in ('', 'inst') else ''}")
        print(name, "|", " ".join(vals))


if __name__ == "__main__":
    main(sys.argv[1])
