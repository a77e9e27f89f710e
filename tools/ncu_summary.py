"""Summarise an ncu --set full report (raw page) into the metrics we track."""
import csv, io, subprocess, sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum', 'launch__registers_per_thread',
        'launch__grid_size', 'launch__block_size', 'sm__maximum_warps_per_active_cycle_pct', 'launch__occupancy_limit_registers',
        'smsp__thread_inst_executed_per_inst_executed.ratio', 'smsp__thread_inst_executed.sum']


def summarize(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, data = rows[0], rows[1], rows[2:]
    ki = h.index('Kernel Name')
    lines = []
    for r in data:
        lines.append(f"kernel: {r[ki][:90]}")
        for w in WANT:
            if w in h:
                i = h.index(w)
                lines.append(f"  {w}: {r[i]} {units[i]}")
    return "\n".join(lines)


if __name__ == '__main__':
    for p in sys.argv[1:]:
        print(f"# {p}")
        print(summarize(p))
