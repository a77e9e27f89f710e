"""Per-kernel roofline table from ncu --set full captures (one .ncu-rep per kernel).

    python tools/ncu_kernels.py gpurun_out/ncu_k_*.ncu-rep > profiles/r1_ncu_kernels.json

For each kernel: duration, DRAM bytes and bandwidth against MEASURED_PEAKS.json
hbm_gbs, FP64-pipe and issue utilization, achieved occupancy, and the bound
that applies (hbm when DRAM throughput dominates, else fp64/issue/latency).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
M = {
    "dur_us": ("gpu__time_duration.sum", 1e-3),
    "dram_read": ("dram__bytes_read.sum", 1.0),
    "dram_write": ("dram__bytes_write.sum", 1.0),
    "fp64_pipe_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "issue_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
    "alu_pct": ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 1.0),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "mem_pct": ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "regs": ("launch__registers_per_thread", 1.0),
    "grid": ("launch__grid_size", 1.0),
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3,
        "msecond": 1e6, "ms": 1e6}


def read(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, data = rows[0], rows[1], rows[2:]
    r = data[0]
    name = r[h.index("Kernel Name")]
    d = {"kernel": name.split("(")[0].replace("void ", "").replace("pumpg::", "")}
    for k, (m, scale) in M.items():
        if m not in h:
            continue
        i = h.index(m)
        v = float(r[i].replace(",", ""))
        v *= UNIT.get(units[i], 1.0)
        if k == "dur_us":
            v *= 1e-3  # ns -> us
        d[k] = round(v, 3)
    return d


def main():
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    hbm = float(peaks["hbm_gbs"])
    out = []
    for p in sys.argv[1:]:
        d = read(p)
        b = d.get("dram_read", 0) + d.get("dram_write", 0)
        gbs = b / (d["dur_us"] * 1e-6) / 1e9 if d.get("dur_us") else 0.0
        d["dram_gbs"] = round(gbs, 1)
        d["hbm_frac"] = round(gbs / hbm, 4)
        # the bound that applies: the most utilized of HBM bandwidth, the FP64
        # pipe and instruction issue; below 25% on all three the kernel is
        # latency-bound (dependent memory round trips, barriers)
        cand = {"hbm": d["hbm_frac"], "fp64": d.get("fp64_pipe_pct", 0) / 100, "issue": d.get("issue_pct", 0) / 100}
        b = max(cand, key=cand.get)
        d["bound"] = b if cand[b] >= 0.25 else "latency"
        d["frac"] = round(cand[b], 4)
        d["source"] = os.path.basename(p)
        out.append(d)
    print(json.dumps({"peak_hbm_gbs": hbm, "note": "ncu --set full --clock-control none, one launch per kernel "
                      f"({os.environ.get('NCU_WORKLOAD', 'quad3d_forest')} warm solve); frac = the utilization of "
                      "the bound that applies",
                      "kernels": out}, indent=1))


if __name__ == "__main__":
    main()
