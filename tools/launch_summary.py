"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of tools/prof_solve.py.

    python tools/launch_summary.py gpurun_out/launches.csv 2 > profiles/r1_launches_latest.txt

With R solves in the profiled process, the last 1/R of the launches (the final, warm solve) is summarised.
"""
import collections
import csv
import sys


def load(path):
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    return [(r[ki], float(r[vi]) / 1e3) for r in rows[1:] if r[mi] == "gpu__time_duration.sum"]


def short(name):
    name = name.replace("void ", "")
    p = name.find("(")
    return name[:p] if p > 0 else name


def main():
    path = sys.argv[1]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    launches = load(path)
    per = len(launches) // reps
    last = launches[len(launches) - per:]
    agg = collections.OrderedDict()
    for n, us in last:
        a = agg.setdefault(short(n), [0, 0.0])
        a[0] += 1
        a[1] += us
    total = sum(v[1] for v in agg.values())
    cmd = sys.argv[3] if len(sys.argv) > 3 else f"tools/one_solve.py quad3d_forest {reps}"
    print(f"# ncu --metrics gpu__time_duration.sum --clock-control none python {cmd}")
    print("# last (warm) solve of the process; ncu serializes launches (bank / MC-table side-stream kernels included)")
    print(f"# {len(last)} launches, kernel time sum {total:.1f} us")
    print(f"{'kernel':<54}{'n':>3}{'avg_us':>10}{'total_us':>10}{'share':>8}")
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:53]:<54}{n:>3}{us / n:>10.2f}{us:>10.1f}{100 * us / total:>7.1f}%")


if __name__ == "__main__":
    main()
