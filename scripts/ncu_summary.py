"""Summaries of the ncu evidence committed under profiles/.

usage:
  python scripts/ncu_summary.py launches LAUNCHES.csv "COMMAND"   # per-kernel totals + step shares
  python scripts/ncu_summary.py full REPORT.ncu-rep N_POINTS       # key --set full metrics per launch
"""
import collections
import csv
import io
import subprocess
import sys

STEP = ("ring_kernel<512, 2, 2", "zline_kernel<512, 4, 0, double2, 0", "tile_kernel<512, 0, 0, 0, 0",
        "tile_kernel<512, 1, 0, 0, 0")


def launches(path, cmd):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    name, val, unit, met = (h.index(k) for k in ("Kernel Name", "Metric Value", "Metric Unit", "Metric Name"))
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[1:]:
        if r[met] != "gpu__time_duration.sum":
            continue
        v = float(r[val].replace(",", ""))
        ms = {"ns": v / 1e6, "us": v / 1e3, "ms": v, "s": v * 1e3}[r[unit]]
        k = r[name].split("(")[0]
        tot[k] += ms
        cnt[k] += 1
    print(f"# command: {cmd}")
    print("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised)")
    print("# total_ms  launches  mean_ms  kernel")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{v:10.3f} {cnt[k]:5d} {v / cnt[k]:9.4f}  {k}")
    step = {k: tot[k] / cnt[k] for k in tot if any(s in k for s in STEP)}
    s = sum(step.values())
    print(f"\n# per split step (mean launch of each of the 4 step kernels): {s:.3f} ms")
    for k, v in step.items():
        print(f"#   share {k:60s} {100 * v / s:5.1f}%")


FULL = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__shared_mem_per_block_dynamic"]


def full(rep, npts):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(FULL)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(h, r))
        print("---")
        print(f"  Kernel Name = {d['Kernel Name'].split('(')[0]}")
        for k in FULL:
            if k in d:
                print(f"  {k} = {d[k]} {units[h.index(k)]}")
        rd, wr = float(d["dram__bytes_read.sum"]), float(d["dram__bytes_write.sum"])
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
        b = rd * scale[units[h.index("dram__bytes_read.sum")]] + wr * scale[units[h.index("dram__bytes_write.sum")]]
        print(f"  dram_bytes_per_point = {b / npts:.2f}")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], int(sys.argv[3]))
