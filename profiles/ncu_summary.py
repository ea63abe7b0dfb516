"""Summarise ncu captures for profiles/: the launch list (per-kernel share of the device time)
and the key `--set full` metrics of the top kernel, including its DRAM traffic per launch.
  python profiles/ncu_summary.py launches <launches.csv>
  python profiles/ncu_summary.py full <prof.ncu-rep> <out.json>"""
import collections
import csv
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
        "launch__block_size", "launch__registers_per_thread", "launch__occupancy_limit_shared_mem",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "lts__t_bytes.sum", "smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3}


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        agg[r[ki].split("(")[0][:90]].append(float(r[vi].replace(",", "")) / 1e3)
    tot = sum(sum(v) for v in agg.values())
    print(f"{'kernel':90s} {'n':>5s} {'sum_us':>10s} {'avg_us':>9s} share")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"{k:90s} {len(v):5d} {sum(v):10.1f} {sum(v) / len(v):9.2f} {100 * sum(v) / tot:5.1f}%")


def full(rep, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")]}
        for k in KEYS:
            if k in h:
                i = h.index(k)
                v = r[i].replace(",", "")
                try:
                    d[k] = float(v) * UNIT.get(units[i], 1)
                    if units[i] in UNIT:
                        d[k + ".unit"] = "us" if units[i] in ("ns", "us", "ms") else "byte"
                except ValueError:
                    d[k] = v
        d["traffic_bytes"] = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        res.append(d)
    json.dump(res, open(out, "w"), indent=1)
    for d in res:
        print(d["kernel"][:80], f"{d['gpu__time_duration.sum']:.2f} us", f"traffic {d['traffic_bytes'] / 1e6:.3f} MB")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], sys.argv[3])
