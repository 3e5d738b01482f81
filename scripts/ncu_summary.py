"""Summarise ncu outputs into profiles/.

  python scripts/ncu_summary.py launches <launches.csv>          per-kernel share of one step
  python scripts/ncu_summary.py full <prof.ncu-rep> [tag]         key metrics of the full capture
Writes nothing by itself; prints markdown (redirect into profiles/).  `full`
also updates profiles/ncu_summary.json (dram bytes per launch by kernel tag),
which bench.py reads for roofline.traffic.
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _csv_rows(text):
    lines = text.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    return list(csv.reader(io.StringIO("\n".join(lines[start:]))))


def launches(path):
    rows = _csv_rows(open(path).read())
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        k = r[ki].split("(")[0]
        tot[k] += float(r[vi].replace(",", ""))
        cnt[k] += 1
    T = sum(tot.values())
    print("| kernel | launches | total ms (ncu, serialised, cold) | share |")
    print("|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"| {k} | {cnt[k]} | {v / 1e6:.2f} | {100 * v / T:.2f}% |")
    print(f"| total | {sum(cnt.values())} | {T / 1e6:.2f} | 100% |")


KEYS = [
    "Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
    "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__t_sector_hit_rate.pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second",
]


def full(path, tag=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = _csv_rows(out)
    h, units = rows[0], rows[1]
    js_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        js = json.load(open(js_path))
    except Exception:
        js = {}
    for r in rows[2:]:
        d = dict(zip(h, r))
        name = d["Kernel Name"].split("(")[0]
        print(f"### {name}\n")
        print("| metric | value | unit |\n|---|---|---|")
        for k in KEYS:
            if k in d:
                print(f"| {k} | {d[k]} | {units[h.index(k)]} |")

        def val(k):
            v = float(d[k].replace(",", ""))
            u = units[h.index(k)]
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
            return v * mult

        try:
            b = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
            js[tag or name] = {"dram_bytes_per_launch": b, "source": os.path.basename(path),
                               "duration": d.get("gpu__time_duration.sum")}
            print(f"\nDRAM read+write per launch: {b / 1e9:.3f} GB")
        except Exception:
            pass
        print()
    with open(js_path, "w") as f:
        json.dump(js, f, indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
