"""Summarise ncu outputs into profiles/.

  python scripts/ncu_summary.py launches <launches.csv> [key]    per-kernel share of one step
                                                                 (key: record the totals in the json)
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


UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def launches(path, record=None):
    """Per-kernel time (and DRAM bytes when the list carries dram__bytes_*) of one step.
    With `record`, the per-step totals go to profiles/ncu_summary.json[record]."""
    rows = _csv_rows(open(path).read())
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    ui = h.index("Metric Unit") if "Metric Unit" in h else None
    tot = collections.defaultdict(float)
    dram = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[1:]:
        k = r[ki].split("(")[0]
        v = float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            tot[k] += v
            cnt[k] += 1
        elif r[mi] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            dram[k] += v * (UNIT.get(r[ui], 1) if ui is not None else 1)
    T = sum(tot.values())
    has_dram = bool(dram)
    print("| kernel | launches | total ms (ncu, serialised, cold) | share |" + (" DRAM GB |" if has_dram else ""))
    print("|---|---|---|---|" + ("---|" if has_dram else ""))
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"| {k} | {cnt[k]} | {v / 1e6:.2f} | {100 * v / T:.2f}% |" + (f" {dram[k] / 1e9:.2f} |" if has_dram else ""))
    D = sum(dram.values())
    print(f"| total | {sum(cnt.values())} | {T / 1e6:.2f} | 100% |" + (f" {D / 1e9:.2f} |" if has_dram else ""))
    if record:
        js_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
        try:
            js = json.load(open(js_path))
        except Exception:
            js = {}
        js[record] = {"dram_bytes_per_step": D if has_dram else None, "ms_per_step": T / 1e6,
                      "launches": sum(cnt.values()), "source": os.path.relpath(path, ROOT),
                      "per_kernel": {k: {"launches": cnt[k], "ms": tot[k] / 1e6, "dram_bytes": dram.get(k)}
                                     for k in tot}}
        with open(js_path, "w") as f:
            json.dump(js, f, indent=1)


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
        launches(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
    else:
        full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
