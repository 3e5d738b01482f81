"""Summarise a ROTOR_TRACE timeline of one tile-DAG fill (per tile task: host
enqueue time, GPU start of its middle, GPU end of its dependent phase; us from
the fill's start).  Usage: python scripts/dag_timeline.py <trace.csv>
Prints markdown: per tile diagonal the tasks' start / end spread and mean task
duration, and the wall time each diagonal's front takes."""
import collections
import csv
import sys


def main(path):
    lines = [l for l in open(path) if not l.startswith("#")]
    tail = [l for l in open(path) if l.startswith("#")]
    rows = [{k: float(v) for k, v in r.items()} for r in csv.DictReader(lines)]
    by = collections.defaultdict(list)
    for r in rows:
        by[int(r["J"] - r["I"])].append(r)
    print("| delta | tiles | first start (us) | last end (us) | front span (us) | mean task (us) | last host enqueue (us) |")
    print("|---|---|---|---|---|---|---|")
    prev_end = 0.0
    for d in sorted(by):
        rs = by[d]
        s0 = min(x["start_us"] for x in rs)
        e1 = max(x["end_us"] for x in rs)
        mean = sum(x["end_us"] - x["start_us"] for x in rs) / len(rs)
        print(f"| {d} | {len(rs)} | {s0:.0f} | {e1:.0f} | {e1 - prev_end:.0f} | {mean:.0f} | {max(x['host_us'] for x in rs):.0f} |")
        prev_end = e1
    for l in tail:
        print(l.strip())


if __name__ == "__main__":
    main(sys.argv[1])
