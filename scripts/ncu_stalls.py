"""Per-source-line warp-stall samples of one kernel in an ncu report.

  python scripts/ncu_stalls.py <prof.ncu-rep> [top]
Prints the source lines holding the most samples with their top stall reasons.
"""
import collections
import csv
import io
import subprocess
import sys


def main(path, top=25):
    txt = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    hdr, cur = None, None
    agg = collections.Counter()
    reasons = collections.defaultdict(collections.Counter)
    text = {}
    for r in csv.reader(io.StringIO(txt)):
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr) or not r[0]:
            continue  # SASS rows carry no line number; the CUDA line rows aggregate them
        d = dict(zip(hdr, r))
        try:
            n = int(d["Warp Stall Sampling (All Samples)"] or 0)
        except ValueError:
            continue
        key = (cur, int(d["Line No"]))
        agg[key] += n
        text[key] = r[1].strip()[:70]
        for k, v in d.items():
            if k.startswith("stall_"):
                try:
                    reasons[key][k[6:]] += int(v or 0)
                except ValueError:
                    pass
    tot = sum(agg.values()) or 1
    print(f"total samples {tot}")
    for key, n in agg.most_common(top):
        rs = ", ".join(f"{k} {100 * v / n:.0f}%" for k, v in reasons[key].most_common(3) if v)
        print(f"{100 * n / tot:5.1f}%  {key[0]}:{key[1]}  {text[key]}  [{rs}]")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
