"""Warp-stall breakdown of an `ncu --page source --csv` export (all samples):

    python tools/ncu_stalls.py gpurun_out/<name>_source.csv [top-N instructions]
"""
import collections
import csv
import sys


def main(path, top=0):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    agg = collections.Counter()
    for r in data:
        for h in stalls:
            agg[h] += int(r[hdr.index(h)] or 0)
    tot = sum(agg.values()) or 1
    print("| stall reason | samples | share |")
    print("|---|---:|---:|")
    for k, v in agg.most_common(8):
        print(f"| {k[6:]} | {v} | {100 * v / tot:.1f}% |")
    if top:
        i_s, i_src = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
        best = sorted(range(len(data)), key=lambda i: -int(data[i][i_s] or 0))[:top]
        print("\n| SASS | samples |\n|---|---:|")
        for i in sorted(best):
            print(f"| `{data[i][i_src].strip()[:70]}` | {data[i][i_s]} |")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
