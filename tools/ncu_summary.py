"""Summarise ncu outputs for profiles/:

    python tools/ncu_summary.py launches gpurun_out/launches.csv   # per-kernel share of a step
    python tools/ncu_summary.py report gpurun_out/prof.ncu-rep      # key metrics of a --set full capture
    python tools/ncu_summary.py report gpurun_out/prof_raw.csv      # same, from `ncu -i ... --page raw --csv`
"""
import collections
import csv
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "smsp__warps_issue_stalled_long_scoreboard_per_warp_active.pct",
    "smsp__warps_issue_stalled_barrier_per_warp_active.pct",
    "smsp__warps_issue_stalled_membar_per_warp_active.pct",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"])
        unit = d["Metric Unit"]
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
        name = d["Kernel Name"].split("(")[0][:80]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print("| kernel | launches | total us | share |")
    print("|---|---:|---:|---:|")
    for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k}` | {n} | {us:.1f} | {100 * us / tot:.1f}% |")
    print(f"\ntotal {tot:.1f} us over {sum(v[0] for v in agg.values())} launches (cold-cache, serialised by ncu)")


def report(path):
    if path.endswith(".csv"):  # `ncu -i rep --page raw --csv` output, converted on the GPU box
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    idx = {}
    for i, h in enumerate(hdr):  # raw-page names may carry a section prefix
        idx.setdefault(h, i)
        idx.setdefault(h.split(".", 2)[-1] if h.count(".") >= 3 and h.split(".")[0].isupper() else h, i)
    for r in rows[2:]:
        print(f"### {r[idx['Kernel Name']][:100]}")
        for k in KEYS:
            if k in idx:
                print(f"- {k}: {r[idx[k]]} {units[idx[k]]}")
        print()


if __name__ == "__main__":
    {"launches": launches, "report": report}[sys.argv[1]](sys.argv[2])
