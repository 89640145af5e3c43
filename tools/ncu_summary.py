"""Summarise ncu captures for profiles/.

  python tools/ncu_summary.py full REPORT.ncu-rep      # key metrics of a --set full capture
  python tools/ncu_summary.py launches LAUNCHES.csv    # per-kernel share of a launch list

The "full" summary lists, per captured kernel: duration, DRAM bytes read/written (the roofline
`traffic`), DMMA / shared (fp64+tensor) pipe activity, shared-memory wavefronts and bank
conflicts, registers, warps active, and the top warp-stall reasons.
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "lts__t_bytes.sum",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.sum",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "sm__cycles_elapsed.avg.per_second",
]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for v in rows[2:]:
        d = dict(zip(hdr, v))
        print(f"kernel: {d.get('Kernel Name', '?')}")
        for k in KEYS:
            if k in d:
                print(f"  {k:80s} {d[k]:>20s} {units[hdr.index(k)]}")
        stalls = []
        for i, n in enumerate(hdr):
            if n.startswith("smsp__average_warp_latency_issue_stalled_") and n.endswith(".ratio"):
                try:
                    stalls.append((float(v[i]), n))
                except ValueError:
                    pass
            if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("_not_issued"):
                try:
                    stalls.append((float(v[i].replace(",", "")), n))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        print("  top stall reasons:")
        for val, n in stalls[:10]:
            print(f"    {n:80s} {val:g}")


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                per[d["Kernel Name"]].append(float(d["Metric Value"]) * (1e-3 if d["Metric Unit"] == "ns" else
                                                                          1.0 if d["Metric Unit"] == "us" else 1e3))
    tot = sum(sum(v) for v in per.values())
    print(f"{'launches':>8s} {'mean us':>12s} {'share':>7s}  kernel")
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        print(f"{len(v):8d} {sum(v) / len(v):12.1f} {100 * sum(v) / tot:6.2f}%  {k}")


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2])
