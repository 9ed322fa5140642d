"""Digest of an ncu --set full report: key throughput metrics, stall reasons
and the hottest SASS lines (by warp-stall samples).

    python scripts/ncu_digest.py report.ncu-rep [--top 20]
"""
import argparse
import csv
import io
import re
import subprocess

KEYS = [r"gpu__time_duration.sum$", r"launch__grid_size$", r"launch__registers_per_thread$",
        r"launch__occupancy_limit_(registers|shared_mem|warps)$", r"sm__warps_active.avg.pct_of_peak_sustained_active$",
        r"sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active$", r"sm__inst_executed_pipe_fp64.avg.pct",
        r"smsp__issue_active.avg.pct_of_peak_sustained_active$", r"dram__bytes_(read|write).sum$",
        r"lts__t_sector_hit_rate.pct$", r"sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active$",
        r"smsp__average_warps_issue_stalled_\w+_per_issue_active.ratio$"]


def ncu(args):
    return subprocess.run(["ncu"] + args, capture_output=True, text=True, check=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=20)
    a = ap.parse_args()
    rows = list(csv.reader(io.StringIO(ncu(["-i", a.rep, "--page", "raw", "--csv"]))))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print("kernel:", r[hdr.index("Kernel Name")][:110])
        for k, u, v in zip(hdr, units, r):
            if any(re.search(p, k) for p in KEYS):
                if "stalled" in k and float(v or 0) < 0.05:
                    continue
                print(f"  {k} = {v} {u}")
    src = list(csv.reader(io.StringIO(ncu(["-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    h = src[1]
    ia, isrc, iss, ie = (h.index(c) for c in ("Address", "Source", "Warp Stall Sampling (All Samples)",
                                               "Instructions Executed"))
    # first kernel's section only (later sections repeat the header)
    data = []
    for r in src[2:]:
        if len(r) <= iss or r[iss] == h[iss] or r[0] == "Kernel Name":
            if data:
                break
            continue
        data.append(r)
    tot = sum(float(r[iss] or 0) for r in data)
    print(f"stall samples: {tot:.0f}")
    for r in sorted(data, key=lambda r: -float(r[iss] or 0))[:a.top]:
        print(f"  {r[ia][-5:]} {float(r[iss] or 0) / tot * 100:5.1f}%  exec {r[ie]:>10}  {r[isrc][:70]}")


if __name__ == "__main__":
    main()
