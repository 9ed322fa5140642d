"""Build profiles/<round>/ from a gpurun_out capture directory:

    python scripts/profile_summary.py gpurun_out/r01c profiles/r01

Reads the ncu launch list (launches_c3.csv: `--metrics gpu__time_duration.sum`)
and the `--set full` reports (*.ncu-rep), writes
  * <out>/launches_c3.csv   : the launch list itself
  * <out>/<name>_details.csv: ncu --page details for each report (text)
  * <out>/summary.json      : launch_share (per-kernel share of the step) and
                              per-kernel duration, DRAM bytes, pipe use
and profiles/ncu_summary.json (the file bench.py reads for roofline.traffic).
"""
import csv
import io
import json
import os
import re
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

METRICS = {
    "duration_ms": "gpu__time_duration.sum",
    "dram_read_mb": "dram__bytes_read.sum",
    "dram_write_mb": "dram__bytes_write.sum",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "dmma_pipe_pct": "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "smem_per_block_kb": "launch__shared_mem_per_block_allocated",
}


def short(name):
    m = re.search(r"(k_\w+)(<[^>]*>)?", name)
    return (m.group(1) + (m.group(2) or "")) if m else name[:60]


def to_unit(v, unit, want):
    v = float(v)
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3,
             "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
    if want in ("mb", "ms"):
        return v * scale.get(unit, 1.0)
    return v


# launched by bench.py outside the evaluation step: the FP64 peak probe and
# the plan's geometry-only precompute
NOT_STEP = ("k_dfma", "k_dmma", "k_periodic_gen", "k_jacobi_svd", "k_svd_factors", "k_m2l_pack",
            "k_inst_count", "k_inst_write")


def launch_share(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[hdr_i + 1:]:
        if len(r) <= iv:
            continue
        t = to_unit(r[iv].replace(",", ""), r[iu], "ms")
        k = short(r[ik])
        tot[k] += t
        cnt[k] += 1
    s = sum(v for k, v in tot.items() if not k.startswith(NOT_STEP))
    return {k: {"launches": cnt[k], "total_ms": round(tot[k], 4),
                "share_of_step": None if k.startswith(NOT_STEP) else round(tot[k] / s, 4)}
            for k in sorted(tot, key=lambda k: -tot[k])}


def report(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": short(r[hdr.index("Kernel Name")])}
        for key, m in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                v = r[i].replace(",", "")
                if key.endswith("_mb"):
                    d[key] = round(to_unit(v, units[i], "mb"), 3)
                elif key == "duration_ms":
                    d[key] = round(to_unit(v, units[i], "ms"), 4)
                else:
                    try:
                        d[key] = round(float(v), 2)
                    except ValueError:
                        d[key] = v
        res.append(d)
    return res


def main():
    src, dst = sys.argv[1], sys.argv[2]
    os.makedirs(dst, exist_ok=True)
    summary = {"source": src}
    lc = os.path.join(src, "launches_c3.csv")
    if os.path.exists(lc):
        summary["launch_share"] = launch_share(lc)
        with open(os.path.join(dst, "launches_c3.csv"), "w") as f:
            f.write(open(lc).read())
    kernels = []
    for fn in sorted(os.listdir(src)):
        if fn.endswith(".ncu-rep"):
            rep = os.path.join(src, fn)
            kernels += report(rep)
            det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                                 text=True, check=True).stdout
            with open(os.path.join(dst, fn.replace(".ncu-rep", "_details.csv")), "w") as f:
                f.write(det)
    summary["kernels"] = kernels
    with open(os.path.join(dst, "summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    p2p = [k for k in kernels if k["kernel"].startswith("k_p2p") and not k["kernel"].startswith("k_p2p_force")]
    if p2p:
        k = p2p[0]
        traffic = {"p2p": {"kernel": k["kernel"], "dram_bytes_per_launch":
                           int(round((k["dram_read_mb"] + k["dram_write_mb"]) * 1e6)),
                           "duration_ms_ncu": k["duration_ms"], "source": os.path.join(dst, "summary.json")}}
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w") as f:
            json.dump(traffic, f, indent=1)
    print(json.dumps(summary.get("launch_share", {}), indent=1)[:2000])
    for k in kernels:
        print(k)


if __name__ == "__main__":
    main()
