"""Summarise one `ncu --set full` capture of the hot kernel into profiles/.

    python scripts/ncu_summary.py gpurun_out/prof_full.ncu-rep [round] [tag]
    (NCU_SUMMARY_DIR=gpurun_out: write there instead of profiles/, on the box)

Writes profiles/r<round>_ncu_summary.json (the numbers bench.py quotes:
DRAM bytes per launch, L2 read GB/s, pipe utilisations) and the raw/details
CSV pages next to it; with a tag (e.g. "lidar") r<round>_ncu_<tag>_summary.json
and r<round>_ncu_full_<tag>_{raw,details}.csv.
"""

import csv
import io
import json
import os
import subprocess
import sys

CAPTURES = {
    None: ("ncu --set full --clock-control none --import-source on -k regex:k_ray_policy2 "
           "-s 1 -c 1 python scripts/profile_target.py (4096 poses x 65536 rays, C1 map)"),
    "lidar": ("ncu --set full --clock-control none --import-source on -k regex:k_lidar_warp "
              "-s 1 -c 1 python scripts/profile_lidar.py (1024 C3 scans x 131072 beams)"),
}

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3,
         "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}

FIELDS = {
    "dram_bytes_read": "dram__bytes_read.sum",
    "dram_bytes_write": "dram__bytes_write.sum",
    "l2_read_sectors_from_l1": "lts__t_sectors_srcunit_tex_op_read.sum",
    "l2_hit_rate_pct": "lts__t_sector_hit_rate.pct",
    "l1_hit_rate_pct": "l1tex__t_sector_hit_rate.pct",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "fp64_pipe_active_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "xu_pipe_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "threads_per_inst": "smsp__thread_inst_executed_per_inst_executed.ratio",
    "registers": "launch__registers_per_thread",
    "inst_executed": "smsp__inst_executed.sum",
}


def ncu_page(rep, page):
    return subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], check=True,
                          capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    rnd = sys.argv[2] if len(sys.argv) > 2 else "01"
    tag = sys.argv[3] if len(sys.argv) > 3 else None
    raw = ncu_page(rep, "raw")
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, vals = rows[0], rows[1], rows[2]
    col = {n: i for i, n in enumerate(head)}

    def get(name):
        i = col[name]
        x = float(vals[i].replace(",", ""))
        return x * SCALE.get(units[i], 1.0)

    out = {"kernel": vals[col["Kernel Name"]].split("(")[0], "capture": CAPTURES.get(tag),
           "duration_ms": get("gpu__time_duration.sum")}
    for k, name in FIELDS.items():
        if name in col:
            out[k] = get(name)
    out["dram_bytes_per_launch"] = out["dram_bytes_read"] + out["dram_bytes_write"]
    out["l2_read_GBps"] = out["l2_read_sectors_from_l1"] * 32 / (out["duration_ms"] * 1e-3) / 1e9
    out["dram_GBps"] = out["dram_bytes_per_launch"] / (out["duration_ms"] * 1e-3) / 1e9
    outdir = os.environ.get("NCU_SUMMARY_DIR", "profiles")
    summ = (f"{outdir}/r{rnd}_ncu_{tag}_summary.json" if tag
            else f"{outdir}/r{rnd}_ncu_summary.json")
    stem = f"{outdir}/r{rnd}_ncu_full_{tag or 'k_ray_policy2'}"
    with open(summ, "w") as fh:
        json.dump(out, fh, indent=1)
        fh.write("\n")
    with open(stem + "_raw.csv", "w") as fh:
        fh.write(raw)
    with open(stem + "_details.csv", "w") as fh:
        fh.write(ncu_page(rep, "details"))
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
