"""Summarise ncu reports (gpurun_out/prof_<config>.ncu-rep) into profiles/r<NN>_<config>_ncu_summary.json
and update profiles/ncu_traffic.json (DRAM bytes per launch of the dominant kernel)."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(rnd, configs):
    tr_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = json.load(open(tr_path)) if os.path.exists(tr_path) else {}
    for c in configs:
        src = os.environ.get("PROF_DIR", os.path.join(ROOT, "gpurun_out"))
        rep = os.path.join(src, f"prof_{c}.ncu-rep")
        raw_csv = os.path.join(src, f"prof_{c}_raw.csv")
        if os.path.exists(raw_csv):  # exported on the GPU box (reports exceed gpurun's copy-back limit)
            out = open(raw_csv).read()
        else:
            out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        hdr, units = rows[0], rows[1]
        kernels = []
        for vals in rows[2:]:
            d = dict(zip(hdr, vals))
            m = {k: f"{d[k]} {units[hdr.index(k)]}".strip() for k in KEYS if k in d}
            rb = float(d["dram__bytes_read.sum"]) * SCALE[units[hdr.index("dram__bytes_read.sum")]]
            wb = float(d["dram__bytes_write.sum"]) * SCALE[units[hdr.index("dram__bytes_write.sum")]]
            kernels.append({"kernel": d.get("Kernel Name"), "dram_bytes": rb + wb, "metrics": m})
        json.dump({"config": c, "tool": "ncu --set full --clock-control none (scripts/gpu_profile.sh)",
                   "kernels": kernels}, open(os.path.join(ROOT, "profiles", f"r{rnd}_{c}_ncu_summary.json"), "w"),
                  indent=1)
        if not kernels:
            print(c, "no kernels in report (graph-launched?)")
            continue
        # dominant kernel(s): those within 2x of the longest launch (AA/EsoTwist: the even and odd kernels)
        def dur(k):
            v, u = k["metrics"]["gpu__time_duration.sum"].split()
            return float(v) * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(u, 1.0)
        tmax = max(dur(k) for k in kernels)
        dom = [k for k in kernels if dur(k) >= 0.5 * tmax]
        traffic[c] = sum(k["dram_bytes"] for k in dom) / len(dom)
        print(c, [(k["kernel"][:40], k["dram_bytes"]) for k in kernels])
    json.dump(traffic, open(tr_path, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
