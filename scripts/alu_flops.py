"""Per-cell floating-point work of the update kernels from an ncu metrics CSV (SASS instruction counts:
FLOP = add + mul + 2 fma, per precision), for the `alu` block of bench.py.

  python scripts/alu_flops.py <config> <cells_per_launch> gpurun_out/<name>_alu.csv >> profiles/alu_flops.jsonl
"""
import csv
import io
import json
import sys

M = {"dadd": "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
     "dmul": "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
     "dfma": "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
     "fadd": "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum",
     "fmul": "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum",
     "ffma": "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum"}


def main(config, cells, path):
    text = open(path).read()
    rows = list(csv.reader(io.StringIO(text[text.index('"ID"'):])))
    hdr = rows[0]
    col = {h: i for i, h in enumerate(hdr)}
    per = {}
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        name, metric, val = r[col["Kernel Name"]], r[col["Metric Name"]], r[col["Metric Value"]]
        k = (r[col["ID"]], name)
        per.setdefault(k, {})[metric] = float(val.replace(",", ""))
    # dominant kernel = the update kernel with the most FP work per launch
    best = None
    for (lid, name), m in per.items():
        f64 = m.get(M["dadd"], 0) + m.get(M["dmul"], 0) + 2 * m.get(M["dfma"], 0)
        f32 = m.get(M["fadd"], 0) + m.get(M["fmul"], 0) + 2 * m.get(M["ffma"], 0)
        if best is None or f64 + f32 > best[2] + best[3]:
            best = (lid, name, f64, f32, m)
    lid, name, f64, f32, m = best
    print(json.dumps({"config": config, "kernel": name.split("(")[0][:80], "fp64_flops_per_cell": f64 / cells,
                      "fp32_flops_per_cell": f32 / cells, "cells_per_launch": cells,
                      "fp64_pipe_pct": m.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                      "issue_active_pct": m.get("smsp__issue_active.avg.pct_of_peak_sustained_active")}))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), sys.argv[3])
