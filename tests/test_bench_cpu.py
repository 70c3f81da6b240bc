"""Host-side pieces of bench.py that need no GPU: workload table, algorithmic bytes per cell,
geometries, the ALU block's FLOP table and the reference arm (the oracle on a bounded sample)."""
import importlib.util
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_algorithmic_bytes_per_cell(bench):
    C = bench.CONFIGS
    assert bench.bytes_per_cell(C["c4"], None) == 304          # D3Q19 fp64: 2 * 19 * 8
    assert bench.bytes_per_cell(C["c2"], None) == 152          # D3Q19 fp32
    assert bench.bytes_per_cell(C["op_cumulant27"], None) == 432
    fl, per = bench.flags_for(C["c3"], (8, 8, 8))
    assert per == (0, 0, 0) and bench.bytes_per_cell(C["c3_flags"], fl) == 433          # + 1 B flag (split mode)
    assert bench.bytes_per_cell(C["c3"], fl) == 432                                      # index lists: flag-free
    assert bench.bytes_per_cell(C["c3"], fl, "links") == 432                             # separate link kernel
    assert bench.bytes_per_cell(C["c3"], fl, "links_fused") == 433                       # in-kernel links: + flag byte
    assert bench.bytes_per_cell(C["c1_f64"], bench.flags_for(C["c1_f64"], (8, 8, 8))[0], "faces") == 304


def test_workloads_match_baseline_configs(bench):
    C = bench.CONFIGS
    assert C["c4"]["shape"] == (512, 512, 512) and C["c4"]["weak"] and C["c4"]["job_steps"] == 200
    assert C["c1_f64"]["force"] == (1e-6, 0, 0) and C["c1_f64"]["job_steps"] == 2000
    assert C["c2"]["pattern"] == "aa" and C["c2"]["dtype"] == "f32" and C["c2"]["job_steps"] == 500
    assert C["c3"]["Q"] == 27 and C["c3"]["op"] == "cumulant" and C["c3"]["job_steps"] == 1000
    assert C["c0"]["shape"] == (32, 32, 32) and C["c0"]["rates"] == (1.8,)
    assert C["c4_strong"]["shape"] == (1024, 1024, 1024) and not C["c4_strong"]["weak"]


def test_alu_table_entries(bench):
    for cfg in ("c4", "c3", "op_cumulant27", "op_kbc_exact"):
        d = bench.load_alu(cfg)
        assert d is not None and d["cells_per_launch"] > 0
        assert (d["fp64_flops_per_cell"] or d["fp32_flops_per_cell"]) > 100


def test_host_info(bench):
    h = bench.host_info()
    assert h["host_logical_cores"] >= 1 and (h["ram_gib"] is None or h["ram_gib"] > 0)


def test_reference_arm_runs_the_oracle_on_cpu():
    """`bench.py --impl reference` (the oracle on the host cores) prints one JSON line with the contract's keys."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c0",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert d["impl"] == "reference" and d["unit"] == "MLUPS" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
