#!/usr/bin/env python
"""Benchmark of the fused LB stream-collide step on B200 (BASELINE.json metric: MLUPS per GPU and
per box, and fraction of the HBM roofline).

Default workload = BASELINE config 4 (weak scaling): D3Q19 TRT fp64, 512^3 cells per GPU in a
z-slab decomposition (512 x 512 x 512N), periodic, seeded near-equilibrium init, one ghost plane
per side, NCCL halo exchange overlapped with the interior update. A bench "step" is one LB time
step over the whole domain (every kernel of lbm_step(1)). Inputs (41 GB per GPU) are far larger
than L2 (126 MB), so no flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4|c0|c1_f64|c1_f32|c2|c3]
  python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
  python bench.py --impl reference     # the CPU oracle on the host cores (bounded sample)

Prints one JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# ---------------------------------------------------------------------------------------------
# Workloads (BASELINE.json configs). bytes/cell = 2 q s (+1 B flag where a flag field exists).
# ---------------------------------------------------------------------------------------------
CONFIGS = {
    "c4": dict(desc="D3Q19 TRT fp64 512^3/GPU z-slab weak scaling, periodic, random near-eq init (BASELINE config 4)",
               shape=(512, 512, 512), weak=True, Q=19, op="trt", rates=(1.6, 0.5), dtype="f64", pattern="pull",
               force=(0, 0, 0), geometry="periodic", init=("random", 1e-3, 0.01), job_steps=200),
    "c0": dict(desc="D3Q19 SRT fp64 32^3 periodic omega=1.8 (BASELINE config 0; L2-resident, launch-bound)",
               shape=(32, 32, 32), weak=False, Q=19, op="srt", rates=(1.8,), dtype="f64", pattern="pull",
               force=(0, 0, 0), geometry="periodic", init=("random", 1e-3, 0.01), job_steps=100),
    "c1_f64": dict(desc="D3Q19 TRT+Guo fp64 256^3 channel (BASELINE config 1)", shape=(256, 256, 256), weak=False,
                   Q=19, op="trt", rates=(1.6, 0.5), dtype="f64", pattern="pull", force=(1e-6, 0, 0),
                   geometry="channel", init=("rest",), job_steps=2000),
    "c1_f32": dict(desc="D3Q19 TRT+Guo fp32 256^3 channel (BASELINE config 1)", shape=(256, 256, 256), weak=False,
                   Q=19, op="trt", rates=(1.6, 0.5), dtype="f32", pattern="pull", force=(1e-6, 0, 0),
                   geometry="channel", init=("rest",), job_steps=2000),
    "c2": dict(desc="D3Q19 weighted MRT fp32 AA 512^3 shear wave (BASELINE config 2)", shape=(512, 512, 512),
               weak=False, Q=19, op="mrt", rates=(1.9, 1.0, 1.0, 1.0), dtype="f32", pattern="aa", force=(0, 0, 0),
               geometry="periodic", init=("shear", 0.0, 1e-4), job_steps=500),
    "c3": dict(desc="D3Q27 cumulant fp64 384^3 lid-driven cavity (BASELINE config 3)", shape=(384, 384, 384),
               weak=False, Q=27, op="cumulant", rates=(1.95,), dtype="f64", pattern="pull", force=(0, 0, 0),
               geometry="cavity", init=("rest",), job_steps=1000, ubb=(0.05, 0, 0)),
}
CONFIGS["c4_strong"] = dict(CONFIGS["c4"], shape=(1024, 1024, 1024), weak=False, dtype="f32",
                           desc="D3Q19 TRT fp32 1024^3 strong scaling (BASELINE config 4, second part); needs >= 2 GPUs "
                                "for the 32-bit slab offsets (81.6 GB/GPU at P = 2)")
CONFIGS["c3_aa"] = dict(CONFIGS["c3"], pattern="aa", desc="D3Q27 cumulant fp64 384^3 lid-driven cavity, AA pattern")
# C1 fp32 / C3 run with index-list boundaries (the fastest boundary implementation there on the B200,
# DESIGN.md section 6.3); the *_flags lines keep the split flag handling for comparison.
CONFIGS["c3_aa_links"] = dict(CONFIGS["c3_aa"], boundary_mode="links",
                              desc="D3Q27 cumulant fp64 384^3 lid-driven cavity, AA pattern, index-list boundaries")
CONFIGS["c3_flags"] = dict(CONFIGS["c3"], desc=CONFIGS["c3"]["desc"] + ", split bulk + near-wall edge kernel flag boundaries")
CONFIGS["c3"] = dict(CONFIGS["c3"], boundary_mode="links", desc=CONFIGS["c3"]["desc"] + ", index-list boundaries")
CONFIGS["c1_f64_flags"] = dict(CONFIGS["c1_f64"], desc=CONFIGS["c1_f64"]["desc"] + ", compiled-in flag boundaries")
CONFIGS["c1_f32_flags"] = dict(CONFIGS["c1_f32"], desc=CONFIGS["c1_f32"]["desc"] + ", split bulk + near-wall edge kernel flag boundaries")
CONFIGS["c1_f64_links"] = dict(CONFIGS["c1_f64"], boundary_mode="links", desc=CONFIGS["c1_f64"]["desc"] + ", index-list boundaries")
CONFIGS["c1_f64_flags"] = dict(CONFIGS["c1_f64_flags"], faces=False,
                               desc=CONFIGS["c1_f64"]["desc"] + ", split bulk + near-wall edge kernel flag boundaries")
# C1 fp64: the face-aligned-wall kernels (walls from coordinates) measured fastest
CONFIGS["c1_f64"] = dict(CONFIGS["c1_f64"], desc=CONFIGS["c1_f64"]["desc"] + ", flag field, face-aligned-wall kernels")
CONFIGS["c1_f32"] = dict(CONFIGS["c1_f32"], boundary_mode="links", desc=CONFIGS["c1_f32"]["desc"] + ", index-list boundaries")
CONFIGS["c3_periodic"] = dict(CONFIGS["c3"], geometry="periodic", init=("random", 1e-3, 0.01),
                              desc="D3Q27 cumulant fp64 384^3 periodic pull (C3 without walls, diagnostic)")
# Operator comparison in the spirit of Fig. 9: the same D3Q19 AA fp64 periodic
# domain (512^3 instead of the paper's 300x100x100 so the B200 is HBM-bound) for each operator.
for _name, _op, _q, _rates in [("trt", "trt", 19, (1.6, 0.5)), ("smagorinsky", "smagorinsky", 19, (1.95, 0.17)),
                               ("mrt", "mrt", 19, (1.9, 1.0, 1.0, 1.0)), ("kbc", "kbc", 19, (1.95,)),
                               ("cumulant27", "cumulant", 27, (1.95,)), ("cumulant19", "cumulant", 19, (1.95,)),
                               ("kbc27", "kbc", 27, (1.95,)), ("kbc_exact", "kbc_exact", 19, (1.95,)),
                               ("kbc27_exact", "kbc_exact", 27, (1.95,)), ("gen_trt", "gen_trt", 19, (1.6, 0.5)),
                               ("gen_mrt", "gen_mrt", 19, (1.9, 1.0, 1.0, 1.0)), ("gen_srt27", "gen_srt", 27, (1.8,)),
                               ("gen_smagorinsky", "gen_smagorinsky", 19, (1.95, 0.17)), ("trt27", "trt", 27, (1.6, 0.5)),
                               ("srt27", "srt", 27, (1.8,)), ("gen_mrt27", "gen_mrt", 27, (1.9, 1.0, 1.0, 1.0))]:
    CONFIGS[f"op_{_name}"] = dict(desc=f"D3Q{_q} {_op} fp64 AA 512^3 periodic (Fig. 9-style operator comparison)",
                                  shape=(512, 512, 512), weak=False, Q=_q, op=_op, rates=_rates, dtype="f64",
                                  pattern="aa", force=(0, 0, 0), geometry="periodic", init=("random", 1e-3, 0.01),
                                  job_steps=200)

for _k in ("op_kbc_exact", "op_kbc27_exact"):
    CONFIGS[_k]["note"] = ("FP64-ALU bound, not HBM-bound: per-cell Newton iterations with two ln(1+x) per "
                           "direction pair; roofline = measured DFMA ceiling (DESIGN.md section 6.2)")
    CONFIGS[_k]["alu_bound"] = True

# Generated operators (codegen/): C4 and C2 with the generated TRT / weighted MRT.
CONFIGS["c4_gen"] = dict(CONFIGS["c4"], op="gen_trt", desc=CONFIGS["c4"]["desc"] + ", generated TRT operator")
CONFIGS["c2_gen"] = dict(CONFIGS["c2"], op="gen_mrt", desc=CONFIGS["c2"]["desc"] + ", generated weighted MRT operator")

# Equilibrium variants: C4's D3Q19 TRT fp64 512^3 pull with the incompressible
# and the moment-matched equilibria; C2's MRT fp32 AA with the incompressible one.
CONFIGS["eq_inc_c4"] = dict(CONFIGS["c4"], equilibrium="incompressible",
                            desc="D3Q19 TRT fp64 512^3 periodic, incompressible Eq. (3) (rho0 = 1)")
CONFIGS["eq_mm_c4"] = dict(CONFIGS["c4"], equilibrium="moment_matched",
                           desc="D3Q19 TRT fp64 512^3 periodic, moment-matched equilibrium")
# Index-list boundaries (Fig. 8 analog: separate boundary kernel vs compiled-in handling)
# EsoTwist (Fig. 7 analog with the other single-array pattern)
CONFIGS["eso_c4"] = dict(CONFIGS["c4"], pattern="esotwist", desc="D3Q19 TRT fp64 512^3 periodic, EsoTwist single array")
CONFIGS["eso_c3"] = dict(CONFIGS["c3_flags"], pattern="esotwist", desc="D3Q27 cumulant fp64 384^3 cavity, EsoTwist single array")
CONFIGS["eso_c2"] = dict(CONFIGS["c2"], pattern="esotwist", desc="D3Q19 weighted MRT fp32 512^3 shear wave, EsoTwist")
# Paper-shaped workloads (SURVEY §8(d) extras; reported, not gated): Fig. 5 / Fig. 7 domain 300x100x100
# (P:1091), Fig. 8 walled channel (walls on all non-periodic sides) compiled-in vs separate boundary
# kernels, Fig. 10 small per-GPU blocks of the weighted-MRT AA channel.
_paper = dict(shape=(300, 100, 100), weak=False, Q=19, force=(0, 0, 0), geometry="periodic",
              init=("random", 1e-3, 0.01), job_steps=500, dtype="f64")
CONFIGS["fig5_srt_pull"] = dict(_paper, op="srt", rates=(1.8,), pattern="pull",
                                desc="D3Q19 SRT fp64 two-array pull 300x100x100 (Fig. 5 analog)")
CONFIGS["fig7_trt_aa"] = dict(_paper, op="trt", rates=(1.6, 0.5), pattern="aa",
                              desc="D3Q19 TRT fp64 AA 300x100x100 (Fig. 7 analog)")
CONFIGS["fig7_trt_aa_q27"] = dict(_paper, Q=27, op="trt", rates=(1.6, 0.5), pattern="aa",
                                  desc="D3Q27 TRT fp64 AA 300x100x100 (Fig. 7 analog, D3Q27)")
CONFIGS["fig7_mrt_aa_f32"] = dict(_paper, op="mrt", rates=(1.9, 1.0, 1.0, 1.0), pattern="aa", dtype="f32",
                                  desc="D3Q19 weighted MRT fp32 AA 300x100x100 (C2's method on the Fig. 7 domain)")
CONFIGS["fig8_channel_flags"] = dict(_paper, op="trt", rates=(1.6, 0.5), pattern="aa", geometry="box",
                                     desc="D3Q19 TRT fp64 AA 300x100x100 channel, walls on the y and z faces, "
                                          "split bulk + near-wall edge kernel flag boundaries (Fig. 8 analog)")
CONFIGS["fig8_channel_links"] = dict(CONFIGS["fig8_channel_flags"], boundary_mode="links",
                                     desc="D3Q19 TRT fp64 AA 300x100x100 channel, walls on the y and z faces, "
                                          "separate index-list boundary kernel (Fig. 8 analog)")
CONFIGS["fig8_channel_inline"] = dict(CONFIGS["fig8_channel_flags"], boundary_mode="inline",
                                      desc="D3Q19 TRT fp64 AA 300x100x100 channel, walls on the y and z faces, "
                                           "compiled-in conditionals in every cell, no boundary launch (Fig. 8 analog)")
CONFIGS["c1_f64_inline"] = dict(CONFIGS["c1_f64_flags"], boundary_mode="inline",
                                desc="D3Q19 TRT+Guo fp64 256^3 channel (BASELINE config 1), flags tested in every cell (inline)")
CONFIGS["c3_inline"] = dict(CONFIGS["c3_flags"], boundary_mode="inline",
                            desc="D3Q27 cumulant fp64 384^3 lid-driven cavity (BASELINE config 3), flags tested in every cell (inline)")
CONFIGS["fig10_small"] = dict(_paper, shape=(128, 128, 128), weak=True, op="mrt", rates=(1.9, 1.0, 1.0, 1.0),
                              pattern="aa", desc="D3Q19 weighted MRT fp64 AA 128^3 per GPU, weak scaling "
                                                 "(Fig. 10 small-block analog; report ms_per_step)")
# collide-stream-push, two arrays
CONFIGS["push_c4"] = dict(CONFIGS["c4"], pattern="push", desc="D3Q19 TRT fp64 512^3 periodic, collide-stream-push")
CONFIGS["push_c3"] = dict(CONFIGS["c3"], pattern="push",
                          desc="D3Q27 cumulant fp64 384^3 cavity, collide-stream-push, index-list boundaries")
CONFIGS["eq_inc_c2"] = dict(CONFIGS["c2"], equilibrium="incompressible",
                            desc="D3Q19 weighted MRT fp32 AA 512^3 shear wave, incompressible Eq. (3)")


def flags_for(cfg, shape):
    import lbminputs as LI
    nx, ny, nz = shape
    if cfg["geometry"] == "channel":
        return LI.channel_flags(nx, ny, nz), (1, 0, 1)
    if cfg["geometry"] == "cavity":
        return LI.cavity_flags(nx), (0, 0, 0)
    if cfg["geometry"] == "box":  # channel along x, NoSlip on the y and z faces (Fig. 8)
        fl = np.zeros((nz, ny, nx), np.uint8)
        fl[:, 0, :] = fl[:, -1, :] = LI.NOSLIP
        fl[0, :, :] = fl[-1, :, :] = LI.NOSLIP
        return fl, (1, 0, 0)
    return None, (1, 1, 1)


def fluid_cells(cfg, shape, flags):
    return int(np.prod(shape)) if flags is None else int((flags == 0).sum())


def bytes_per_cell(cfg, flags, impl=None):
    """2 q s, + 1 B flag where the update kernel reads a flag field (not with the separate
    index-list kernel, whose update kernels are flag-free, nor with face-aligned walls, recognised from
    coordinates; the in-kernel index lists read one flag byte per cell)."""
    s = 8 if cfg["dtype"] == "f64" else 4
    reads_flags = flags is not None and ((cfg.get("boundary_mode", "flags") in ("flags", "inline") and impl != "faces")
                                         or impl == "links_fused")
    return 2 * cfg["Q"] * s + (1 if reads_flags else 0)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def load_traffic(config_name):
    """dram bytes per launch of the dominant kernel from a committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        v = d.get(config_name)
        if v:
            return v
    return None


def load_alu(config_name):
    """FP work per cell of the config's dominant update kernel (SASS instruction counts from an ncu metrics
    pass, scripts/alu_flops.py -> profiles/alu_flops.jsonl; the last entry per config wins)."""
    p = os.path.join(ROOT, "profiles", "alu_flops.jsonl")
    found = None
    if os.path.exists(p):
        with open(p) as fh:
            for line in fh:
                line = line.strip()
                if line:
                    d = json.loads(line)
                    if d.get("config") == config_name:
                        found = d
    return found


def alu_block(config_name, dtype, kernel_ms_per_step, device):
    """Achieved FP throughput of the dominant kernel against the measured FMA-chain ceiling of the dtype
    (lbm_probe_fma, run live: DFMA for fp64, FFMA for fp32)."""
    d = load_alu(config_name)
    if d is None:
        return None
    from paper_2001_11806_b200 import lbm as L
    key = "fp64_flops_per_cell" if dtype == "f64" else "fp32_flops_per_cell"
    try:
        peak = L.probe_fma(dtype, device)
    except L.LBMError:
        return None
    achieved = d[key] * d["cells_per_launch"] / (kernel_ms_per_step / 1e3) / 1e12
    return {"flops_per_cell": d[key], "achieved_tflops": achieved, "peak_tflops": peak, "frac": achieved / peak,
            "peak_source": f"measured live (lbm_probe_fma, {'DFMA' if dtype == 'f64' else 'FFMA'} chains)",
            "flops_source": "ncu SASS counts add + mul + 2 fma (profiles/alu_flops.jsonl)",
            "fp64_pipe_pct_ncu": d.get("fp64_pipe_pct"), "issue_active_pct_ncu": d.get("issue_active_pct")}


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([s.strip() for s in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > i + 2 and s[i + 2] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline and --impl reference)
# ---------------------------------------------------------------------------------------------
def oracle_sample(cfg, target_s=15.0, max_steps=None):
    """Time the oracle (as it stands) on a bounded sample of the workload: a z-sub-slab of the
    config's x-y extent, periodic in z, same operator and dtype-independent fp64 arithmetic."""
    import oracle as O
    nx, ny, nz = cfg["shape"]
    threads = os.cpu_count() or 1
    m = O.Method(Q=cfg["Q"], op=cfg["op"].removeprefix("gen_"), rates=cfg["rates"], force=cfg["force"], ubb_u=cfg.get("ubb", (0, 0, 0)),
                 equilibrium=cfg.get("equilibrium", "compressible"),
                 nthreads=threads)
    per_cell = 1.0 / (2.0e6 if cfg["op"] in ("srt", "trt") else 0.6e6 if cfg["op"] == "mrt" else 0.17e6)
    planes = max(2, min(nz, int(target_s / (per_cell * nx * ny * 2))))
    d = O.Domain(m, nx, ny, planes)
    f = np.empty(d.shape)
    _, w, _ = O.stencil_arrays(cfg["Q"])
    f[:] = w[:, None, None, None]
    g = f.copy()
    steps, t0 = 0, time.perf_counter()
    while True:
        d.step_pull(f, g)
        f, g = g, f
        steps += 1
        el = time.perf_counter() - t0
        if el > target_s / 2 or (max_steps and steps >= max_steps):
            break
    cells = nx * ny * planes
    # the same oracle on one core, on a 2-plane sample (the paper's per-core view)
    m1 = O.Method(Q=m.Q, op=m.op, rates=m.rates, force=m.force, ubb_u=m.ubb_u, equilibrium=m.equilibrium, nthreads=1)
    d1 = O.Domain(m1, nx, ny, 2)
    f1 = np.empty(d1.shape)
    f1[:] = w[:, None, None, None]
    g1 = f1.copy()
    s1, t1 = 0, time.perf_counter()
    while True:
        d1.step_pull(f1, g1)
        f1, g1 = g1, f1
        s1 += 1
        e1 = time.perf_counter() - t1
        if e1 > target_s / 4:
            break
    return {"value": cells * steps / el / 1e6, "unit": "MLUPS", "cores": threads, "kind": "oracle",
            "sample": f"{nx}x{ny}x{planes} sub-slab of {cfg['desc'].split(' (')[0]}, {steps} pull steps, fp64, "
                      f"{threads} OpenMP threads, {el:.1f} s",
            "value_1core": nx * ny * 2 * s1 / e1 / 1e6,
            "sample_1core": f"{nx}x{ny}x2 sub-slab, {s1} pull steps, 1 thread, {e1:.1f} s",
            **host_info()}


def host_info():
    """CPU model, logical cores and RAM of the host the oracle ran on (SURVEY §8(d) oracle timing)."""
    model, ram = None, None
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
        with open("/proc/meminfo") as fh:
            for line in fh:
                if line.startswith("MemTotal"):
                    ram = round(int(line.split()[1]) / 2 ** 20, 1)
                    break
    except OSError:
        pass
    return {"cpu_model": model, "host_logical_cores": os.cpu_count(), "ram_gib": ram}


# ---------------------------------------------------------------------------------------------
def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle as O
    nx, ny, nz = cfg["shape"]
    threads = os.cpu_count() or 1
    m = O.Method(Q=cfg["Q"], op=cfg["op"].removeprefix("gen_"), rates=cfg["rates"], force=cfg["force"], ubb_u=cfg.get("ubb", (0, 0, 0)),
                 equilibrium=cfg.get("equilibrium", "compressible"),
                 nthreads=threads)
    # each reference step = one pull step of a sub-slab with one z plane per host thread (the
    # oracle parallelises over z), a bounded sample of the workload
    planes = max(2, min(nz, threads))
    d = O.Domain(m, nx, ny, planes)
    f = np.empty(d.shape)
    _, w, _ = O.stencil_arrays(cfg["Q"])
    f[:] = w[:, None, None, None]
    g = f.copy()
    for _ in range(args.warmup):
        d.step_pull(f, g)
        f, g = g, f
    t0 = time.perf_counter()
    for _ in range(args.steps):
        d.step_pull(f, g)
        f, g = g, f
    el = time.perf_counter() - t0
    cells = nx * ny * planes
    val = cells * args.steps / el / 1e6
    line = {"impl": "reference", "metric": "MLUPS (fluid-cell updates per second, whole job)", "value": val,
            "unit": "MLUPS", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": el / args.steps * 1e3, "higher_is_better": True, "scaling": "weak" if cfg["weak"] else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "desc": cfg["desc"], "sample": f"{nx}x{ny}x{planes} sub-slab per step"},
            "cpu_baseline": {"value": val, "unit": "MLUPS", "cores": threads, "kind": "oracle",
                             "sample": f"{nx}x{ny}x{planes} sub-slab, one pull step per bench step", **host_info()},
            "e2e": {"value": val, "unit": "MLUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-reps", type=int, default=4)
    ap.add_argument("--e2e-steps", type=int, default=0, help="LB steps per e2e job (0 = the config's step count)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-probe", action="store_true", help="skip the copy-q roofline probe")
    ap.add_argument("--halo-mode", type=int, default=-1, help="0 zero-copy NCCL (default), 1 packed NCCL, 2 fused NVLink peer stores")
    ap.add_argument("--nccl-self", type=int, default=0,
                    help="N=1 only: ghost planes exchanged through a 1-rank NCCL communicator (times the multi-GPU path)")
    ap.add_argument("--block-x", type=int, default=0)
    ap.add_argument("--graph", type=int, default=-1,
                    help="small-domain launch mode: 0 plain launches, 1 CUDA graph, 2 persistent cooperative kernel "
                         "(default: 2 for domains of <= 2^21 cells per GPU, else 0)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2001_11806_b200 import build
    if rank == 0:
        build.build()
    if world > 1:
        dist.barrier()
    from paper_2001_11806_b200 import lbm as L

    nx, ny, nz1 = cfg["shape"]
    P = world
    nzg = nz1 * P if cfg["weak"] else nz1
    gshape = (nx, ny, nzg)
    flags, periodic = flags_for(cfg, gshape)
    nccl_id = None
    if world > 1:
        buf = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            buf.copy_(torch.frombuffer(bytearray(L.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(buf, 0)
        nccl_id = bytes(buf.cpu().numpy().tobytes())
    # a dedicated (non-default) torch stream: the library launches every kernel on it, so CUDA
    # events recorded on it bracket exactly our kernels (the legacy default stream's handle is 0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    # (persistent kernel vs graph, profiles/r03i_launch_modes.jsonl: 32^3 3.4 vs 4.2 us per step, 128^3 108 vs 99 us
    # = 0.90 vs 0.98 of copy BW; the grid barrier and the grid-strided tail cost more than a kernel boundary once
    # a step takes tens of microseconds)
    small = np.prod(gshape) / P <= 2 ** 18
    # small domains: one persistent kernel per lbm_step call; large single-slab domains: the captured two-step
    # CUDA graph (removes the per-launch CPU overhead and gaps: C1 fp32 0.945 -> 0.958 of copy BW; the roofline
    # then uses the timed region's time per step, gaps included)
    use_graph = (2 if small else 1) if args.graph < 0 else args.graph
    nccl_self = bool(args.nccl_self) and world == 1
    use_graph = 0 if (nccl_self or world > 1) else use_graph  # graphs / persistent kernels: single-slab runs only
    exchanging = world > 1 or nccl_self
    halo_mode = args.halo_mode
    if halo_mode < 0:
        # default: zero-copy NCCL send/recv overlapped with the interior. The fused NVLink peer-store halo
        # (--halo-mode 2) is bit-identical and as fast on one GPU (1-rank communicator) but has not run
        # across GPUs in this build (tests/test_multigpu.py runs it on the first multi-GPU box), and the
        # C4 halo is ~0.2 % of a step, so the default favours the transport that cannot hang a scaling run.
        halo_mode = L.HALO_ZEROCOPY

    if cfg.get("faces") is False:  # the split flag kernels even where the face-aligned ones would run
        os.environ["LBM_FACES"] = "0"

    def make(mode):
        return L.Simulation(gshape, stencil=cfg["Q"], collision=cfg["op"], rates=cfg["rates"], dtype=cfg["dtype"],
                            pattern=cfg["pattern"], force=cfg["force"], flags=flags,
                            ubb_velocity=cfg.get("ubb", (0, 0, 0)), periodic=periodic, rank=rank, nranks=world,
                            nccl_id=nccl_id, device=local, stream=stream.cuda_stream, halo_mode=mode,
                            use_graph=use_graph, block_x=args.block_x, nccl_self=nccl_self,
                            equilibrium=cfg.get("equilibrium", "compressible"),
                            boundary_mode=cfg.get("boundary_mode", "flags"))

    sim, err = None, None
    try:
        sim = make(halo_mode)
    except L.LBMError as e:
        err = str(e)
    if world > 1:  # every rank must agree before falling back (creation is collective)
        ok = torch.tensor([0 if sim is None else 1], dtype=torch.int32, device="cuda")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok) == 0 and sim is not None:
            sim.close()
            sim = None
    if sim is None:
        if halo_mode != L.HALO_FUSED:
            raise RuntimeError(err or "lbm_create failed on another rank")
        if rank == 0:
            print(f"# fused halo unavailable ({err}); falling back to zero-copy NCCL", file=sys.stderr)
        halo_mode = L.HALO_ZEROCOPY
        if world > 1:  # fresh NCCL id for the second communicator
            buf = torch.zeros(128, dtype=torch.uint8, device="cuda")
            if rank == 0:
                buf.copy_(torch.frombuffer(bytearray(L.nccl_unique_id()), dtype=torch.uint8))
            dist.broadcast(buf, 0)
            nccl_id = bytes(buf.cpu().numpy().tobytes())
        sim = make(halo_mode)
    args.halo_mode = halo_mode
    kind = cfg["init"][0]
    if kind == "rest":
        sim.init_equilibrium(torch.ones(sim.cells, dtype=torch.float64, device="cuda"),
                             torch.zeros(3 * sim.cells, dtype=torch.float64, device="cuda"))
    else:
        sim.init_random(0, cfg["init"][1], cfg["init"][2], 1 if kind == "shear" else 0, 0.01)

    # ---- device-timed region ------------------------------------------------------------
    sim.step(args.warmup)
    sim.sync()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sim.enable_kernel_timing() if use_graph != 1 else None
    l0 = sim.launches
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        sim.step(args.steps)
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_ms = ev0.elapsed_time(ev1)
    launches = sim.launches - l0
    if use_graph != 1:
        kms, klaunch = sim.kernel_time_ms()
    else:
        kms, klaunch = t_ms, launches
    if world > 1:
        t = torch.tensor([t_ms, kms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_ms, kms_max = float(t[0]), float(t[1])
    else:
        kms_max = kms
    fl_local = None
    if flags is not None:
        fl_local = flags[sim.z0: sim.z0 + sim.nz_local]
    nf_local = fluid_cells(cfg, (nx, ny, sim.nz_local), fl_local)
    nf_total = nf_local * world if cfg["weak"] else fluid_cells(cfg, gshape, flags)
    mlups = nf_total * args.steps / (t_ms / 1e3) / 1e6
    bpc = bytes_per_cell(cfg, flags, sim.boundary_impl)
    # dominant kernel: the fused stream-collide kernel (the only kernel of a single-GPU step)
    kernel_ms_per_step = kms_max / args.steps
    achieved = nf_local * bpc / (kernel_ms_per_step / 1e3) / 1e9
    peak, peak_src = load_peaks()
    clocks = clk.summary()
    phases = None
    if exchanging and use_graph != 1:  # one timed step's phase timeline (boundary / exchange / interior), after the timed region
        sim.enable_kernel_timing()
        sim.step(1)
        try:
            ph = sim.step_phases_ms()
            (b0, b1), (x0, x1), (i0, i1) = ph["boundary"], ph["exchange"], ph["interior"]
            phases = {"boundary_ms": [b0, b1], "exchange_ms": [x0, x1], "interior_ms": [i0, i1],
                      "exchange_hidden_by_interior": bool(x1 <= i1 and x0 >= i0 - 1e-3),
                      "note": "CUDA events per phase on the stream it runs on (lbm_step_phases_ms)"}
        except L.LBMError:
            phases = None

    # ---- end-to-end through the public API with host buffers ------------------------------
    e2e = None
    job = args.e2e_steps or cfg["job_steps"]
    if args.e2e_reps > 0:
        rho_h = torch.empty(sim.cells, dtype=torch.float64, pin_memory=True)
        u_h = torch.empty(3 * sim.cells, dtype=torch.float64, pin_memory=True)
        if kind == "rest":
            rho_h.fill_(1.0)
            u_h.zero_()
        else:
            import lbminputs as LI
            r, u = LI.random_fields(0, nx, ny, nzg, cfg["init"][1], cfg["init"][2], 1 if kind == "shear" else 0, 0.01,
                                    z0=sim.z0, nz=sim.nz_local)
            rho_h.copy_(torch.from_numpy(r.reshape(-1)))
            u_h.copy_(torch.from_numpy(u.reshape(-1)))
        rho_o = torch.empty(sim.cells, dtype=torch.float64, pin_memory=True)
        u_o = torch.empty(3 * sim.cells, dtype=torch.float64, pin_memory=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        # jobs through the asynchronous host I/O (LBM_HOST_ASYNC): job i+1's upload and job i's download run on
        # their own streams during the steps; every byte still crosses PCIe inside the timed region
        sim.sync()
        t0 = time.perf_counter()
        for _ in range(args.e2e_reps):
            L._check(L.lbm_init_equilibrium(sim.h, rho_h.data_ptr(), u_h.data_ptr(), L.HOST_ASYNC), sim.h, "init")
            L._check(L.lbm_step(sim.h, job), sim.h, "lbm_step")
            L._check(L.lbm_get_macroscopic(sim.h, rho_o.data_ptr(), u_o.data_ptr(), L.HOST_ASYNC), sim.h, "get_macroscopic")
        sim.sync()
        torch.cuda.synchronize()
        te = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([te], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te = float(t[0])
        # bytes copied per job (rho + u up, rho + u down), and per LB step of that job
        h2d_job = d2h_job = int(4 * 8 * sim.cells)
        e2e = {"value": nf_total * job * args.e2e_reps / te / 1e6, "unit": "MLUPS",
               "h2d_bytes_per_step": h2d_job / job, "d2h_bytes_per_step": d2h_job / job,
               "h2d_bytes_per_job": h2d_job, "d2h_bytes_per_job": d2h_job, "lb_steps_per_job": job,
               "step": f"one job: init_equilibrium from pinned host rho/u, lbm_step({job}), get_macroscopic to host "
                       "(LBM_HOST_ASYNC: uploads / downloads on their own streams, overlapped with the previous / next "
                       "job's steps); bytes per step = bytes per job / LB steps per job",
               "reps": args.e2e_reps}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_sample(cfg)

    if rank == 0:
        # copy-q probe (paper Table III analogue): the LB gather streams without collision, same local
        # shape; run after the timed region with the simulation's arrays still resident
        copyq = None
        if not args.no_probe:
            try:
                copyq = L.probe_copy(cfg["Q"], cfg["dtype"], True, (nx, ny, sim.nz_local), reps=5, device=local)
            except L.LBMError:
                copyq = None
        alu = alu_block(args.config, cfg["dtype"], kernel_ms_per_step, local)
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": load_traffic(args.config), "peak_source": peak_src,
                    "algorithmic_bytes_per_cell": bpc, "cells_per_launch": nf_local,
                    "kernel_ms_per_step": kernel_ms_per_step, "kernel_launches_timed": klaunch,
                    "kernel_time_source": ("CUDA events around the timed region on the launching stream, per step "
                                           "(CUDA-graph replay: launch gaps included)") if use_graph == 1 else
                                          "CUDA events around every launch on its stream, summed per step",
                    "frac_of_nominal_8tbs": achieved / 8000.0,
                    "note": ("L2-resident launch/latency-bound domain: the HBM roofline does not bind "
                             "(one persistent kernel per lbm_step call)")
                            if (cfg["Q"] * np.prod(gshape) / P * (8 if cfg["dtype"] == "f64" else 4)
                                * (2 if cfg["pattern"] in ("pull", "push") else 1)) < 100e6 else cfg.get("note"),
                    "copy_q_gbs": copyq, "frac_of_copy_q": (achieved / copyq) if copyq else None,
                    "boundary_mode": cfg.get("boundary_mode", "flags") if flags is not None else "none",
                    "boundary_impl": sim.boundary_impl,
                    "kernel_path": L.kernel_path()}
        if cfg.get("alu_bound") and alu is not None:
            # the FP64-ALU-bound operators (exact KBC): the roofline is the measured DFMA ceiling; the HBM
            # figures stay beside it
            roofline = {"bound": "alu", "achieved": alu["achieved_tflops"], "peak": alu["peak_tflops"],
                        "unit": "TFLOP/s", "frac": alu["frac"], "traffic": load_traffic(args.config),
                        "peak_source": alu["peak_source"], "flops_per_cell": alu["flops_per_cell"],
                        "hbm_achieved_gbs": achieved, "hbm_frac": achieved / peak, "kernel_ms_per_step": kernel_ms_per_step,
                        "kernel_launches_timed": klaunch, "cells_per_launch": nf_local, "kernel_path": L.kernel_path(),
                        "note": cfg.get("note")}
        line = {
            "metric": "MLUPS (fluid-cell updates per second, whole job)",
            "value": mlups, "unit": "MLUPS", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "weak" if cfg["weak"] else "strong", "vs_baseline": None, "dtype": cfg["dtype"],
            "data": "synthetic",
            "config": {"workload": args.config, "desc": cfg["desc"], "global": list(gshape),
                       "per_gpu_mlups": mlups / world, "pattern": cfg["pattern"],
                       "parallelism": f"z-slab x{world}" if world > 1 else
                       ("single GPU, NCCL self-exchange of ghost planes" if nccl_self else "single GPU"),
                       "l2": "inputs larger than L2 (no flush)" if not small else "L2-resident (launch-bound config)",
                       "halo_mode": {0: "zerocopy NCCL send/recv", 1: "packed NCCL send/recv", 2: "fused NVLink peer stores (NCCL LSA windows)"}[args.halo_mode] if (world > 1 or nccl_self) else "none (single slab, z wraps in-kernel)", "launch_mode": {0: "plain launches", 1: "CUDA graph (2-step cycle)", 2: "persistent cooperative kernel"}[use_graph]},
            "roofline": roofline,
            "alu": alu,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "phases": phases,
            "clocks": clocks,
        }
        print(json.dumps(line))
    sim.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
