"""Diagnostic: shear-wave viscosity fit of config 2 on the GPU for dtype x noise x kernel path x pattern."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2001_11806_b200 import lbm as L
from tests import closed_forms as CF
import lbminputs as LI

def run(dtype, amp, path, pattern, shape=(512, 512, 512), op="mrt", rates=(1.9, 1.0, 1.0, 1.0)):
    L.set_kernel_path(path)
    sim = L.Simulation(shape, 19, op, rates, dtype, pattern)
    sim.init_random(0, 0.0, amp, 1, 0.01)
    A = {}
    for t0, t1 in ((0, 100), (100, 500)):
        sim.step(t1 - t0)
        rho = torch.empty((shape[2], shape[1], shape[0]), dtype=torch.float64, device="cuda")
        u = torch.empty((3,) + tuple(rho.shape), dtype=torch.float64, device="cuda")
        sim.macroscopic(rho, u)
        A[t1] = CF.shear_wave_amplitude(u[0].mean(dim=(1, 2)).cpu().numpy())
        del rho, u
    sim.close()
    L.set_kernel_path("auto")
    nu = CF.lattice_viscosity(rates[0])
    return CF.fitted_viscosity(A[100], A[500], 100, 500, shape[2]) / nu - 1

for args in [("f32", 1e-4, "auto", "aa"), ("f32", 0.0, "auto", "aa"), ("f64", 1e-4, "auto", "aa"), ("f64", 0.0, "auto", "aa"),
             ("f32", 1e-4, "plain", "aa"), ("f32", 1e-4, "auto", "pull"), ("f32", 0.0, "auto", "aa", (8, 8, 512)),
             ("f32", 1e-4, "auto", "aa", (32, 32, 512)), ("f32", 1e-4, "auto", "aa", (512, 512, 512), "srt", (1.9,)),
             ("f32", 1e-4, "auto", "aa", (512, 512, 512), "trt", (1.9, 1.9))]:
    print(args, run(*args), flush=True)
