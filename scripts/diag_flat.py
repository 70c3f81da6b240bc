"""Diagnostic: where do the flat-row and box-block launches of the fp32 AA channel with index-list boundaries differ?"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.gpu_common import Case, fluid_mask, init_sim, make_sim, oracle_run
from paper_2001_11806_b200 import lbm as L

def run(case, kw, env=None, steps=(3, 2)):
    if env is not None:
        os.environ["LBM_FLAT"] = env
    else:
        os.environ.pop("LBM_FLAT", None)
    sim = make_sim(case, boundary_mode="links", **kw)
    init_sim(sim, case)
    out = []
    for n in steps:
        sim.step(n)
        out.append((sim.populations(raw=True).copy(), sim.populations().copy()))
    impl = sim.boundary_impl
    sim.close()
    return out, impl

for dtype in ("f32", "f64"):
    for path in ("plain", "auto"):
        L.set_kernel_path(path)
        case = Case("flat", (44, 11, 6), 19, "trt", (1.6, 0.5), dtype, pattern="aa", geometry="channel", force=(1e-5, 0, 0), steps=5)
        mask = fluid_mask(case, 19)
        runs = {"flat1": run(case, {}), "box1": run(case, {"block_x": 32}), "box2": run(case, {"block_x": 32}),
                "flat2": run(case, {}), "envbox": run(case, {}, env="0"), "box64": run(case, {"block_x": 64})}
        print(dtype, path, {k: v[1] for k, v in runs.items()})
        ref = runs["box1"][0]
        for k, (o, _) in runs.items():
            for s in range(2):
                for kind in (0, 1):
                    d = (o[s][kind] != ref[s][kind]) & mask
                    if d.any():
                        idx = np.argwhere(d)
                        print(f"  {k} step-set {s} {'raw' if kind == 0 else 'canonical'}: {len(idx)} differ", idx[:12].tolist(),
                              o[s][kind][d][:6], ref[s][kind][d][:6])
        orc = oracle_run(case, 5)
        for k, (o, _) in runs.items():
            e = np.abs(o[1][1][mask] - orc[mask]) / np.abs(orc[mask])
            print(f"  {k} vs oracle after 5 steps: max rel err {e.max():.3e}")
L.set_kernel_path("auto")
