"""Measured ceilings on the box: copy-q / update-q bandwidth probes and the DFMA / FFMA ALU probe
(include/lbm.h lbm_probe_copy / lbm_probe_update / lbm_probe_fma). Prints one JSON object."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2001_11806_b200 import lbm as L

out = {"fma_tflops": {d: L.probe_fma(d) for d in ("f64", "f32")}}
for d in ("f64", "f32"):
    for Q in (19, 27):
        shape = (512, 512, 512 if (Q == 19 or d == "f32") else 384)
        out[f"copy_q{Q}_{d}"] = L.probe_copy(Q, d, True, shape, reps=5)
        for mode, name in ((0, "even"), (1, "odd"), (2, "pair")):
            out[f"update_q{Q}_{d}_{name}"] = L.probe_update(Q, d, mode, shape, reps=6)
print(json.dumps(out))
