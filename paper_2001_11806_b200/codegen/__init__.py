"""Symbolic derivation, FLOP-minimising simplification and CUDA emission of collision operators
(the paper's kernel-generation pipeline).

The generated header ``csrc/generated/gen_collide.cuh`` is committed and compiled into
``liblbm_b200.so`` as the collision ids ``LBM_GEN_SRT / LBM_GEN_TRT / LBM_GEN_MRT``; the stream,
boundary and halo code around it are the same hand-written kernels as for the other operators.
"""
from __future__ import annotations

import os

from . import derive, emit, methods  # noqa: F401

HERE = os.path.dirname(os.path.abspath(__file__))
GENERATED = os.path.join(os.path.dirname(HERE), "csrc", "generated", "gen_collide.cuh")

# (Q, op) generated into the library
OPERATORS = [(19, "srt"), (19, "trt"), (19, "mrt"), (27, "srt"), (27, "trt")]

# Table II: (only CSE, custom with direction CSE, custom default CSE); compressible,
# D3Q19 / D3Q27; "mrt" = the weighted MRT row.
PAPER_TABLE2 = {(19, "srt"): (261, 193, 193), (19, "trt"): (262, 233, 214), (19, "mrt"): (406, 947, 903),
                (27, "srt"): (444, 293, 389), (27, "trt"): (446, 379, 516), (27, "mrt"): (786, 3290, 3984)}


def generate_all(operators=OPERATORS):
    """Returns (header text, FLOP table rows)."""
    ops, table = [], []
    for Q, op in operators:
        res = derive.strategies(Q, op)
        name, best = derive.best(res)
        paper = PAPER_TABLE2.get((Q, op))
        ops.append((best, name, min(paper) if paper else None))
        table.append({"Q": Q, "op": op, "initial": res["only_cse"].history[0][1].total,
                      **{k: v.flops().total for k, v in res.items()},
                      "custom_steps": [(lbl, f.total) for lbl, f in res["custom"].history],
                      "chosen": name, "chosen_flops": best.flops().total,
                      "chosen_detail": best.flops().as_dict(),
                      "paper": dict(zip(("only_cse", "custom_direction_cse", "custom"), paper)) if paper else None})
    return emit.emit_file(ops), table
