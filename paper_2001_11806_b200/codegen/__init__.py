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

# (Q, op, equilibrium) generated into the library
C, I = "compressible", "incompressible"
OPERATORS = [(19, "srt", C), (19, "trt", C), (19, "mrt", C), (19, "smagorinsky", C), (19, "srt", I), (19, "trt", I),
             (27, "srt", C), (27, "trt", C), (27, "mrt", C), (27, "smagorinsky", C), (27, "srt", I), (27, "trt", I)]
# FLOP-table rows that are not compiled into the library
TABLE_ONLY = []

# Table II: (only CSE, custom with direction CSE, custom default CSE), D3Q19 / D3Q27;
# "mrt" = the weighted MRT row.
PAPER_TABLE2 = {(19, "srt", C): (261, 193, 193), (19, "srt", I): (252, 162, 162), (19, "smagorinsky", C): (306, 251, 251),
                (19, "trt", C): (262, 233, 214), (19, "trt", I): (253, 225, 206), (19, "mrt", C): (406, 947, 903),
                (27, "srt", C): (444, 293, 389), (27, "srt", I): (435, 289, 346), (27, "smagorinsky", C): (510, 370, 370),
                (27, "trt", C): (446, 379, 516), (27, "trt", I): (437, 374, 482), (27, "mrt", C): (786, 3290, 3984)}


def generate_all(operators=OPERATORS, table_only=()):
    """Returns (header text, FLOP table rows)."""
    ops, table = [], []
    for Q, op, eq in list(operators) + list(table_only):
        res = derive.strategies(Q, op, eq)
        name, best = derive.best(res)
        paper = PAPER_TABLE2.get((Q, op, eq))
        if (Q, op, eq) in operators:
            ops.append((best, name, min(paper) if paper else None))
        table.append({"Q": Q, "op": op, "equilibrium": eq, "initial": res["only_cse"].history[0][1].total,
                      **{k: v.flops().total for k, v in res.items()},
                      "custom_steps": [(lbl, f.total) for lbl, f in res["custom"].history],
                      "chosen": name, "chosen_flops": best.flops().total,
                      "chosen_detail": best.flops().as_dict(),
                      "paper": dict(zip(("only_cse", "custom_direction_cse", "custom"), paper)) if paper else None})
    return emit.emit_file(ops), table
