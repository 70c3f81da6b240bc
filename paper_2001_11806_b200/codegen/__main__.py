"""Regenerate csrc/generated/gen_collide.cuh and the FLOP table (profiles/codegen_flops.json).

Usage: python -m paper_2001_11806_b200.codegen [--check]
  --check: exit 1 if the committed header differs from a fresh generation.
"""
from __future__ import annotations

import json
import os
import sys

from . import GENERATED, OPERATORS, TABLE_ONLY, generate_all


def main(argv=None) -> int:
    argv = sys.argv[1:] if argv is None else argv
    text, table = generate_all(OPERATORS, TABLE_ONLY if "--check" not in argv else ())
    if "--check" in argv:
        with open(GENERATED) as fh:
            same = fh.read() == text
        print("up to date" if same else "STALE: regenerate with python -m paper_2001_11806_b200.codegen")
        return 0 if same else 1
    os.makedirs(os.path.dirname(GENERATED), exist_ok=True)
    with open(GENERATED, "w") as fh:
        fh.write(text)
    root = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    with open(os.path.join(root, "profiles", "codegen_flops.json"), "w") as fh:
        json.dump(table, fh, indent=1)
    for row in table:
        print(f"D3Q{row['Q']} {row['op'][:5]:5s} {row['equilibrium'][:5]} only_cse {row['only_cse']:5d}  custom+dir {row['custom_direction_cse']:5d}"
              f"  custom {row['custom']:5d}  -> {row['chosen']} ({row['chosen_flops']}); paper {row['paper']}")
    print("wrote", GENERATED)
    return 0


if __name__ == "__main__":
    sys.exit(main())
