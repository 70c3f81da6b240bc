"""Worker of tests/test_multigpu.py, one process per GPU (torchrun): the z-slab decomposition over NCCL ranks
 must reproduce the single-GPU run bit for bit, for every storage pattern and halo transport.

  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tests/multigpu_worker.py \
      --pattern pull --halo 2 --steps 13

Every rank runs its slab; rank 0 gathers the slabs' stored states (NCCL all-gather of the canonical
populations), runs the same configuration on one GPU, compares and prints one JSON line
{"ok": bool, ...}. Exit code 0 iff identical.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--pattern", default="pull")
    ap.add_argument("--halo", type=int, default=0)
    ap.add_argument("--steps", type=int, default=13)
    ap.add_argument("--geometry", default="channel")
    ap.add_argument("--links", type=int, default=0)
    args = ap.parse_args()

    import numpy as np
    import torch
    import torch.distributed as dist

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2001_11806_b200 import lbm as L
    from tests.gpu_common import Case, init_sim, make_sim

    case = Case("mgpu", (32, 24, 8 * world), 19, "trt", (1.6, 0.5), "f64", pattern=args.pattern,
                force=(1e-5, 0, 0), geometry=args.geometry, ubb=(0.02, -0.01, 0.03), steps=args.steps)
    buf = torch.zeros(128, dtype=torch.uint8, device="cuda")
    if rank == 0:
        buf.copy_(torch.frombuffer(bytearray(L.nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(buf, 0)
    nccl_id = bytes(buf.cpu().numpy().tobytes())
    bm = "links" if args.links else "flags"
    sim = make_sim(case, rank=rank, nranks=world, nccl_id=nccl_id, device=local, halo_mode=args.halo, boundary_mode=bm)
    init_sim(sim, case)
    sim.step(case.steps)
    sim.sync()
    local_pops = torch.from_numpy(sim.populations()).cuda()  # (Q, nz_local, ny, nx), canonical
    parts = [torch.empty_like(local_pops) for _ in range(world)]
    dist.all_gather(parts, local_pops)
    ok, err = True, 0.0
    if rank == 0:
        got = torch.cat(parts, dim=1).cpu().numpy()
        one = make_sim(case, device=local, boundary_mode=bm)
        init_sim(one, case)
        one.step(case.steps)
        ref = one.populations()
        fl = case.flags()
        mask = np.ones(ref.shape, bool) if fl is None else np.broadcast_to(fl == 0, ref.shape)
        ok = bool(np.array_equal(got[mask], ref[mask]))
        err = float(np.abs(got[mask] - ref[mask]).max())
        print(json.dumps({"ok": ok, "world": world, "pattern": args.pattern, "halo": args.halo, "links": args.links,
                          "max_abs_diff": err}))
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.broadcast(flag, 0)
    sim.close()
    dist.destroy_process_group()
    return 0 if int(flag) == 1 else 1


if __name__ == "__main__":
    sys.exit(main())
