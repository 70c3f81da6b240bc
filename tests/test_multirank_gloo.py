"""Multi-rank host logic on CPU (world_size 2 and 4, gloo): each rank computes its slab with the
oracle, and the halo exchange executes the PRODUCT's decomposition plan (lbm_slab_plan) and
zero-copy NCCL schedule (lbm_halo_schedule) with torch.distributed point-to-point messages. The
gathered result must be bit-identical to the undecomposed oracle run."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import lbminputs as LI
import oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASES = {
    "trt_channel_force": dict(Q=19, op="trt", rates=(1.6, 0.5), force=(1e-4, 0, 0), geom="channel"),
    "cumulant_periodic": dict(Q=27, op="cumulant", rates=(1.95,), force=(0, 0, 0), geom="periodic"),
}
NX, NY, NZ, STEPS = 6, 5, 8, 3


def _setup(case):
    c = CASES[case]
    fl = LI.channel_flags(NX, NY, NZ) if c["geom"] == "channel" else None
    m = O.Method(Q=c["Q"], op=c["op"], rates=c["rates"], force=c["force"], nthreads=1)
    return c, fl, m


def _worker(rank, world, port, case, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2001_11806_b200 import lbm as L
    c, fl, m = _setup(case)
    z0, nzl, down, up = L.slab_plan(NZ, world, rank)
    zg = [(z0 + k) % NZ for k in range(-1, nzl + 1)]
    d = O.Domain(m, NX, NY, nzl, zghost=1, flags=None if fl is None else np.ascontiguousarray(fl[zg]))
    # initial state on the slab incl. ghost planes: equilibrium of the seeded fields at global z
    zz, yy, xx = np.meshgrid(np.array(zg), np.arange(NY), np.arange(NX), indexing="ij")
    rho, u = LI.fields_at(0, NX, NY, NZ, xx, yy, zz, 1e-3, 0.01)
    full = O.Domain(m, NX, NY, nzl + 2)  # equilibrium of every storage plane
    a = np.ascontiguousarray(full.init_equilibrium(rho, u))
    b = a.copy()
    sched = L.halo_schedule(c["Q"], nzl, rank, world)
    for _ in range(STEPS):
        d.step_pull(a, b)
        # post the schedule: gloo isend/irecv in the same order NCCL would see them
        reqs, bufs = [], []
        for kind, peer, q, plane in sched:
            if kind == 0:
                t = torch.from_numpy(np.ascontiguousarray(b[q, plane]))
                bufs.append(t)
                reqs.append(dist.isend(t, peer))
            else:
                t = torch.empty((NY, NX), dtype=torch.float64)
                bufs.append((t, q, plane))
                reqs.append(dist.irecv(t, peer))
        for r in reqs:
            r.wait()
        for item in bufs:
            if isinstance(item, tuple):
                t, q, plane = item
                b[q, plane] = t.numpy()
        a, b = b, a
    np.save(os.path.join(out_path, f"rank{rank}.npy"), a[:, 1:-1])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("case", sorted(CASES))
def test_decomposed_oracle_with_product_schedule_bit_identical(tmp_path, world, case):
    from paper_2001_11806_b200 import build
    build.build()
    mp.spawn(_worker, args=(world, _free_port(), case, str(tmp_path)), nprocs=world, join=True)
    c, fl, m = _setup(case)
    ref_d = O.Domain(m, NX, NY, NZ, flags=fl)
    rho, u = LI.random_fields(0, NX, NY, NZ, 1e-3, 0.01)
    ref = ref_d.run_pull(ref_d.init_equilibrium(rho, u), STEPS)
    got = np.concatenate([np.load(tmp_path / f"rank{r}.npy") for r in range(world)], axis=1)
    mask = np.ones(ref.shape, bool) if fl is None else np.broadcast_to(fl == 0, ref.shape)
    np.testing.assert_array_equal(got[mask], ref[mask])


def test_schedule_shape():
    from paper_2001_11806_b200 import lbm as L
    for Q, n in ((19, 5), (27, 9)):
        s = L.halo_schedule(Q, 7, 1, 3)
        assert len(s) == 4 * n
        sends = [op for op in s if op[0] == 0]
        recvs = [op for op in s if op[0] == 1]
        assert {op[3] for op in sends} == {1, 7} and {op[3] for op in recvs} == {0, 8}
        assert all(op[1] in (0, 2) for op in s)
