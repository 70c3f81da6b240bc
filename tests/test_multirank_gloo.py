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
    "trt_channel_force": dict(Q=19, op="trt", rates=(1.6, 0.5), force=(1e-4, 0, 0), geom="channel", pattern="pull"),
    "cumulant_periodic": dict(Q=27, op="cumulant", rates=(1.95,), force=(0, 0, 0), geom="periodic", pattern="pull"),
    "aa_trt_periodic": dict(Q=19, op="trt", rates=(1.6, 0.5), force=(1e-4, 0, 0), geom="periodic", pattern="aa"),
    "aa_cumulant_periodic": dict(Q=27, op="cumulant", rates=(1.95,), force=(0, 0, 0), geom="periodic", pattern="aa"),
    "eso_trt_periodic": dict(Q=19, op="trt", rates=(1.6, 0.5), force=(1e-4, 0, 0), geom="periodic", pattern="esotwist"),
    "eso_mrt_periodic": dict(Q=19, op="mrt", rates=(1.9, 1.3, 1.1, 0.8), force=(0, 0, 0), geom="periodic",
                             pattern="esotwist"),
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

    def exchange(arr, phase):
        # post the product's schedule: gloo isend/irecv in the same order NCCL would see them
        reqs, bufs = [], []
        for kind, peer, q, plane in L.halo_schedule(c["Q"], nzl, rank, world, phase):
            if kind == 0:
                t = torch.from_numpy(np.ascontiguousarray(arr[q, plane]))
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
                arr[q, plane] = t.numpy()

    if c["pattern"] == "pull":
        for _ in range(STEPS):
            d.step_pull(a, b)
            exchange(b, L.PHASE_PULL)
            a, b = b, a
        out = a[:, 1:-1]
    elif c["pattern"] == "aa":
        # AA: even step (local), ghost fill, odd step, return of the ghost-plane pushes
        for t in range(STEPS):
            if t % 2 == 0:
                d.aa_even(a)
                exchange(a, L.PHASE_AA_FILL)
            else:
                d.aa_odd(a)
                exchange(a, L.PHASE_AA_RETURN)
        out = a[:, 1:-1]
    else:
        # EsoTwist: the slab's own cells write the arriving populations of the first step, lower ghost included
        e = np.zeros_like(a)
        canon = a[:, 1:-1]
        _, _, _ = O.stencil_arrays(c["Q"])
        cq, _, _ = O.stencil_arrays(c["Q"])
        opp = O.stencil_arrays(c["Q"])[2]
        cp = np.maximum(cq, 0)
        for q in range(c["Q"]):  # a(x - c_q^+)(q) = f_q(x) for interior x (storage plane z + 1)
            for z in range(nzl):
                e[q, z + 1 - cp[q, 2]] = np.roll(canon[q, z], shift=(-cp[q, 1], -cp[q, 0]), axis=(0, 1))
        for t in range(STEPS):
            d.eso_step(e, t % 2)
            exchange(e, L.PHASE_ESO_AFTER_ODD if t % 2 else L.PHASE_ESO_AFTER_EVEN)
        out = np.zeros_like(canon)
        for q in range(c["Q"]):  # canonical F_q(x) = a(x - c_q^+)(q or qbar)
            slot = opp[q] if STEPS % 2 else q
            for z in range(nzl):
                out[q, z] = np.roll(e[slot, z + 1 - cp[q, 2]], shift=(cp[q, 1], cp[q, 0]), axis=(0, 1))
    np.save(os.path.join(out_path, f"rank{rank}.npy"), out)
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
    f0 = ref_d.init_equilibrium(rho, u)
    ref = ref_d.run_pull(f0, STEPS) if c["pattern"] == "pull" else ref_d.run_push(f0, STEPS)
    if c["pattern"] == "aa" and STEPS % 2:  # raw AA array after an odd step count: gather
        got_raw = np.concatenate([np.load(tmp_path / f"rank{r}.npy") for r in range(world)], axis=1)
        cq, _, opp = O.stencil_arrays(c["Q"])
        got = np.stack([np.roll(got_raw[opp[q]], shift=(cq[q, 2], cq[q, 1], cq[q, 0]), axis=(0, 1, 2))
                        for q in range(c["Q"])])
        np.testing.assert_array_equal(got, ref)
        return
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
