"""C-ABI library checks that need no GPU: the shared library loads, exports every symbol declared
in include/lbm.h, and its host-only functions (decomposition plan, crossing directions, stencil
table, validation errors) agree with the oracle / the paper."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lbm.h")


@pytest.fixture(scope="module")
def L():
    from paper_2001_11806_b200 import build
    build.build()
    from paper_2001_11806_b200 import lbm
    return lbm


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(lbm_[a-z_0-9]+)\s*\(", src, flags=re.M)))


def test_every_declared_symbol_is_exported(L):
    names = declared_functions()
    assert "lbm_create" in names and "lbm_step" in names and "lbm_get_macroscopic" in names
    out = subprocess.run(["nm", "-D", "--defined-only", L.LIBPATH], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (lbm_[a-z_0-9]+)$", out, flags=re.M))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    # the binding wraps every declared function under the same name
    assert sorted(set(L.EXPORTED)) == names


def test_library_is_sm100a(L):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", L.LIBPATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_stencil_table_matches_oracle(L):
    import oracle as O
    for Q in (19, 27):
        c, w = L.stencil_table(Q)
        co, wo, _ = O.stencil_arrays(Q)
        np.testing.assert_array_equal(c, co)
        np.testing.assert_array_equal(w, wo)


def test_crossing_directions(L):
    import oracle as O
    for Q, n in ((19, 5), (27, 9)):
        c, _, _ = O.stencil_arrays(Q)
        for d in (1, -1):
            got = L.crossing_directions(Q, d)
            assert len(got) == n and got == [q for q in range(Q) if c[q, 2] == d]


def test_slab_plan(L):
    for P in (1, 2, 4, 8):
        spans = [L.slab_plan(512 * P, P, r) for r in range(P)]
        assert [s[0] for s in spans] == [512 * r for r in range(P)]
        assert all(s[1] == 512 for s in spans)
        assert [s[2] for s in spans] == [(r - 1) % P for r in range(P)]
        assert [s[3] for s in spans] == [(r + 1) % P for r in range(P)]
    with pytest.raises(L.LBMError):
        L.slab_plan(10, 3, 0)
    with pytest.raises(L.LBMError):
        L.slab_plan(8, 8, 0)  # one plane per slab is too thin


@pytest.mark.parametrize("kw,code", [
    (dict(rates=(2.5,)), -1),                                   # rate outside (0, 2)
    (dict(collision="trt", rates=(1.6,)), -1),                  # TRT needs two rates
    (dict(stencil=27, collision="mrt", rates=(1.9,)), -2),      # MRT is D3Q19 only
    (dict(collision="mrt", rates=(1.9,), force=(1e-5, 0, 0)), -2),
    (dict(collision="smagorinsky", rates=(1.9,)), -1),             # needs [omega_0, C_S]
    (dict(n_local_slabs=3), -1),                                # nz % slabs != 0
    (dict(periodic=(1, 0, 1)), -1),                             # non-periodic axis without walls
    (dict(nccl_self=True, n_local_slabs=2), -1),                # self-exchange is single-slab
    (dict(equilibrium=3), -1),                                  # unknown equilibrium kind
    (dict(shape=(0, 8, 8)), -1),                                # empty lattice
    (dict(shape=(8, 8, 0)), -1),
    (dict(boundary_mode=3), -1),                                # unknown boundary mode
    (dict(boundary_mode="inline", nccl_self=True, halo_mode=2), -2),  # inline: no fused halo
    (dict(collision="trt", rates=(1.0,) * 15), -1),             # per-moment rates are for MRT
    (dict(collision="mrt", rates=(1.0,) * 14 + (2.0,)), -1),    # per-moment rate outside (0, 2)
    (dict(collision="mrt", rates=(1.0,) * 15, equilibrium="incompressible"), -2),
    (dict(stencil=27, collision="cumulant", rates=(1.9,), equilibrium="incompressible"), -2),
    (dict(collision="kbc", rates=(1.9,), equilibrium="moment_matched"), -2),
    (dict(collision="kbc_exact", rates=(1.9,), force=(1e-5, 0, 0)), -2),   # forcing is SRT/TRT only
    (dict(collision=12), -1),                                   # unknown collision id
    (dict(collision="gen_srt", rates=(1.8,), equilibrium="moment_matched"), -2),
    (dict(collision="gen_smagorinsky", rates=(1.9,)), -1),        # needs [omega_0, C_S]
    (dict(collision="gen_trt", rates=(1.6, 0.5), force=(1e-5, 0, 0)), -2),
])
def test_create_validation_errors(L, kw, code):
    """Validation happens before any CUDA call, so these run on a CPU-only host."""
    args = dict(shape=(8, 8, 8))
    args.update(kw)
    with pytest.raises(L.LBMError) as e:
        L.Simulation(**args)
    assert e.value.status == code


def test_nonperiodic_axis_requires_walls(L):
    import lbminputs as LI
    fl = LI.channel_flags(8, 8, 8)
    fl[:, -1, 3] = 0  # hole in the top wall
    with pytest.raises(L.LBMError) as e:
        L.Simulation((8, 8, 8), periodic=(1, 0, 1), flags=fl)
    assert e.value.status == -1


def test_binding_constants_match_header(L):
    """Every enum constant of the binding equals the #define of include/lbm.h (collision ids incl.
    LBM_KBC_EXACT and the generated operators, boundary modes, equilibria, patterns)."""
    import re
    defs = dict(re.findall(r"^#define (LBM_[A-Z0-9_]+) (-?\d+)", open(HEADER).read(), re.M))
    names = {"KBC_EXACT": "LBM_KBC_EXACT", "GEN_SRT": "LBM_GEN_SRT", "GEN_TRT": "LBM_GEN_TRT",
             "GEN_MRT": "LBM_GEN_MRT", "GEN_SMAGORINSKY": "LBM_GEN_SMAGORINSKY", "KBC": "LBM_KBC",
             "SMAGORINSKY": "LBM_SMAGORINSKY", "CUMULANT": "LBM_CUMULANT", "MRT": "LBM_MRT", "TRT": "LBM_TRT",
             "SRT": "LBM_SRT", "IDENTITY": "LBM_IDENTITY", "BOUNDARY_FLAGS": "LBM_BOUNDARY_FLAGS",
             "BOUNDARY_LINKS": "LBM_BOUNDARY_LINKS", "BOUNDARY_INLINE": "LBM_BOUNDARY_INLINE"}
    for py, c in names.items():
        assert getattr(L, py) == int(defs[c]), (py, c)
    for name, v in L.COLLISIONS.items():
        assert v == int(defs["LBM_" + name.upper()]), name
    for name, v in L.BOUNDARY_MODES.items():
        assert v == int(defs["LBM_BOUNDARY_" + name.upper()]), name


def _cfg(L, **kw):
    import ctypes as C
    cfg = L.lbm_config()
    L.lbm_config_default(C.byref(cfg))
    for k, v in kw.items():
        if k == "pdf_dev":
            cfg.pdf_dev[0], cfg.pdf_dev[1] = v
        elif k == "global_":
            cfg.global_[0], cfg.global_[1], cfg.global_[2] = v
        else:
            setattr(cfg, k, v)
    return cfg


def test_buffer_sizes_and_borrowed_buffer_validation(L):
    """lbm_buffer_sizes (host-only) and the ownership rules of borrowed device buffers (include/lbm.h
    "Ownership"): sizes follow the SoA layout with ghost planes; validation happens before any
    CUDA call, so fake (never dereferenced) device addresses exercise it on a CPU-only host."""
    import ctypes as C
    out = np.zeros(3, np.int64)
    cfg = _cfg(L, stencil=19, dtype=L.F64, global_=(32, 16, 8))
    assert L.lbm_buffer_sizes(C.byref(cfg), out.ctypes.data) == 0
    assert list(out) == [32 * 16 * 8 * 19 * 8, 0, 0]
    fl = np.zeros((8, 16, 32), np.uint8)
    fl[:, 0, :] = fl[:, -1, :] = 1
    cfg = _cfg(L, stencil=27, dtype=L.F32, global_=(32, 16, 8), nccl_self=1, flags=fl.ctypes.data)
    cfg.periodic[1] = 0
    assert L.lbm_buffer_sizes(C.byref(cfg), out.ctypes.data) == 0
    assert list(out) == [32 * 16 * 10 * 27 * 4, 32 * 16 * 10, 4 * 32 * 16 * 9 * 4]
    bad = [
        (dict(pdf_dev=(0x1000, 0)), -1),                               # pull needs both arrays
        (dict(pattern=L.AA, pdf_dev=(0x1000, 0x2000)), -1),             # AA has one array
        (dict(pdf_dev=(0x1008, 0x2000)), -1),                           # not 16-byte aligned
        (dict(pdf_dev=(0x1000, 0x2000), n_local_slabs=2), -2),          # one slab per process
        (dict(pdf_dev=(0x1000, 0x2000), nccl_self=1, halo_mode=L.HALO_FUSED), -2),  # fused owns its windows
        (dict(flags_dev=0x1000), -1),                                   # no flag field
        (dict(halo_dev=0x1000), -1),                                    # no decomposition
    ]
    for kw, code in bad:
        cfg = _cfg(L, global_=(32, 16, 8), **kw)
        assert L.lbm_buffer_sizes(C.byref(cfg), out.ctypes.data) == code, kw
    cfg = _cfg(L, global_=(32, 16, 8), pattern=L.AA, pdf_dev=(0x1000, 0))
    assert L.lbm_buffer_sizes(C.byref(cfg), out.ctypes.data) == 0


@pytest.mark.parametrize("geometry,periodic,expect", [
    ("channel", (1, 0, 1), [0, 0, 1, 1, 0, 0]),
    ("cavity", (0, 0, 0), [1, 1, 1, 1, 1, 2]),   # lid = UBB face; its edges belong to the x/y faces (G9)
    ("cavity_z_first", (0, 0, 0), None),        # lid edges UBB: not the -x,+x,-y,+y,-z,+z precedence
    ("obstacles", (1, 1, 1), None),
    ("channel_hole", (1, 0, 1), None),
])
def test_face_aligned_wall_detection(L, geometry, periodic, expect):
    """lbm_detect_faces (host-only): the flag fields of C1 (channel) and C3 (cavity) are face-aligned and run
    the FM_FACES kernels; other geometries keep the flag kernels."""
    import ctypes as C
    import lbminputs as LI
    n = 12
    if geometry == "channel":
        fl = LI.channel_flags(n, n, n)
    elif geometry.startswith("cavity"):
        fl = LI.cavity_flags(n)
        if geometry == "cavity_z_first":
            fl[n - 1, :, :] = LI.UBB
    elif geometry == "channel_hole":
        fl = LI.channel_flags(n, n, n)
        fl[3, 5, 5] = LI.NOSLIP  # an interior obstacle
    else:
        fl = LI.random_obstacles(0, n, n, n)
    fl = np.ascontiguousarray(fl, np.uint8)
    cfg = _cfg(L, global_=(n, n, n), flags=fl.ctypes.data)
    for d in range(3):
        cfg.periodic[d] = periodic[d]
    out = np.zeros(6, np.int8)
    r = L.lbm_detect_faces(C.byref(cfg), out.ctypes.data)
    if expect is None:
        assert r == 0
    else:
        assert r == 1 and out.tolist() == expect
