"""The C ABI from plain C (examples/lbm_demo.c): it compiles and links against liblbm_b200.so without Python
or torch headers (CPU), and on a GPU its channel-flow result matches the oracle (x/z-invariant flow: a
1 x 34 x 1 oracle column) to the fp64 bar."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    from paper_2001_11806_b200 import build
    build.build()
    exe = str(tmp_path / "lbm_demo")
    libdir = os.path.join(ROOT, "paper_2001_11806_b200")
    cmd = ["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "examples", "lbm_demo.c"),
           "-L", libdir, "-llbm_b200", f"-Wl,-rpath,{libdir}", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_example_compiles_and_links(tmp_path):
    exe = _build(tmp_path)
    out = subprocess.run(["nm", "-u", exe], capture_output=True, text=True).stdout
    assert "lbm_create" in out and "lbm_step" in out and "lbm_get_macroscopic" in out


@pytest.mark.gpu
def test_c_example_runs_and_matches_oracle(tmp_path):
    import lbminputs as LI
    import oracle as O
    exe = _build(tmp_path)
    r = subprocess.run([exe, "200"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    m = re.search(r"mass=(\S+) umax=(\S+) launches=(\d+)", r.stdout)
    mass, umax, launches = float(m.group(1)), float(m.group(2)), int(m.group(3))
    assert launches > 0
    nx, ny, nz = 32, 34, 16
    d = O.Domain(O.Method(Q=19, op="trt", rates=(1.6, 0.5), force=(1e-6, 0, 0)), 1, ny, 1, flags=LI.channel_flags(1, ny, 1))
    f = d.run_pull(d.init_equilibrium(np.ones((1, ny, 1)), np.zeros((3, 1, ny, 1))), 200)
    rho, u = d.macroscopic(f, post_collision=True)
    assert abs(umax / u[0, 0, 1:ny - 1, 0].max() - 1) <= 1e-12
    assert abs(mass / (rho[0, 1:ny - 1, 0].sum() * nx * nz) - 1) <= 1e-13
