"""The zernkit installer (paper_2409_19156_b200.zernkit_plugin) rebinds the
reference's hot-path names. CPU part: binding mechanics against the real
reference when it is importable (build container only). GPU part: the
installer's GPU wrappers exercised through a stand-in package laid out like
zernkit (the reference itself is not on the GPU box)."""

import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"


@pytest.fixture
def zernkit():
    if not os.path.isdir(REF):
        pytest.skip("reference package not present (GPU box)")
    sys.path.insert(0, REF)
    try:
        import zernkit as zk
    finally:
        sys.path.remove(REF)
    return zk


def test_install_rebinds_every_hot_path_name(zernkit):
    from paper_2409_19156_b200.zernkit_plugin import install, uninstall
    import zernkit.batch as zb_ref
    import zernkit.evaluate as ze_ref
    before = ze_ref.radial_jacobi
    done = install(zernkit)
    try:
        for name in ("radial_jacobi", "zernike_eval"):
            assert f"zernkit.evaluate.{name}" in done
            assert getattr(zernkit, name) is getattr(ze_ref, name) is done[f"zernkit.evaluate.{name}"]
        for name in ("batch_cached", "batch_independent", "evaluate_batch"):
            assert getattr(zb_ref, name) is done[f"zernkit.batch.{name}"]
        assert ze_ref.radial_jacobi is not before
        # validation happens before any device work, with the reference's exception types
        with pytest.raises(zernkit.ModeError):
            zernkit.radial_jacobi(3, 2, [0.5])
        with pytest.raises(zernkit.GridError):
            zernkit.radial_jacobi(2, 0, [1.5])
        req = zb_ref.BatchRequest(modes=zernkit.full_mode_set(2), grid=[0.5], strategy="independent")
        with pytest.raises(ValueError):
            zernkit.batch_cached(req)
    finally:
        uninstall(zernkit)
    assert ze_ref.radial_jacobi is before


def _stand_in_package(name):
    """A package laid out like zernkit (evaluate / batch / tables / modes
    submodules) whose types are this repository's API mirrors and whose
    original hot-path functions are the oracle's -- so the installer's GPU
    wrappers can be exercised on the B200, where the reference is absent."""
    import types

    import paper_2409_19156_b200 as zb
    import zk_oracle as orc
    from paper_2409_19156_b200 import batch as mb, modes as mm, tables as mt

    pkg = types.ModuleType(name)
    pkg.__path__ = []
    subs = {}
    for sub in ("evaluate", "batch", "tables", "modes"):
        mod = types.ModuleType(f"{name}.{sub}")
        subs[sub] = mod
        sys.modules[f"{name}.{sub}"] = mod
        setattr(pkg, sub, mod)
    sys.modules[name] = pkg
    subs["tables"].radial_grid, subs["tables"].angular_grid = mt.radial_grid, mt.angular_grid
    subs["tables"].EvalMatrix, subs["tables"].GridError = mt.EvalMatrix, mt.GridError
    subs["modes"].make_mode = mm.make_mode
    subs["batch"].StepCounter, subs["batch"].BatchRequest = mb.StepCounter, mb.BatchRequest
    subs["evaluate"].radial_jacobi = lambda n, m, g, k=0: orc.radial_single(n, m, np.asarray(g), k)
    subs["evaluate"].zernike_eval = lambda md, g, t, k=0: orc.zernike_2d(md.n, md.m, g, t, k)
    for fn in ("batch_cached", "batch_independent", "evaluate_batch"):
        setattr(subs["batch"], fn, getattr(zb, fn))
    for fn in ("radial_jacobi", "zernike_eval"):
        setattr(pkg, fn, getattr(subs["evaluate"], fn))
    for fn in ("batch_cached", "batch_independent", "evaluate_batch"):
        setattr(pkg, fn, getattr(subs["batch"], fn))
    return pkg


@pytest.mark.gpu
def test_installed_wrappers_compute_on_the_gpu():
    import numpy as np

    import paper_2409_19156_b200 as zb
    import zk_oracle as orc
    from paper_2409_19156_b200.zernkit_plugin import install, uninstall

    pkg = _stand_in_package("zk_stand_in")
    try:
        before = pkg.evaluate.radial_jacobi
        done = install(pkg)
        assert pkg.radial_jacobi is pkg.evaluate.radial_jacobi is done["zk_stand_in.evaluate.radial_jacobi"]
        grid = np.linspace(0.0, 1.0, 257)
        got = pkg.radial_jacobi(12, 4, grid, 2)
        want = orc.radial_batch([(12, 4)], grid, 2, power=orc.cr_power)[:, 0]
        assert np.array_equal(got, want)
        th = np.linspace(-3.0, 3.0, 257)
        z = pkg.zernike_eval(zb.make_mode(9, -3), grid, th, 1)
        zr = orc.zernike_2d(9, -3, grid, th, 1)
        assert np.abs(z - zr).max() <= 1e-12 * max(1.0, np.abs(zr).max())
        req = zb.BatchRequest(modes=zb.full_mode_set(25), grid=grid, deriv_order=1)
        table, counter = pkg.evaluate_batch(req)
        assert isinstance(table, zb.EvalMatrix) and isinstance(counter, zb.StepCounter)
        ref, cref = zb.evaluate_batch(req)
        assert np.array_equal(table.values, ref.values) and counter == cref
        with pytest.raises(zb.GridError):
            pkg.radial_jacobi(2, 0, [1.5])
        with pytest.raises(ValueError):
            pkg.zernike_eval(zb.make_mode(2, 0), grid, th[:5])
        uninstall(pkg)
        assert pkg.evaluate.radial_jacobi is before
    finally:
        for key in [k for k in sys.modules if k == "zk_stand_in" or k.startswith("zk_stand_in.")]:
            del sys.modules[key]
