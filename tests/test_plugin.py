"""The zernkit installer (paper_2409_19156_b200.zernkit_plugin) rebinds the
reference's hot-path names. CPU part: binding mechanics against the real
reference when it is importable (build container only). GPU part: the
installed names return the reference's own result types with GPU values."""

import os
import sys

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
