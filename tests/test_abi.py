"""CPU-side checks of the C-ABI boundary (no compute calls without a GPU):
libdem.so builds for sm_100a, loads, exports every function include/dem.h
declares, and refuses to run without a CUDA device (no CPU fallback)."""
import ctypes as C
import subprocess

import pytest

from paper_1301_1714_b200 import build as B
from paper_1301_1714_b200 import dem


@pytest.fixture(scope="module")
def libdem():
    B.build()
    return dem.lib()


def test_header_declares_the_survey_entry_points():
    names = dem.exported_symbols()
    for must in ("dem_create", "dem_destroy", "dem_set_particles", "dem_set_contacts", "dem_step",
                 "dem_get_state", "dem_get_contacts", "dem_get_grid", "dem_get_stats",
                 "dem_strerror", "dem_last_error", "dem_sync", "dem_profile"):
        assert must in names


def test_library_exports_every_declared_symbol(libdem):
    out = subprocess.check_output(["nm", "-D", "--defined-only", B.LIB], text=True)
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [s for s in dem.exported_symbols() if s not in exported]
    assert not missing, missing
    for s in dem.exported_symbols():
        assert hasattr(libdem, s)


def test_library_is_sm100a(libdem):
    out = subprocess.check_output(["cuobjdump", "--list-elf", B.LIB], text=True)
    assert "sm_100a" in out


def test_strerror_table(libdem):
    for code in range(0, -11, -1):
        assert libdem.dem_strerror(code)
    assert libdem.dem_strerror(dem.DEM_EOVERFLOW) == b"contact history capacity exceeded"


def test_params_struct_matches_header_abi_version(libdem):
    from paper_1301_1714_b200 import scenes
    p = dem.params_from(scenes.SimParams())
    assert p.abi_version == dem.DEM_ABI_VERSION
    bad = dem.params_from(scenes.SimParams())
    bad.abi_version = 999
    h = C.c_void_p()
    assert libdem.dem_create(C.byref(bad), C.byref(h)) == dem.DEM_EABI
    bad = dem.params_from(scenes.SimParams(dt=-1.0))
    assert libdem.dem_create(C.byref(bad), C.byref(h)) == dem.DEM_EINVAL


def test_no_cpu_fallback_without_device(libdem):
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1301_1714_b200 import scenes
    with pytest.raises(dem.DemError) as e:
        dem.Dem(scenes.SimParams(), torch_allocator=False)
    assert e.value.code == dem.DEM_ECUDA


def test_ablations_only_in_their_build(libdem):
    """The product library carries only the default path: the ablation flags
    (the paper's fused mapping, half lists, one lane per particle) are
    rejected there and accepted by libdem_ablations.so, which exports the
    same symbols."""
    from paper_1301_1714_b200 import scenes
    abl = dem.lib(dem.ABLATIONS_PATH)
    for s in dem.exported_symbols():
        assert hasattr(abl, s)
    for f in (dem.DEM_F_THREAD_PER_PARTICLE, dem.DEM_F_HALF_LISTS, dem.DEM_F_FORCE_LANES,
              dem.DEM_F_FORCE_WS):
        p = dem.params_from(scenes.SimParams(), flags=f)
        h = C.c_void_p()
        assert libdem.dem_create(C.byref(p), C.byref(h)) == dem.DEM_EINVAL
        rc = abl.dem_create(C.byref(p), C.byref(h))
        assert rc != dem.DEM_EINVAL  # (DEM_ECUDA without a device)
        if rc == dem.DEM_OK:
            abl.dem_destroy(h)
