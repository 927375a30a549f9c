"""CPU checks of the C-ABI boundary: libosam.so loads and exports every symbol include/osam.h declares."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "osam.h")
LIB = os.path.join(ROOT, "paper_2511_20687_b200", "libosam.so")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(osam_[a-z_]+)\s*\(", src)))


def test_header_declares_the_five_calls():
    names = declared_functions()
    for required in ("osam_create_subdomain", "osam_set_ic", "osam_step", "osam_get_state", "osam_destroy"):
        assert required in names


@pytest.mark.skipif(not os.path.exists(LIB), reason="libosam.so not built (run __graft_entry__.build())")
def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    for name in declared_functions():
        assert hasattr(lib, name), name
    from paper_2511_20687_b200 import osam
    assert set(osam.EXPORTS) >= set(declared_functions())


@pytest.mark.skipif(not os.path.exists(LIB), reason="libosam.so not built")
def test_no_gpu_fails_loudly_not_silently():
    """Without a GPU the library must refuse (OSAM_ECUDA), never fall back to a CPU path."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2511_20687_b200 import osam
    with pytest.raises(osam.OsamError) as e:
        osam.Subdomain(osam.OSAM_FOM, (0, 0, 0), (1, 1, 1), (2, 2, 2), 1e9, 0.25, 1000.0)
    assert e.value.code == -3


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2511_20687_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f


@pytest.mark.skipif(not os.path.exists(LIB), reason="libosam.so not built")
@pytest.mark.parametrize("case", ["fom_implicit", "rom_material", "bad_material", "neg_substeps", "bad_integrator",
                                  "cbar_without_hbar"])
def test_descriptor_validation_before_any_gpu_work(case):
    """Invalid descriptors are rejected with OSAM_EINVAL by host-side validation (GPU or not): the FOM is explicit,
    a ROM has no material model, n_substeps in 0..4096, integrator / material enums, COpInf needs Hbar."""
    import numpy as np
    from paper_2511_20687_b200 import osam
    d = osam.osam_subdomain_desc()
    d.kind = osam.OSAM_FOM
    d.lo[:] = [0.0, 0.0, 0.0]
    d.hi[:] = [1.0, 1.0, 1.0]
    d.nel[:] = [2, 2, 2]
    d.E, d.nu, d.rho = 1e9, 0.25, 1000.0
    d.batch = 1
    keep = []
    if case == "fom_implicit":
        d.integrator = osam.OSAM_IMPLICIT
    elif case == "rom_material":
        d.kind = osam.OSAM_ROM
        d.material = osam.OSAM_SVK
    elif case == "bad_material":
        d.material = 7
    elif case == "neg_substeps":
        d.n_substeps = -1
    elif case == "bad_integrator":
        d.integrator = 5
    elif case == "cbar_without_hbar":
        d.kind = osam.OSAM_ROM
        r = 2
        mats = [np.asfortranarray(np.eye(r)), np.asfortranarray(np.zeros((r, 4)))]
        keep += mats
        d.r, d.r_b, d.n_free, d.n_s = r, 0, r, 0
        d.Phi = osam._dptr(mats[0])
        d.Kbar = osam._dptr(mats[0])
        d.Cbar = osam._dptr(mats[1])
    h = ctypes.c_void_p()
    rc = osam.lib().osam_create_subdomain(ctypes.byref(d), None, ctypes.byref(h))
    assert rc == -1, (case, rc, osam.lib().osam_last_error())
    assert not h.value


@pytest.mark.skipif(not os.path.exists(LIB), reason="libosam.so not built")
@pytest.mark.parametrize("rows", [[3, 1, 5], [0, 2, 9], [0, -1, 2], [0, 1]])
def test_phi_row_subset_validation_before_any_gpu_work(rows):
    """phi_rows (Phi given on the rows the transfer lifts) must be strictly ascending free-row indices in
    [0, n_free) with at least r rows: anything else is OSAM_EINVAL from host-side validation (GPU or not)."""
    import numpy as np
    from paper_2511_20687_b200 import osam
    r, n_free = 3, 9
    d = osam.osam_subdomain_desc()
    d.kind = osam.OSAM_ROM
    d.lo[:] = [0.0, 0.0, 0.0]
    d.hi[:] = [1.0, 1.0, 1.0]
    d.nel[:] = [2, 2, 2]
    d.E, d.nu, d.rho = 1e9, 0.25, 1000.0
    d.batch = 1
    ids = np.asarray(rows, dtype=np.int64)
    Phi = np.asfortranarray(np.ones((len(rows), r)))
    K = np.asfortranarray(np.eye(r))
    d.r, d.r_b, d.n_free, d.n_s = r, 0, n_free, 0
    d.Phi, d.Kbar = osam._dptr(Phi), osam._dptr(K)
    d.phi_rows = ids.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
    d.n_phi_rows = len(rows)
    h = ctypes.c_void_p()
    rc = osam.lib().osam_create_subdomain(ctypes.byref(d), None, ctypes.byref(h))
    assert rc == -1, (rows, rc, osam.lib().osam_last_error())
    assert not h.value


def test_binding_rejects_wrong_buffers():
    """The binding checks dtype, contiguity and element count before handing a pointer to the library."""
    import numpy as np
    from paper_2511_20687_b200 import osam
    with pytest.raises(ValueError):
        osam._ptr(np.zeros(4, dtype=np.float32))
    with pytest.raises(ValueError):
        osam._ptr(np.zeros(4), numel=5)
    with pytest.raises(ValueError):
        osam._ptr(np.zeros((4, 4))[:, 1])
    assert osam._ptr(np.zeros(4), numel=4) is not None
