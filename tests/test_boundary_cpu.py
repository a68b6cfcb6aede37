"""CPU-only checks of the C-ABI boundary: the library builds for sm_100a, loads without a
GPU, and exports every function include/qdpb.h declares; host-side argument validation
that needs no device."""
import ctypes
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def q():
    from paper_1408_5925_b200 import build as b
    b.build()
    from paper_1408_5925_b200 import qdpb
    return qdpb


def test_exports_every_declared_symbol(q):
    names = q.header_symbols()
    assert len(names) >= 25
    L = q.lib()
    for n in names:
        assert hasattr(L, n), n
    # and the binding wraps every one of them under the same name
    for n in names:
        assert hasattr(q, n), n
    out = subprocess.run(["nm", "-D", q.LIB_PATH], capture_output=True, text=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert set(names) <= exported


def test_no_cuda_runtime_dependency_and_sm100a(q):
    out = subprocess.run(["ldd", q.LIB_PATH], capture_output=True, text=True).stdout
    assert "libcudart" not in out and "libtorch" not in out
    sass = subprocess.run(["cuobjdump", "--list-elf", q.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in sass


def test_strerror_and_init_validation_without_gpu(q):
    assert q.qdp_strerror(q.QDP_ESHAPE) == "shape mismatch"
    assert q.qdp_strerror(q.QDP_OK) == "ok"
    L = q.lib()
    out = ctypes.c_void_p()
    four = lambda *v: (ctypes.c_int * 4)(*v)
    # odd extent, non-divisible grid, odd local extent, wrong rank count: rejected before touching a device
    assert L.qdp_init(four(4, 4, 4, 5), four(1, 1, 1, 1), 0, 1, None, None, ctypes.byref(out)) == q.QDP_ESHAPE
    assert L.qdp_init(four(4, 4, 4, 8), four(1, 1, 1, 3), 0, 3, None, None, ctypes.byref(out)) == q.QDP_ESHAPE
    assert L.qdp_init(four(4, 4, 4, 6), four(1, 1, 1, 2), 0, 2, None, None, ctypes.byref(out)) == q.QDP_ESHAPE
    assert L.qdp_init(four(4, 4, 4, 8), four(1, 1, 1, 2), 0, 1, None, None, ctypes.byref(out)) == q.QDP_ESHAPE
    assert L.qdp_init(four(4, 4, 4, 8), four(1, 1, 1, 1), 1, 1, None, None, ctypes.byref(out)) == q.QDP_EINVAL
    assert L.qdp_finalize(None) == q.QDP_EINVAL
    assert L.qdp_dslash(None, None, None, 0) == q.QDP_EINVAL


def test_oracle_is_not_imported_by_product():
    """The product package must not reference oracle/ (it fails loudly instead)."""
    pkg = os.path.join(ROOT, "paper_1408_5925_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cpp", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "oracle.c" not in txt, f


def test_binding_constants_match_header(q):
    """Every QDP_OPT_* / QDP_PK_* / status constant of the binding equals the header's enum value."""
    import re
    hdr = open(os.path.join(ROOT, "include", "qdpb.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)  # comments mention values too
    found = 0
    for body in re.findall(r"enum\s*\{(.*?)\}", hdr, flags=re.S):
        nxt = 0
        for item in body.split(","):
            item = item.strip()
            if not item:
                continue
            name, _, val = item.partition("=")
            name = name.strip()
            nxt = int(val.strip(), 0) if val.strip() else nxt
            if name.startswith("QDP_"):
                assert getattr(q, name) == nxt, name
                found += 1
            nxt += 1
    assert found >= 30 and q.QDP_OPT_PDL == 10
