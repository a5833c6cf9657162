"""libccm.so builds, loads and exports every symbol include/libccm.h declares; host-only
entry points (workspace sizing, validation that fails before touching the GPU) behave.
No compute calls here: this container has no GPU."""
import ctypes as C
import os
import re

import pytest

from paper_2011_11082_b200 import build as B
from paper_2011_11082_b200 import libccm

HEADER = os.path.join(B.INCLUDE, "libccm.h")


@pytest.fixture(scope="module")
def lib():
    B.build()
    return libccm.load()


def declared_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(edm_[a-z_A-Z]+)\s*\(", txt)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for n in ("edm_embed_knn", "edm_simplex_optimal_E", "edm_ccm_all_pairs", "edm_workspace_bytes",
              "edm_last_error", "edm_causal_map_host"):
        assert n in names
    assert set(names) == set(libccm.EXPORTS)


def test_every_declared_symbol_is_exported(lib):
    raw = C.CDLL(B.LIB)
    for n in declared_functions():
        assert hasattr(raw, n), n


def test_built_for_sm100a():
    out = os.popen(f"cuobjdump --list-elf {B.LIB} 2>&1").read()
    assert "sm_100a" in out, out


def test_version_and_workspace_sizes(lib):
    assert b"sm_100a" in lib.edm_version()
    assert lib.edm_workspace_bytes(0, 1000, 1000, 20, 1, 1) > 0
    w1 = lib.edm_workspace_bytes(1, 1000, 1000, 20, 1, 1)
    w2 = lib.edm_workspace_bytes(1, 2000, 1000, 20, 1, 1)
    assert 0 < w1 < w2
    assert lib.edm_workspace_bytes(0, 0, 1000, 20, 1, 1) == 0       # N < 1
    assert lib.edm_workspace_bytes(1, 10, 1000, 21, 1, 1) == 0      # E_max > cap
    assert lib.edm_workspace_bytes(2, 10, 1000, 20, 1, 1) == 0      # unknown which


def test_validation_before_device(lib):
    # null pointers / bad sizes are rejected synchronously (EINVAL) without any GPU work
    assert lib.edm_embed_knn(None, 100, 2, 1, 1, 1, None, None, None, None) == libccm.EDM_EINVAL
    assert b"null" in lib.edm_last_error()
    fake = C.c_void_p(16)
    assert lib.edm_embed_knn(fake, 100, 0, 1, 1, 1, fake, fake, None, None) == libccm.EDM_EINVAL
    assert lib.edm_embed_knn(fake, 100, 21, 1, 1, 1, fake, fake, None, None) == libccm.EDM_EINVAL
    assert lib.edm_embed_knn(fake, 5, 3, 1, 1, 1, fake, fake, None, None) == libccm.EDM_ETOOSHORT
    ds = libccm.edm_dataset(16, 10, 100, 10)
    assert lib.edm_simplex_optimal_E(ds, 25, 1, 0, 10, fake, None, fake, 1 << 30, None) == libccm.EDM_EINVAL
    assert lib.edm_simplex_optimal_E(ds, 5, 1, 0, 11, fake, None, fake, 1 << 30, None) == libccm.EDM_EINVAL
    assert lib.edm_simplex_optimal_E(ds, 5, 1, 0, 10, fake, None, fake, 16, None) == libccm.EDM_EWORKSPACE
    assert lib.edm_ccm_all_pairs(ds, fake, 1, 1, 7, 1, 0, 10, fake, fake, 1 << 30, None) == libccm.EDM_EINVAL
    assert lib.edm_ccm_all_pairs(ds, fake, 1, 1, 0, 1, 3, 2, fake, fake, 1 << 30, None) == libccm.EDM_EINVAL
    # convergence test: sizes must be >= 1 and every order a permutation of 0..L-1 (host arrays)
    import numpy as np
    sizes = np.array([10, 50], np.int32)
    orders = np.tile(np.arange(100, dtype=np.int32), (2, 1))
    sp, op = sizes.ctypes.data, orders.ctypes.data
    assert lib.edm_ccm_convergence_workspace_bytes(10, 100, 1, 1, 2, 2) > 0
    assert lib.edm_ccm_convergence_workspace_bytes(10, 100, 1, 1, 0, 2) == 0
    orders[1, 3] = 4
    assert lib.edm_ccm_convergence(ds, fake, 1, 1, 0, 1, sp, 2, op, 2, 0, 10, fake, None, fake, 1 << 40,
                                   None) == libccm.EDM_EINVAL
    assert b"permutation" in lib.edm_last_error()
    orders[1, 3] = 3
    sizes[1] = 0
    assert lib.edm_ccm_convergence(ds, fake, 1, 1, 0, 1, sp, 2, op, 2, 0, 10, fake, None, fake, 1 << 40,
                                   None) == libccm.EDM_EINVAL
    sizes[1] = 50
    assert lib.edm_ccm_convergence(ds, fake, 1, 1, 0, 1, sp, 2, op, 2, 0, 10, fake, None, fake, 16,
                                   None) == libccm.EDM_EWORKSPACE


def test_product_path_does_not_touch_the_oracle():
    # the product package never imports / links / executes anything under oracle/
    pkg = os.path.dirname(B.__file__)
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(root, f)).read()
                assert "oracle" not in src.replace("oracle's", "").replace("the oracle", "").lower() or \
                    "import oracle" not in src and "from oracle" not in src, f
                assert "import oracle" not in src and "from oracle" not in src and "liboracle" not in src, f
                # nor the host comparison implementation (no CPU fallback anywhere in the product)
                assert "cpu_baseline" not in src and "mpedm_cpu" not in src, f
