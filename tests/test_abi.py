"""CPU-only checks of the C-ABI boundary (no compute calls without a GPU):
libhfr.so loads, exports every function include/hfr.h declares, validates
arguments before touching the GPU, and its (host-side) double binary tree
equals the oracle's — two independent constructions of reading R9."""
import ctypes
import os
import re

import pytest

import paper_2408_14158_b200 as hfr
from oracle import hfr_oracle as O
from paper_2408_14158_b200 import _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    _build.build()


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "hfr.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hfr_[a-z_]+)\s*\(", src)) - {"hfr_allgather_fn"})


def test_exports_every_declared_symbol():
    L = hfr.lib()
    declared = _declared_functions()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(L, name), name
    assert sorted(hfr.EXPORTS) == declared


def test_nm_shows_c_linkage():
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", hfr.LIB_PATH], capture_output=True, text=True).stdout
    for name in _declared_functions():
        assert re.search(rf"\bT {name}$", out, re.M), name


def test_status_strings():
    for s in range(9):
        assert hfr.status_string(s)
    assert "protocol" in hfr.status_string(hfr.ERR_PROTOCOL)


def test_config_default():
    c = hfr._Config()
    hfr.lib().hfr_config_default(ctypes.byref(c))
    assert c.algo == hfr.ALGO_AUTO and c.scale == 1.0
    assert c.chunk_elems == 0 and c.threads == 0 and c.timeout_ms > 0
    assert c.oneshot_max_bytes == 4 << 20


def test_argument_validation_without_gpu():
    L = hfr.lib()
    h = ctypes.c_void_p()
    null_ag = hfr._AG_FN()
    assert L.hfr_init(None, 0, 1, 0, null_ag, None, None) == hfr.ERR_INVALID_ARGUMENT
    assert L.hfr_init(ctypes.byref(h), 2, 2, 0, null_ag, None, None) == hfr.ERR_INVALID_ARGUMENT
    assert L.hfr_init(ctypes.byref(h), 0, 0, 0, null_ag, None, None) == hfr.ERR_INVALID_ARGUMENT
    assert L.hfr_init(ctypes.byref(h), 0, 17, 0, null_ag, None, None) == hfr.ERR_INVALID_ARGUMENT
    assert L.hfr_init(ctypes.byref(h), 0, 2, 0, null_ag, None, None) == hfr.ERR_INVALID_ARGUMENT  # no allgather
    bad = hfr.Config(chunk_elems=100)._c()
    assert L.hfr_init_virtual(ctypes.byref(h), 2, 0, ctypes.byref(bad)) == hfr.ERR_INVALID_ARGUMENT
    bad = hfr.Config(threads=1000)._c()
    assert L.hfr_init_virtual(ctypes.byref(h), 2, 0, ctypes.byref(bad)) == hfr.ERR_INVALID_ARGUMENT
    assert L.hfr_allreduce(None, None, 0, 0, 0, None, None) == hfr.ERR_NOT_INITIALIZED
    assert L.hfr_wait(None, None) == hfr.SUCCESS
    assert L.hfr_finalize(None) == hfr.ERR_NOT_INITIALIZED
    assert L.hfr_comm_status(None) == hfr.ERR_NOT_INITIALIZED
    assert L.hfr_tree_query(0, 0, None, None, None) == hfr.ERR_INVALID_ARGUMENT


@pytest.mark.parametrize("n", list(range(1, 65)) + [100, 255, 256, 257, 1000, 1024])
def test_library_tree_equals_oracle_tree(n):
    want = O.build_double_binary_tree(n)
    for which in (0, 1):
        parent, children = hfr.tree_query(n, which)
        assert parent == want[which][0]
        assert children == want[which][1]


def test_config_struct_matches_header():
    """The ctypes mirror of hfr_config_t has the header's fields in the
    header's order with matching C types (the ABI of every call taking a
    config)."""
    src = open(os.path.join(ROOT, "include", "hfr.h")).read()
    body = re.search(r"typedef struct \{(.*?)\} hfr_config_t;", src, re.S).group(1)
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = re.findall(r"^\s*(int|size_t|float)\s+(\w+);", body, re.M)
    ctype = {"int": ctypes.c_int, "size_t": ctypes.c_size_t, "float": ctypes.c_float}
    assert [(n, ctype[t]) for t, n in fields] == [(n, t) for n, t in hfr._Config._fields_]
    assert [f for f in hfr.Config.__dataclass_fields__] == [n for _, n in fields]


def test_tree_staging_validated():
    L = hfr.lib()
    h = ctypes.c_void_p()
    bad = hfr.Config(tree_staging=3)._c()
    assert L.hfr_init_virtual(ctypes.byref(h), 2, 0, ctypes.byref(bad)) == hfr.ERR_INVALID_ARGUMENT
