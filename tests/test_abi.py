"""C-ABI boundary checks that need no GPU: the library loads, exports every
entry point include/infllm_b200.h declares, and its host-only entry points
(config defaults / validation, error codes, last_error) behave like the
reference's EngineConfig (types.hpp:84-109) and ModelShape (types.hpp:45-48).
No compute calls are made here.
"""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2402_04617_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "infllm_b200.h")
PKG = os.path.join(ROOT, "paper_2402_04617_b200")


def declared_functions():
    s = open(HEADER).read()
    s = re.sub(r"/\*.*?\*/", "", s, flags=re.S)
    s = re.sub(r"//[^\n]*", "", s)
    return sorted(set(re.findall(r"(?<![\w*])(infllm_\w+)\s*\(", s)))


@pytest.fixture(scope="module")
def L():
    if not os.path.exists(_lib.LIB_PATH):
        subprocess.check_call(["make", "-s", "-C", PKG])
    return _lib.lib()


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ["infllm_engine_create", "infllm_engine_destroy", "infllm_encode_chunk", "infllm_decode_step",
                 "infllm_finish", "infllm_retrieved_ids", "infllm_lookup", "infllm_select_representatives",
                 "infllm_get_layer_metrics", "infllm_trace", "infllm_unit_info", "infllm_last_error"]:
        assert must in names


def test_library_exports_every_declared_symbol(L):
    missing = [n for n in declared_functions() if not hasattr(L, n)]
    assert not missing, f"declared in {HEADER} but not exported: {missing}"


def test_exports_match_nm():
    if not os.path.exists(_lib.LIB_PATH):
        subprocess.check_call(["make", "-s", "-C", PKG])
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (infllm_\w+)", out))
    assert set(declared_functions()) <= exported
    # extern "C": no mangled public names leak the C++ engine types
    assert not [s for s in re.findall(r"\bT (\S+)", out) if s.startswith("_Z") and "infllm_" in s]


def test_ctypes_signatures_cover_header(L):
    assert set(declared_functions()) <= set(_lib.SIGNATURES)


def test_version_string(L):
    v = L.infllm_version().decode()
    assert "sm_100a" in v


def test_config_defaults_match_reference(L):
    c = _lib.EngineConfig()
    assert L.infllm_config_default(C.byref(c)) == 0
    # types.hpp:85-94
    assert (c.chunk_size, c.unit_size, c.n_repr, c.local_size, c.init_size, c.n_lookup, c.hot_capacity) == (
        512, 128, 4, 4096, 128, 32, 32)
    assert c.decay == 0.1
    assert c.lookup_mode == 0 and c.position_mode == 0


# one row per throw in EngineConfig::validate (types.hpp:96-109), same messages
BAD_CONFIGS = [
    (dict(chunk_size=0), "chunk_size must be >= 1"),
    (dict(unit_size=0), "unit_size must be >= 1"),
    (dict(n_repr=0), "n_repr must be >= 1"),
    (dict(local_size=0), "local_size must be >= 1"),
    (dict(init_size=-1), "init_size must be >= 0"),
    (dict(n_lookup=-1), "n_lookup must be >= 0"),
    (dict(n_repr=129), "n_repr must not exceed unit_size"),
    (dict(hot_capacity=8, n_lookup=9), "hot_capacity must be >= n_lookup"),
    (dict(decay=-0.01), "decay must lie in [0, 1]"),
    (dict(decay=1.5), "decay must lie in [0, 1]"),
]


@pytest.mark.parametrize("bad,msg", BAD_CONFIGS)
def test_config_validate_mirrors_reference(L, bad, msg):
    c = _lib.EngineConfig()
    L.infllm_config_default(C.byref(c))
    for k, v in bad.items():
        setattr(c, k, v)
    rc = L.infllm_config_validate(C.byref(c), None)
    assert rc == _lib.ERR_CONFIG
    assert msg in L.infllm_last_error().decode()


def test_config_validate_accepts_edges(L):
    c = _lib.EngineConfig()
    L.infllm_config_default(C.byref(c))
    c.n_lookup, c.hot_capacity, c.decay, c.init_size, c.n_repr, c.unit_size = 0, 0, 1.0, 0, 7, 7
    assert L.infllm_config_validate(C.byref(c), None) == 0


@pytest.mark.parametrize("shape,ok", [
    ((1, 32, 8, 128, 128), True),
    ((1, 4, 4, 64, 0), True),      # value_dim <= 0 -> head_dim
    ((1, 32, 5, 128, 128), False),  # n_heads % n_kv_heads != 0
    ((0, 32, 8, 128, 128), False),
    ((1, 0, 8, 128, 128), False),
    ((1, 8, 8, 0, 128), False),
])
def test_shape_validate(L, shape, ok):
    c = _lib.EngineConfig()
    L.infllm_config_default(C.byref(c))
    s = _lib.ModelShape(*shape)
    rc = L.infllm_config_validate(C.byref(c), C.byref(s))
    assert (rc == 0) == ok
    if not ok:
        assert rc == _lib.ERR_CONFIG and L.infllm_last_error()


def test_create_rejects_bad_config_before_touching_cuda(L):
    c = _lib.EngineConfig()
    L.infllm_config_default(C.byref(c))
    c.decay = 2.0
    s = _lib.ModelShape(1, 8, 2, 128, 128)
    h = C.c_void_p()
    assert L.infllm_engine_create(C.byref(c), C.byref(s), 1, 0, 0, 0, C.byref(h)) == _lib.ERR_CONFIG
    assert not h.value


def test_null_arguments_are_errors_not_crashes(L):
    assert L.infllm_config_validate(None, None) != 0
    assert L.infllm_engine_destroy(None) in (0, _lib.ERR_ARG)


def test_product_never_imports_the_oracle():
    """The product path has no CPU fallback: nothing under the package
    imports, loads or links oracle/ (only tests, smoke and bench may)."""
    offenders = []
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")) or f == "Makefile":
                text = open(os.path.join(dirpath, f), errors="replace").read()
                if re.search(r"^\s*(from|import)\s+oracle\b|liboracle|oracle/_ref|infllm_oracle", text, re.M):
                    offenders.append(f)
    assert not offenders, offenders
