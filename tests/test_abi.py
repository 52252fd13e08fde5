"""C-ABI library checks that need no GPU: it loads, exports every symbol that
include/remoe.h declares, validates arguments before touching the device, and
the binding names match the header."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "remoe.h")
HEADERS = sorted(os.path.join(ROOT, "include", f) for f in os.listdir(os.path.join(ROOT, "include"))
                 if f.endswith(".h"))


def declared():
    src = "".join(open(h).read() for h in HEADERS)
    return re.findall(r"REMOE_API\s+[\w\s\*]+?\b(remoe_\w+)\s*\(", src)


@pytest.fixture(scope="module")
def lib(remoe_lib_built):
    import paper_2512_18674_b200 as remoe
    return remoe.lib()


def test_header_declares_the_boundary():
    names = set(declared())
    for n in ("remoe_sps_build", "remoe_sps_query", "remoe_expert_plan", "remoe_sps_destroy",
              "remoe_nccl_unique_id", "remoe_status_string", "remoe_last_error"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    import paper_2512_18674_b200 as remoe
    out = subprocess.run(["nm", "-D", "--defined-only", remoe.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT\s+(remoe_\w+)", out))
    for n in declared():
        assert n in exported, n
        assert hasattr(lib, n)
    assert set(remoe.ABI_FUNCTIONS) | set(remoe.PLANNER_FUNCTIONS) == set(declared())


def test_status_strings_and_defaults(lib):
    import paper_2512_18674_b200 as remoe
    assert lib.remoe_status_string(0) == b"ok"
    assert lib.remoe_status_string(1) == b"invalid argument"
    c = remoe.remoe_sps_config_default()
    assert abs(c.sigma - 1e-6) < 1e-12 and c.temperature == 1.0 and c.world == 1


def test_argument_errors_are_synchronous(lib):
    """Invalid configs are rejected before any CUDA call (works without a GPU)."""
    import paper_2512_18674_b200 as remoe
    c = remoe.remoe_sps_config_default()
    h = ctypes.c_void_p()
    dummy = (ctypes.c_uint16 * 64)()
    act = (ctypes.c_float * 64)()
    c.n_local, c.dim, c.n_layers, c.n_experts = 8, 12, 1, 1   # dim % 8 != 0
    assert lib.remoe_sps_build(ctypes.byref(c), dummy, act, ctypes.byref(h)) == 1
    assert b"dim" in lib.remoe_last_error()
    c.dim = 8
    c.sigma = 0.0
    assert lib.remoe_sps_build(ctypes.byref(c), dummy, act, ctypes.byref(h)) == 1
    c.sigma = 1e-6
    c.max_k = 300
    assert lib.remoe_sps_build(ctypes.byref(c), dummy, act, ctypes.byref(h)) == 5
    c.max_k = 8
    c.world = 2  # world > 1 without an NCCL id
    assert lib.remoe_sps_build(ctypes.byref(c), dummy, act, ctypes.byref(h)) == 1
    assert lib.remoe_sps_query(None, None, 1, 1, None, None, None, None) == 6
    assert lib.remoe_expert_plan(None, 1, 1, 4, 5, None, None) == 1   # n_cold > E
    assert h.value is None


def test_binding_fails_loudly_without_library(monkeypatch, tmp_path):
    import paper_2512_18674_b200.sps as sps
    monkeypatch.setattr(sps, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(sps, "_LIB", None)
    with pytest.raises(RuntimeError, match="no fallback"):
        sps.lib()
