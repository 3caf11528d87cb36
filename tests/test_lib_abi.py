"""CPU-side checks of the C ABI: libbf.so is built for sm_100a, loads, and exports
every function include/bf.h declares; host-only calls behave (no GPU needed)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bf.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\**\s+\**(bf_[a-z_0-9]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    __graft_entry__.build()
    from paper_1907_08607_b200 import bf
    return bf


def test_header_parses():
    names = declared_functions()
    for want in ("bf_graph_create", "bf_rank", "bf_count_total", "bf_count_vertex", "bf_count_edge",
                 "bf_wedge_count", "bf_nccl_unique_id", "bf_nccl_comm_create", "bf_graph_destroy",
                 "bf_status_str"):
        assert want in names


def test_exports_every_declared_symbol(lib):
    so = ctypes.CDLL(lib.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(so, n)]
    assert not missing, missing
    assert set(declared_functions()) <= set(lib.EXPORTED)


def test_built_for_sm100a(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_host_only_calls(lib):
    o = lib.bf_options_default()
    assert o.world_size == 1 and o.device == 0 and o.orient == lib.BF_ORIENT_AUTO
    assert lib._lib.bf_status_str(lib.BF_EDUP) == b"BF_EDUP"
    # argument checks happen before any CUDA call
    h = ctypes.c_void_p()
    assert lib._lib.bf_graph_create(1, 1, None, 5, None, ctypes.byref(h)) == lib.BF_EINVAL
    assert lib._lib.bf_graph_create(1, 1, None, 0, None, None) == lib.BF_EINVAL
    assert lib._lib.bf_graph_create(1, 1, None, 1 << 31, None, ctypes.byref(h)) == lib.BF_EINVAL
    assert lib._lib.bf_rank(None, 0) == lib.BF_EINVAL
    assert lib._lib.bf_count_total(None, None) == lib.BF_EINVAL
    w = ctypes.c_uint64()
    assert lib._lib.bf_wedge_count(None, ctypes.byref(w)) == lib.BF_EINVAL
    lib.bf_graph_destroy(None)


def test_product_does_not_import_oracle():
    """The product path never routes through the oracle (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_1907_08607_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "oracle.c" not in txt, f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".c")):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            assert "import paper_1907_08607_b200" not in txt and "from paper_1907_08607_b200" not in txt, f
            assert not re.search(r'#include\s+"[^"]*(bf|csrc)', txt), f
